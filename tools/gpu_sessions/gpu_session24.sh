#!/bin/bash
# gather4 probe; parity after the fp32 gate rewrite and K-aware raster; switch + synthetic lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 60 ./tools/probes/gather4_probe >> gpurun_out/summary.txt 2>&1; echo "probe rc=$?" >> gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py tests/test_predictor_gpu.py -q -x > gpurun_out/pytest_s24.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_s24.txt >> gpurun_out/summary.txt
timeout 300 python bench.py --config switch > gpurun_out/bench_switch24.txt 2>&1; echo "switch rc=$?" >> gpurun_out/summary.txt
timeout 300 python bench.py --config synthetic > gpurun_out/bench_synth24.txt 2>&1; echo "synth rc=$?" >> gpurun_out/summary.txt
for f in bench_switch24 bench_synth24; do
  tail -1 gpurun_out/$f.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('$f', L['value'], L['ms_per_step'], L['stages_ms'], L['roofline']['frac'], L['e2e']['value'], L['clocks']['sm_mhz'])" >> gpurun_out/summary.txt 2>&1
done
cat gpurun_out/summary.txt
