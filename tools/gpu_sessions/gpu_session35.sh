#!/bin/bash
# EP fault status tests; small-T fp32 gate; config-1 line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_ep.py tests/test_forward_gpu.py tests/test_edge_cases_gpu.py -q -x > gpurun_out/pytest_s35.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/pytest_s35.txt >> gpurun_out/summary.txt
timeout 300 python bench.py --config synthetic > gpurun_out/bench_synth35.txt 2>&1; echo "synth rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_synth35.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('synthetic', L['value'], L['ms_per_step'], L['stages_ms'])" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
