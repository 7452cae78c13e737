#!/bin/bash
# split-K 3xTF32 for small batches: parity + config-1 line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s57
rm -f gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py tests/test_random_shapes_gpu.py -q -x -k "fp32 or config1 or random or stage_api" > gpurun_out/s57/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s57/pytest.txt >> gpurun_out/summary.txt
timeout 300 python bench.py --config synthetic > gpurun_out/s57/bench.txt 2>&1; echo "synth rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/s57/bench.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('synthetic', L['value'], L['ms_per_step'], L['stages_ms'], L['roofline']['frac'], L['roofline']['achieved'])" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
