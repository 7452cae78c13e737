#!/bin/bash
# shared stack workspace: serving tests + BASELINE config 4 (32-layer stack) bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s49
rm -f gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_serving_gpu.py tests/test_boundary.py -q -x > gpurun_out/s49/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s49/pytest.txt >> gpurun_out/summary.txt
timeout 900 python bench.py --config stack --steps 6 > gpurun_out/s49/bench_stack.txt 2>&1; echo "stack rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s49/bench_stack.txt | cut -c1-2500 >> gpurun_out/summary.txt
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
