#!/bin/bash
# first GPU session: correctness of every stage, then a short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 120 python tools/gemm_check.py 1024 512 1024 8 2 4 > gpurun_out/gemm_check_small.txt 2>&1; echo "gemm_check_small rc=$?" >> gpurun_out/summary.txt
timeout 120 python tools/gemm_check.py 8192 4096 14336 8 2 4 > gpurun_out/gemm_check_big.txt 2>&1; echo "gemm_check_big rc=$?" >> gpurun_out/summary.txt
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
