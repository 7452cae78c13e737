#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
for cg in 1 2; do
  timeout 120 python tools/gemm_check.py 1024 512 1024 8 2 4 $cg > gpurun_out/gemm_check_small_cg$cg.txt 2>&1; echo "gemm_check_small cg$cg rc=$?" >> gpurun_out/summary.txt
  timeout 180 python tools/gemm_check.py 16384 4096 14336 8 2 4 $cg > gpurun_out/gemm_check_big_cg$cg.txt 2>&1; echo "gemm_check_big cg$cg rc=$?" >> gpurun_out/summary.txt
done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --gemm-cta-group 1 --no-cpu-baseline > gpurun_out/bench_cg1.txt 2>&1; echo "bench cg1 rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --gemm-cta-group 2 --no-cpu-baseline > gpurun_out/bench_cg2.txt 2>&1; echo "bench cg2 rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
