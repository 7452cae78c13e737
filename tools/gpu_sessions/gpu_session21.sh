#!/bin/bash
# peer-memory expert parallelism (2 ranks sharing the B200) + ncu of the Switch GEMM1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_ep.py tests/test_forward_gpu.py -q -x > gpurun_out/pytest_s21.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/pytest_s21.txt >> gpurun_out/summary.txt
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:grouped_gemm_kernel<1' --launch-skip 3 --launch-count 1 \
  -o gpurun_out/switch_gemm1 -f python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu21.txt 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/ncu21.txt >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
