#!/bin/bash
# EP over peer memory with the return pushed from GEMM2's epilogue (2 ranks on one B200)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_ep.py tests/test_forward_gpu.py -q -x > gpurun_out/pytest_s29.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/pytest_s29.txt >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
