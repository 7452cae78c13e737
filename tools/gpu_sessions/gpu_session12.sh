#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 900 python -m pytest tests -q -m gpu -x --ignore=tests/test_dropin_gpu.py > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --config switch --no-cpu-baseline > gpurun_out/bench_switch.txt 2>&1; echo "switch rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
