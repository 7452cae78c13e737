#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 1200 python -m pytest tests -q -m gpu -x --ignore=tests/test_dropin_gpu.py > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --config stream --stream-layers 8 --stream-prompts 80 > gpurun_out/bench_stream8.txt 2>&1; echo "stream8 rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --config stream --stream-layers 32 --stream-prompts 120 > gpurun_out/bench_stream32.txt 2>&1; echo "stream32 rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
