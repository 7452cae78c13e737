#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/e2e.txt
timeout 900 python -m pytest tests -q -m gpu -x --ignore=tests/test_dropin_gpu.py > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --config switch --no-cpu-baseline > gpurun_out/bench_switch.txt 2>&1; echo "switch rc=$?" >> gpurun_out/summary.txt
for c in 2 4 8; do
  EMOE_H2D_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 10 > gpurun_out/e_tmp.txt 2>&1
  echo "chunks$c $(tail -1 gpurun_out/e_tmp.txt)" >> gpurun_out/e2e.txt
done
cat gpurun_out/summary.txt
