#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/panel.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
for i in 1 2; do
  for mb in 24 48 96; do
    EMOE_GEMM_PANEL_MB=$mb timeout 300 python bench.py --no-cpu-baseline --steps 40 --e2e-steps 1 > gpurun_out/p_tmp.txt 2>&1
    echo "panel$mb $(tail -1 gpurun_out/p_tmp.txt)" >> gpurun_out/panel.txt
  done
done
timeout 600 python bench.py --config switch --no-cpu-baseline > gpurun_out/bench_switch.txt 2>&1; echo "bench switch rc=$?" >> gpurun_out/summary.txt
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.txt 2>&1; echo "bench ref rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
