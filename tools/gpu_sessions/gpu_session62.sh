#!/bin/bash
# after the tile-decode fix: Switch bench line, ncu --set full of the Switch GEMMs,
# the K probe again (the per-tile fixed cost should be gone)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s62
rm -f gpurun_out/summary.txt
timeout 900 python bench.py --config switch > gpurun_out/s62/bench_switch.txt 2>&1; echo "switch rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_kernel --launch-skip 4 --launch-count 2 \
  -o gpurun_out/s62/switch_gemms -f python bench.py --config switch --graph off --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
  > gpurun_out/s62/ncu_switch.txt 2>&1; echo "ncu switch rc=$?" >> gpurun_out/summary.txt
timeout 900 python tools/pitch_probe.py 512 768 1024 1280 > gpurun_out/s62/k_probe.txt 2>&1; echo "probe rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
