#!/bin/bash
# ncu full capture of the 3xTF32 GEMMs (config 1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s56
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tf32x3_kernel --launch-skip 4 --launch-count 2 \
  -o gpurun_out/s56/tf32_gemms -f python bench.py --config synthetic --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s56/ncu.txt 2>&1
echo "ncu rc=$?"
