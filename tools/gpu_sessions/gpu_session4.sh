#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/ab.txt
for i in 1 2 3; do
  for cg in 1 2; do
    timeout 300 python bench.py --gemm-cta-group $cg --no-cpu-baseline --steps 60 --e2e-steps 1 > gpurun_out/ab_tmp.txt 2>&1
    echo "cg$cg $(tail -1 gpurun_out/ab_tmp.txt)" >> gpurun_out/ab.txt
  done
done
for cg in 1 2; do
timeout 900 ncu --set full --clock-control none -k regex:grouped_gemm_kernel -s 6 -c 2 \
  -o gpurun_out/gemm_full_cg$cg python bench.py --gemm-cta-group $cg --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_cg$cg.txt 2>&1; echo "ncu cg$cg rc=$?" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
