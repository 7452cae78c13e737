#!/bin/bash
# final round-1 measurements: headline bench line + reference arm, other configs,
# ncu --set full of the config-2 GEMMs and HBM-bound kernels (timed-step launches)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s34
rm -f gpurun_out/summary.txt
timeout 900 python bench.py > gpurun_out/s34/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/s34/bench.txt >> gpurun_out/summary.txt
timeout 900 python bench.py --impl reference > gpurun_out/s34/bench_ref.txt 2>&1; echo "ref rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/s34/bench_ref.txt >> gpurun_out/summary.txt
for c in switch synthetic; do
  timeout 600 python bench.py --config $c > gpurun_out/s34/bench_$c.txt 2>&1; echo "$c rc=$?" >> gpurun_out/summary.txt
done
timeout 900 python bench.py --config stream > gpurun_out/s34/bench_stream.txt 2>&1; echo "stream rc=$?" >> gpurun_out/summary.txt
# full captures: launches 3..4 of each kernel family are warm-up forwards at full T
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_kernel --launch-skip 3 --launch-count 2 \
  -o gpurun_out/s34/mixtral_gemms -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s34/ncu_gemm.txt 2>&1; echo "ncu gemm rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gate_route|permute_kernel|combine_bf16" --launch-skip 3 --launch-count 3 \
  -o gpurun_out/s34/mixtral_hbm -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s34/ncu_hbm.txt 2>&1; echo "ncu hbm rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
