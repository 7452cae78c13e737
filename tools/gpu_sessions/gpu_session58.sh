#!/bin/bash
# end-of-round measurements of the final state: headline line + reference arm,
# Switch and synthetic configs, launch list of the bench, ncu --set full of
# the config-2 GEMMs (one warm launch each), smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s58
rm -f gpurun_out/summary.txt
timeout 900 python bench.py > gpurun_out/s58/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --impl reference > gpurun_out/s58/bench_ref.txt 2>&1; echo "ref rc=$?" >> gpurun_out/summary.txt
for c in switch synthetic; do
  timeout 600 python bench.py --config $c > gpurun_out/s58/bench_$c.txt 2>&1; echo "$c rc=$?" >> gpurun_out/summary.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:gemm_kernel|route|permute|scan|seg_offsets|combine|hist|prompt_trans|save_last" \
  --csv --log-file gpurun_out/s58/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline \
  > gpurun_out/s58/ncu_launches.txt 2>&1; echo "ncu launches rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_kernel --launch-skip 3 --launch-count 2 \
  -o gpurun_out/s58/mixtral_gemms -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s58/ncu_gemm.txt 2>&1; echo "ncu gemm rc=$?" >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s58/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
