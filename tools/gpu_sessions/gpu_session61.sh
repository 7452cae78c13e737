#!/bin/bash
# final refresh: default bench line of every config (3 repetitions of the headline
# for the run-to-run spread), the stack and stream configs, ncu --set full of the
# Switch and 3xTF32 GEMMs under the final code
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s61
rm -f gpurun_out/summary.txt
for rep in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/s61/bench_$rep.txt 2>&1; echo "bench $rep rc=$?" >> gpurun_out/summary.txt
done
for c in switch synthetic stack; do
  timeout 900 python bench.py --config $c > gpurun_out/s61/bench_$c.txt 2>&1; echo "$c rc=$?" >> gpurun_out/summary.txt
done
timeout 1200 python bench.py --config stream > gpurun_out/s61/bench_stream.txt 2>&1; echo "stream rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_kernel --launch-skip 4 --launch-count 2 \
  -o gpurun_out/s61/switch_gemms -f python bench.py --config switch --graph off --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
  > gpurun_out/s61/ncu_switch.txt 2>&1; echo "ncu switch rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3_kernel|splitk_reduce" --launch-skip 6 --launch-count 3 \
  -o gpurun_out/s61/tf32_gemms -f python bench.py --config synthetic --graph off --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
  > gpurun_out/s61/ncu_tf32.txt 2>&1; echo "ncu tf32 rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
