#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/switch_launches.csv \
  -k regex:"route|scan|seg_offsets|permute|grouped_gemm|combine|hist" python bench.py --config switch --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu switch rc=$?" >> gpurun_out/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"route_from_logits|permute_kernel" -s 6 -c 2 -o gpurun_out/switch_full \
  python bench.py --config switch --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu switch full rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
