python -m pytest tests/test_forward_gpu.py -m gpu -q -k "multicast or bulk" 2>&1 | tail -4 > gpurun_out/r2_gputest_7.txt
ncu --set full --clock-control none --import-source on -k regex:gate_route_tc -c 1 -o gpurun_out/r2_gate_tc7 python bench.py --config switch --steps 3 --warmup 3 --e2e-steps 2 --graph off --no-cpu-baseline > /dev/null 2>&1
for i in 1 2; do
python bench.py --no-cpu-baseline > gpurun_out/r2_mc1_$i.json 2>&1
EMOE_GEMM_MC=2 python bench.py --no-cpu-baseline > gpurun_out/r2_mc2_$i.json 2>&1
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:grouped_gemm -c 4 --csv --log-file gpurun_out/r2_gemm_traffic_mc1.csv python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
EMOE_GEMM_MC=2 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:grouped_gemm -c 4 --csv --log-file gpurun_out/r2_gemm_traffic_mc2.csv python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
