python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py tests/test_random_shapes_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x 2>&1 | tail -8 > gpurun_out/r2_gputest_6.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate_route|route_from|grouped_gemm|permute|scan|seg_off|hist|combine" -c 40 --csv --log-file gpurun_out/r2_switch_launches_6.csv python bench.py --config switch --steps 3 --warmup 3 --e2e-steps 2 --graph off --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate_route|route_from|permute|scan|seg_off|hist|combine" -c 30 --csv --log-file gpurun_out/r2_mixtral_launches_6.csv python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
python bench.py --config switch > gpurun_out/r2_bench_switch_6.json 2> gpurun_out/r2_bench_switch_6.err
python bench.py > gpurun_out/r2_bench_mixtral_6.json 2> gpurun_out/r2_bench_mixtral_6.err
