python -m pytest tests/test_fullsize_gpu.py tests/test_fullshape_stack_gpu.py -m gpu -q -s > gpurun_out/r2_gputest_4b.txt 2>&1
python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py tests/test_random_shapes_gpu.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r2_gputest_4.txt
python bench.py --config switch > gpurun_out/r2_bench_switch_4.json 2> gpurun_out/r2_bench_switch_4.err
EMOE_GATE_ROUTE=split python bench.py --config switch > gpurun_out/r2_bench_switch_4split.json 2>&1
EMOE_GATE_CLUSTER=1 python bench.py --config switch > gpurun_out/r2_bench_switch_4c1.json 2>&1
EMOE_GATE_CLUSTER=4 python bench.py --config switch > gpurun_out/r2_bench_switch_4c4.json 2>&1
