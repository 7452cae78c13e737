python -m pytest tests/test_ep.py tests/test_forward_gpu.py tests/test_serving_gpu.py tests/test_bench_contract.py -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r2_gputest_2.txt
python bench.py --config stack --steps 4 --warmup 3 --e2e-steps 2 > gpurun_out/r2_bench_stack_2.json 2> gpurun_out/r2_bench_stack_2.err
