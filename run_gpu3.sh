python -m pytest tests/test_ep.py tests/test_forward_gpu.py tests/test_serving_gpu.py tests/test_bench_contract.py -m gpu -q 2>&1 | tail -30 > gpurun_out/r2_gputest_3.txt
python -m pytest tests/test_fullsize_gpu.py tests/test_fullshape_stack_gpu.py -m gpu -q -s 2>&1 | tail -40 > gpurun_out/r2_gputest_3b.txt
