python -m pytest tests/test_ep.py -m gpu -q 2>&1 | tail -15 > gpurun_out/r2_gputest_11.txt
python -m pytest tests/test_forward_gpu.py -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/r2_gputest_11.txt
