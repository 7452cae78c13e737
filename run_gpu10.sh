./tools/probes/tma_stream_probe 768 > gpurun_out/r2_tma_probe_768.txt 2>&1
./tools/probes/tma_stream_probe 4096 > gpurun_out/r2_tma_probe_4096.txt 2>&1
python -m pytest tests/test_forward_gpu.py -m gpu -q -k "fused_gate" 2>&1 | tail -3 > gpurun_out/r2_gputest_10.txt
