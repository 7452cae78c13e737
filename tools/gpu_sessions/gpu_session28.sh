#!/bin/bash
# full GPU suite; compute-sanitizer on the new kernels (3xTF32, fused top-1 combine,
# column-split permute); config-1 line; ncu launch list + GEMM DRAM traffic of the headline command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s28
rm -f gpurun_out/summary.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s28/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s28/pytest.txt >> gpurun_out/summary.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_forward_gpu.py -q -m gpu -k "mixtral_small or switch_small or fp32 or config1 or host_pipelined" > gpurun_out/s28/sanitizer_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/s28/sanitizer_memcheck.txt >> gpurun_out/summary.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_forward_gpu.py -q -m gpu -k "switch_small_cta2 or fp32_relu" > gpurun_out/s28/sanitizer_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/s28/sanitizer_racecheck.txt >> gpurun_out/summary.txt
timeout 300 python bench.py --config synthetic > gpurun_out/s28/bench_synth.txt 2>&1; echo "synth rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/s28/bench_synth.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('synthetic', L['value'], L['ms_per_step'], L['stages_ms'], L['roofline']['frac'])" >> gpurun_out/summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s28/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s28/ncu_launch_bench.txt 2>&1; echo "ncu launches rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:grouped_gemm --launch-skip 6 --launch-count 2 --log-file gpurun_out/s28/gemm_traffic.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s28/ncu_traffic_bench.txt 2>&1; echo "ncu traffic rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
