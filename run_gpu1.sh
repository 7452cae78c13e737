set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest_1.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_1.txt 2>&1
python bench.py > gpurun_out/r2_bench_mixtral_1.json 2> gpurun_out/r2_bench_mixtral_1.err
python bench.py --config switch > gpurun_out/r2_bench_switch_1.json 2> gpurun_out/r2_bench_switch_1.err
python bench.py --config synthetic > gpurun_out/r2_bench_synth_1.json 2> gpurun_out/r2_bench_synth_1.err
tail -3 gpurun_out/r2_gputest_1.txt
