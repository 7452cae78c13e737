#!/bin/bash
# routing prefetch + per-block fallback; Switch launch list and full ncu of one Switch step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 600 python -m pytest tests -q -m gpu -x --ignore=tests/test_dropin_gpu.py > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_gpu.txt >> gpurun_out/summary.txt
timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_switch.txt 2>&1; echo "switch rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_switch.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print(L['value'], L['ms_per_step'], L['stages_ms'], L['clocks']['sm_mhz'], L['config']['gemm_cta_group'])" >> gpurun_out/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/switch_launches15.csv \
  python bench.py --config switch --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu15a.txt 2>&1; echo "ncu list rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:route_from_logits_kernel|seg_offsets_kernel|permute_kernel|grouped_gemm_kernel' \
  --launch-skip 18 --launch-count 6 -o gpurun_out/switch_step15 -f \
  python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu15b.txt 2>&1; echo "ncu full rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
