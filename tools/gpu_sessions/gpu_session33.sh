#!/bin/bash
# kernel-time vs step-time (launch gaps) for the Switch and config-1 shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s33
rm -f gpurun_out/summary.txt
for c in switch synthetic; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 3 > gpurun_out/s33/bench_$c.txt 2>&1
  tail -1 gpurun_out/s33/bench_$c.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('$c', L['value'], L['ms_per_step'], L['stages_ms'], L['gpu_launches'])" >> gpurun_out/summary.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s33/launches_$c.csv python bench.py --config $c --steps 4 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
cat gpurun_out/summary.txt
