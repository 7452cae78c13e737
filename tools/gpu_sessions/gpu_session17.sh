#!/bin/bash
# on-demand (dynamic) residency baseline vs predicted residency on the config-5 stream
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 600 python -m pytest tests/test_serving_gpu.py tests/test_forward_gpu.py -q -x > gpurun_out/pytest_s17.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_s17.txt >> gpurun_out/summary.txt
timeout 900 python bench.py --config stream --residency predicted > gpurun_out/bench_stream_pred.txt 2>&1; echo "pred rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --config stream --residency dynamic > gpurun_out/bench_stream_dyn.txt 2>&1; echo "dyn rc=$?" >> gpurun_out/summary.txt
for f in bench_stream_pred bench_stream_dyn; do
  tail -1 gpurun_out/$f.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); s=L['stream']; print('$f', L['value'], L['ms_per_step'], s.get('hit_rate'), s.get('planned_loads'), s.get('load_gbs'), L['clocks']['sm_mhz'])" >> gpurun_out/summary.txt 2>&1
done
cat gpurun_out/summary.txt
