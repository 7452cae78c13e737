#!/bin/bash
# full GPU suite with the column-panel GEMM2 default + headline bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s39
rm -f gpurun_out/summary.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s39/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s39/pytest.txt >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/summary.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py > gpurun_out/s39/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/s39/bench.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('bench', L['value'], L['ms_per_step'], L['stages_ms'], L['roofline']['frac'], L['roofline']['traffic'], L['e2e']['value'], L['clocks'])" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
