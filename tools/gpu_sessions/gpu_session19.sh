#!/bin/bash
# re-entry check: full GPU suite, smoke, config-2 and config-3 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_s19.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_s19.txt >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/summary.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py > gpurun_out/bench_s19.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_s19.txt >> gpurun_out/summary.txt
timeout 600 python bench.py --config switch > gpurun_out/bench_switch_s19.txt 2>&1; echo "switch rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_switch_s19.txt >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
