#!/bin/bash
# final lines on the final code: configs 1-3 (the tile-decode fix and the fused
# tf32 split came after session 61), the GPU suite and smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s65
rm -f gpurun_out/summary.txt
for c in mixtral switch synthetic; do
  timeout 900 python bench.py --config $c > gpurun_out/s65/bench_$c.txt 2>&1; echo "$c rc=$?" >> gpurun_out/summary.txt
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s65/suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/s65/suite.log >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s65/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
