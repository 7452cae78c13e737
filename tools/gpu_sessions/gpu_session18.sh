#!/bin/bash
# measured reference CostModel on the B200 (config-5 stack)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 600 python -m pytest tests/test_serving_gpu.py -q -x > gpurun_out/pytest_s18.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_s18.txt >> gpurun_out/summary.txt
timeout 900 python tools/profile_cost_model.py --layers 32 > gpurun_out/cost_model.json 2> gpurun_out/cost_model.err; echo "cost rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/cost_model.json >> gpurun_out/summary.txt
tail -5 gpurun_out/cost_model.err >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
