#!/bin/bash
# predictor invocation on its own stream with a persistent arena: parity suites + measured cost model
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
timeout 1200 python -m pytest tests/test_predictor_gpu.py tests/test_serving_gpu.py tests/test_dropin_gpu.py -q -x > gpurun_out/pytest_s32.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_s32.txt >> gpurun_out/summary.txt
timeout 900 python tools/profile_cost_model.py --layers 32 > gpurun_out/cost_model_s32.json 2> gpurun_out/cost_model_s32.err; echo "cost rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/cost_model_s32.json >> gpurun_out/summary.txt
tail -3 gpurun_out/cost_model_s32.err >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
