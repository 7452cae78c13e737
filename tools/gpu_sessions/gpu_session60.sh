#!/bin/bash
# compute-sanitizer memcheck over this round's new device code: route_from_logits
# staging, gate tensor map over the real rows, combine column split, 3xTF32 split /
# split-K bounds, fused top-2 combine (opt-in), device predictor tallies
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s60
rm -f gpurun_out/summary.txt
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py -q -m gpu \
  -k "not fused and not raster and not host_async" > gpurun_out/s60/memcheck_forward.txt 2>&1; echo "memcheck forward rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s60/memcheck_forward.txt >> gpurun_out/summary.txt
EMOE_FUSED_COMBINE=2 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_edge_cases_gpu.py -q -m gpu \
  -k "ragged or stage_api" > gpurun_out/s60/memcheck_fused_top2.txt 2>&1; echo "memcheck fused top2 rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s60/memcheck_fused_top2.txt >> gpurun_out/summary.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_predictor_sync.py -q -m gpu > gpurun_out/s60/memcheck_predictor_sync.txt 2>&1; echo "memcheck predictor sync rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/s60/memcheck_predictor_sync.txt >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
