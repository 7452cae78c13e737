#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/e2e.txt gpurun_out/cg.txt
timeout 900 python -m pytest tests/test_edge_cases_gpu.py tests/test_forward_gpu.py -q -m gpu > gpurun_out/pytest_edge.txt 2>&1; echo "pytest edge rc=$?" >> gpurun_out/summary.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_forward_gpu.py -q -m gpu -k "mixtral_small or switch_small or host_pipelined" > gpurun_out/sanitizer_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/summary.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_forward_gpu.py -q -m gpu -k "mixtral_small and not cta1" > gpurun_out/sanitizer_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/summary.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_predictor_gpu.py -q -m gpu -k "invocation or golden" > gpurun_out/sanitizer_predictor.txt 2>&1; echo "memcheck predictor rc=$?" >> gpurun_out/summary.txt
for c in 8 16; do
  EMOE_H2D_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 5 > gpurun_out/e_tmp.txt 2>&1
  echo "chunks$c $(tail -1 gpurun_out/e_tmp.txt)" >> gpurun_out/e2e.txt
done
for cg in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --steps 40 --e2e-steps 1 --gemm-cta-group $cg > gpurun_out/c_tmp.txt 2>&1
  echo "cg$cg $(tail -1 gpurun_out/c_tmp.txt)" >> gpurun_out/cg.txt
done
cat gpurun_out/summary.txt
