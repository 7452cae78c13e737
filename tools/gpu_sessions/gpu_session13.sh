#!/bin/bash
# TMA-store epilogue: parity + A/B against the direct-store epilogue + ncu of the Switch GEMMs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/ab13.jsonl
timeout 600 python -m pytest tests -q -m gpu -x --ignore=tests/test_dropin_gpu.py > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_gpu.txt >> gpurun_out/summary.txt
for rep in 1 2; do
  for ts in 1 0; do
    EMOE_GEMM_TMA_STORE=$ts timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
    echo "{\"tma_store\": $ts, \"config\": \"switch\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/ab13.jsonl
  done
done
for ts in 1 0; do
  EMOE_GEMM_TMA_STORE=$ts timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"tma_store\": $ts, \"config\": \"mixtral\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/ab13.jsonl
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_kernel --launch-skip 8 --launch-count 2 \
  -o gpurun_out/switch_gemm_tma -f python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu13.txt 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/ab13.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["tma_store"], d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"], L["roofline"]["achieved"])
    except Exception as e:
        print("bad", l[:200], e)
PY
cat gpurun_out/summary.txt
