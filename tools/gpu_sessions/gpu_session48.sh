#!/bin/bash
# L2 policy of the epilogue TMA stores: none vs evict-first vs evict-last (alternating reps)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/summary.txt gpurun_out/sh48.jsonl
for rep in 1 2; do
for h in 0 1 2; do
  EMOE_GEMM_STORE_HINT=$h timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"store_hint\": $h, \"config\": \"mixtral\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/sh48.jsonl
  EMOE_GEMM_STORE_HINT=$h timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"store_hint\": $h, \"config\": \"switch\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/sh48.jsonl
done
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/sh48.jsonl"):
    d = json.loads(l); L = d["line"]; s = L["stages_ms"]
    print(d["store_hint"], d["config"], L["value"], L["ms_per_step"], s["gemm1"], s["gemm2"], L["clocks"]["sm_mhz"])
PY
cat gpurun_out/summary.txt
