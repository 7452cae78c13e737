#!/bin/bash
# top-1 combine fused into GEMM2: full GPU suite + A/B on the Switch shape
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/fused26.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_s26.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/pytest_s26.txt >> gpurun_out/summary.txt
for rep in 1 2; do
for g in 1 0; do
  EMOE_FUSED_COMBINE=$g timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"fused_combine\": $g, \"config\": \"switch\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/fused26.jsonl
done
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/fused26.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["fused_combine"], d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
