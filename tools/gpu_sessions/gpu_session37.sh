#!/bin/bash
# GEMM2 column panel 8 vs off, alternating repetitions on one box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s37
rm -f gpurun_out/summary.txt gpurun_out/s37/ab.jsonl
for rep in 1 2 3; do
for g2 in 0 8; do
  EMOE_GEMM2_NPANEL=$g2 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"g2\": $g2, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s37/ab.jsonl
done
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/s37/ab.jsonl"):
    d = json.loads(l); L = d["line"]; s = L["stages_ms"]; mhz = L["clocks"]["sm_mhz"]
    print(d["g2"], L["value"], L["ms_per_step"], s["gemm1"], s["gemm2"], mhz, "gemm2*MHz", round(s["gemm2"] * mhz), "gemm1*MHz", round(s["gemm1"] * mhz), L["clocks"].get("power_w_median"))
PY
cat gpurun_out/summary.txt
