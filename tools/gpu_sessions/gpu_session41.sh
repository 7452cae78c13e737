#!/bin/bash
# Switch shape: column panels for the short-K GEMM1, CTA group re-check
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s41
rm -f gpurun_out/summary.txt gpurun_out/s41/ab.jsonl
for cfg in "0 0" "4 0" "6 0" "3 0" "0 1"; do
  set -- $cfg
  if [ $2 = 1 ]; then CG="--gemm-cta-group 1"; else CG=""; fi
  EMOE_GEMM1_NPANEL=$1 timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 $CG > gpurun_out/b_tmp.txt 2>&1
  echo "{\"g1\": $1, \"cg1\": $2, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s41/ab.jsonl
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/s41/ab.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["g1"], d["cg1"], L["value"], L["ms_per_step"], L["stages_ms"], L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:200], e)
PY
cat gpurun_out/summary.txt
