#!/bin/bash
# CTA-pair ring depth sensitivity of the short-K Switch GEMM1 (compile-time variants)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/summary.txt gpurun_out/stages31.jsonl
for v in 6 5 4 3; do
  if [ $v = 6 ]; then L=""; else L=$GRAFT_REPO_ROOT/paper_2503_06823_b200/lib/var_s$v/libemoe.so; fi
  EMOE_LIB_PATH=$L timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"cg2_stages\": $v, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/stages31.jsonl
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/stages31.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["cg2_stages"], L["value"], L["ms_per_step"], L["stages_ms"], L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
