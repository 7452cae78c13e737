#!/bin/bash
# e2e (host-buffer API) chunk sweep with 20 e2e steps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s40
rm -f gpurun_out/summary.txt gpurun_out/s40/ab.jsonl
for rep in 1 2; do
for c in 1 2 4; do
  EMOE_H2D_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --e2e-steps 20 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"chunks\": $c, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s40/ab.jsonl
done
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/s40/ab.jsonl"):
    d = json.loads(l); L = d["line"]
    print(d["chunks"], L["value"], L["ms_per_step"], "e2e", round(L["e2e"]["value"]), round(L["e2e"]["ms_per_step"], 3), L["clocks"]["sm_mhz"])
PY
cat gpurun_out/summary.txt
