#!/bin/bash
# raster group sweep (exact group_m) on the Switch and Mixtral shapes; config-1 (fp32) bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/group23.jsonl
for gm in 1 2 4 10; do
  EMOE_GEMM_GROUP_M=$gm timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"group_m\": $gm, \"config\": \"switch\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/group23.jsonl
done
for gm in 2 8 24; do
  EMOE_GEMM_GROUP_M=$gm timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"group_m\": $gm, \"config\": \"mixtral\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/group23.jsonl
done
timeout 300 python bench.py --config synthetic > gpurun_out/bench_synth23.txt 2>&1; echo "synthetic rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/bench_synth23.txt >> gpurun_out/summary.txt
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/group23.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["group_m"], d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:200], e)
PY
cat gpurun_out/summary.txt
