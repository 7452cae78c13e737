#!/bin/bash
# GEMM1 row gather (fused permute): parity + A/B on both bf16 configs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/gather25.jsonl
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py tests/test_ep.py -q -x > gpurun_out/pytest_s25.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/pytest_s25.txt >> gpurun_out/summary.txt
for rep in 1 2; do
for g in 1 0; do
  EMOE_GATHER_A=$g timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"gather\": $g, \"config\": \"switch\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/gather25.jsonl
  EMOE_GATHER_A=$g timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"gather\": $g, \"config\": \"mixtral\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/gather25.jsonl
done
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/gather25.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["gather"], d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
