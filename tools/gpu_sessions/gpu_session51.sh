#!/bin/bash
# routing fused into the gate GEMM epilogue (E >= 32): parity + A/B on the Switch shape
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s51
rm -f gpurun_out/summary.txt gpurun_out/s51/ab.jsonl
timeout 900 python -m pytest tests/test_edge_cases_gpu.py tests/test_forward_gpu.py -q -x > gpurun_out/s51/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -15 gpurun_out/s51/pytest.txt >> gpurun_out/summary.txt
for rep in 1 2; do
for g in 1 0; do
  EMOE_FUSED_GATE_ROUTE=$g timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"fused_gate\": $g, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s51/ab.jsonl
done
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/s51/ab.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["fused_gate"], L["value"], L["ms_per_step"], L["stages_ms"], L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
