#!/bin/bash
# fused top-2 combine: GPU suite + A/B against the separate combine kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_suite.log 2>&1; echo rc=$? >> gpurun_out/gpu_suite.log
out=gpurun_out/fused_top2_ab.jsonl; : > $out
for rep in 1 2 3; do
  for fc in 2 1; do
    line=$(EMOE_FUSED_COMBINE=$fc timeout 400 python bench.py --e2e-steps 40 --no-cpu-baseline 2>/dev/null | tail -1)
    python - "$fc" "$line" >> $out <<'PY'
import json, sys
d = json.loads(sys.argv[2])
print(json.dumps(dict(fused_combine=sys.argv[1], value=d["value"], ms_per_step=d["ms_per_step"],
                      e2e=d["e2e"]["value"], stages_ms=d["stages_ms"], sm_mhz=d["clocks"]["sm_mhz"],
                      power_w=d["clocks"].get("power_w_median"))))
PY
  done
done
