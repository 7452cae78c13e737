#!/bin/bash
# A/B: L2 prefetch of the next tile's operand boxes in the grouped GEMM producer
# (the prefetch code was reverted after this A/B: profiles/r01_gemm_l2_prefetch_ab.jsonl)
mkdir -p gpurun_out
out=gpurun_out/prefetch_ab.jsonl; : > $out
EMOE_GEMM_PREFETCH=1 timeout 600 python -m pytest tests/test_forward_gpu.py -m gpu -x -q > gpurun_out/prefetch_tests.log 2>&1; echo rc=$? >> gpurun_out/prefetch_tests.log
for rep in 1 2; do
  for cfg in switch mixtral; do
    for pf in 0 1; do
      arg=""; [ $cfg = switch ] && arg="--config switch"
      line=$(EMOE_GEMM_PREFETCH=$pf timeout 400 python bench.py $arg --e2e-steps 4 2>/dev/null | tail -1)
      python - "$pf" "$cfg" "$line" >> $out <<'PY'
import json, sys
d = json.loads(sys.argv[3])
print(json.dumps(dict(prefetch=int(sys.argv[1]), config=sys.argv[2], value=d["value"], ms_per_step=d["ms_per_step"],
                      stages_ms=d["stages_ms"], sm_mhz=d["clocks"]["sm_mhz"])))
PY
    done
  done
done
