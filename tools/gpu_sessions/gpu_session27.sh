#!/bin/bash
# fp32 (config 1) on tcgen05 3xTF32: parity at 1e-5 + A/B against the SIMT FFMA kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/tf32_27.jsonl
timeout 900 python -m pytest tests/test_forward_gpu.py -q -x -k "fp32 or config1" > gpurun_out/pytest_s27.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -25 gpurun_out/pytest_s27.txt >> gpurun_out/summary.txt
for m in tf32 ffma; do
  EMOE_F32_GEMM=$m timeout 300 python bench.py --config synthetic --no-cpu-baseline --e2e-steps 5 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"f32_gemm\": \"$m\", \"config\": \"synthetic\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/tf32_27.jsonl
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/tf32_27.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["f32_gemm"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["roofline"]["achieved"], L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
