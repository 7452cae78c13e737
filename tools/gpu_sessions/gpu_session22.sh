#!/bin/bash
# Switch GEMM1: ncu full capture + raster panel sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/panel22.jsonl
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:grouped_gemm_kernel<\(int\)1,' --launch-skip 3 --launch-count 1 \
  -o gpurun_out/switch_gemm1 -f python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu22.txt 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
for mb in 4 8 16 24 64; do
  EMOE_GEMM_PANEL_MB=$mb timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"panel_mb\": $mb, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/panel22.jsonl
done
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/panel22.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["panel_mb"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"])
    except Exception as e:
        print("bad", l[:200], e)
PY
cat gpurun_out/summary.txt
