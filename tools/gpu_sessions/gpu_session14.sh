#!/bin/bash
# cta_group 1 vs 2 with the TMA-store epilogue (Switch + Mixtral), ncu of the Switch GEMM1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/ab14.jsonl
for rep in 1 2; do
  for cg in 1 2; do
    for cfg in switch mixtral; do
      timeout 300 python bench.py --config $cfg --gemm-cta-group $cg --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
      echo "{\"cg\": $cg, \"config\": \"$cfg\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/ab14.jsonl
    done
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:grouped_gemm_kernel<1, 1>' --launch-skip 3 --launch-count 1 \
  -o gpurun_out/switch_gemm1_tma -f python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu14.txt 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/ab14.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["cg"], d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"], L["clocks"].get("power_w_median"), L["roofline"]["achieved"])
    except Exception as e:
        print("bad", l[:200], e)
PY
cat gpurun_out/summary.txt
