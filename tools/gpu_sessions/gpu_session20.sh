#!/bin/bash
# 8 vs 4 epilogue warps in the grouped GEMM: parity (incl. long-K cases) + A/B + ncu of the Switch GEMM1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/ab20.jsonl
timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_edge_cases_gpu.py -q -x > gpurun_out/pytest_s20.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_s20.txt >> gpurun_out/summary.txt
for rep in 1 2; do
  for ew in 8 4; do
    EMOE_GEMM_EPI_WARPS=$ew timeout 300 python bench.py --config switch --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
    echo "{\"ew\": $ew, \"config\": \"switch\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/ab20.jsonl
  done
done
for ew in 8 4; do
  EMOE_GEMM_EPI_WARPS=$ew timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"ew\": $ew, \"config\": \"mixtral\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/ab20.jsonl
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_kernel --launch-skip 8 --launch-count 2 \
  -o gpurun_out/switch_gemm_ew8 -f python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu20.txt 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/ab20.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["ew"], d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"], L["roofline"]["achieved"])
    except Exception as e:
        print("bad", l[:200], e)
PY
cat gpurun_out/summary.txt
