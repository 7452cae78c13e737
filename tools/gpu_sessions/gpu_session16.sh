#!/bin/bash
# smem-staged routing, flat permute gather, 64-col TMA store boxes + relaxed TMEM-empty arrive
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/ab16.jsonl
timeout 600 python -m pytest tests -q -m gpu -x --ignore=tests/test_dropin_gpu.py > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_gpu.txt >> gpurun_out/summary.txt
for cfg in switch mixtral switch; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"config\": \"$cfg\", \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/ab16.jsonl
done
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:route_from_logits_kernel|seg_offsets_kernel|permute_kernel|grouped_gemm_kernel' \
  --launch-skip 18 --launch-count 6 -o gpurun_out/switch_step16 -f \
  python bench.py --config switch --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu16.txt 2>&1; echo "ncu full rc=$?" >> gpurun_out/summary.txt
python - <<'PY' >> gpurun_out/summary.txt
import json
for l in open("gpurun_out/ab16.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        print(d["config"], L["value"], L["ms_per_step"], L.get("stages_ms"), L["clocks"]["sm_mhz"], L["roofline"]["achieved"], L["e2e"]["value"])
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
