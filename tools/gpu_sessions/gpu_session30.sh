#!/bin/bash
# GEMM DRAM re-reads: L2 eviction hints (A panel evict-last, weights evict-first) x raster panel size
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s30
rm -f gpurun_out/summary.txt gpurun_out/s30/ab.jsonl
for cfg in "2 24" "2 48" "2 12" "0 12"; do
  set -- $cfg
  EMOE_GEMM_L2_HINTS=$1 EMOE_GEMM_PANEL_MB=$2 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"hints\": $1, \"panel_mb\": $2, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s30/ab.jsonl
  EMOE_GEMM_L2_HINTS=$1 EMOE_GEMM_PANEL_MB=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:grouped_gemm --launch-skip 6 --launch-count 2 --log-file gpurun_out/s30/traffic_h$1_p$2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
python - <<'PY' >> gpurun_out/summary.txt
import json, csv
for l in open("gpurun_out/s30/ab.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        tr = {}
        for r in csv.reader(open(f"gpurun_out/s30/traffic_h{d['hints']}_p{d['panel_mb']}.csv")):
            if len(r) > 14 and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tr[(r[0], r[12])] = float(r[14].replace(",", ""))
        tot = sum(tr.values()) / 1e9
        print(d["hints"], d["panel_mb"], L["value"], L["ms_per_step"], L["stages_ms"]["gemm1"], L["stages_ms"]["gemm2"], L["clocks"]["sm_mhz"], "traffic GB", round(tot, 2), {k: round(v / 1e9, 2) for k, v in tr.items()})
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
