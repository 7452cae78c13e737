#!/bin/bash
# column panels with row blocks evict-normal instead of evict-first
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s38
rm -f gpurun_out/summary.txt gpurun_out/s38/ab.jsonl
for cfg in "0 8 0" "0 8 1" "16 8 1" "28 8 1" "0 4 1"; do
  set -- $cfg
  EMOE_GEMM1_NPANEL=$1 EMOE_GEMM2_NPANEL=$2 EMOE_GEMM_PANEL_A_NORMAL=$3 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"g1\": $1, \"g2\": $2, \"anorm\": $3, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s38/ab.jsonl
  EMOE_GEMM1_NPANEL=$1 EMOE_GEMM2_NPANEL=$2 EMOE_GEMM_PANEL_A_NORMAL=$3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:grouped_gemm --launch-skip 6 --launch-count 2 --log-file gpurun_out/s38/traffic_$1_$2_$3.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
python - <<'PY' >> gpurun_out/summary.txt
import json, csv
for l in open("gpurun_out/s38/ab.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        tr = {}
        for r in csv.reader(open(f"gpurun_out/s38/traffic_{d['g1']}_{d['g2']}_{d['anorm']}.csv")):
            if len(r) > 14 and r[12] not in ("Metric Name",):
                tr[("G1" if r[0] == "0" else "G2") + ":" + r[12].split("__")[1][:10]] = round(float(r[14].replace(",", "")) / (1e9 if "bytes" in r[12] else 1e6), 2)
        print(d["g1"], d["g2"], d["anorm"], L["value"], L["ms_per_step"], L["stages_ms"]["gemm1"], L["stages_ms"]["gemm2"], L["clocks"]["sm_mhz"], tr)
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
