#!/bin/bash
# column-panel raster for the FFN GEMMs (weights evict-last, rows evict-first): parity + traffic/time sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s36
rm -f gpurun_out/summary.txt gpurun_out/s36/ab.jsonl
EMOE_GEMM1_NPANEL=3 EMOE_GEMM2_NPANEL=1 timeout 900 python -m pytest tests/test_forward_gpu.py -q -x -k "not fp32 and not config1" > gpurun_out/s36/pytest.txt 2>&1; echo "pytest (panels 3/1) rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/s36/pytest.txt >> gpurun_out/summary.txt
for cfg in "0 0" "0 8" "0 4" "16 0" "28 8"; do
  set -- $cfg
  EMOE_GEMM1_NPANEL=$1 EMOE_GEMM2_NPANEL=$2 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
  echo "{\"g1\": $1, \"g2\": $2, \"line\": $(tail -1 gpurun_out/b_tmp.txt)}" >> gpurun_out/s36/ab.jsonl
  EMOE_GEMM1_NPANEL=$1 EMOE_GEMM2_NPANEL=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k regex:grouped_gemm --launch-skip 6 --launch-count 2 --log-file gpurun_out/s36/traffic_$1_$2.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
python - <<'PY' >> gpurun_out/summary.txt
import json, csv
for l in open("gpurun_out/s36/ab.jsonl"):
    try:
        d = json.loads(l); L = d["line"]
        tr = {}
        for r in csv.reader(open(f"gpurun_out/s36/traffic_{d['g1']}_{d['g2']}.csv")):
            if len(r) > 14 and r[12] not in ("Metric Name",):
                tr[("G1" if r[0] == "0" else "G2") + ":" + r[12].split("__")[1][:12]] = r[14]
        print(d["g1"], d["g2"], L["value"], L["ms_per_step"], L["stages_ms"]["gemm1"], L["stages_ms"]["gemm2"], L["clocks"]["sm_mhz"], tr)
    except Exception as e:
        print("bad", l[:300], e)
PY
cat gpurun_out/summary.txt
