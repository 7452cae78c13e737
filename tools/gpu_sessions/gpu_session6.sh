#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt gpurun_out/panel.txt
timeout 1800 python -m pytest tests/test_dropin_gpu.py -q -m gpu > gpurun_out/pytest_dropin.txt 2>&1; echo "dropin rc=$?" >> gpurun_out/summary.txt
for i in 1 2; do
  for mb in 8 16 24; do
    EMOE_GEMM_PANEL_MB=$mb timeout 300 python bench.py --no-cpu-baseline --steps 40 --e2e-steps 1 > gpurun_out/p_tmp.txt 2>&1
    echo "panel$mb $(tail -1 gpurun_out/p_tmp.txt)" >> gpurun_out/panel.txt
  done
done
for mb in 8 24; do
EMOE_GEMM_PANEL_MB=$mb timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm_kernel -s 6 -c 2 \
  --csv --log-file gpurun_out/gemm_traffic_p$mb.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu traffic p$mb rc=$?" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
