#!/bin/bash
# correctness suite + smoke + ncu launch list + ncu full capture of the FFN GEMMs + full bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  -k regex:"route|scan|permute|grouped_gemm|combine|hist|prompt_trans|save_last|set_tables" \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1; echo "ncu launches rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 6 -c 2 \
  -o gpurun_out/gemm_full python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full_bench.txt 2>&1; echo "ncu full rc=$?" >> gpurun_out/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gate_route|permute_kernel|combine_bf16" -s 9 -c 3 \
  -o gpurun_out/hbm_full python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_hbm_bench.txt 2>&1; echo "ncu hbm rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
