#!/bin/bash
# diagnostic: grouped GEMMs without output stores (Switch and Mixtral shapes)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/summary.txt
for v in normal nostore; do
  if [ $v = normal ]; then L=""; else L=$GRAFT_REPO_ROOT/paper_2503_06823_b200/lib/var_nostore/libemoe.so; fi
  for c in switch mixtral; do
    EMOE_LIB_PATH=$L timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_tmp.txt 2>&1
    tail -1 gpurun_out/b_tmp.txt | python -c "import json,sys; L=json.loads(sys.stdin.read()); print('$v', '$c', L['ms_per_step'], L['stages_ms'], L['clocks']['sm_mhz'])" >> gpurun_out/summary.txt
  done
done
cat gpurun_out/summary.txt
