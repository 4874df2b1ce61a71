#!/bin/bash
R=gpurun_out/r02c
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_nlmc.py -m gpu -x -q > $R/pytest_nlmc.log 2>&1; tail -3 $R/pytest_nlmc.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.log 2>&1; tail -2 $R/smoke.log
for v in 0 1; do
  MC_RECORDS=$v timeout 600 python scripts/prof_graph.py 4 100 fracture > $R/plain_rec$v.log 2>&1 && \
  MC_RECORDS=$v timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o $R/fracture_only_rec$v \
    python scripts/prof_graph.py 4 100 fracture > $R/ncu_rec$v.log 2>&1
  tail -1 $R/plain_rec$v.log; tail -2 $R/ncu_rec$v.log
done
