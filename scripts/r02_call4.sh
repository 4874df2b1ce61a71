#!/bin/bash
R=gpurun_out/r02d
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for v in 1 0; do
  MC_BLOCKED=$v timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/prof_graph4_fracture_blk$v.log 2>&1; tail -1 $R/prof_graph4_fracture_blk$v.log
done
for v in 1 0; do
  MC_BLOCKED=$v timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/prof_graph2_fracture_blk$v.log 2>&1; tail -1 $R/prof_graph2_fracture_blk$v.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming_jacobi or config2_full_size_parity_D or config4_full_size_residuals or ragged" > $R/pytest_blk.log 2>&1; tail -3 $R/pytest_blk.log
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_checked.py -m gpu -x -q > $R/pytest_precond_checked.log 2>&1; tail -3 $R/pytest_precond_checked.log
timeout 600 python scripts/prof_graph.py 4 100 fracture > $R/plain_blk1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o $R/fracture_only_blk1 \
    python scripts/prof_graph.py 4 100 fracture > $R/ncu_blk1.log 2>&1
tail -1 $R/plain_blk1.log; tail -2 $R/ncu_blk1.log
