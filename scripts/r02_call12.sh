#!/bin/bash
R=gpurun_out/r02l
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for rep in 1 2; do
timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_c.$rep.log 2>&1; echo "compact88 $(tail -1 $R/pg4_c.$rep.log)"
MC_COMPACT=0 timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_b96.$rep.log 2>&1; echo "blocked96 $(tail -1 $R/pg4_b96.$rep.log)"
done
timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_c.log 2>&1; echo "compact88 $(tail -1 $R/pg2_c.log)"
MC_COMPACT=0 timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_b96.log 2>&1; echo "blocked96 $(tail -1 $R/pg2_b96.log)"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming or config2_full_size_parity_D" > $R/pytest_streaming.log 2>&1; tail -3 $R/pytest_streaming.log
