#!/bin/bash
R=gpurun_out/r02i
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
echo "--- config 4 fracture: compact, 96-byte blocked"
timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_c.log 2>&1; tail -1 $R/pg4_c.log
MC_COMPACT=0 timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_b96.log 2>&1; tail -1 $R/pg4_b96.log
echo "--- config 2 fracture: same"
timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_c.log 2>&1; tail -1 $R/pg2_c.log
MC_COMPACT=0 timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_b96.log 2>&1; tail -1 $R/pg2_b96.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming or config2_full_size_parity_D or ragged or config4_cropped" > $R/pytest_parity.log 2>&1; tail -3 $R/pytest_parity.log
timeout 600 python scripts/nlmc_bench.py --oracle --out $R/nlmc.json > $R/nlmc.log 2>&1; tail -3 $R/nlmc.log
