#!/bin/bash
R=gpurun_out/r02h
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
echo "--- config 4 fracture: compact (3 stages), compact (2 stages), 96-byte blocked"
timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_c3.log 2>&1; tail -1 $R/pg4_c3.log
MC_LIB=paper_2209_01158_b200/libmc_c2.so timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_c2.log 2>&1; tail -1 $R/pg4_c2.log
MC_COMPACT=0 timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/pg4_b96.log 2>&1; tail -1 $R/pg4_b96.log
echo "--- config 2 fracture: same"
timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_c3.log 2>&1; tail -1 $R/pg2_c3.log
MC_LIB=paper_2209_01158_b200/libmc_c2.so timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_c2.log 2>&1; tail -1 $R/pg2_c2.log
MC_COMPACT=0 timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/pg2_b96.log 2>&1; tail -1 $R/pg2_b96.log
echo "--- config 1 fracture (resident, records)"
timeout 300 python scripts/prof_graph.py 1 3000 fracture > $R/pg1.log 2>&1; tail -1 $R/pg1.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not config1_full and not config3 and not LU_config1" > $R/pytest_parity.log 2>&1; tail -3 $R/pytest_parity.log
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_checked.py -m gpu -x -q > $R/pytest_pc.log 2>&1; tail -3 $R/pytest_pc.log
timeout 1500 python tests/tools/parity_full.py --config 4 --scheme D --steps 2 --load .oracle_ship --out $R/r02_parity_config4_D.json > $R/parity4.log 2>&1; tail -4 $R/parity4.log
