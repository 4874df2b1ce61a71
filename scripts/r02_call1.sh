#!/bin/bash
# round-2 GPU call 1: new tests, config-2 full-size D parity, perf baselines, fracture-dominated ncu capture
R=gpurun_out/r02a
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming_jacobi or run_bitwise or run_failure or config2_full_size_parity_D or run_with_snapshots or worked_example or noconv" > $R/pytest_new.log 2>&1
tail -5 $R/pytest_new.log
timeout 900 python -m pytest tests/test_gpu_precond.py -m gpu -x -q > $R/pytest_precond.log 2>&1
tail -3 $R/pytest_precond.log
timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/prof_graph4_fracture.log 2>&1; tail -2 $R/prof_graph4_fracture.log
timeout 600 python scripts/prof_graph.py 4 60 grid > $R/prof_graph4_grid.log 2>&1; tail -2 $R/prof_graph4_grid.log
timeout 300 python scripts/prof_graph.py 1 3000 fracture > $R/prof_graph1_fracture.log 2>&1; tail -2 $R/prof_graph1_fracture.log
timeout 900 python scripts/parity_full.py --config 2 --scheme D --steps 3 --out $R/r02_parity_config2_D.json > $R/parity2D.log 2>&1; tail -4 $R/parity2D.log
timeout 600 python scripts/prof_step.py 4 D 2000 1 > $R/prof4_frac_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o $R/step_config4_fracture2000 \
  python scripts/prof_step.py 4 D 2000 1 > $R/prof4_frac_ncu.log 2>&1
tail -3 $R/prof4_frac_plain.log $R/prof4_frac_ncu.log
