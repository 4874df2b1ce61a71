#!/bin/bash
R=gpurun_out/r02f
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for v in 1 0; do
  MC_BLOCKED=$v timeout 300 python scripts/prof_graph.py 1 3000 fracture > $R/pg1_blk$v.log 2>&1; echo "blocked=$v $(tail -1 $R/pg1_blk$v.log)"
done
MC_LIB=paper_2209_01158_b200/libmc_prof.so timeout 300 python scripts/prof_phases.py 1 3000 fracture > $R/phases1.log 2>&1; tail -2 $R/phases1.log
MC_BLOCKED=0 MC_LIB=paper_2209_01158_b200/libmc_prof.so timeout 300 python scripts/prof_phases.py 1 3000 fracture > $R/phases1_old.log 2>&1; tail -1 $R/phases1_old.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config0 or ragged or sigma_zero or neumann or deterministic or cta_count or paper_analogue or LU_config0 or wells or run_" > $R/pytest_res2.log 2>&1; tail -3 $R/pytest_res2.log
timeout 600 python bench.py --config 1 --steps 10 --warmup 4 --no-cpu-baseline > $R/bench1.json 2>$R/bench1.err; python -c "
import json; d=json.load(open('$R/bench1.json')); print(d['value'], d['ms_per_step'], d['config']['cg_iters_per_step'], d['roofline']['per_solve'], d['e2e'])"
timeout 600 python scripts/run_trace.py --out $R/run_trace.json > $R/run_trace.log 2>&1; cat $R/run_trace.log
