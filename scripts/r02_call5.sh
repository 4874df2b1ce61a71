#!/bin/bash
R=gpurun_out/r02e
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for lib in libmc_nsub1.so libmc.so; do
  for rep in 1 2; do
  MC_LIB=paper_2209_01158_b200/$lib timeout 300 python scripts/prof_graph.py 1 3000 fracture > $R/pg1_$lib.$rep.log 2>&1; echo "$lib cfg1 $(tail -1 $R/pg1_$lib.$rep.log)"
  done
  MC_LIB=paper_2209_01158_b200/$lib timeout 300 python scripts/prof_graph.py 3 400 fracture > $R/pg3_$lib.log 2>&1; echo "$lib cfg3 $(tail -1 $R/pg3_$lib.log)"
  MC_LIB=paper_2209_01158_b200/$lib timeout 300 python scripts/prof_graph.py 4 300 fracture > $R/pg4_$lib.log 2>&1; echo "$lib cfg4 $(tail -1 $R/pg4_$lib.log)"
  MC_LIB=paper_2209_01158_b200/$lib timeout 600 python bench.py --config 1 --steps 10 --warmup 4 --no-cpu-baseline --no-e2e > $R/bench1_$lib.json 2>$R/bench1_$lib.err; python -c "
import json; d=json.load(open('$R/bench1_$lib.json')); print('$lib', d['value'], d['ms_per_step'], d['config']['cg_iters_per_step'], d['roofline']['per_solve'])"
done
timeout 900 python -m pytest tests/test_gpu_checked.py -m gpu -q > $R/pytest_checked.log 2>&1; tail -4 $R/pytest_checked.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deterministic or cta_count or config0 or run_bitwise" > $R/pytest_det.log 2>&1; tail -3 $R/pytest_det.log
