#!/bin/bash
R=gpurun_out/r02p
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for lib in libmc.so libmc_nopre.so; do
for rep in 1 2; do
MC_LIB=paper_2209_01158_b200/$lib timeout 300 python scripts/prof_graph.py 1 3000 fracture > $R/pg1_$lib.$rep.log 2>&1; echo "$lib $(tail -1 $R/pg1_$lib.$rep.log)"
done
MC_LIB=paper_2209_01158_b200/$lib timeout 300 python scripts/prof_graph.py 4 300 fracture > $R/pg4_$lib.log 2>&1; echo "$lib $(tail -1 $R/pg4_$lib.log)"
MC_LIB=paper_2209_01158_b200/$lib timeout 300 python scripts/prof_graph.py 4 60 grid > $R/pg4g_$lib.log 2>&1; echo "$lib $(tail -1 $R/pg4g_$lib.log)"
MC_LIB=paper_2209_01158_b200/$lib timeout 600 python bench.py --config 1 --steps 10 --warmup 4 --no-cpu-baseline --no-e2e > $R/b1_$lib.json 2>$R/b1_$lib.err; python -c "
import json; d=json.load(open('$R/b1_$lib.json')); print('$lib', d['value'], d['ms_per_step'], [round(p['us_per_iteration'],2) for p in d['roofline']['per_solve']])"
MC_LIB=paper_2209_01158_b200/$lib timeout 600 python bench.py --config 0 --steps 20 --warmup 4 --no-cpu-baseline --no-e2e > $R/b0_$lib.json 2>$R/b0_$lib.err; python -c "
import json; d=json.load(open('$R/b0_$lib.json')); print('$lib', d['value'], d['ms_per_step'], [round(p['us_per_iteration'],2) for p in d['roofline']['per_solve']])"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config0 or ragged or sigma_zero or neumann or deterministic or cta_count or paper_analogue or LU_config0 or wells or run_" > $R/pytest_res.log 2>&1; tail -3 $R/pytest_res.log
