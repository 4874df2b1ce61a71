#!/bin/bash
R=gpurun_out/r02b
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for v in 0 1; do
  MC_RECORDS=$v timeout 600 python scripts/prof_graph.py 4 300 fracture > $R/prof_graph4_fracture_rec$v.log 2>&1; tail -1 $R/prof_graph4_fracture_rec$v.log
done
MC_RECORDS=1 timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/prof_graph2_fracture_rec1.log 2>&1; tail -1 $R/prof_graph2_fracture_rec1.log
MC_RECORDS=0 timeout 600 python scripts/prof_graph.py 2 2000 fracture > $R/prof_graph2_fracture_rec0.log 2>&1; tail -1 $R/prof_graph2_fracture_rec0.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming_jacobi or config2_full_size_parity_D or config4_full_size_residuals" > $R/pytest_rec.log 2>&1; tail -3 $R/pytest_rec.log
timeout 900 python -m pytest tests/test_gpu_precond.py -m gpu -x -q > $R/pytest_precond.log 2>&1; tail -2 $R/pytest_precond.log
timeout 1500 python bench.py --steps 3 --warmup 3 > $R/bench_config4_short.json 2> $R/bench_config4_short.err; tail -c 3000 $R/bench_config4_short.json
bash scripts/sanitize.sh
