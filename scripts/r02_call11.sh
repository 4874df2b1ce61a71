#!/bin/bash
R=gpurun_out/r02k
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 1200 python tests/tools/parity_full.py --config 2 --scheme coupled --steps 2 --load .oracle_ship --out $R/r02_parity_config2_coupled.json > $R/parity2c.log 2>&1; tail -3 $R/parity2c.log
timeout 900 python -m pytest tests/test_gpu_precond.py -m gpu -x -q > $R/pytest_precond.log 2>&1; tail -3 $R/pytest_precond.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming" > $R/pytest_streaming.log 2>&1; tail -3 $R/pytest_streaming.log
for c in 2 4 1; do
  for v in 1 0; do
    MC_BLOCKED=$v timeout 900 python bench.py --config $c --steps 3 --warmup 4 --precond block --no-cpu-baseline --no-e2e > $R/bench_config${c}_block_blk$v.json 2> $R/bench_config${c}_block_blk$v.err; python -c "
import json; d=json.load(open('$R/bench_config${c}_block_blk$v.json')); print($c, 'block blocked=$v', d['value'], d['ms_per_step'], d['config']['cg_iters_per_step'], [round(p['us_per_iteration'],2) for p in d['roofline']['per_solve']])"
  done
done
