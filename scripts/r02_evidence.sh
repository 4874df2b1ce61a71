#!/bin/bash
# Regenerates the committed evidence (supersedes round 1's gpu_profiles.sh): under gpurun_out/$1 (copy what is judged to profiles/):
#   gpurun --timeout 6000 -- 'bash scripts/r02_evidence.sh r02final'
R=gpurun_out/${1:-r02final}
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.log 2>&1; tail -1 $R/smoke.log
timeout 2400 python bench.py --steps 20 --warmup 5 > $R/bench_config4.json 2> $R/bench_config4.err; tail -c 1800 $R/bench_config4.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/plain4.json 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $R/launches_config4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/ncu_launch4.log 2>&1
timeout 1500 python tests/tools/parity_full.py --config 4 --scheme D --steps 2 --load .oracle_ship --out $R/r02_parity_config4_D.json > $R/parity4.log 2>&1; tail -3 $R/parity4.log
timeout 900 python tests/tools/parity_full.py --config 2 --scheme D --steps 3 --out $R/r02_parity_config2_D.json > $R/parity2.log 2>&1; tail -2 $R/parity2.log
[ -f .oracle_ship/config2_coupled_step2.npy ] && { timeout 900 python tests/tools/parity_full.py --config 2 --scheme coupled --steps 2 --load .oracle_ship --out $R/r02_parity_config2_coupled.json > $R/parity2c.log 2>&1; tail -3 $R/parity2c.log; }
for c in 0 1 2 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 4 > $R/bench_config$c.json 2> $R/bench_config$c.err; python -c "
import json; d=json.load(open('$R/bench_config$c.json')); print($c, d['value'], d['ms_per_step'], d['config']['cg_iters_per_step'], [ (p['path'], round(p['us_per_iteration'],2)) for p in d['roofline']['per_solve']], d['e2e']['value'], d['cpu_baseline']['value'])"
done
for c in 1 2 4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 4 --precond block --no-cpu-baseline > $R/bench_config${c}_block.json 2> $R/bench_config${c}_block.err; python -c "
import json; d=json.load(open('$R/bench_config${c}_block.json')); print($c, 'block', d['value'], d['ms_per_step'], d['config']['cg_iters_per_step'])"
done
timeout 600 python scripts/paper_analogue.py --out $R/paper_analogue > $R/paper_analogue.log 2>&1; tail -8 $R/paper_analogue.log
timeout 600 python scripts/paper_analogue.py --precond block --out $R/paper_analogue_block > $R/paper_analogue_block.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $R/pytest_gpu.log 2>&1; tail -4 $R/pytest_gpu.log
