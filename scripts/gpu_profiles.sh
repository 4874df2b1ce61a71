#!/bin/bash
# Regenerates the round's evidence under gpurun_out/rNN (copy what is judged to profiles/):
# GPU tests, bench lines (all configs, block-Jacobi option), the ncu launch list of the
# default bench command, a full ncu capture of a capped config-4 step, the NLMC build and
# coarse schemes, the paper analogue, the capped config-4 coupled comparator.
#   gpurun --timeout 5400 -- 'bash scripts/gpu_profiles.sh r01'
R=gpurun_out/${1:-r01}
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1800 2>&1 | tail -4 > $R/pytest_gpu.log
timeout 900 python bench.py > $R/bench_config1.json 2> $R/bench_config1.err
timeout 600 python bench.py --precond block --no-cpu-baseline > $R/bench_config1_block.json 2> $R/bench_config1_block.err
timeout 600 python bench.py --config 0 --steps 20 --warmup 3 > $R/bench_config0.json 2> $R/bench_config0.err
timeout 1200 python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > $R/bench_config2.json 2> $R/bench_config2.err
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 > $R/bench_config3.json 2> $R/bench_config3.err
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $R/bench_config4.json 2> $R/bench_config4.err
timeout 900 python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --precond block > $R/bench_config2_block.json 2> $R/bench_config2_block.err
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --precond block > $R/bench_config4_block.json 2> $R/bench_config4_block.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $R/launches_config1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/ncu_launch.log 2>&1
timeout 600 python scripts/prof_step.py 4 D 40 1 > $R/prof4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o $R/step_config4_capped \
  python scripts/prof_step.py 4 D 40 1 > $R/prof4_ncu.log 2>&1
timeout 600 python scripts/nlmc_bench.py --oracle --out $R/nlmc.json > $R/nlmc.log 2>&1
timeout 600 python scripts/paper_analogue.py --out $R/paper_analogue > $R/paper_analogue.log 2>&1
timeout 600 python scripts/paper_analogue.py --precond block --out $R/paper_analogue_block > $R/paper_analogue_block.log 2>&1
timeout 600 python scripts/coupled_cfg4.py 400 --out $R/coupled_config4_capped.json > $R/coupled_cfg4.log 2>&1
cat $R/pytest_gpu.log
