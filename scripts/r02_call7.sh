#!/bin/bash
R=gpurun_out/r02g
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 2400 python bench.py --steps 20 --warmup 5 > $R/bench_config4.json 2> $R/bench_config4.err; tail -c 2500 $R/bench_config4.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/plain4.json 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $R/launches_config4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $R/ncu_launch4.log 2>&1
tail -3 $R/launches_config4.csv
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $R/bench_reference.json 2> $R/bench_reference.err; tail -c 1200 $R/bench_reference.json
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $R/pytest_gpu.log 2>&1; tail -5 $R/pytest_gpu.log
