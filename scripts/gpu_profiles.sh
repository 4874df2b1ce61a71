#!/bin/bash
# round-1 evidence: GPU tests, full bench lines, launch list of the bench command, one full ncu capture
mkdir -p gpurun_out/r01f
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1800 2>&1 | tail -4 > gpurun_out/r01f/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r01f/bench_config1.json 2> gpurun_out/r01f/bench_config1.err
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01f/bench_config4.json 2> gpurun_out/r01f/bench_config4.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01f/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01f/launches_config1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01f/ncu_launch.log 2>&1
timeout 600 python scripts/prof_step.py 4 D 40 1 > gpurun_out/r01f/prof4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/r01f/step_config4_capped python scripts/prof_step.py 4 D 40 1 > gpurun_out/r01f/prof4_ncu.log 2>&1
cat gpurun_out/r01f/pytest_gpu.log
