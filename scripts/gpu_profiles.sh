#!/bin/bash
# round-1 evidence: full bench line, launch list of the same command, one full ncu capture
mkdir -p gpurun_out/r01
timeout 900 python bench.py > gpurun_out/r01/bench_config1.json 2> gpurun_out/r01/bench_config1.err
echo "bench rc=$?"
timeout 1500 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01/bench_config4.json 2> gpurun_out/r01/bench_config4.err
echo "bench4 rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01/launches_config1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
timeout 600 python scripts/prof_step.py 4 D 40 1 > gpurun_out/r01/prof4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/r01/step_config4_capped python scripts/prof_step.py 4 D 40 1 > gpurun_out/r01/prof4_ncu.log 2>&1
echo "ncu4 rc=$?"
