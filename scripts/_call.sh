#!/bin/bash
R=gpurun_out/r02z
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.log 2>&1; tail -1 $R/smoke.log
timeout 900 python bench.py --config 3 --steps 10 --warmup 4 > $R/bench_config3.json 2> $R/bench_config3.err; tail -c 600 $R/bench_config3.json
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $R/pytest_gpu.log 2>&1; tail -4 $R/pytest_gpu.log
