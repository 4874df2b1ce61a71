#!/bin/bash
for v in libmc libmc_old32; do
  echo "== $v"
  export MC_LIB=$PWD/paper_2209_01158_b200/$v.so
  timeout 300 python scripts/prof_graph.py 1 3000 fracture | tail -1
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['cg_iters_per_step'], d['config']['ms_per_solve'])"
done
unset MC_LIB
timeout 300 python scripts/prof_graph.py 4 100 fracture | tail -1
timeout 300 python scripts/prof_graph.py 4 60 grid | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cta_count or ragged or worked or deterministic or sigma_zero or config0 or config2_standin or cropped" 2>&1 | tail -2
