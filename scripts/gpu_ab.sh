#!/bin/bash
timeout 300 python scripts/probe.py 3 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "nlmc or config3 or LU_config0 or cta_count or worked or deterministic or host_and" 2>&1 | tail -2
timeout 300 python bench.py --scheme U --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | cut -c1-300
