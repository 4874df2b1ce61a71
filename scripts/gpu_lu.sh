#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "LU or ragged" 2>&1 | tail -4
timeout 300 python bench.py --scheme U --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | cut -c1-400
