#!/bin/bash
# dev: paper-analogue parity + experiment table, U/L bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "analogue or wells" 2>&1 | tail -4
timeout 600 python scripts/paper_analogue.py --out gpurun_out/r01_paper_analogue 2>&1 | tail -20
for s in U L D; do timeout 300 python bench.py --scheme $s --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-300; done
