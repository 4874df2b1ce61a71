#!/bin/bash
# dev: quick correctness + timing pass
timeout 300 python scripts/probe.py 0 3 2>&1 | tee gpurun_out/quick_probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cta_count or ragged or worked or deterministic or nlmc_ragged or sigma_zero or neumann or config2_standin or snapshots or noconv or host_and or config1" 2>&1 | tail -3
timeout 300 python scripts/prof_graph.py 1 3000 fracture | tail -1
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-800
