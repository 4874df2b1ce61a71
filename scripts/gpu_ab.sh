#!/bin/bash
timeout 300 python scripts/prof_graph.py 4 100 fracture | tail -1
timeout 300 python scripts/prof_graph.py 1 3000 fracture | tail -1
timeout 300 python scripts/prof_graph.py 4 60 grid | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cta_count or ragged or worked or deterministic or nlmc_ragged or sigma_zero or config0 or config2_standin or cropped" 2>&1 | tail -2
