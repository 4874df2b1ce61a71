#!/bin/bash
# dev: A/B tuning variants of libmc on isolated solves
for v in libmc_s2b2 libmc_s3b2; do
  for nc in 0 1; do
  echo "== $v MC_NO_CHAIN=$nc"
  export MC_LIB=$PWD/paper_2209_01158_b200/$v.so MC_NO_CHAIN=$nc
  timeout 300 python scripts/prof_graph.py 1 3000 fracture | tail -1
  timeout 300 python scripts/prof_graph.py 4 100 fracture | tail -1
  done
  timeout 300 python scripts/prof_graph.py 4 60 grid | tail -1
done
