#!/bin/bash
# compute-sanitizer runs: memcheck, racecheck, synccheck over the step kernel's
# paths and the NLMC build.  Logs -> gpurun_out/r02_sanitize/ (copy to profiles/).
#   gpurun --timeout 3600 -- 'bash scripts/sanitize.sh'
R=gpurun_out/r02_sanitize
mkdir -p $R
python -m paper_2209_01158_b200.build > /dev/null
for case in cfg0 cfg3 ell_stream bjs bj run nlmc; do
  timeout 300 python scripts/sanitize_target.py $case > $R/plain_$case.log 2>&1 || { echo "plain $case failed"; tail -3 $R/plain_$case.log; continue; }
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_target.py $case > $R/${tool}_$case.log 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $R/${tool}_$case.log | tail -1)"
  done
done | tee $R/summary.txt
