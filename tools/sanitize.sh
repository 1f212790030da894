#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck,
# synccheck, initcheck.  Logs to gpurun_out/sanitize_<tool>.log; the
# summaries are copied to profiles/ by hand.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
      python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?" | tee -a gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|Invalid|hazard" gpurun_out/sanitize_$tool.log | tail -5 \
      | tee -a gpurun_out/sanitize_summary.txt
done
