#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, synccheck, racecheck
# (shared-memory hazards), initcheck.  Logs: gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  # racecheck/initcheck are slow: derive-only subset
  arg=""
  [ $tool = racecheck ] && arg="derive"
  [ $tool = initcheck ] && arg="derive"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 \
    python tools/sanitize_cases.py $arg > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
