#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (GPU box).  Logs: gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|case " gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
