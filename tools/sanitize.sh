#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck (shared-memory hazards),
# synccheck (barrier misuse).  Logs under gpurun_out/; summary lines printed.
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
