#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck (shared-memory hazards),
# synccheck (barrier misuse).  Logs under gpurun_out/; summary lines printed.
cd "$(dirname "$0")/.."
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
# synccheck stops a process at its first reported kernel: one process per case
for i in 0 1 2 3 4 5 6 7; do
  timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 4 \
      python tools/sanitize_cases.py $i > gpurun_out/sanitize_synccheck_$i.log 2>&1
  echo "synccheck case $i exit=$? $(grep '^ok' gpurun_out/sanitize_synccheck_$i.log) $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_synccheck_$i.log | tail -1) $(grep -m1 'Device Frame' gpurun_out/sanitize_synccheck_$i.log | sed 's/.*Frame: //' | cut -c1-90)"
done
