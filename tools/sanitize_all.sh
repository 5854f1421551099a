#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_check.py); logs -> gpurun_out/sanitize_*.log
for tool in memcheck racecheck synccheck; do
  for fam in map slices rows skinny coop scan stream; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_check.py $fam \
      > gpurun_out/sanitize_${tool}_${fam}.log 2>&1
    echo "$tool $fam rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${fam}.log | tail -1)"
  done
done
