#!/bin/bash
# compute-sanitizer over the kernel families; run under gpurun.
# Writes gpurun_out/${TAG}_sanitize_<tool>_<case>.txt and a summary.
cd "$(dirname "$0")/.."
T=${1:-san}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in c1 c2 c3 c4 ibk m5 fuse c5 sweep fit; do
    out=gpurun_out/${T}_sanitize_${tool}_${case}.txt
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $case > $out 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out | tail -1)" >> gpurun_out/${T}_sanitize_summary.txt
  done
done
cat gpurun_out/${T}_sanitize_summary.txt
