#!/bin/bash
# compute-sanitizer tiers on the GPU box; logs under gpurun_out/sanitizer/
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 \
      python tools/sanitize_run.py tiny small5k > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer/summary.txt
done
