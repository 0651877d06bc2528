#!/bin/bash
# compute-sanitizer over every kernel family (small shapes); summaries to gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 700 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
