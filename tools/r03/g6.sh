#!/bin/bash
# compute-sanitizer over the pipelined class loops of the tuned plane kernels (both on) vs off
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for v in 0 1; do
    TFNO_PLANE_SKEW=$v TFNO_PLANE_ISKEW=$v timeout 900 compute-sanitizer --tool $tool --print-limit 2000 python tools/r03/skew_cases.py > gpurun_out/skew_${tool}_$v.log 2>&1
    echo "$tool skew=$v rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/skew_${tool}_$v.log | tail -1) $(grep -c '^ok' gpurun_out/skew_${tool}_$v.log)"
  done
done | tee gpurun_out/skew_sanitizer_summary.txt
for v in 0 1; do
  grep -oE '(Read|Write) access at .* in [a-z0-9_]+\.cu[h]?:[0-9]+' gpurun_out/skew_racecheck_$v.log | sed -E 's/\(.*\)//' | sort | uniq -c | sort -rn > gpurun_out/skew_racecheck_sites_$v.txt
  echo "== skew=$v sites"; head -20 gpurun_out/skew_racecheck_sites_$v.txt
done
