#!/bin/bash
# compute-sanitizer over every kernel family (small shapes); summaries to gpurun_out/
#   memcheck / racecheck / synccheck on tools/sanitize_cases.py (default schedules), and again with
#   TFNO_PLANE_FUSEDMIX=1 (the fused inverse + channel mix kernel on the small rank-2 shapes);
#   racecheck on tools/probes/racecheck_mbar_probe (the mbarrier / TMA hand-off patterns in isolation)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for fm in -1 1; do
    TFNO_PLANE_FUSEDMIX=$fm timeout 900 compute-sanitizer --tool $tool --print-limit 2000 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_fm$fm.log 2>&1
    echo "$tool fusedmix=$fm rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_fm$fm.log | tail -1)"
  done
done
for f in gpurun_out/sanitize_racecheck_fm*.log; do
  grep -oE '(Read|Write) access at .* in [a-z0-9_]+\.cu[h]?:[0-9]+' $f | sed -E 's/\(.*\)//' | sort | uniq -c | sort -rn > ${f%.log}_sites.txt
done
P=tools/probes/racecheck_mbar_probe
[ -x $P ] || nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o $P $P.cu
timeout 300 compute-sanitizer --tool racecheck --print-limit 50 ./$P > gpurun_out/sanitize_probe.log 2>&1
echo "probe rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/sanitize_probe.log | tail -1)"
grep -oE '(Read|Write) access at .* in [a-z0-9_]+\.cu:[0-9]+' gpurun_out/sanitize_probe.log | sort | uniq -c > gpurun_out/sanitize_probe_sites.txt
cat gpurun_out/sanitize_probe_sites.txt
