#!/bin/bash
# ncu evidence for one workload: launch list of the bench command + full capture of the hot kernels
WL=${1:-C4}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$WL.csv \
  python bench.py --workload $WL --steps 2 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_bench_$WL.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"plane_|cgemm|fused_rows" -s 3 -c 3 \
  -o gpurun_out/prof_$WL -f python bench.py --workload $WL --steps 1 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_full_$WL.log 2>&1
echo done
