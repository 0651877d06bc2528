#!/bin/bash
# ncu --set full of the final C4 kernels (forward + fused inverse/mix) and the launch list
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_C4_final6.csv \
  python bench.py --steps 2 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_bench_C4_6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"plane_" -s 2 -c 2 \
  -o gpurun_out/prof_C4_final6 -f python bench.py --workload C4 --steps 1 --warmup 3 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_full_C4_6.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_C4_final6.ncu-rep > gpurun_out/ncu_C4_final6.txt 2>&1
python tools/ncu_opmix.py gpurun_out/prof_C4_final6.ncu-rep > gpurun_out/opmix_C4_final6.txt 2>&1
head -40 gpurun_out/ncu_C4_final6.txt
