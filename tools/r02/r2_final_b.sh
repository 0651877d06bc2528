#!/bin/bash
# round-2 final B: ncu launch list of the C4 bench, full captures of the C4 / C3 kernels, N3 re-capture, sweep
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_C4_r2.csv \
  python bench.py --workload C4 --steps 2 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_launch_C4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"plane_" -s 2 -c 2 \
  -o gpurun_out/prof_C4_final -f python bench.py --workload C4 --steps 1 --warmup 1 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_C4_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plane_|cgemm" -s 3 -c 3 \
  -o gpurun_out/prof_C3_final -f python bench.py --workload C3 --steps 1 --warmup 1 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_C3_final.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/n3_raw.csv python tools/n3_traffic.py run C3 C4 C5L C1 C2-N1024-H64-B1024 > gpurun_out/n3_run.log 2>&1
python tools/n3_traffic.py summarize gpurun_out/n3_raw.csv > gpurun_out/n3_traffic.json 2>gpurun_out/n3_sum.err
tail -2 gpurun_out/n3_run.log; head -c 300 gpurun_out/n3_traffic.json
bash tools/r02/r2_sweep.sh r2b
