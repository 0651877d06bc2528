#!/bin/bash
# stage split of the contraction-bound / N4096 C2 points + ncu of the mode CGEMM and the team FFTs
mkdir -p gpurun_out
timeout 900 python tools/stages.py --workloads C2-N4096-H256-B1024,C2-N4096-H64-B1024,C2-N1024-H256-B256,C2-N4096-H256-B64 --modes fully_fused,staged > gpurun_out/stages23.txt 2>&1
cat gpurun_out/stages23.txt | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cgemm_modes|team_fft" -c 3 \
  -o gpurun_out/prof_n4096 -f python bench.py --workload C2-N4096-H256-B1024 --steps 1 --warmup 1 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu23.log 2>&1
tail -1 gpurun_out/ncu23.log
