#!/bin/bash
mkdir -p gpurun_out
TFNO_PLANE_GENERIC=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane_ -s 2 -c 2 -o gpurun_out/gen_C4 -f \
  python bench.py --steps 1 --warmup 1 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_gen.log 2>&1; tail -2 gpurun_out/ncu_gen.log
