#!/bin/bash
# C1: bench line with baselines (PDL default) + ncu of the fused 1D kernel; C5 chain with PDL level 1
mkdir -p gpurun_out
timeout 300 python bench.py --workload C1 --no-e2e --no-cpu > gpurun_out/bench_C1.json 2>gpurun_out/b13.err; tail -c 1500 gpurun_out/bench_C1.json
timeout 300 python bench.py --workload C5 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>>gpurun_out/b13.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused1d" -s 5 -c 1 \
  -o gpurun_out/prof_C1 -f python bench.py --workload C1 --steps 1 --warmup 1 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_C1.log 2>&1
tail -1 gpurun_out/ncu_C1.log
