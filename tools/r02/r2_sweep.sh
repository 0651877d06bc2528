#!/bin/bash
# full sweep (every BASELINE config + the 27-point C2 grid x 5 modes + TF32 variants + baselines + parity)
mkdir -p gpurun_out
timeout 3000 python tools/sweep.py --out gpurun_out/sweep_${1:-r2}.json > gpurun_out/sweep_${1:-r2}.log 2>&1
tail -3 gpurun_out/sweep_${1:-r2}.log
