#!/bin/bash
# final-code sweeps: every BASELINE config + 27-point C2 grid, and the 2D shapes beyond the configs
mkdir -p gpurun_out
timeout 3000 python tools/sweep.py --out gpurun_out/sweep_r2e.json > gpurun_out/sweep_r2e.log 2>&1; tail -1 gpurun_out/sweep_r2e.log | cut -c1-300
timeout 1500 python tools/sweep2d.py --out gpurun_out/sweep2d_r2e.json > gpurun_out/sweep2d_r2e.log 2>&1; tail -2 gpurun_out/sweep2d_r2e.log | cut -c1-300
