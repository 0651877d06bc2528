#!/bin/bash
# session-4 GPU call 1: state check after the container rebuild (GPU suite, C4 bench line),
# then the A/B of the 4-slot / register-accumulator forward at 512^2 (TFNO_PG_S4)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/g1_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_gpu_tests.log 2>&1; tail -2 gpurun_out/g1_gpu_tests.log
timeout 600 python bench.py > gpurun_out/g1_bench_C4.json 2>gpurun_out/g1_bench_C4.err; tail -c 600 gpurun_out/g1_bench_C4.json
DEFS=TFNO_PG_S4 WL=C4 MODES=fully_fused timeout 1500 bash tools/ab_build.sh > gpurun_out/g1_ab_s4.txt 2>&1; cat gpurun_out/g1_ab_s4.txt
