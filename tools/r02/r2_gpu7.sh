#!/bin/bash
# round-2 checkpoint: full GPU suite, default bench line, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
timeout 600 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; tail -c 3000 gpurun_out/bench_C4.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json
