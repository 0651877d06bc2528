#!/bin/bash
# generic plane kernels: parity, then A/B timing vs the tuned kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu > gpurun_out/gen_tests.txt 2>&1; tail -30 gpurun_out/gen_tests.txt
timeout 600 python tools/sweep2d.py --out gpurun_out/sweep2d_a.json > gpurun_out/sweep2d_a.log 2>&1; cat gpurun_out/sweep2d_a.log | cut -c1-400
TFNO_PLANE_GENERIC=1 timeout 600 python tools/sweep2d.py --out gpurun_out/sweep2d_g.json --no-torch --modes fully_fused --shapes "32,64,64,256,256,32,32;256,64,64,256,256,16,16;32,128,128,512,512,64,64" > gpurun_out/sweep2d_g.log 2>&1; cat gpurun_out/sweep2d_g.log | cut -c1-400
TFNO_PLANE_GENERIC=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/bench_C4_gen.json 2>gpurun_out/bench_C4_gen.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_C4_gen.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages'])"
