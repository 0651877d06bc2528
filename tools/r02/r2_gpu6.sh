#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/tc_tests.txt 2>&1; tail -5 gpurun_out/tc_tests.txt
for p in bf16 tf32x3; do timeout 300 python bench.py --steps 10 --warmup 3 --precision $p --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])"; done
