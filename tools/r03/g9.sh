#!/bin/bash
# A/B: 64 x 64 mode-CGEMM tiles for N <= 64 (TFNO_CGEMM_SMALL) on the C3 / C5 layers + parity with it on
mkdir -p gpurun_out
TFNO_CGEMM_SMALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/g9_tests_small.log 2>&1; tail -1 gpurun_out/g9_tests_small.log
VAR=TFNO_CGEMM_SMALL VALS="0 1" WL=C3,C5L MODES=fully_fused,fft_optimized timeout 900 bash tools/ab_env.sh > gpurun_out/g9_small_ab.txt 2>&1; cat gpurun_out/g9_small_ab.txt
for r in 1 2; do for v in 0 1; do
TFNO_CGEMM_SMALL=$v timeout 300 python bench.py --workload C3 --no-baselines --no-e2e --no-cpu --steps 50 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C3 small=$v', d['ms_per_step'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], [(s['kernel'], s['ms']) for s in d['stages']])"
done; done 2>&1 | tee gpurun_out/g9_c3_bench_small.txt
