#!/bin/bash
# tiny1d for N = 128 / 256 / 1024: parity + A/B vs fused1d on the batch-64 C2 points and C1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused1d.py -q -m gpu -x > gpurun_out/t25.txt 2>&1; tail -2 gpurun_out/t25.txt
out=gpurun_out/tiny2_ab.txt; : > $out
for rep in 1 2; do for wl in C1 C2-N256-H64-B64 C2-N256-H128-B64 C2-N1024-H64-B64; do for t in 0 -1; do
  TFNO_TINY1D=$t timeout 300 python bench.py --workload $wl --steps 50 --warmup 10 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl tiny=$t', d['ms_per_step'], d['schedule'], d['baselines']['cufft_cublas_staged']['ms'], d['baselines']['speedup_vs_best_unfused'], d.get('max_rel_error'))" >> $out
done; done; done
cat $out
