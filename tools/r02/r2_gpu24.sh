#!/bin/bash
# tiny1d (C1-sized 1D layers): parity + A/B vs fused1d (TFNO_TINY1D=0) incl. the staged baseline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused1d.py -q -m gpu -x > gpurun_out/t24.txt 2>&1; tail -2 gpurun_out/t24.txt
out=gpurun_out/tiny_ab.txt; : > $out
for rep in 1 2 3; do for t in 0 1; do
  TFNO_TINY1D=$t timeout 300 python bench.py --workload C1 --steps 50 --warmup 10 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 tiny=$t', d['ms_per_step'], d['schedule'], d['baselines']['cufft_cublas_staged']['ms'], d['baselines']['speedup_vs_best_unfused'])" >> $out
done; done
cat $out
