#!/bin/bash
# K5 with output-channel split at any batch: parity + timing vs the unfused schedule
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused1d.py -q -k "channel_split or partial_modes" > gpurun_out/k5split_tests.log 2>&1; tail -3 gpurun_out/k5split_tests.log
for wl in C2-N1024-H128-B256 C2-N1024-H128-B1024 C2-N1024-H256-B64 C2-N1024-H256-B256 C2-N1024-H256-B1024; do
  for m in fused_gemm_ifft fft_optimized; do
  timeout 600 python bench.py --workload $wl --mode $m --no-baselines --no-e2e --no-cpu > gpurun_out/b39.json 2>gpurun_out/b39.err
  python -c "
import json; d=json.loads(open('gpurun_out/b39.json').read().strip().splitlines()[-1])
print('$wl', '$m', d['ms_per_step'], d['schedule'], [(s['kernel'], s['ms']) for s in d['stages']])"
  done
done
