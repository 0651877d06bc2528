#!/bin/bash
# K4 / K5 on the fused 1D kernel: parity (fused1d file + golden parity) + sweep of the partial modes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fused1d.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t32.txt 2>&1; tail -2 gpurun_out/t32.txt
timeout 1800 python tools/sweep.py --workloads C1,C2-N256-H64-B64,C2-N256-H64-B1024,C2-N256-H256-B1024,C2-N1024-H64-B1024,C2-N1024-H128-B64,C2-N256-H128-B256 --out gpurun_out/sweep_k45.json > gpurun_out/sweep_k45.log 2>&1
python -c "
import json
d=json.load(open('gpurun_out/sweep_k45.json'))
for r in d['rows']: print(r['workload'], 'ff', r['fully_fused'], 'fo', r['fft_optimized'], 'ffg', r['fused_fft_gemm'], r['fused_fft_gemm_schedule'], 'fgi', r['fused_gemm_ifft'], r['fused_gemm_ifft_schedule'], 'st', r['staged'])"
