#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_plane_generic.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t33.txt 2>&1; tail -2 gpurun_out/t33.txt
timeout 1200 python tools/sweep.py --workloads C3,C4,C5L --out gpurun_out/sweep_2dmodes.json > gpurun_out/sweep_2dmodes.log 2>&1
python -c "
import json
d=json.load(open('gpurun_out/sweep_2dmodes.json'))
for r in d['rows']: print(r['workload'], 'ff', r['fully_fused'], 'fo', r['fft_optimized'], 'ffg', r['fused_fft_gemm'], r['fused_fft_gemm_schedule'], 'fgi', r['fused_gemm_ifft'], r['fused_gemm_ifft_schedule'], 'st', r['staged'])"
