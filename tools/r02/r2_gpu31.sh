#!/bin/bash
# mode CGEMM 128x128 tile with 512 threads (8x4 per thread): parity + A/B on the contraction-bound points
mkdir -p gpurun_out
TFNO_CGEMM_NTH512=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused1d.py -q -m gpu -x -k "cgemm or golden or fused1d_vs" > gpurun_out/t31.txt 2>&1; tail -2 gpurun_out/t31.txt
for e in 0 1; do
  TFNO_CGEMM_NTH512=$e timeout 900 python tools/stages.py --workloads C2-N4096-H256-B1024,C2-N1024-H256-B256,C2-N4096-H256-B64,C2-N1024-H256-B64 --modes fully_fused > gpurun_out/stages31_$e.txt 2>&1
  echo "nth512=$e"; cut -c1-260 gpurun_out/stages31_$e.txt
done
