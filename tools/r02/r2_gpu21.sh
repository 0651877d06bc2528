#!/bin/bash
# fused mix reading A from L2 into registers (TFNO_MIX_DIRECT=1): parity + same-box A/B on C4
mkdir -p gpurun_out
TFNO_MIX_DIRECT=1 timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x -k "fused_mix" > gpurun_out/t21.txt 2>&1; tail -2 gpurun_out/t21.txt
out=gpurun_out/mixdirect_ab.txt; : > $out
for rep in 1 2 3; do for d in 0 1; do
  TFNO_MIX_DIRECT=$d timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 direct=$d', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
done; done
cat $out
