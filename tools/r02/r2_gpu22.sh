#!/bin/bash
# fused mix with tasks of 4 output channels (TFNO_MIX_GN=4): parity + same-box A/B
mkdir -p gpurun_out
TFNO_MIX_GN=4 timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x -k "fused_mix and fp32" > gpurun_out/t22.txt 2>&1; tail -2 gpurun_out/t22.txt
out=gpurun_out/mixgn_ab.txt; : > $out
for rep in 1 2 3; do for gn in 8 4; do
  TFNO_MIX_GN=$gn timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 gn=$gn', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
  TFNO_PLANE_FUSEDMIX=1 TFNO_MIX_GN=$gn timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 fused gn=$gn', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
done; done
cat $out
