#!/bin/bash
# A/B of tuned vs generic plane kernels per geometry: stage times from bench.py (TFNO_PLANE_GENERIC bits: 1 fwd, 2 inv)
out=${1:-gpurun_out/plane_mix.txt}
: > $out
for wl in C4 C3 C5L; do
  for mix in 0 3; do
    TFNO_PLANE_GENERIC=$mix timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl mix=$mix', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
  done
done
cat $out
