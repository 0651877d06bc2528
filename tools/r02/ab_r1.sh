#!/bin/bash
# same-box A/B: round-1 final tree (_ab_r1) vs HEAD (tuned / generic plane-kernel mixes); stage times per run
out=${1:-gpurun_out/ab_r1.txt}
: > $out
st() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d.get('stages', [])])" >> $out; }
for rep in 1 2; do
  for wl in C4 C3; do
    (cd _ab_r1 && timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null) | st "r1   $wl"
    for mix in 0 1 3; do
      TFNO_PLANE_GENERIC=$mix timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | st "HEAD $wl mix=$mix"
    done
  done
done
cat $out
