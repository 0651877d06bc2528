#!/bin/bash
# generic forward, 2 rows per team: parity + same-box A/B on C4 and generic-kernel shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x -k "two_rows" > gpurun_out/t19.txt 2>&1; tail -2 gpurun_out/t19.txt
out=gpurun_out/grpt_ab.txt; : > $out
for rep in 1 2; do for r in 1 2; do
  TFNO_PLANE_GRPT=$r timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 rpt=$r', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
  for wl in C3 C5L; do
  TFNO_PLANE_GENERIC=1 TFNO_PLANE_GRPT=$r timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl genfwd rpt=$r', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
  done
done; done
cat $out
