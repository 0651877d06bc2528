#!/bin/bash
# PDL: full GPU suite, then same-box A/B (TFNO_PDL=0/1) on C1 / C3 / C5 / C2 points / C4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t12.txt 2>&1; tail -3 gpurun_out/t12.txt
out=gpurun_out/pdl_ab.txt; : > $out
for rep in 1 2; do for wl in C1 C3 C5 C2-N256-H64-B64 C2-N1024-H128-B64 C4; do for p in 0 1; do
  TFNO_PDL=$p timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-baselines --no-e2e --no-cpu 2>gpurun_out/b12.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl pdl=$p', d['ms_per_step'], d['schedule'], d.get('launch'))" >> $out
done; done; done
cat $out; tail -3 gpurun_out/b12.err
