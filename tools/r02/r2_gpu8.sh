#!/bin/bash
# plane-kernel mix per geometry (C5L) + ncu full capture of the generic C4 kernels (mix=3)
mkdir -p gpurun_out
out=gpurun_out/mix_c5.txt; : > $out
for rep in 1 2; do for mix in 0 1 2 3; do
  TFNO_PLANE_GENERIC=$mix timeout 300 python bench.py --workload C5L --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5L mix=$mix', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
done; done
cat $out
TFNO_PLANE_GENERIC=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plane_" -s 2 -c 2 \
  -o gpurun_out/prof_C4g -f python bench.py --workload C4 --steps 1 --warmup 1 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_C4g.log 2>&1
tail -2 gpurun_out/ncu_C4g.log
