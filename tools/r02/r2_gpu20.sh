#!/bin/bash
# generic forward via L2 prefetch + register loads (no smem ring): parity + same-box A/B
mkdir -p gpurun_out
TFNO_PLANE_GDLD=1 timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x -k "generic_plane_layer or deterministic or zero_and" > gpurun_out/t20.txt 2>&1; tail -2 gpurun_out/t20.txt
out=gpurun_out/gdld_ab.txt; : > $out
for rep in 1 2; do for d in 0 1; do
  TFNO_PLANE_GDLD=$d timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 dld=$d', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
  for wl in C3 C5L; do
  TFNO_PLANE_GENERIC=1 TFNO_PLANE_GDLD=$d timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl genfwd dld=$d', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
  done
done; done
cat $out
TFNO_PLANE_GDLD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plane_fwd" -s 1 -c 1 \
  -o gpurun_out/prof_gdld -f python bench.py --workload C4 --steps 1 --warmup 1 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_gdld.log 2>&1
tail -1 gpurun_out/ncu_gdld.log
