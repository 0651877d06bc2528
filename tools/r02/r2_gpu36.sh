#!/bin/bash
# per-mode mix kernel: parity + timing; stage breakdown of the C2 points below 1.5x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_permode.py tests/test_gpu_symmetric.py -q > gpurun_out/permode_tests.log 2>&1; tail -3 gpurun_out/permode_tests.log
timeout 300 python tools/permode_time.py > gpurun_out/permode_time.json 2>&1; cat gpurun_out/permode_time.json | tail -2
for wl in C2-N4096-H256-B64 C2-N1024-H256-B64 C2-N1024-H128-B64; do
  timeout 600 python bench.py --workload $wl --no-baselines --no-e2e --no-cpu > gpurun_out/b36_$wl.json 2>gpurun_out/b36_$wl.err
  python -c "
import json; d=json.loads(open('gpurun_out/b36_$wl.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], [(s['kernel'], s['ms'], s.get('GBps')) for s in d['stages']])"
done
