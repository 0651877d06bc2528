#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "host_pipeline or device_api" > gpurun_out/t16.txt 2>&1; tail -2 gpurun_out/t16.txt
for wl in C4 C3 C5 C1; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_r2d.json 2>gpurun_out/b16_$wl.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_${wl}_r2d.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), d['e2e'].get('ms_per_step'))"
done
