#!/bin/bash
# last-tree check: full GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_final5.log 2>&1; tail -2 gpurun_out/gpu_tests_final5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final5.log 2>&1; tail -2 gpurun_out/smoke_final5.log
timeout 900 python bench.py > gpurun_out/bench_C4_final5.json 2>gpurun_out/bf5_C4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_C4_final5.json').read().strip().splitlines()[-1])
print('C4', d['ms_per_step'], d['schedule'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), 'err', d.get('max_rel_error'), d['clocks'])"
