#!/bin/bash
# round-2 final A: full GPU suite, smoke, bench lines for C4 (default) / C1 / C3 / C5, reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_final.log 2>&1; tail -3 gpurun_out/gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -3 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_C4_final.json 2>gpurun_out/bf_C4.err
for wl in C1 C3 C5; do timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_final.json 2>gpurun_out/bf_$wl.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final.json 2>gpurun_out/bf_ref.err
for wl in C4 C1 C3 C5; do python -c "
import json; d=json.loads(open('gpurun_out/bench_${wl}_final.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), 'err', d.get('max_rel_error'), d['clocks'])"; done
tail -c 600 gpurun_out/bench_ref_final.json
