#!/bin/bash
# last tree (loaded twiddle companions): full GPU suite, smoke, bench lines C4 / C1 / C3 / C5, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_final6.log 2>&1; tail -2 gpurun_out/gpu_tests_final6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final6.log 2>&1; tail -2 gpurun_out/smoke_final6.log
timeout 900 python bench.py > gpurun_out/bench_C4_final6.json 2>gpurun_out/bf6_C4.err
for wl in C1 C3 C5; do timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_final6.json 2>gpurun_out/bf6_$wl.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final6.json 2>gpurun_out/bf6_ref.err
for wl in C4 C1 C3 C5; do python -c "
import json; d=json.loads(open('gpurun_out/bench_${wl}_final6.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], d['launch'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), 'err', d.get('max_rel_error'), d['clocks'])"; done
tail -c 400 gpurun_out/bench_ref_final6.json
echo done
