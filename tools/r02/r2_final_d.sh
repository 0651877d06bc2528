#!/bin/bash
# round-2 final D (after K4/K5 fused1d parts and rank-2 fused_gemm_ifft): bench lines + sweeps
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_C4_final3.json 2>gpurun_out/bf3_C4.err
for wl in C1 C3 C5; do timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_final3.json 2>gpurun_out/bf3_$wl.err; done
for wl in C4 C1 C3 C5; do python -c "
import json; d=json.loads(open('gpurun_out/bench_${wl}_final3.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), 'err', d.get('max_rel_error'))"; done
timeout 3000 python tools/sweep.py --out gpurun_out/sweep_r2d.json > gpurun_out/sweep_r2d.log 2>&1; tail -1 gpurun_out/sweep_r2d.log | cut -c1-200
timeout 1500 python tools/sweep2d.py --out gpurun_out/sweep2d_r2d.json > gpurun_out/sweep2d_r2d.log 2>&1; tail -2 gpurun_out/sweep2d_r2d.log | cut -c1-300
