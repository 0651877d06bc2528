#!/bin/bash
# round-2 final C (after tiny1d): full GPU suite, smoke, bench lines, sweeps, N3, ncu of the C1 kernel
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_final2.log 2>&1; tail -3 gpurun_out/gpu_tests_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; tail -3 gpurun_out/smoke_final2.log
timeout 900 python bench.py > gpurun_out/bench_C4_final2.json 2>gpurun_out/bf2_C4.err
for wl in C1 C3 C5; do timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_final2.json 2>gpurun_out/bf2_$wl.err; done
for wl in C4 C1 C3 C5; do python -c "
import json; d=json.loads(open('gpurun_out/bench_${wl}_final2.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), 'err', d.get('max_rel_error'))"; done
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/n3_raw2.csv python tools/n3_traffic.py run C1 C3 C4 C5L C2-N1024-H64-B1024 > gpurun_out/n3_run2.log 2>&1
python tools/n3_traffic.py summarize gpurun_out/n3_raw2.csv > gpurun_out/n3_traffic2.json 2>gpurun_out/n3_sum2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tiny1d" -s 2 -c 1 \
  -o gpurun_out/prof_C1_tiny -f python bench.py --workload C1 --steps 2 --warmup 2 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_C1_tiny.log 2>&1
timeout 3000 python tools/sweep.py --out gpurun_out/sweep_r2c.json > gpurun_out/sweep_r2c.log 2>&1; tail -1 gpurun_out/sweep_r2c.log | cut -c1-200
timeout 1500 python tools/sweep2d.py --out gpurun_out/sweep2d_r2c.json > gpurun_out/sweep2d_r2c.log 2>&1; tail -2 gpurun_out/sweep2d_r2c.log | cut -c1-300
