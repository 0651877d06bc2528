#!/bin/bash
# session-4 final evidence: full GPU suite, smoke, bench lines C4 (default) / C1 / C3 / C5,
# reference arm, ncu launch list of the default bench + full captures of the C4 and C3 kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_final4.log 2>&1; tail -2 gpurun_out/gpu_tests_final4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final4.log 2>&1; tail -2 gpurun_out/smoke_final4.log
timeout 900 python bench.py > gpurun_out/bench_C4_final4.json 2>gpurun_out/bf4_C4.err
for wl in C1 C3 C5; do timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_final4.json 2>gpurun_out/bf4_$wl.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_final4.json 2>gpurun_out/bf4_ref.err
for wl in C4 C1 C3 C5; do python -c "
import json; d=json.loads(open('gpurun_out/bench_${wl}_final4.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['schedule'], d['launch'], 'roof', d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], 'x', d['baselines']['speedup_vs_best_unfused'], 'e2e', d['e2e'].get('value'), 'err', d.get('max_rel_error'), d['clocks'])"; done
tail -c 400 gpurun_out/bench_ref_final4.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_C4_final4.csv \
  python bench.py --steps 2 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_bench_C4.log 2>&1
for wl in C4 C3; do
ncu --set full --clock-control none --import-source on -k regex:"plane_|cgemm" -s 3 -c 3 \
  -o gpurun_out/prof_${wl}_final4 -f python bench.py --workload $wl --steps 1 --warmup 3 --graph off --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_full_$wl.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_${wl}_final4.ncu-rep > gpurun_out/ncu_${wl}_final4.txt 2>&1
done
echo done
