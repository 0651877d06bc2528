#!/bin/bash
# session-4 GPU call 3: skewed class tail of the tuned forward (TFNO_PLANE_SKEW):
# parity (plane tests incl. the bitwise skew test, full-size slices), then C3 / C5 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g3_tests.log 2>&1; tail -1 gpurun_out/g3_tests.log
VAR=TFNO_PLANE_SKEW VALS="0 1" WL=C3,C5L timeout 900 bash tools/ab_env.sh > gpurun_out/g3_skew_ab.txt 2>&1; cat gpurun_out/g3_skew_ab.txt
for r in 1 2; do for v in 0 1; do
TFNO_PLANE_SKEW=$v timeout 300 python bench.py --workload C3 --no-baselines --no-e2e --no-cpu --steps 50 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C3 skew=$v', d['ms_per_step'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], [(s['kernel'], s['ms']) for s in d['stages']])"
done; done 2>&1 | tee gpurun_out/g3_c3_bench_skew.txt
for wl in C3 C5L; do timeout 600 python bench.py --workload $wl > gpurun_out/g3_bench_$wl.json 2>gpurun_out/g3_bench_$wl.err; python -c "
import json; d=json.loads(open('gpurun_out/g3_bench_$wl.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['launch'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], d['baselines'].get('speedup_vs_best_unfused'), d['roofline']['frac'], d.get('max_rel_error'))"; done
