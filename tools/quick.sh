#!/bin/bash
# quick GPU iteration: plane/fused parity subset + layer timings (no baselines/e2e/cpu)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "${TESTS:-plane2d or golden}" 2>&1 | tail -4
for wl in ${WLS:-C4 C3 C5L}; do
  timeout 300 python bench.py --workload $wl --steps 10 --no-baselines --no-e2e --no-cpu > gpurun_out/q_$wl.json 2> gpurun_out/q_$wl.err || tail -5 gpurun_out/q_$wl.err
  python -c "
import json; d=json.loads(open('gpurun_out/q_$wl.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], 'ms', d['value'], 'GFLOP/s', 'roof', d['layer_roofline']['frac_of_measured_hbm'], [(s['kernel'], s['ms'], s['GBps']) for s in d['stages']])"
done
if [ -n "$NCU" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 3 -c ${NCUC:-2} -o gpurun_out/prof_q -f \
    python bench.py --workload ${NCUWL:-C4} --steps 1 --warmup 3 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_q.log 2>&1
  tail -2 gpurun_out/ncu_q.log
fi
