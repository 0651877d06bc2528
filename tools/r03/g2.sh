#!/bin/bash
# session-4 GPU call 2: S4 default (C4 plane tests + bench line), C3 A/Bs:
# eager vs CUDA-graph step, PDL off/on, generic vs tuned forward, tuned variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_plane_generic.py -m gpu -x -q > gpurun_out/g2_tests.log 2>&1; tail -1 gpurun_out/g2_tests.log
timeout 600 python bench.py > gpurun_out/g2_bench_C4.json 2>gpurun_out/g2_bench_C4.err
python -c "
import json; d=json.loads(open('gpurun_out/g2_bench_C4.json').read().strip().splitlines()[-1])
print('C4', d['ms_per_step'], d['roofline']['frac'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], [(s['kernel'], s['ms']) for s in d['stages']], d['clocks']['sm_mhz'])"
for r in 1 2; do
 for g in off on; do
  for pdl in 1 2; do
   TFNO_PDL=$pdl timeout 300 python bench.py --workload C3 --no-baselines --no-e2e --no-cpu --graph $g --steps 50 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C3 graph=$g pdl=$pdl', d['ms_per_step'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], [(s['kernel'], s['ms']) for s in d['stages']])"
  done
 done
done 2>&1 | tee gpurun_out/g2_c3_graph_pdl.txt
VAR=TFNO_PLANE_GENERIC VALS="0 1 3" WL=C3 timeout 600 bash tools/ab_env.sh > gpurun_out/g2_c3_generic.txt 2>&1; cat gpurun_out/g2_c3_generic.txt
VAR=TFNO_PLANE_VARIANT VALS="0 1 2 3" WL=C3 timeout 600 bash tools/ab_env.sh > gpurun_out/g2_c3_variant.txt 2>&1; cat gpurun_out/g2_c3_variant.txt
