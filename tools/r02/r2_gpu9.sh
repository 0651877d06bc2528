#!/bin/bash
# fused inverse + channel mix: parity, then same-box A/B (TFNO_PLANE_FUSEDMIX=0/1) on C4 / C3 / C5L
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t9.txt 2>&1; tail -3 gpurun_out/t9.txt
out=gpurun_out/fusedmix_ab.txt; : > $out
for rep in 1 2; do for wl in C4 C3 C5L; do for fm in 0 1; do
  TFNO_PLANE_FUSEDMIX=$fm timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>gpurun_out/b9.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl fm=$fm', d['ms_per_step'], d['schedule'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
done; done; done
cat $out; tail -3 gpurun_out/b9.err
