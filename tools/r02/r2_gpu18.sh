#!/bin/bash
# tcgen05 fused mix: parity (fused-mix tests, tensor-core tests) + A/B on C4 / C3 / C5L for tf32x3 / tf32
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x -k "fused_mix" > gpurun_out/t18.txt 2>&1; tail -3 gpurun_out/t18.txt
timeout 1200 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/t18b.txt 2>&1; tail -3 gpurun_out/t18b.txt
out=gpurun_out/tcmix_ab.txt; : > $out
for wl in C4 C3 C5L; do for p in tf32x3 tf32; do for fm in 0 1; do
  TFNO_PLANE_FUSEDMIX=$fm timeout 300 python bench.py --workload $wl --precision $p --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>gpurun_out/b18.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $p fm=$fm', d['ms_per_step'], d['schedule'], [(s['kernel'], s['ms']) for s in d['stages']], d.get('max_rel_error'))" >> $out
done; done; done
cat $out; tail -3 gpurun_out/b18.err
