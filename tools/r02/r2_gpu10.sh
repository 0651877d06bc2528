#!/bin/bash
# fused inverse + channel mix (deeper A ring): parity + same-box A/B on C4 / C3 / C5L
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py -q -m gpu -x -k "fused_mix or generic_plane_layer" > gpurun_out/t10.txt 2>&1; tail -3 gpurun_out/t10.txt
out=gpurun_out/fusedmix_ab2.txt; : > $out
for rep in 1 2; do for wl in C4 C3; do for fm in 0 1; do
  TFNO_PLANE_FUSEDMIX=$fm timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>gpurun_out/b10.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl fm=$fm', d['ms_per_step'], d['schedule'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
done; done; done
cat $out
TFNO_PLANE_FUSEDMIX=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"invmix" -s 1 -c 1 \
  -o gpurun_out/prof_invmix -f python bench.py --workload C4 --steps 1 --warmup 1 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_invmix.log 2>&1
tail -1 gpurun_out/ncu_invmix.log
