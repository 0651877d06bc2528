#!/bin/bash
# session-4 GPU call 4: pipelined class head of the tuned inverse (TFNO_PLANE_ISKEW) +
# forward tail (TFNO_PLANE_SKEW): parity, bitwise test, C3 / C5L A/B, bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plane_generic.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g4_tests.log 2>&1; tail -1 gpurun_out/g4_tests.log
for r in 1 2; do for v in "-1 0" "-1 1"; do set -- $v
 echo "== SKEW=$1 ISKEW=$2 round $r"
 TFNO_PLANE_SKEW=$1 TFNO_PLANE_ISKEW=$2 timeout 300 python tools/stages.py --workloads C3,C5L --modes fully_fused 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d.get('workload'), d.get('mode'), d.get('ms'), d.get('stages_ms'))"
done; done 2>&1 | tee gpurun_out/g4_skew_ab.txt
for wl in C3 C5L C5; do timeout 600 python bench.py --workload $wl > gpurun_out/g4_bench_$wl.json 2>gpurun_out/g4_bench_$wl.err; python -c "
import json; d=json.loads(open('gpurun_out/g4_bench_$wl.json').read().strip().splitlines()[-1])
print('$wl', d['ms_per_step'], d['launch'], d['layer_roofline']['frac_of_roof_8TBps_74TF'], d['baselines'].get('speedup_vs_best_unfused'), d['roofline']['frac'], d.get('max_rel_error'))"; done
