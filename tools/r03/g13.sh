#!/bin/bash
# A/B: loaded twiddle companions in the fused inverse + mix (default) vs rebuilt per use (TFNO_TWP_REBUILD_INV)
mkdir -p gpurun_out
for round in 1 2; do
  for defs in "" "TFNO_TWP_REBUILD_INV"; do
    TFNO_NVCC_DEFS=$defs python -c "from paper_2504_11681_b200 import build; build.build(force=True)" || exit 1
    echo "== defs='$defs' round $round"
    timeout 300 python tools/stages.py --workloads C4 --modes fully_fused 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d.get('workload'), d.get('mode'), d.get('ms'), d.get('stages_ms'))"
  done
done 2>&1 | tee gpurun_out/g13_twp_ab.txt
python -c "from paper_2504_11681_b200 import build; build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_plane_generic.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/g13_tests.log 2>&1; tail -1 gpurun_out/g13_tests.log
