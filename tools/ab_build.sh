#!/bin/bash
# A/B of a compile-time switch: time WL (tools/stages.py) with the default build and with
# TFNO_NVCC_DEFS=$DEFS, alternating twice.  Usage: DEFS=TFNO_F1_NO_ACOMP WL=... MODES=... bash tools/ab_build.sh
WL=${WL:-C2-N256-H256-B1024}
MODES=${MODES:-fully_fused}
for round in 1 2; do
  for defs in "" "$DEFS"; do
    TFNO_NVCC_DEFS=$defs python -c "from paper_2504_11681_b200 import build; build.build(force=True)" || exit 1
    echo "== defs='$defs' round $round"
    timeout 300 python tools/stages.py --workloads $WL --modes $MODES 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(d.get('workload'), d.get('mode'), d.get('ms'))"
  done
done
python -c "from paper_2504_11681_b200 import build; build.build(force=True)"
