#!/bin/bash
# A/B of a runtime env switch: VAR=name VALS="0 1 2" WL=... MODES=... bash tools/ab_env.sh
WL=${WL:-C2-N4096-H64-B1024}
MODES=${MODES:-fully_fused}
for round in 1 2; do
  for v in $VALS; do
    echo "== $VAR=$v round $round"
    env $VAR=$v timeout 300 python tools/stages.py --workloads $WL --modes $MODES 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print(d.get('workload'), d.get('mode'), d.get('ms'), d.get('stages_ms'))"
  done
done
