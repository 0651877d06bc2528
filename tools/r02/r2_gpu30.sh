#!/bin/bash
# generic forward with rows straight into a 2-deep register queue (TFNO_PLANE_GDLD=1): parity + A/B + ncu
mkdir -p gpurun_out
TFNO_PLANE_GDLD=1 PYTHONPATH=. timeout 600 python -c "
import numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
for s in [(2, 3, 4, 512, 512, 64, 64), (150, 2, 2, 512, 512, 64, 64), (1, 5, 9, 512, 512, 40, 64)]:
    cfg = T.FnoLayerConfig(*s, rank=2); x, w = O.random_inputs(cfg, 11)
    out, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    print(s, T.max_rel_error(out.data, O.reference_layer(cfg, x, w)))
"
out=gpurun_out/gdld2_ab.txt; : > $out
for rep in 1 2 3; do for d in 0 1; do
  TFNO_PLANE_GDLD=$d timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-baselines --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 dld=$d', d['ms_per_step'], [(s['kernel'], s['ms']) for s in d['stages']])" >> $out
done; done
cat $out
TFNO_PLANE_GDLD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plane_fwd" -s 1 -c 1 \
  -o gpurun_out/prof_gdld2 -f python bench.py --workload C4 --steps 1 --warmup 1 --no-baselines --no-e2e --no-cpu > gpurun_out/ncu_gdld2.log 2>&1
tail -1 gpurun_out/ncu_gdld2.log
