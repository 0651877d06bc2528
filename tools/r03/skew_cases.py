"""Small invocations of the tuned plane kernels (C3 / C5 / 128^2 planes, several planes per CTA)
for compute-sanitizer over the pipelined class loops: run with TFNO_PLANE_SKEW / TFNO_PLANE_ISKEW
set (tools/r03/g6.sh)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2504_11681_b200 as T  # noqa: E402
from oracle import fnofuse_port as O  # noqa: E402

for s in [(1, 2, 2, 256, 256, 16, 16), (1, 2, 2, 256, 256, 32, 32), (2, 2, 2, 128, 128, 16, 16), (200, 1, 1, 256, 256, 16, 16)]:
    cfg = T.FnoLayerConfig(*s, rank=2)
    x, w = O.random_inputs(cfg, 5)
    out, _ = T.run_fused(cfg, T.SpectralTensor(x), T.ComplexMatrix(w))
    err = T.max_rel_error(out.data, O.reference_layer(cfg, x, w))
    assert err < 1e-5, (s, err)
print("ok")
