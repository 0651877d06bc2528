import numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
cases = [(16, 64, 64, 1, 128, 1, 32, 1), (3, 64, 64, 1, 128, 1, 32, 1), (5, 37, 21, 1, 128, 1, 20, 1),
         (2, 128, 8, 1, 128, 1, 64, 1), (4, 16, 30, 1, 128, 1, 1, 1), (1, 200, 3, 1, 128, 1, 33, 1)]
for rep in range(2):
    for case in cases:
        cfg = T.FnoLayerConfig(*case)
        x, w = O.random_inputs(cfg, 3000 + sum(case))
        out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
        ref = O.run_layer_values(cfg, x, w)
        print(rep, case, "err %.2e" % T.max_rel_error(out.data, ref), flush=True)
