import numpy as np, paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
for case in [(2, 128, 8, 1, 128, 1, 64, 1), (2, 64, 8, 1, 128, 1, 64, 1), (2, 128, 8, 1, 128, 1, 32, 1), (2, 16, 8, 1, 128, 1, 64, 1), (2, 128, 8, 1, 128, 1, 48, 1)]:
    cfg = T.FnoLayerConfig(*case)
    x, w = O.random_inputs(cfg, 3000 + sum(case))
    out, _ = T.run_layer(cfg, T.SpectralTensor(x), T.ComplexMatrix(w), mode="fully_fused")
    ref = O.run_layer_values(cfg, x, w)
    d = np.abs(out.data - ref)[:, :, 0, :]
    print(case, T.layer_schedule(cfg, "fully_fused")[1], "err", T.max_rel_error(out.data, ref),
          "per-n max", np.round(d.max(axis=(0, 2)) / np.abs(ref).max(), 4), "per-b", np.round(d.max(axis=(1, 2)) / np.abs(ref).max(), 4))
