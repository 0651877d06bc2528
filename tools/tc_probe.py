"""Probe the tcgen05 contraction on given shapes / precisions."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_11681_b200 as T  # noqa: E402

for (M, N, K, B) in [(300, 37, 20, 2), (256, 37, 16, 1), (256, 64, 20, 1), (300, 64, 16, 1), (4096, 128, 128, 2)]:
    rng = np.random.default_rng(0)
    a = (rng.standard_normal((B, K, M)) + 1j * rng.standard_normal((B, K, M))).astype(np.complex64)
    w = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
    A = torch.from_numpy(a).cuda().transpose(1, 2)
    W = torch.from_numpy(w).cuda()
    want = np.einsum("bkm,kn->bmn", a.astype(np.complex128), w.astype(np.complex128))
    for prec in ("tf32", "tf32x3"):
        out = torch.full((B, N, M), 7.0, dtype=torch.complex64, device="cuda").transpose(1, 2)
        C = T.cgemm_device(A, W, out=out, precision=prec).cpu().numpy()
        d = np.abs(C - want)
        bad = np.argwhere(d > 1e-3 * np.abs(want).max())
        print((M, N, K, B), prec, "err", T.max_rel_error(C, want), "nbad", len(bad), bad[:4].tolist())
