"""Generate the golden fixtures by importing the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``fnofuse`` from /root/reference/pkg/src (read-only; nothing is
copied), runs the reference's own public API (``run_layer`` in every mode,
``fft.plan``/``fft.execute``, ``layer_op_stats``, the ledger) on seeded
inputs, and writes small ``.npz`` / ``.json`` fixtures next to this script.
The GPU box has no /root/reference; tests there read only these fixtures.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (name, batch, hidden, out, dim_x, dim_y, keep_x, keep_y, rank, seed)
LAYER_CASES = [
    ("c1", 16, 64, 64, 1, 128, 1, 32, 1, 1001),            # BASELINE configs[0]
    ("r1_ragged", 3, 20, 37, 1, 64, 1, 13, 1, 11),
    ("r1_keepall", 3, 8, 8, 1, 64, 1, 64, 1, 12),
    ("r1_dy1", 4, 5, 3, 1, 1, 1, 1, 1, 13),
    ("r1_dy2_keep1", 2, 3, 4, 1, 2, 1, 1, 1, 14),
    ("r1_h1n1", 5, 1, 1, 1, 256, 1, 32, 1, 15),
    ("r1_n1024", 2, 16, 24, 1, 1024, 1, 128, 1, 16),
    ("r1_n4096", 1, 8, 8, 1, 4096, 1, 512, 1, 17),
    ("r2_small", 2, 16, 24, 32, 64, 8, 16, 2, 21),
    ("r2_nonsquare", 2, 6, 5, 8, 64, 3, 20, 2, 22),
    ("r2_dx1", 2, 4, 6, 1, 32, 1, 8, 2, 23),
    ("r2_keepall", 1, 4, 4, 16, 16, 16, 16, 2, 24),
    ("r2_128", 1, 8, 8, 128, 128, 16, 16, 2, 25),
    ("r2_c3like", 1, 4, 4, 256, 256, 32, 32, 2, 26),
]

FFT_NS = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]


def main():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import fnofuse
    from fnofuse import fft
    from fnofuse.cgemm import ComplexMatrix
    from fnofuse.core import FnoLayerConfig, random_spectral
    from fnofuse.pipeline import MODES, layer_op_stats, run_layer

    meta = {"reference": "fnofuse " + fnofuse.__version__, "numpy": np.__version__,
            "layers": {}, "plans": [], "fft_cases": []}
    arrays = {}
    for (name, b, h, n, dx, dy, kx, ky, rank, seed) in LAYER_CASES:
        cfg = FnoLayerConfig(b, h, n, dx, dy, kx, ky, rank=rank)
        rng = np.random.default_rng(seed)
        x = random_spectral(cfg, rng)
        w = ComplexMatrix.random(h, n, rng)
        outs, ledgers, stats = {}, {}, {}
        for mode in MODES:
            out, led = run_layer(cfg, x, w, mode=mode)
            outs[mode] = out.data
            ledgers[mode] = led.to_json_dict()
            stats[mode] = layer_op_stats(cfg, mode)
        bitwise = all(np.array_equal(outs[m], outs["fully_fused"]) for m in MODES)
        arrays[f"{name}__x"] = x.data
        arrays[f"{name}__w"] = np.ascontiguousarray(w.values)
        arrays[f"{name}__out_fully_fused"] = outs["fully_fused"]
        if not bitwise:
            for m in MODES:
                arrays[f"{name}__out_{m}"] = outs[m]
        meta["layers"][name] = {"cfg": cfg.to_json_dict(), "seed": seed,
                                "modes_bitwise_equal": bitwise,
                                "ledgers": ledgers, "op_stats": stats}
    for nn in FFT_NS:
        keeps = sorted(k for k in {1, 2, 3, max(1, nn // 8), max(1, nn // 4), max(1, nn // 2), nn - 1, nn} if 1 <= k <= nn)
        for keep in keeps:
            for src in sorted({1, max(1, nn // 8), max(1, nn // 2), nn}):
                for d in (fft.FORWARD, fft.INVERSE):
                    p = fft.plan(nn, d, keep=keep, src_len=src)
                    meta["plans"].append({"n": nn, "direction": d, "keep": keep, "src_len": src,
                                          "op_budget": p.op_budget,
                                          "twiddle_budget": p.twiddle_budget,
                                          "full_ops": p.full_ops})
    rng = np.random.default_rng(77)
    for i, (nn, d, keep, src) in enumerate([(8, "forward", 8, 8), (64, "forward", 16, 64),
                                            (256, "forward", 64, 256), (1024, "forward", 128, 1024),
                                            (64, "inverse", 64, 16), (256, "inverse", 256, 64),
                                            (512, "inverse", 512, 64), (4096, "forward", 512, 4096),
                                            (4096, "inverse", 4096, 512), (2, "forward", 1, 2),
                                            (1, "inverse", 1, 1)]):
        p = fft.plan(nn, d, keep=keep, src_len=src)
        xin = (rng.standard_normal((5, src)) + 1j * rng.standard_normal((5, src))).astype(np.complex64)
        out, cnt = fft.batched_execute(p, xin)
        arrays[f"fft{i}__in"] = xin
        arrays[f"fft{i}__out"] = out
        meta["fft_cases"].append({"id": i, "n": nn, "direction": d, "keep": keep,
                                  "src_len": src, "butterflies": cnt.butterflies,
                                  "twiddle_muls": cnt.twiddle_muls})
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(meta["plans"]), "plans")


if __name__ == "__main__":
    main()
