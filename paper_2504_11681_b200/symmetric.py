"""Symmetric (+-mode) truncation — SURVEY.md §8f row 4, beyond the reference.

The reference keeps the FIRST keep_x x keep_y bins (Appendix A).  Neural-operator
codes keep the low frequencies of both signs, bins [-k/2, k/2) per axis.  That is
the reference layer conjugated by a plane modulation (``tfno_modulate``):

    DFT(x * e^{+2 pi i s n / N})[j] = DFT(x)[j - s]

so with s = keep // 2 per axis, the first-keep bins of the modulated input are
the bins [-s, keep - s) of x, and the zero-padded inverse of those bins equals
e^{+2 pi i s n / N} times the inverse we want — undone by modulating the output
with -s.  ``run_layer_symmetric`` = modulate(+s) -> first-keep layer (shared W or
per-mode W, any mode/precision) -> modulate(-s).  Per-mode weight index p' in
[0, keep) is frequency p' - s.  Pinned by its own float64 oracle
(``tests/test_gpu_symmetric.py``).
"""

from __future__ import annotations

from . import _device
from ._lib import check, lib
from .core import FnoLayerConfig
from .pipeline import run_layer_device


def shifts(cfg: FnoLayerConfig):
    return (cfg.keep_x // 2 if cfg.rank == 2 else 0), cfg.keep_y // 2


def modulate(t_in, cfg: FnoLayerConfig, sign: int, out=None, scale: float = 1.0, stream=None):
    """out = scale * t_in * exp(sign * 2 pi i (sx x / dx + sy y / dy)) over the last two axes."""
    t = _device.torch()
    sx, sy = shifts(cfg)
    src = t_in.contiguous()
    dst = t.empty_like(src) if out is None else out
    planes = src.numel() // (cfg.dim_x * cfg.dim_y)
    check(lib().tfno_modulate(planes, cfg.dim_x, cfg.dim_y, sx, sy, int(sign), src.data_ptr(), dst.data_ptr(),
                              float(scale), _device.stream_ptr(stream)), "tfno_modulate")
    return dst


def run_layer_symmetric(cfg: FnoLayerConfig, x, w=None, w_modes=None, mode: str = "fully_fused",
                        precision: str = "fp32", stream=None):
    """Fourier layer keeping bins [-keep/2, keep/2) on each transformed axis.
    w: shared [H,N] weights (reference contraction) or w_modes: [H,N,kx,ky]."""
    xm = modulate(x, cfg, +1, stream=stream)
    if w_modes is not None:
        from .permode import run_layer_permode
        y = run_layer_permode(cfg, xm, w_modes, stream=stream)
    else:
        y = run_layer_device(cfg, xm, w, mode=mode, precision=precision, stream=stream)
    return modulate(y, cfg, -1, out=y, stream=stream)
