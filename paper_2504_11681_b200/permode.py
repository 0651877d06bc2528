"""Per-mode spectral weights — the FNO contraction of neural-operator codes,
``out_hat[b,n,p,q] = sum_h x_hat[b,h,p,q] * W[h,n,p,q]`` (einsum
``bhpq,hnpq->bnpq``), SURVEY.md §8f row 4.  The reference ``fnofuse`` shares
one W[H,N] across all modes (Appendix A) and has no per-mode variant, so this
extension is pinned by its own float64 oracle (``tests/test_gpu_permode.py``).

Same first-``keep``-bin truncation, zero padding and 1/(dx*dy) inverse as the
reference layer; the transforms are the sm_100a spectrum kernels of the
forward path (per-plane 2D kernels for the plane shapes, row/pencil FFTs
otherwise) and the channel mix is the FP32 SIMT mode CGEMM batched over the
kx*ky modes (M = batch, K = H, N = N_out) on mode-major copies of the
spectra.  Mode-major weights are prepared once per weight tensor
(``prepare_weights``).
"""

from __future__ import annotations

from . import _device
from ._lib import check, lib
from .core import FnoLayerConfig, ShapeMismatch
from .multigpu import spectrum_forward, spectrum_inverse


def prepare_weights(w_modes):
    """[H, N, kx, ky] complex64 (CUDA) -> mode-major [kx*ky, H, N] contiguous."""
    H, N, kx, ky = w_modes.shape
    return w_modes.permute(2, 3, 0, 1).reshape(kx * ky, H, N).contiguous()


def run_layer_permode(cfg: FnoLayerConfig, x, w_modes=None, w_prepared=None, stream=None):
    """y[B,N,dx,dy] = iDFT_pad( einsum(bhpq,hnpq->bnpq, DFT_trunc(x), W) ) / (dx*dy).

    x: [B,H,dx,dy] complex64 CUDA tensor; w_modes: [H,N,kx,ky] (or its
    ``prepare_weights`` form in ``w_prepared``)."""
    t = _device.torch()
    B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
    kx, ky = cfg.keep_x, cfg.keep_y
    MQ = kx * ky
    if tuple(x.shape) != (B, H, cfg.dim_x, cfg.dim_y):
        raise ShapeMismatch(f"x shape {tuple(x.shape)} != {(B, H, cfg.dim_x, cfg.dim_y)}")
    if w_prepared is None:
        if w_modes is None or tuple(w_modes.shape) != (H, N, kx, ky):
            raise ShapeMismatch(f"w_modes must be [{H}, {N}, {kx}, {ky}]")
        w_prepared = prepare_weights(w_modes)
    A = spectrum_forward(cfg, x.contiguous(), stream)                  # [B,H,kx,ky]
    Aq = A.reshape(B, H, MQ).permute(2, 1, 0).contiguous()             # [q][h][b]
    Cq = t.empty((MQ, N, B), dtype=t.complex64, device=x.device)       # [q][n][b]
    # per mode q: C[q] (B x N, b fastest) = A[q]^T (B x H) * W[q] (H x N)
    rc = lib().tfno_cgemm(B, N, H, MQ, Aq.data_ptr(), 1, B, H * B, w_prepared.data_ptr(), N, 1, H * N,
                          Cq.data_ptr(), 1, B, N * B, 1.0, _device.stream_ptr(stream))
    check(rc, "tfno_cgemm")
    C = Cq.permute(2, 1, 0).reshape(B, N, kx, ky).contiguous()         # [B,N,kx,ky]
    return spectrum_inverse(cfg, C, (B, N), scale=1.0, stream=stream)
