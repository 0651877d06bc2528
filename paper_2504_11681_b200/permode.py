"""Per-mode spectral weights — the FNO contraction of neural-operator codes,
``out_hat[b,n,p,q] = sum_h x_hat[b,h,p,q] * W[h,n,p,q]`` (einsum
``bhpq,hnpq->bnpq``), SURVEY.md §8f row 4.  The reference ``fnofuse`` shares
one W[H,N] across all modes (Appendix A) and has no per-mode variant, so this
extension is pinned by its own float64 oracle (``tests/test_gpu_permode.py``).

Same first-``keep``-bin truncation, zero padding and 1/(dx*dy) inverse as the
reference layer; the transforms are the sm_100a spectrum kernels of the
forward path (per-plane 2D kernels for the plane shapes, row/pencil FFTs
otherwise) and the channel mix is ``tfno_permode_mix`` (csrc/permode.cu): a
mode-parallel FP32 contraction that reads the spectrum [B][H][kx*ky] and the
weights [H][N][kx][ky] in their natural layouts and writes the [B][N][kx][ky]
modes the inverse consumes, so there are no mode-major copies on the path.
"""

from __future__ import annotations

from . import _device
from ._lib import check, lib
from .core import FnoLayerConfig, ShapeMismatch
from .multigpu import _on, spectrum_forward, spectrum_inverse


def prepare_weights(w_modes):
    """[H, N, kx, ky] complex64 (CUDA) -> the contiguous [H, N, kx*ky] the mix kernel reads
    (a no-op view for contiguous complex64 weights)."""
    H, N, kx, ky = w_modes.shape
    return w_modes.to(_device.torch().complex64).reshape(H, N, kx * ky).contiguous()


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
    if (tuple(w_prepared.shape) != (H, N, MQ) or not w_prepared.is_contiguous()
            or w_prepared.dtype != t.complex64):
        raise ShapeMismatch(f"w_prepared must be a contiguous complex64 [{H}, {N}, {MQ}] tensor (prepare_weights)")
    A = spectrum_forward(cfg, x.contiguous(), stream)                  # [B,H,kx,ky]
    with _on(stream):
        C = t.empty((B, N, kx, ky), dtype=t.complex64, device=x.device)
    # C[b][n][q] = sum_h A[b][h][q] W[h][n][q]
    rc = lib().tfno_permode_mix(B, H, N, MQ, A.data_ptr(), w_prepared.data_ptr(), C.data_ptr(), 1.0,
                                _device.stream_ptr(stream))
    check(rc, "tfno_permode_mix")
    return spectrum_inverse(cfg, C, (B, N), scale=1.0, stream=stream)

