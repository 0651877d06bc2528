"""Symmetric (+-mode) truncation (paper_2504_11681_b200.symmetric, SURVEY §8f
row 4) vs a float64 oracle that gathers bins [-k/2, k/2) explicitly with
torch.fft in complex128.  FP32 bar 1e-5."""

import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _bins(n, k):
    s = k // 2
    return [(j - s) % n for j in range(k)]  # frequency j - s at storage index j


def _ref(x, w, cfg, per_mode):
    import torch
    x = x.to(torch.complex128)
    w = w.to(torch.complex128)
    by = _bins(cfg.dim_y, cfg.keep_y)
    if cfg.rank == 2:
        bx = _bins(cfg.dim_x, cfg.keep_x)
        X = torch.fft.fft2(x)[:, :, bx][:, :, :, by]
    else:
        X = torch.fft.fft(x, dim=-1)[..., by]
    C = torch.einsum("bhpq,hnpq->bnpq" if per_mode else "bhpq,hn->bnpq", X, w)
    S = torch.zeros((cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y), dtype=torch.complex128)
    if cfg.rank == 2:
        for i, p in enumerate(bx):
            S[:, :, p, by] = C[:, :, i, :]
        return torch.fft.ifft2(S)
    S[..., by] = C
    return torch.fft.ifft(S, dim=-1)


CASES = [
    ((3, 8, 6, 1, 256, 1, 32, 1), False),
    ((2, 4, 5, 64, 64, 8, 8, 2), False),
    ((1, 2, 3, 256, 256, 32, 32, 2), False),    # plane kernels
    ((64, 4, 4, 1, 128, 1, 20, 1), True),       # per-mode weights
    ((2, 4, 5, 32, 64, 6, 10, 2), True),
]


@pytest.mark.parametrize("case,per_mode", CASES)
def test_symmetric_vs_float64(case, per_mode):
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200.symmetric import run_layer_symmetric
    cfg = T.FnoLayerConfig(*case)
    g = torch.Generator().manual_seed(sum(case) + per_mode)
    x = torch.view_as_complex(torch.randn((cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y, 2), generator=g))
    wshape = (cfg.hidden_dim, cfg.output_dim) + ((cfg.keep_x, cfg.keep_y) if per_mode else ())
    w = torch.view_as_complex(torch.randn(wshape + (2,), generator=g))
    if per_mode:
        y = run_layer_symmetric(cfg, x.cuda(), w_modes=w.cuda())
    else:
        y = run_layer_symmetric(cfg, x.cuda(), w.cuda().contiguous())
    torch.cuda.synchronize()
    ref = _ref(x, w, cfg, per_mode)
    assert T.max_rel_error(y.cpu().numpy(), ref.numpy()) < TOL
