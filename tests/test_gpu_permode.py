"""Per-mode spectral weights (paper_2504_11681_b200.permode, SURVEY.md §8f
row 4) vs a float64 oracle: torch.fft in complex128 of
iDFT_pad(einsum(bhpq,hnpq->bnpq, DFT_trunc(x), W)) — the reference has no
per-mode variant, so this is the extension's own oracle.  FP32 bar 1e-5."""

import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _ref(x, w, cfg):
    import torch
    x = x.to(torch.complex128)
    w = w.to(torch.complex128)
    if cfg.rank == 2:
        X = torch.fft.fft2(x)[..., :cfg.keep_x, :cfg.keep_y]
        return torch.fft.ifft2(torch.einsum("bhpq,hnpq->bnpq", X, w), s=(cfg.dim_x, cfg.dim_y))
    X = torch.fft.fft(x, dim=-1)[..., :cfg.keep_y]
    return torch.fft.ifft(torch.einsum("bhpq,hnpq->bnpq", X, w), n=cfg.dim_y, dim=-1)


CASES = [
    (64, 8, 6, 1, 256, 1, 32, 1),        # 1D, mode CGEMM fast path (M = batch = 64)
    (5, 4, 3, 1, 128, 1, 20, 1),         # 1D, general CGEMM (small batch, ragged keep)
    (2, 4, 5, 64, 64, 8, 8, 2),          # 2D generic spectra
    (128, 4, 4, 256, 256, 32, 32, 2),    # 2D plane kernels, fast mode CGEMM (batch 128)
]


@pytest.mark.parametrize("case", CASES)
def test_permode_vs_float64(case):
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200.permode import prepare_weights, run_layer_permode
    cfg = T.FnoLayerConfig(*case)
    g = torch.Generator().manual_seed(sum(case))
    x = torch.view_as_complex(torch.randn((cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y, 2), generator=g))
    w = torch.view_as_complex(torch.randn((cfg.hidden_dim, cfg.output_dim, cfg.keep_x, cfg.keep_y, 2),
                                          generator=g))
    y = run_layer_permode(cfg, x.cuda(), w.cuda())
    y2 = run_layer_permode(cfg, x.cuda(), w_prepared=prepare_weights(w.cuda()))
    torch.cuda.synchronize()
    ref = _ref(x, w, cfg)
    assert T.max_rel_error(y.cpu().numpy(), ref.numpy()) < TOL
    assert torch.equal(y, y2)


def test_permode_equals_shared_weights_when_modes_repeat():
    """W[h,n,p,q] = W[h,n] for all modes reduces to the reference layer."""
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200.permode import run_layer_permode
    cfg = T.FnoLayerConfig(64, 8, 8, 1, 256, 1, 32, 1)
    x = torch.randn(64, 8, 1, 256, dtype=torch.complex64, device="cuda")
    w = torch.randn(8, 8, dtype=torch.complex64, device="cuda")
    y1 = run_layer_permode(cfg, x, w[:, :, None, None].expand(8, 8, 1, 32).contiguous())
    y2 = T.run_layer_device(cfg, x, w)
    torch.cuda.synchronize()
    assert T.max_rel_error(y1.cpu().numpy(), y2.cpu().numpy()) < TOL
