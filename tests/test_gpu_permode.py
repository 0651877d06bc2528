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
    (128, 4, 4, 256, 256, 32, 32, 2),    # 2D plane kernels (batch 128)
    (19, 7, 21, 1, 128, 1, 37, 1),       # ragged batch / channels / modes (every tile edge masked)
    (3, 9, 5, 128, 64, 9, 7, 2),         # 2D ragged keeps: 63 modes
    (40, 70, 33, 64, 64, 16, 16, 2),     # H not a multiple of the 4-deep chunk, several b / n tiles
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
    y3 = run_layer_permode(cfg, x.cuda(), w.cuda())
    torch.cuda.synchronize()
    ref = _ref(x, w, cfg)
    assert T.max_rel_error(y.cpu().numpy(), ref.numpy()) < TOL
    assert torch.equal(y, y2) and torch.equal(y, y3)  # deterministic


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


def test_permode_mix_abi_vs_einsum():
    """tfno_permode_mix straight through the C-ABI: C = alpha * einsum(bhq,hnq->bnq) in float64,
    natural layouts, alpha applied, zero-size problems are no-ops, bad sizes are rejected."""
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200._lib import lib
    g = torch.Generator().manual_seed(3)
    for B, H, N, MQ in [(17, 13, 35, 100), (64, 128, 16, 32), (1, 1, 1, 1)]:
        A = torch.view_as_complex(torch.randn((B, H, MQ, 2), generator=g))
        W = torch.view_as_complex(torch.randn((H, N, MQ, 2), generator=g))
        C = torch.empty((B, N, MQ), dtype=torch.complex64, device="cuda")
        Ad, Wd = A.cuda(), W.cuda()
        assert lib().tfno_permode_mix(B, H, N, MQ, Ad.data_ptr(), Wd.data_ptr(), C.data_ptr(), 0.5, None) == 0
        torch.cuda.synchronize()
        ref = 0.5 * torch.einsum("bhq,hnq->bnq", A.to(torch.complex128), W.to(torch.complex128))
        assert T.max_rel_error(C.cpu().numpy(), ref.numpy()) < TOL
    assert lib().tfno_permode_mix(0, 3, 3, 3, None, None, None, 1.0, None) == 0
    assert lib().tfno_permode_mix(-1, 3, 3, 3, None, None, None, 1.0, None) != 0
