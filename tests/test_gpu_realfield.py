"""Real-field layer and FNO block (paper_2504_11681_b200.realfield, SURVEY.md §8f
row 4) vs a float64 oracle written with torch.fft.rfft2 / irfft2 (the reference is
complex-to-complex only, so this extension has its own oracle):

    y = act(irfft2(rfft2(x)[..., :kx, :ky] W, s=(dx, dy)) + einsum(bhxy,hn->bnxy, x, Wb) + bias)

FP32 bar 1e-5 (max_rel_error), as for the complex layer."""

import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _ref(x, w, cfg, wb=None, bias=None, act=None):
    import torch
    x = x.double()
    w = w.to(torch.complex128)
    if cfg.rank == 2:
        X = torch.fft.rfft2(x)[..., :cfg.keep_x, :cfg.keep_y]
        y = torch.fft.irfft2(torch.einsum("bhpq,hn->bnpq", X, w), s=(cfg.dim_x, cfg.dim_y))
    else:
        X = torch.fft.rfft(x, dim=-1)[..., :cfg.keep_y]
        y = torch.fft.irfft(torch.einsum("bhpq,hn->bnpq", X, w), n=cfg.dim_y, dim=-1)
    if wb is not None:
        y = y + torch.einsum("bhxy,hn->bnxy", x, wb.double())
    if bias is not None:
        y = y + bias.double()[None, :, None, None]
    if act == "relu":
        y = torch.relu(y)
    elif act == "gelu":
        y = torch.nn.functional.gelu(y)
    return y


CASES = [
    (4, 8, 6, 1, 256, 1, 32, 1),        # 1D
    (3, 4, 4, 1, 128, 1, 65, 1),        # 1D, keep = dy/2 + 1 (Nyquist bin kept)
    (2, 4, 5, 64, 64, 8, 8, 2),         # 2D generic row/pencil kernels
    (2, 4, 4, 256, 256, 32, 32, 2),     # 2D plane kernels (C3 plane shape)
    (1, 2, 3, 16, 8, 16, 5, 2),         # 2D keep_y = dy/2 + 1, keep_x = dx
]


@pytest.mark.parametrize("case", CASES)
def test_real_layer_vs_float64(case):
    import torch

    import paper_2504_11681_b200 as T
    cfg = T.FnoLayerConfig(*case)
    g = torch.Generator().manual_seed(sum(case))
    x = torch.randn((cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), generator=g)
    w = torch.view_as_complex(torch.randn((cfg.hidden_dim, cfg.output_dim, 2), generator=g))
    y = T.real_layer(cfg, x.cuda(), w.cuda())
    torch.cuda.synchronize()
    assert y.dtype == torch.float32
    err = T.max_rel_error(y.cpu().numpy(), _ref(x, w, cfg).numpy())
    assert err < TOL, err


@pytest.mark.parametrize("act", [None, "relu", "gelu"])
@pytest.mark.parametrize("case", [CASES[0], CASES[3]])
def test_fno_block_vs_float64(case, act):
    import torch

    import paper_2504_11681_b200 as T
    cfg = T.FnoLayerConfig(*case)
    g = torch.Generator().manual_seed(7 + sum(case))
    x = torch.randn((cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), generator=g)
    w = torch.view_as_complex(torch.randn((cfg.hidden_dim, cfg.output_dim, 2), generator=g))
    wb = torch.randn((cfg.hidden_dim, cfg.output_dim), generator=g)
    bias = torch.randn((cfg.output_dim,), generator=g)
    y = T.fno_block(cfg, x.cuda(), w.cuda(), bypass_w=wb.cuda(), bias=bias.cuda(), activation=act)
    torch.cuda.synchronize()
    err = T.max_rel_error(y.cpu().numpy(), _ref(x, w, cfg, wb, bias, act).numpy())
    assert err < TOL, err


def test_real_epilogue_scalar_path_and_launches():
    """P % 4 != 0 takes the scalar epilogue; every stage is one of this library's kernels."""
    import torch

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200._lib import lib
    cfg = T.FnoLayerConfig(3, 2, 3, 1, 2, 1, 2, 1)
    x = torch.randn(3, 2, 1, 2)
    w = torch.randn(2, 3, dtype=torch.complex64)
    n0 = lib().tfno_launch_count()
    y = T.fno_block(cfg, x.cuda(), w.cuda(), bias=torch.ones(3).cuda(), activation="relu")
    torch.cuda.synchronize()
    assert lib().tfno_launch_count() - n0 >= 5
    assert T.max_rel_error(y.cpu().numpy(), _ref(x, w, cfg, None, torch.ones(3), "relu").numpy()) < TOL


def test_real_layer_rejects_bad_inputs():
    import torch

    import paper_2504_11681_b200 as T
    cfg = T.FnoLayerConfig(1, 2, 2, 1, 16, 1, 10, 1)
    with pytest.raises(T.FnofuseError):
        T.real_layer(cfg, torch.randn(1, 2, 1, 16).cuda(), torch.randn(2, 2, dtype=torch.complex64).cuda())
    cfg = T.FnoLayerConfig(1, 2, 2, 1, 16, 1, 4, 1)
    with pytest.raises(T.ShapeMismatch):
        T.real_layer(cfg, torch.randn(1, 2, 1, 16, dtype=torch.float64).cuda(),
                     torch.randn(2, 2, dtype=torch.complex64).cuda())
    with pytest.raises(T.FnofuseError):
        T.fno_block(cfg, torch.randn(1, 2, 1, 16).cuda(), torch.randn(2, 2, dtype=torch.complex64).cuda(),
                    activation="tanh")
