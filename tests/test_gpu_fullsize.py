"""GPU parity at BASELINE.json's full sizes.  The CPU oracle cannot run the
whole batch (C4 would need ~190 GB of host RAM and ~14 min), so each full-size
run is checked (a) on batch slices against the oracle — batch elements are
independent, SURVEY.md §8c — and (b) through size-independent properties:
linearity, bitwise determinism, and batch-shard consistency.
FP32 tolerance 1e-5 (max_rel_error)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2504_11681_b200 as T
    from oracle import fnofuse_port as O
    return T, O, torch


def _rand(torch, shape, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.view_as_complex(torch.randn(tuple(shape) + (2,), generator=g, device="cuda"))


def _slice_check(T, O, cfg, x, w, y, idx):
    from types import SimpleNamespace
    wh = w.cpu().numpy()
    for b in idx:
        c1 = SimpleNamespace(**{**cfg.__dict__, "batch": 1})
        ref = O.run_layer_values(c1, x[b:b + 1].cpu().numpy(), wh)
        err = T.max_rel_error(y[b:b + 1].cpu().numpy(), ref)
        assert err < TOL, (cfg, b, err)


@pytest.mark.parametrize("name,shape,idx", [
    ("C3", (32, 64, 64, 256, 256, 32, 32, 2), (0, 17, 31)),
    ("C4", (128, 128, 128, 512, 512, 64, 64, 2), (0, 127)),
    ("C5-layer", (256, 64, 64, 256, 256, 16, 16, 2), (0, 255)),
    ("C2-max", (1024, 256, 256, 1, 4096, 1, 512, 1), (0, 1023)),
    ("C1", (16, 64, 64, 1, 128, 1, 32, 1), tuple(range(16))),
])
def test_full_size_batch_slices_vs_oracle(env, name, shape, idx):
    T, O, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x = _rand(torch, (cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), 11)
    w = _rand(torch, (cfg.hidden_dim, cfg.output_dim), 12).contiguous()
    y = T.run_layer_device(cfg, x, w)
    torch.cuda.synchronize()
    _slice_check(T, O, cfg, x, w, y, idx)
    y2 = T.run_layer_device(cfg, x, w)
    assert torch.equal(y, y2), "not bitwise deterministic"
    del x, y, y2
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,shape,idx", [
    ("C4", (128, 128, 128, 512, 512, 64, 64, 2), (0, 127)),
    ("C5-layer", (256, 64, 64, 256, 256, 16, 16, 2), (0, 255)),
])
def test_full_size_tensorcore_precisions(env, name, shape, idx):
    """The tcgen05 contraction variants at full C4 / C5-layer size, batch slices vs
    the oracle at the stated tolerances (3xTF32 1e-5, TF32 1e-3, BF16 5e-3)."""
    from types import SimpleNamespace
    T, O, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x = _rand(torch, (cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), 31)
    w = _rand(torch, (cfg.hidden_dim, cfg.output_dim), 32).contiguous()
    wh = w.cpu().numpy()
    c1 = SimpleNamespace(**{**cfg.__dict__, "batch": 1})
    refs = {b: O.run_layer_values(c1, x[b:b + 1].cpu().numpy(), wh) for b in idx}
    for prec, tol in (("tf32x3", 1e-5), ("tf32", 1e-3), ("bf16", 5e-3)):
        y = T.run_layer_device(cfg, x, w, precision=prec)
        torch.cuda.synchronize()
        for b in idx:
            err = T.max_rel_error(y[b:b + 1].cpu().numpy(), refs[b])
            assert err < tol, (name, prec, b, err)
        del y
    del x
    torch.cuda.empty_cache()


def test_c4_linearity_and_shards(env):
    """C4 layer shape (batch 16): L(x1 + 2 x2) == L(x1) + 2 L(x2) and two
    batch shards == the whole batch (bitwise)."""
    T, O, torch = env
    cfg = T.FnoLayerConfig(16, 128, 128, 512, 512, 64, 64, 2)
    x1 = _rand(torch, (16, 128, 512, 512), 21)
    x2 = _rand(torch, (16, 128, 512, 512), 22)
    w = _rand(torch, (128, 128), 23).contiguous()
    y1 = T.run_layer_device(cfg, x1, w).clone()
    y2 = T.run_layer_device(cfg, x2, w).clone()
    y12 = T.run_layer_device(cfg, x1 + 2 * x2, w)
    assert T.max_rel_error(y12.cpu().numpy(), (y1 + 2 * y2).cpu().numpy()) < TOL
    half = T.FnoLayerConfig(8, 128, 128, 512, 512, 64, 64, 2)
    a = T.run_layer_device(half, x1[:8].contiguous(), w).clone()
    b = T.run_layer_device(half, x1[8:].contiguous(), w)
    assert torch.equal(torch.cat([a, b]), y1)


def test_c5_chain_full_batch(env):
    """4-layer chain at full C5 batch (256) in one CUDA graph, slice vs the
    oracle's chained layers."""
    T, O, torch = env
    from types import SimpleNamespace

    from paper_2504_11681_b200.chain import FnoChain
    cfg = T.FnoLayerConfig(256, 64, 64, 256, 256, 16, 16, 2)
    x = _rand(torch, (256, 64, 256, 256), 31)
    ws = [_rand(torch, (64, 64), 40 + i).contiguous() for i in range(4)]
    ch = FnoChain(cfg, ws).capture(x)
    y = ch.forward(x)
    torch.cuda.synchronize()
    c1 = SimpleNamespace(**{**cfg.__dict__, "batch": 1})
    for b in (0, 255):
        ref = x[b:b + 1].cpu().numpy()
        for w in ws:
            ref = O.run_layer_values(c1, ref, w.cpu().numpy())
        assert T.max_rel_error(y[b:b + 1].cpu().numpy(), ref) < TOL
