"""GPU: the tcgen05 (tensor-core) contraction.  Stated tolerances
(BASELINE.md §5): 3xTF32 <= 1e-5 (fp32-level), TF32 <= 1e-3, BF16 <= 5e-3
at the layer (the bare BF16 GEMM vs float64: 1e-2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2504_11681_b200 as T
    from oracle import fnofuse_port as O
    return T, O, torch


@pytest.mark.parametrize("M,N,K,B", [(4096, 128, 128, 2), (512, 256, 256, 2), (200, 300, 40, 1), (1024, 64, 64, 3), (256, 64, 64, 2), (300, 37, 20, 2), (32, 64, 64, 5), (16, 40, 30, 7), (32, 256, 256, 3),
                                     (32, 64, 64, 4), (129, 1, 3, 1), (128, 128, 256, 1)])
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("tf32x3", 1e-5), ("tf32", 2e-3), ("bf16", 1e-2)])
def test_tc_cgemm_vs_float64(env, M, N, K, B, prec, tol):
    T, O, torch = env
    rng = np.random.default_rng(M + N + K)
    a = (rng.standard_normal((B, K, M)) + 1j * rng.standard_normal((B, K, M))).astype(np.complex64)
    w = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
    A = torch.from_numpy(a).cuda().transpose(1, 2)            # [B, M, K] view, m contiguous
    W = torch.from_numpy(w).cuda()
    out = torch.empty((B, N, M), dtype=torch.complex64, device="cuda").transpose(1, 2)
    C = T.cgemm_device(A, W, out=out, alpha=0.5, precision=prec)
    want = 0.5 * np.einsum("bkm,kn->bmn", a.astype(np.complex128), w.astype(np.complex128))
    assert T.max_rel_error(C.cpu().numpy(), want) < tol


@pytest.mark.parametrize("shape", [(2, 8, 8, 512, 512, 64, 64, 2), (3, 16, 8, 256, 256, 32, 32, 2),
                                   (2, 8, 16, 256, 256, 16, 16, 2), (3, 12, 20, 1, 1024, 1, 128, 1), (2, 256, 256, 1, 256, 1, 32, 1)])
def test_layer_tensorcore_precisions(env, shape):
    T, O, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x, w = O.random_inputs(cfg, 8)
    ref = O.run_layer_values(cfg, x, w)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    modes = ["fully_fused"] if cfg.rank == 2 else ["fft_optimized", "fully_fused"]
    for mode in modes:  # rank-1 fully_fused: contraction-heavy shapes take the unfused tcgen05 schedule
        for prec, tol in (("tf32x3", 1e-5), ("tf32", 1e-3), ("bf16", 5e-3)):
            y = T.run_layer_device(cfg, xd, wd, mode=mode, precision=prec)
            assert T.max_rel_error(y.cpu().numpy(), ref) < tol, (mode, prec)


@pytest.mark.parametrize("shape", [(2, 8, 8, 512, 512, 64, 64, 2), (3, 12, 20, 1, 1024, 1, 128, 1),
                                   (2, 16, 8, 128, 256, 40, 24, 2)])
@pytest.mark.parametrize("prec", ["tf32x3", "tf32", "bf16"])
def test_prepared_weights_match_per_call_image(env, shape, prec):
    """tfno_prepare_weights (W' image built once per weight tensor) gives the same
    layer bitwise as the per-call image build, with one launch fewer."""
    T, O, torch = env
    cfg = T.FnoLayerConfig(*shape)
    x, w = O.random_inputs(cfg, 9)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    mode = "fully_fused" if cfg.rank == 2 else "fft_optimized"
    y0 = T.run_layer_device(cfg, xd, wd, mode=mode, precision=prec).clone()
    pw = T.prepare_weights(cfg, wd, prec)
    n0 = T._lib.lib().tfno_launch_count()
    y1 = T.run_layer_device(cfg, xd, wd, mode=mode, precision=prec, packed=pw)
    n1 = T._lib.lib().tfno_launch_count() - n0
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert n1 == T.layer_schedule(cfg, mode, prec)[0] - 1  # no image-build launch
    with pytest.raises(T.FnofuseError):
        T.run_layer_device(cfg, xd, wd, mode=mode, precision="tf32" if prec != "tf32" else "bf16", packed=pw)
