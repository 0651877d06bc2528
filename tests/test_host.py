"""CPU: host logic of the drop-in (validation order, errors, ledger, op
stats, schedule), and that the C-ABI library loads and exports every symbol
include/turbofno.h declares.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2504_11681_b200 as T
from paper_2504_11681_b200 import _lib
from tests import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "turbofno.h")).read()
    declared = set(re.findall(r"\b(tfno_[a-z_0-9]+)\s*\(", hdr))
    lib = _lib.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
    assert b"sm_100a" in lib.tfno_version()


def test_native_plan_counts_equal_reference():
    for p in G.meta()["plans"]:
        pl = T.plan(p["n"], p["direction"], keep=p["keep"], src_len=p["src_len"])
        assert (pl.op_budget, pl.twiddle_budget, pl.full_ops) == (p["op_budget"], p["twiddle_budget"], p["full_ops"])
        assert pl.op_budget == sum(int(m.sum()) for m in pl.prune_mask)


def test_plan_attributes_mirror_reference():
    a = T.plan(64, keep=16, src_len=32)
    assert len(a.stages) == 6 and [s.stride for s in a.stages] == [1, 2, 4, 8, 16, 32]
    assert [s.twiddle_offset for s in a.stages] == [0, 1, 3, 7, 15, 31]
    assert not a.twiddles.flags.writeable
    assert all(m.all() for m in T.plan(32).prune_mask)
    assert T.plan(4, keep=1).op_budget / T.full_op_count(4) == 0.375
    with pytest.raises(T.InvalidLength):
        T.plan(100)
    with pytest.raises(T.InvalidKeep):
        T.plan(8, keep=9)
    with pytest.raises(T.InvalidSrcLen):
        T.plan(8, src_len=0)


@pytest.mark.parametrize("name", G.LAYER_NAMES)
def test_ledger_and_op_stats_equal_reference(name):
    m = G.meta()["layers"][name]
    cfg = T.FnoLayerConfig(**m["cfg"])
    for mode in T.MODES:
        assert T.model_ledger(cfg, T.DEFAULT_TILES, mode).to_json_dict() == m["ledgers"][mode]
        assert T.layer_op_stats(cfg, mode) == m["op_stats"][mode]


def test_launch_counts_and_delta():
    cfg = T.FnoLayerConfig(2, 16, 16, 1, 64, 1, 16, rank=1)
    got = {mode: T.model_ledger(cfg, T.DEFAULT_TILES, mode).kernel_launches for mode in T.MODES}
    assert got == {"staged": 5, "fft_optimized": 3, "fused_fft_gemm": 2, "fused_gemm_ifft": 2, "fully_fused": 1}
    big = T.FnoLayerConfig(1024, 64, 64, 1, 256, 1, 64, rank=1)
    d = T.traffic_delta(T.model_ledger(big, T.DEFAULT_TILES, "staged"), T.model_ledger(big, T.DEFAULT_TILES, "fully_fused"))
    assert d.arrays["A_panel"]["saved_written"] == 1024 * 64 * 64 * 8
    r2 = T.FnoLayerConfig(2, 16, 16, 64, 64, 16, 16, rank=2)
    d2 = T.traffic_delta(T.model_ledger(r2, T.DEFAULT_TILES, "staged"), T.model_ledger(r2, T.DEFAULT_TILES, "fully_fused"))
    assert d2.stage1_write_ratio == 0.25 and d2.stage2_compute_ratio == (16 / 64) ** 2
    with pytest.raises(T.ConfigMismatch):
        T.traffic_delta(T.model_ledger(cfg, T.DEFAULT_TILES, "staged"), T.model_ledger(r2, T.DEFAULT_TILES, "staged"))


def test_validation_order_and_errors_before_any_device_work():
    cfg = T.FnoLayerConfig(2, 16, 16, 1, 64, 1, 16, rank=1)
    x = T.SpectralTensor.zeros(2, 16, 1, 64)
    w = T.ComplexMatrix.zeros(16, 16)
    with pytest.raises(T.FnofuseError):
        T.run_layer(cfg, x, w, mode="bogus")
    with pytest.raises(T.ScheduleInvalid):
        T.run_layer(cfg, x, w, fft_batch_size=4)
    bad = T.FnoLayerConfig(2, 16, 16, 1, 100, 1, 50, rank=1)
    with pytest.raises(T.ConfigError) as ei:
        T.run_layer(bad, x, w)
    assert [v.code for v in ei.value.violations] == ["NonPowerOfTwoLength"]
    with pytest.raises(T.ShapeMismatch):
        T.run_layer(cfg, T.SpectralTensor.zeros(2, 16, 1, 128), w)
    with pytest.raises(T.ShapeMismatch):
        T.run_layer(cfg, x, T.ComplexMatrix.zeros(17, 16))
    # mode error wins over a config error (pipeline.py:133-137 order)
    with pytest.raises(T.FnofuseError) as e2:
        T.run_layer(bad, x, w, mode="bogus")
    assert not isinstance(e2.value, T.ConfigError)


def test_native_violations_match_python():
    cases = [T.FnoLayerConfig(2, 16, 16, 1, 64, 1, 16, rank=1), T.FnoLayerConfig(2, 16, 16, 8, 100, 4, 50, 2),
             T.FnoLayerConfig(0, 16, 16, 1, 64, 1, 16, rank=1), T.FnoLayerConfig(2, 16, 16, 4, 64, 2, 16, rank=1),
             T.FnoLayerConfig(2, 16, 16, 8, 64, 9, 65, rank=2), T.FnoLayerConfig(2, 16, 16, 8, 64, 4, 16, rank=3)]
    tiles = [T.DEFAULT_TILES, T.TileConfig(32, 32, 4, 32, 16, 4, 4), T.TileConfig(32, 30, 8, 32, 16, 4, 4)]
    bits = {v: k for k, v in _lib.VIOLATION_BITS.items()}
    for cfg in cases:
        for t in tiles:
            py = {v.code for v in T.config_violations(cfg, t)}
            c, tt = _lib.cfg_struct(cfg), _lib.tiles_struct(t)
            mask = _lib.lib().tfno_config_violations(ctypes.byref(c), ctypes.byref(tt), 8)
            assert {name for name, bit in bits.items() if mask & bit} == py, (cfg, t)


def test_schedules_and_workspace():
    c4 = T.FnoLayerConfig(128, 128, 128, 512, 512, 64, 64, 2)
    # FP32: the channel mix runs inside the inverse kernel (plane_invmix_g), its C
    # tiles in a per-CTA two-task ring (SMs x 2 x 8 planes; 148 SMs without a device)
    assert T.layer_schedule(c4, "fully_fused") == (2, "plane-fft2d|plane-mix-ifft2d")
    assert T.workspace_bytes(c4, "fully_fused") == (128 * 128 + 148 * 2 * 8) * 64 * 64 * 8
    # tensor-core precisions keep the standalone tcgen05 CGEMM (W' image) between the plane kernels
    # (the tcgen05 mix inside the inverse is opt-in: TFNO_PLANE_FUSEDMIX=1)
    for p in ("tf32x3", "tf32", "bf16"):
        assert T.layer_schedule(c4, "fully_fused", p)[1] == "plane-fft2d|cgemm-modes|plane-ifft2d"
    c1 = T.FnoLayerConfig(16, 64, 64, 1, 128, 1, 32, 1)
    assert T.layer_schedule(c1, "fully_fused") == (1, "tiny1d-fft-cgemm-ifft")  # one launch (tiny1d.cu)
    assert T.layer_schedule(T.FnoLayerConfig(256, 64, 64, 1, 128, 1, 32, 1), "fully_fused") == \
        (1, "fused1d-fft-cgemm-ifft")  # more CTAs than one wave: the persistent fused kernel
    assert T.layer_schedule(c1, "fused_fft_gemm") == (2, "fused1d-fft-cgemm|y-ifft")  # K4 on the fused 1D kernel
    assert T.layer_schedule(c1, "fused_gemm_ifft") == (2, "y-fft|fused1d-cgemm-ifft")  # K5
    c2 = T.FnoLayerConfig(1024, 256, 256, 1, 256, 1, 32, 1)
    assert T.layer_schedule(c2, "fully_fused") == (1, "fused1d-fft-cgemm-ifft")
    c2b = T.FnoLayerConfig(1024, 256, 256, 1, 4096, 1, 512, 1)
    assert T.layer_schedule(c2b, "fully_fused") == (3, "y-fft|cgemm|y-ifft")
    assert T.layer_schedule(c1, "fft_optimized")[0] == 3
    r2 = T.FnoLayerConfig(2, 16, 16, 32, 64, 8, 16, 2)  # generic plane kernels (dy >= 64, KP = 16 <= dx)
    assert T.layer_schedule(r2, "fully_fused") == (3, "plane-fft2d|cgemm-modes|plane-ifft2d")
    # ragged keeps pad to KP = 32 modes per axis in the A / C workspace tensors
    r3 = T.FnoLayerConfig(2, 16, 8, 256, 128, 20, 12, 2)
    assert T.workspace_bytes(r3, "fully_fused") == 2 * (16 + 8) * 32 * 32 * 8
    c3 = T.FnoLayerConfig(32, 64, 64, 256, 256, 32, 32, 2)  # too few mix tasks per CTA: standalone CGEMM
    assert T.layer_schedule(c3, "fully_fused") == (3, "plane-fft2d|cgemm-modes|plane-ifft2d")
    # fused_gemm_ifft on the plane path is the fused channel mix + inverse kernel
    assert T.layer_schedule(c3, "fused_gemm_ifft") == (2, "plane-fft2d|plane-mix-ifft2d")
    r4 = T.FnoLayerConfig(2, 16, 16, 64, 32, 8, 16, 2)  # dy < 64: the paper schedule
    assert T.layer_schedule(r4, "fully_fused") == (3, "x-fft|fused-fft-cgemm-ifft|x-ifft")
    f = T.layer_flops(c4)
    assert f["bytes"] == 8 * (2 * 128 * 128 * 512 * 512 + 128 * 128)


def test_no_cpu_fallback():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    cfg = T.FnoLayerConfig(1, 2, 2, 1, 8, 1, 4, rank=1)
    with pytest.raises(_lib.NativeUnavailable):
        T.run_layer(cfg, T.SpectralTensor.zeros(1, 2, 1, 8), T.ComplexMatrix.zeros(2, 2))
    with pytest.raises(_lib.NativeUnavailable):
        T.execute(T.plan(8), np.zeros(8, np.complex64))
