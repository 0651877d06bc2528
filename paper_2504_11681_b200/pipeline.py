"""The Fourier layer — drop-in for ``fnofuse.pipeline`` (pipeline.py:1-416).

``run_layer(cfg, x, w, tiles, mode, fft_batch_size)`` keeps the reference's
signature, validation order (mode -> schedule -> config -> shapes,
pipeline.py:133-137), exception classes and return value
``(SpectralTensor, TrafficLedger)``.  The values are computed on the GPU by
``libturbofno.so`` (``tfno_layer_forward``); the ledger is the reference's
*modeled* per-array traffic (pipeline.py:143-292), returned identically.
Measured DRAM bytes of the real kernels are reported by ``bench.py`` / ncu
beside it.

``run_layer_device`` is the zero-copy device API (torch CUDA tensors in,
torch CUDA tensor out) used by the benchmark and multi-GPU driver.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device
from ._lib import MODE_CODES, PREC_CODES, cfg_struct, check, lib
from .cgemm import ComplexMatrix
from .core import (COMPLEX_BYTES, DEFAULT_TILES, FFT_BLOCK_BATCH, FnoLayerConfig, FnofuseError,
                   ShapeMismatch, SpectralTensor, TileConfig, validate_config)
from .fft import FORWARD, INVERSE, full_op_count, plan

ARRAY_NAMES = ("input", "spectrum_stage1", "A_panel", "B", "C", "output")
MODES = ("staged", "fft_optimized", "fused_fft_gemm", "fused_gemm_ifft", "fully_fused")


class ScheduleInvalid(FnofuseError):
    pass


class ConfigMismatch(FnofuseError):
    pass


@dataclass
class ArrayTraffic:
    bytes_read: int = 0
    bytes_written: int = 0

    @property
    def total(self) -> int:
        return self.bytes_read + self.bytes_written


@dataclass
class TrafficLedger:
    """Per-array modeled global byte counters plus logical pass count (pipeline.py:53-91)."""

    arrays: dict = field(default_factory=lambda: {n: ArrayTraffic() for n in ARRAY_NAMES})
    kernel_launches: int = 0
    config_key: tuple = ()

    def read(self, name: str, nbytes: int) -> None:
        self.arrays[name].bytes_read += int(nbytes)

    def write(self, name: str, nbytes: int) -> None:
        self.arrays[name].bytes_written += int(nbytes)

    def launch(self) -> None:
        self.kernel_launches += 1

    def total(self, name: str) -> int:
        return self.arrays[name].total

    def total_bytes(self) -> int:
        return sum(t.total for t in self.arrays.values())

    def to_json_dict(self) -> dict:
        return {"arrays": {n: {"bytes_read": t.bytes_read, "bytes_written": t.bytes_written}
                           for n, t in self.arrays.items()},
                "kernel_launches": self.kernel_launches}


@dataclass(frozen=True)
class FusedSchedule:
    panel_rows: int
    panel_cols: int
    k_loop_order: tuple
    epilogue_tiles: tuple


def build_schedule(cfg: FnoLayerConfig, tiles: TileConfig, fft_batch_size: int = FFT_BLOCK_BATCH) -> FusedSchedule:
    """pipeline.py:106-116."""
    if tiles.k_tb != fft_batch_size:
        raise ScheduleInvalid(f"FFT block batch bs={fft_batch_size} must equal k_tb={tiles.k_tb}")
    n_chunks = -(-cfg.hidden_dim // tiles.k_tb)
    n_tiles = tuple((n0, min(cfg.output_dim, n0 + tiles.n_tb)) for n0 in range(0, cfg.output_dim, tiles.n_tb))
    return FusedSchedule(panel_rows=tiles.m_tb, panel_cols=tiles.k_tb,
                         k_loop_order=tuple(range(n_chunks)), epilogue_tiles=n_tiles)


def _check_layer_args(cfg, x_shape, w_shape):
    """pipeline.py:119-126."""
    shape = (cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y)
    if tuple(x_shape) != shape:
        raise ShapeMismatch(f"tensor shape {tuple(x_shape)} != config shape {shape}")
    if tuple(w_shape) != (cfg.hidden_dim, cfg.output_dim):
        raise ShapeMismatch(f"weights are {w_shape[0]}x{w_shape[1]}, config wants "
                            f"{cfg.hidden_dim}x{cfg.output_dim}")


def model_ledger(cfg: FnoLayerConfig, tiles: TileConfig, mode: str) -> TrafficLedger:
    """The reference's modeled traffic for (cfg, mode) — the same counter
    updates, in the same order, as run_layer (pipeline.py:143-292)."""
    E = COMPLEX_BYTES
    B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
    dx, dy, kx, ky = cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y
    fuse_fg = mode in ("fused_fft_gemm", "fully_fused")
    fuse_gi = mode in ("fused_gemm_ifft", "fully_fused")
    builtin = mode != "staged"
    m_size = B * kx * ky
    led = TrafficLedger(config_key=(B, H, N, dx, dy, kx, ky, cfg.rank))
    if cfg.rank == 2:
        led.read("input", B * H * dx * dy * E)
        if builtin:
            led.write("spectrum_stage1", B * H * kx * dy * E)
            led.launch()
        else:
            led.write("spectrum_stage1", B * H * dx * dy * E)
            led.launch()
            led.read("spectrum_stage1", B * H * kx * dy * E)
            led.write("spectrum_stage1", B * H * kx * dy * E)
            led.launch()
        src_name = "spectrum_stage1"
    else:
        src_name = "input"
    src_elems = B * H * kx * dy
    b_read = -(-m_size // tiles.m_tb) * H * N * E
    if fuse_fg:
        for k0 in range(0, H, tiles.k_tb):
            k1 = min(H, k0 + tiles.k_tb)
            led.read(src_name, B * (k1 - k0) * kx * dy * E)
        led.read("B", b_read)
    else:
        if builtin:
            led.read(src_name, src_elems * E)
            led.write("A_panel", m_size * H * E)
            led.launch()
        else:
            led.read(src_name, src_elems * E)
            led.write("spectrum_stage1", src_elems * E)
            led.launch()
            led.read("spectrum_stage1", m_size * H * E)
            led.write("A_panel", m_size * H * E)
            led.launch()
        led.read("A_panel", m_size * H * E)
        led.read("B", b_read)
    mid_elems = B * N * kx * dy
    if fuse_gi:
        led.write("output", mid_elems * E)
        led.launch()
    else:
        led.write("C", m_size * N * E)
        led.launch()
        if builtin:
            led.read("C", m_size * N * E)
            led.write("output", mid_elems * E)
            led.launch()
        else:
            led.read("C", m_size * N * E)
            led.write("output", B * N * dx * dy * E)
            led.launch()
            led.read("output", B * N * dx * dy * E)
            led.write("output", B * N * dx * dy * E)
            led.launch()
    if cfg.rank == 2:
        if builtin:
            led.read("output", mid_elems * E)
        else:
            led.read("output", B * N * dx * dy * E)
        led.write("output", B * N * dx * dy * E)
        led.launch()
    return led


def _validate(cfg, x_shape, w_shape, tiles, mode, fft_batch_size):
    if mode not in MODES:
        raise FnofuseError(f"unknown mode {mode!r}; expected one of {MODES}")
    build_schedule(cfg, tiles, fft_batch_size)
    validate_config(cfg, tiles, fft_batch_size)
    _check_layer_args(cfg, x_shape, w_shape)


def workspace_bytes(cfg: FnoLayerConfig, mode: str = "fully_fused", precision: str = "fp32") -> int:
    c = cfg_struct(cfg)
    return int(lib().tfno_workspace_bytes(ctypes.byref(c), MODE_CODES[mode], PREC_CODES[precision]))


def layer_schedule(cfg: FnoLayerConfig, mode: str = "fully_fused", precision: str = "fp32"):
    """(number of kernel launches, description) of the sm_100a schedule."""
    c = cfg_struct(cfg)
    buf = ctypes.create_string_buffer(256)
    n = lib().tfno_layer_schedule(ctypes.byref(c), MODE_CODES[mode], PREC_CODES[precision], buf, 256)
    return int(n), buf.value.decode()


class PackedWeights:
    """The tcgen05 contraction's real-embedded W' image of one weight tensor
    (tfno_prepare_weights): built once, reused by every run_layer_device call
    with ``packed=`` (no per-call image build launch)."""

    def __init__(self, cfg: FnoLayerConfig, w, precision: str, stream=None):
        t = _device.torch()
        if precision not in ("tf32", "tf32x3", "bf16"):
            raise FnofuseError(f"packed weights are for the tensor-core precisions, not {precision!r}")
        w = w if (w.dtype == t.complex64 and w.is_contiguous()) else w.to(t.complex64).contiguous()
        c = cfg_struct(cfg)
        self.precision, self.hidden_dim, self.output_dim = precision, cfg.hidden_dim, cfg.output_dim
        nbytes = int(lib().tfno_packed_weight_bytes(ctypes.byref(c), PREC_CODES[precision]))
        self.data = t.empty(max(nbytes, 16), dtype=t.uint8, device=w.device)
        self.w = w
        check(lib().tfno_prepare_weights(ctypes.byref(c), PREC_CODES[precision], w.data_ptr(), self.data.data_ptr(),
                                         _device.stream_ptr(stream)), "tfno_prepare_weights")


def prepare_weights(cfg: FnoLayerConfig, w, precision: str = "tf32x3", stream=None) -> PackedWeights:
    """Pack W[H][N] (complex64 CUDA tensor, row-major) for the tensor-core
    contraction once per weight tensor (SURVEY.md §8b tfno_prepare_weights)."""
    return PackedWeights(cfg, w, precision, stream)


def run_layer_device(cfg: FnoLayerConfig, x, w, tiles: TileConfig = DEFAULT_TILES, mode: str = "fully_fused",
                     fft_batch_size: int = FFT_BLOCK_BATCH, out=None, precision: str = "fp32", stream=None,
                     validate: bool = True, workspace=None, packed: "PackedWeights" = None):
    """Device API: x [B,H,dx,dy] and w [H,N] complex64 CUDA tensors (w in
    row-major [H][N]); returns the [B,N,dx,dy] CUDA tensor.  Asynchronous
    on ``stream`` (default: torch's current stream).  ``workspace``: an
    optional caller-owned uint8 CUDA tensor (``workspace_bytes`` large) —
    CUDA graphs capture its pointer, so graph owners pass their own instead
    of the shared per-device scratch (which may be regrown by other calls)."""
    t = _device.torch()
    if validate:
        _validate(cfg, tuple(x.shape), tuple(w.shape), tiles, mode, fft_batch_size)
    if precision not in PREC_CODES:
        raise FnofuseError(f"unknown precision {precision!r}")
    dev = x.device
    if dev.type != "cuda":
        raise FnofuseError("run_layer_device needs CUDA tensors (no CPU fallback)")
    x = x if (x.dtype == t.complex64 and x.is_contiguous()) else x.to(t.complex64).contiguous()
    w = w if (w.dtype == t.complex64 and w.is_contiguous()) else w.to(t.complex64).contiguous()
    # the kernels move rows with 16-byte TMA bulk copies: odd-element views get an aligned copy
    if x.data_ptr() % 16:
        x = x.clone()
    if w.data_ptr() % 16:
        w = w.clone()
    user_out = None
    if out is not None and out.data_ptr() % 16:
        user_out, out = out, None
    if out is None:
        out = t.empty((cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y), dtype=t.complex64, device=dev)
    c = cfg_struct(cfg)
    mcode, pcode = MODE_CODES[mode], PREC_CODES[precision]
    nbytes = int(lib().tfno_workspace_bytes(ctypes.byref(c), mcode, pcode))
    if workspace is not None and workspace.numel() >= nbytes:
        ws = workspace if nbytes else None
    else:
        ws = _device.workspace(nbytes, dev, stream)  # per (device, stream): no sharing across streams
    if packed is not None and precision != "fp32":
        if (packed.precision != precision or packed.hidden_dim != cfg.hidden_dim
                or packed.output_dim != cfg.output_dim):
            raise FnofuseError("packed weights were prepared for another precision or shape")
        rc = lib().tfno_layer_forward_packed(ctypes.byref(c), mcode, pcode, x.data_ptr(), w.data_ptr(),
                                             packed.data.data_ptr(), out.data_ptr(),
                                             ws.data_ptr() if ws is not None else None, nbytes,
                                             _device.stream_ptr(stream))
        check(rc, "tfno_layer_forward_packed")
    else:
        rc = lib().tfno_layer_forward(ctypes.byref(c), mcode, pcode, x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                      ws.data_ptr() if ws is not None else None, nbytes,
                                      _device.stream_ptr(stream))
        check(rc, "tfno_layer_forward")
    if user_out is not None:
        if stream is not None:
            with t.cuda.stream(stream):
                user_out.copy_(out)
        else:
            user_out.copy_(out)
        return user_out
    return out


def run_layer(cfg: FnoLayerConfig, x: SpectralTensor, w: ComplexMatrix, tiles: TileConfig = DEFAULT_TILES,
              mode: str = "fully_fused", fft_batch_size: int = FFT_BLOCK_BATCH, precision: str = "fp32"):
    """Run one spectral layer on the GPU; returns (output tensor, traffic
    ledger) exactly like pipeline.run_layer (pipeline.py:129-294)."""
    xd = x.data if isinstance(x, SpectralTensor) else x
    wv = w.values if isinstance(w, ComplexMatrix) else w
    _validate(cfg, tuple(xd.shape), tuple(wv.shape), tiles, mode, fft_batch_size)
    dev = _device.require_cuda()
    t = _device.torch()
    x_dev = _device.to_device_c64(xd, dev)
    w_dev = _device.to_device_c64(np.ascontiguousarray(_device_np(wv)), dev)
    y = run_layer_device(cfg, x_dev, w_dev, tiles, mode, fft_batch_size, precision=precision, validate=False)
    out = y.cpu().numpy()
    del t
    return SpectralTensor(out), model_ledger(cfg, tiles, mode)


def _device_np(v):
    return v.detach().cpu().numpy() if hasattr(v, "detach") else np.asarray(v)


def run_staged(cfg, x, w, tiles=DEFAULT_TILES, fft_batch_size=FFT_BLOCK_BATCH):
    """pipeline.py:297-300 — the unfused baseline (cuFFT + truncate + cuBLAS + pad + cuFFT^-1)."""
    return run_layer(cfg, x, w, tiles, "staged", fft_batch_size)


def run_fused(cfg, x, w, tiles=DEFAULT_TILES, fft_batch_size=FFT_BLOCK_BATCH):
    """pipeline.py:303-306 — fully fused execution."""
    return run_layer(cfg, x, w, tiles, "fully_fused", fft_batch_size)


@dataclass(frozen=True)
class TrafficDelta:
    arrays: dict
    baseline_launches: int
    fused_launches: int
    stage1_write_ratio: float
    stage2_compute_ratio: float

    def to_json_dict(self) -> dict:
        return {"arrays": self.arrays, "baseline_launches": self.baseline_launches,
                "fused_launches": self.fused_launches, "stage1_write_ratio": self.stage1_write_ratio,
                "stage2_compute_ratio": self.stage2_compute_ratio}


def stage_ratios(cfg_key: tuple) -> tuple:
    """pipeline.py:329-339."""
    _, _, _, dx, dy, kx, ky, rank = cfg_key
    if rank == 2:
        return kx / dx, (kx * ky) / (dx * dy)
    return 1.0, ky / dy


def traffic_delta(staged: TrafficLedger, fused: TrafficLedger) -> TrafficDelta:
    """pipeline.py:342-366."""
    if staged.config_key != fused.config_key:
        raise ConfigMismatch(f"ledgers from different configs: {staged.config_key} vs {fused.config_key}")
    arrays = {}
    for name in ARRAY_NAMES:
        s, f = staged.arrays[name], fused.arrays[name]
        arrays[name] = {"staged_read": s.bytes_read, "staged_written": s.bytes_written,
                        "fused_read": f.bytes_read, "fused_written": f.bytes_written,
                        "saved_read": s.bytes_read - f.bytes_read,
                        "saved_written": s.bytes_written - f.bytes_written,
                        "traffic_ratio": (f.total / s.total) if s.total else 1.0}
    s1, s2 = stage_ratios(staged.config_key)
    return TrafficDelta(arrays=arrays, baseline_launches=staged.kernel_launches,
                        fused_launches=fused.kernel_launches, stage1_write_ratio=s1, stage2_compute_ratio=s2)


def layer_op_stats(cfg: FnoLayerConfig, mode: str) -> dict:
    """pipeline.py:369-416 — canonical FFT op counts of one layer."""
    if mode not in MODES:
        raise FnofuseError(f"unknown mode {mode!r}")
    builtin = mode != "staged"
    B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
    dx, dy, kx, ky = cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y
    stages, base = [], []
    if cfg.rank == 2:
        stages.append((B * H * dy, plan(dx, FORWARD, keep=(kx if builtin else dx))))
        base.append((B * H * dy, dx))
    stages.append((B * H * kx, plan(dy, FORWARD, keep=(ky if builtin else dy))))
    base.append((B * H * kx, dy))
    if builtin:
        stages.append((B * N * kx, plan(dy, INVERSE, src_len=ky)))
    else:
        stages.append((B * N * dx, plan(dy, INVERSE)))
    base.append((B * N * dx, dy))
    if cfg.rank == 2:
        stages.append((B * N * dy, plan(dx, INVERSE, src_len=(kx if builtin else dx))))
        base.append((B * N * dy, dx))
    budget = sum(p * pl.op_budget for p, pl in stages)
    twiddles = sum(p * pl.twiddle_budget for p, pl in stages)
    baseline = sum(p * full_op_count(n) for p, n in base)
    ratio = budget / baseline if baseline else 1.0
    if cfg.rank == 2:
        s2_elems = B * H * kx * (ky if builtin else dy)
        s2_untrunc = B * H * dx * dy
    else:
        s2_elems = B * H * (ky if builtin else dy)
        s2_untrunc = B * H * dy
    return {"fft_op_budget": budget, "fft_twiddle_muls": twiddles, "fft_op_baseline": baseline,
            "fft_op_ratio": ratio, "fft_op_reduction": 1.0 - ratio, "stage2_elements": s2_elems,
            "stage2_elements_untruncated": s2_untrunc}


def layer_flops(cfg: FnoLayerConfig, mode: str = "fully_fused") -> dict:
    """Canonical algorithmic work of one layer (SURVEY.md §8d / BASELINE.md §3):
    flops = 2*fft_op_budget + 6*fft_twiddle_muls + 8*B*kx*ky*H*N,
    bytes = 8*(B*H*dx*dy + B*N*dx*dy + H*N)."""
    st = layer_op_stats(cfg, mode)
    fft = 2 * st["fft_op_budget"] + 6 * st["fft_twiddle_muls"]
    gemm = 8 * cfg.batch * cfg.keep_x * cfg.keep_y * cfg.hidden_dim * cfg.output_dim
    nbytes = 8 * (cfg.batch * cfg.hidden_dim * cfg.dim_x * cfg.dim_y
                  + cfg.batch * cfg.output_dim * cfg.dim_x * cfg.dim_y + cfg.hidden_dim * cfg.output_dim)
    return {"fft_flops": fft, "cgemm_flops": gemm, "flops": fft + gemm, "bytes": nbytes}


class HostPipeline:
    """End-to-end host-buffer execution as a three-stage software pipeline over
    batch chunks: streams per role -- ``ncopy`` H2D streams and ``ncopy`` D2H
    streams (alternating chunks, so each direction keeps more than one copy in
    flight) and one kernel stream -- over ``nbuf`` device chunk buffers, so the
    two PCIe directions and the sm_100a kernels all run back to back:

        H2D(i)     waits for layer(i - nbuf)  (its input buffer is free again)
        layer(i)   waits for H2D(i) and D2H(i - nbuf) (its output buffer is free)
        D2H(i)     waits for layer(i)

    Inputs and outputs are pinned host tensors; device buffers are allocated
    once and reused.  The default chunk is one batch element up to 512 MiB of
    in+out per chunk (small chunks shorten the pipeline fill / drain; the layer
    kernels of a chunk are far shorter than its transfers)."""

    def __init__(self, cfg: FnoLayerConfig, mode: str = "fully_fused", precision: str = "fp32",
                 chunk: int | None = None, nbuf: int = 4, ncopy: int = 2, device=None):
        t = _device.torch()
        self.dev = _device.require_cuda(device)
        self.cfg, self.mode, self.precision = cfg, mode, precision
        self.chunk = chunk or default_pipe_chunk(cfg)
        self.nbuf = max(2, nbuf)
        self.ncopy = max(1, min(ncopy, self.nbuf))
        cc = self.chunk
        self.ccfg = FnoLayerConfig(cc, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                                   cfg.keep_x, cfg.keep_y, cfg.rank)
        self.h2d = [t.cuda.Stream(self.dev) for _ in range(self.ncopy)]
        self.d2h = [t.cuda.Stream(self.dev) for _ in range(self.ncopy)]
        self.comp = t.cuda.Stream(self.dev)
        self.xb = [t.empty((cc, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), dtype=t.complex64, device=self.dev)
                   for _ in range(self.nbuf)]
        self.yb = [t.empty((cc, cfg.output_dim, cfg.dim_x, cfg.dim_y), dtype=t.complex64, device=self.dev)
                   for _ in range(self.nbuf)]
        self.ws = t.empty(max(workspace_bytes(self.ccfg, mode, precision), 1), dtype=t.uint8, device=self.dev)

    def __call__(self, x_host, w, out_host):
        """x_host [B,H,dx,dy] / out_host [B,N,dx,dy]: pinned complex64 CPU
        tensors; w: [H,N] complex64 (CPU or CUDA).  Returns out_host once
        the last D2H copy completed."""
        t = _device.torch()
        cfg = self.cfg
        cur = t.cuda.current_stream(self.dev)
        w_dev = w.to(self.dev, non_blocking=True).contiguous()
        ready = t.cuda.Event()
        ready.record(cur)
        for st in self.h2d + self.d2h + [self.comp]:
            st.wait_event(ready)
        c = cfg_struct(self.ccfg)
        mcode, pcode = MODE_CODES[self.mode], PREC_CODES[self.precision]
        nb_, comp_done, out_done = self.nbuf, [], []
        for i, b0 in enumerate(range(0, cfg.batch, self.chunk)):
            k = i % nb_
            nb = min(self.chunk, cfg.batch - b0)
            xb, yb = self.xb[k][:nb], self.yb[k][:nb]
            hs, ds = self.h2d[i % self.ncopy], self.d2h[i % self.ncopy]
            with t.cuda.stream(hs):
                if i >= nb_:
                    hs.wait_event(comp_done[i - nb_])
                xb.copy_(x_host[b0:b0 + nb], non_blocking=True)
                in_done = t.cuda.Event()
                in_done.record(hs)
            with t.cuda.stream(self.comp):
                self.comp.wait_event(in_done)
                if i >= nb_:
                    self.comp.wait_event(out_done[i - nb_])
                if nb == self.chunk:
                    cc = c
                else:
                    cc = cfg_struct(FnoLayerConfig(nb, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                                                   cfg.keep_x, cfg.keep_y, cfg.rank))
                rc = lib().tfno_layer_forward(ctypes.byref(cc), mcode, pcode, xb.data_ptr(), w_dev.data_ptr(),
                                              yb.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                              self.comp.cuda_stream)
                check(rc, "tfno_layer_forward")
                ev = t.cuda.Event()
                ev.record(self.comp)
                comp_done.append(ev)
            with t.cuda.stream(ds):
                ds.wait_event(comp_done[i])
                out_host[b0:b0 + nb].copy_(yb, non_blocking=True)
                ev = t.cuda.Event()
                ev.record(ds)
                out_done.append(ev)
        for st in self.d2h:
            cur.wait_stream(st)
        cur.synchronize()
        return out_host


def default_pipe_chunk(cfg: FnoLayerConfig) -> int:
    """Batch elements per HostPipeline chunk: up to 512 MiB of input + output."""
    per_b = 8 * cfg.dim_x * cfg.dim_y * (cfg.hidden_dim + cfg.output_dim)
    return max(1, min(cfg.batch, (512 << 20) // max(per_b, 1)))


def run_layer_host(cfg: FnoLayerConfig, x_host, w, out_host=None, mode: str = "fully_fused",
                   precision: str = "fp32", tiles: TileConfig = DEFAULT_TILES,
                   fft_batch_size: int = FFT_BLOCK_BATCH):
    """Host-buffer API: pinned CPU tensors in/out, copies overlapped with
    compute (see HostPipeline)."""
    t = _device.torch()
    _validate(cfg, tuple(x_host.shape), tuple(w.shape), tiles, mode, fft_batch_size)
    if out_host is None:
        out_host = t.empty((cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y), dtype=t.complex64,
                           pin_memory=True)
    return HostPipeline(cfg, mode, precision)(x_host, w, out_host)
