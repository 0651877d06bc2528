"""Multi-GPU drivers: one process per GPU, ``torch.distributed`` for plumbing.

* ``BatchSharded`` — the forward shards naturally on the batch axis (FFT
  pencils are per (b, h), GEMM rows per (b, mode), iFFT pencils per (b, n);
  SURVEY.md §8e), so each rank runs the sm_100a layer on its own contiguous
  batch slice and there is NO collective on the data path.  Timing is the
  max over ranks.
* ``hidden_split_forward`` — optional hidden-dimension split (north_star):
  rank r owns input channels [h0, h1) of every batch element, computes the
  truncated spectrum of its channels and the partial channel mix
  C_r = sum_{h in shard} A[b,h] W[h,:], then the partials are summed over
  NVLink with NCCL (``all_reduce``: every rank gets all N output channels,
  or ``reduce_scatter``: rank r gets output channels [n0, n1)), and the
  padded inverse runs on the reduced modes.  The layer is linear in x, so
  the split is exact up to fp32 summation order.

The reference has no distributed code at all; these are new.
"""

from __future__ import annotations

import ctypes

from . import _device
from ._lib import cfg_struct, check, lib
from .core import FnoLayerConfig
from .pipeline import run_layer_device


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Balanced contiguous split of n items over world ranks: [start, stop)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def local_config(cfg: FnoLayerConfig, world: int, rank: int, axis: str = "batch") -> FnoLayerConfig:
    if axis == "batch":
        b0, b1 = shard_bounds(cfg.batch, world, rank)
        return FnoLayerConfig(b1 - b0, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                              cfg.keep_x, cfg.keep_y, cfg.rank)
    if axis == "hidden":
        h0, h1 = shard_bounds(cfg.hidden_dim, world, rank)
        return FnoLayerConfig(cfg.batch, h1 - h0, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                              cfg.keep_x, cfg.keep_y, cfg.rank)
    raise ValueError(axis)


class BatchSharded:
    """Batch-sharded Fourier layer for rank ``rank`` of ``world``."""

    def __init__(self, cfg: FnoLayerConfig, world: int, rank: int, mode: str = "fully_fused",
                 precision: str = "fp32"):
        self.cfg, self.world, self.rank = cfg, world, rank
        self.bounds = shard_bounds(cfg.batch, world, rank)
        self.local = local_config(cfg, world, rank, "batch")
        self.mode, self.precision = mode, precision

    def forward(self, x_local, w, out=None, stream=None):
        """x_local: this rank's [B_r, H, dx, dy] CUDA tensor; returns [B_r, N, dx, dy]."""
        return run_layer_device(self.local, x_local, w, mode=self.mode, precision=self.precision,
                                out=out, stream=stream)


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


# ---------------------------------------------------------------- hidden split
def _on(stream):
    """Run a helper with `stream` as torch's current stream, so every temporary
    is allocated on (and recycled against) the stream its kernels run on, and
    NCCL collectives issued inside are ordered after those kernels."""
    import contextlib
    t = _device.torch()
    return t.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def spectrum_forward(cfg: FnoLayerConfig, x, stream=None):
    """modes[B][H][kx][ky] (natural order) = first-keep DFT of every plane (GPU)."""
    t = _device.torch()
    c = cfg_struct(cfg)
    with _on(stream):
        modes = t.empty((cfg.batch, cfg.hidden_dim, cfg.keep_x, cfg.keep_y), dtype=t.complex64, device=x.device)
        nb = int(lib().tfno_spectrum_workspace_bytes(ctypes.byref(c), -1))
        ws = _device.workspace(nb, x.device, stream)  # cached per (device, stream): no per-call allocation
        check(lib().tfno_spectrum_forward(ctypes.byref(c), x.data_ptr(), modes.data_ptr(),
                                          ws.data_ptr() if ws is not None else None, nb,
                                          _device.stream_ptr(stream)), "tfno_spectrum_forward")
    return modes


def spectrum_inverse(cfg: FnoLayerConfig, modes, planes_shape, scale: float = 1.0, stream=None):
    """y[planes] = scale * zero-padded normalised inverse of natural-order modes (GPU)."""
    t = _device.torch()
    c = cfg_struct(cfg)
    with _on(stream):
        y = t.empty(tuple(planes_shape) + (cfg.dim_x, cfg.dim_y), dtype=t.complex64, device=modes.device)
        nb = int(lib().tfno_spectrum_workspace_bytes(ctypes.byref(c), 1))
        ws = _device.workspace(nb, modes.device, stream)
        check(lib().tfno_spectrum_inverse(ctypes.byref(c), modes.data_ptr(), y.data_ptr(), float(scale),
                                          ws.data_ptr() if ws is not None else None, nb,
                                          _device.stream_ptr(stream)), "tfno_spectrum_inverse")
    return y


def hidden_split_partial(cfg: FnoLayerConfig, x_shard, w_shard, channel_major: bool = False, stream=None):
    """This rank's partial modes C_r[b, n] = sum_{h in shard} A[b, h] W[h, n].

    x_shard [B, H_r, dx, dy], w_shard [H_r, N] (CUDA).  Returns [B, N, kx, ky]
    (or [N, B, kx, ky] when ``channel_major`` — contiguous per output-channel
    block, the layout reduce_scatter needs)."""
    t = _device.torch()
    lc = FnoLayerConfig(cfg.batch, x_shard.shape[1], cfg.output_dim, cfg.dim_x, cfg.dim_y,
                        cfg.keep_x, cfg.keep_y, cfg.rank)
    with _on(stream):
        A = spectrum_forward(lc, x_shard, stream)
        B, Hr, N = cfg.batch, x_shard.shape[1], cfg.output_dim
        MQ = cfg.keep_x * cfg.keep_y
        w = w_shard.contiguous()
        if channel_major:
            C = t.empty((N, B, cfg.keep_x, cfg.keep_y), dtype=t.complex64, device=x_shard.device)
            c_ns, c_bs = B * MQ, MQ
        else:
            C = t.empty((B, N, cfg.keep_x, cfg.keep_y), dtype=t.complex64, device=x_shard.device)
            c_ns, c_bs = MQ, N * MQ
        rc = lib().tfno_cgemm(MQ, N, Hr, B, A.data_ptr(), 1, MQ, Hr * MQ, w.data_ptr(), N, 1, 0,
                              C.data_ptr(), 1, c_ns, c_bs, 1.0, _device.stream_ptr(stream))
        check(rc, "tfno_cgemm")
    return C


def reduce_partials(C, how: str = "all_reduce", group=None):
    """Sum the ranks' partial modes: all_reduce (full C everywhere) or
    reduce_scatter along dim 0 (rank r keeps block r).  Device-agnostic:
    NCCL for CUDA tensors over NVLink, gloo for CPU tensors (tests)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if how == "all_reduce":
        dist.all_reduce(torch.view_as_real(C), op=dist.ReduceOp.SUM, group=group)
        return C
    if how == "reduce_scatter":
        n = C.shape[0]
        if n % world:
            raise ValueError(f"reduce_scatter needs dim 0 ({n}) divisible by world ({world})")
        out = torch.empty((n // world,) + tuple(C.shape[1:]), dtype=C.dtype, device=C.device)
        if C.is_cuda:
            dist.reduce_scatter_tensor(torch.view_as_real(out), torch.view_as_real(C.contiguous()),
                                       op=dist.ReduceOp.SUM, group=group)
        else:  # gloo has no reduce_scatter: all_reduce then keep this rank's block
            dist.all_reduce(torch.view_as_real(C), op=dist.ReduceOp.SUM, group=group)
            rank = dist.get_rank(group)
            out.copy_(C[rank * (n // world):(rank + 1) * (n // world)])
        return out
    raise ValueError(how)


def hidden_split_forward(cfg: FnoLayerConfig, x_shard, w_shard, how: str = "all_reduce", group=None,
                         stream=None):
    """Full hidden-split layer on this rank (see module doc).  Returns
    y [B, N, dx, dy] (all_reduce) or this rank's channel block
    [N/world, B, dx, dy] (reduce_scatter, channel-major)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    cm = how == "reduce_scatter"
    # one stream for partial -> NCCL reduce -> inverse: the collective (enqueued
    # on torch's current stream) is ordered after the partial CGEMM
    with _on(stream):
        C = hidden_split_partial(cfg, x_shard, w_shard, channel_major=cm, stream=stream)
        C = reduce_partials(C, how, group)
        if cm:
            nr = cfg.output_dim // world
            pc = FnoLayerConfig(1, 1, nr * cfg.batch, cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y, cfg.rank)
            return spectrum_inverse(pc, C, (nr, cfg.batch), 1.0, stream)
        oc = FnoLayerConfig(cfg.batch, 1, cfg.output_dim, cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y, cfg.rank)
        return spectrum_inverse(oc, C, (cfg.batch, cfg.output_dim), 1.0, stream)
