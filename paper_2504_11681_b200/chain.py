"""Chains of Fourier layers (BASELINE configs[4]: 4-layer 2D FNO forward,
Navier-Stokes shape) — SURVEY.md §8f "next" row 1.

The reference has no multi-layer model; its semantics are chained
``run_layer`` calls with independent weights and no activation in between
(SURVEY.md §7 step 9), which is exactly what ``FnoChain`` computes: every
layer runs in full (forward 2D FFT, channel mix, padded inverse) — the chain
is NOT collapsed algebraically even though, without activations, it could
be.  Layers ping-pong between two device buffers; the whole chain can be
captured once into a CUDA graph (``capture()``) so a forward is a single
graph launch (12 kernels for 4 rank-2 layers).
"""

from __future__ import annotations

from . import _device
from .core import FnoLayerConfig, FnofuseError
from .pipeline import run_layer_device, workspace_bytes


class FnoChain:
    def __init__(self, cfg: FnoLayerConfig, weights, mode: str = "fully_fused", precision: str = "fp32"):
        """cfg: one layer's shape (hidden_dim == output_dim for depth > 1);
        weights: list of [H, N] complex64 CUDA tensors, one per layer."""
        if len(weights) > 1 and cfg.hidden_dim != cfg.output_dim:
            raise FnofuseError("a chain needs hidden_dim == output_dim")
        t = _device.torch()
        self.cfg, self.mode, self.precision = cfg, mode, precision
        self.weights = [w.contiguous() for w in weights]
        dev = self.weights[0].device
        shape = (cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y)
        self.buf = [t.empty(shape, dtype=t.complex64, device=dev), t.empty(shape, dtype=t.complex64, device=dev)]
        # the chain owns its workspace: a captured graph keeps this pointer, independent of the
        # shared scratch other calls may regrow
        self.ws = t.empty(max(workspace_bytes(cfg, mode, precision), 1), dtype=t.uint8, device=dev)
        self.graph = None
        self._x = None

    def _run(self, x, stream=None):
        cur = x
        for i, w in enumerate(self.weights):
            out = self.buf[i % 2]
            run_layer_device(self.cfg, cur, w, mode=self.mode, precision=self.precision, out=out,
                             stream=stream, validate=(i == 0), workspace=self.ws)
            cur = out
        return cur

    def forward(self, x, stream=None):
        """Run the chain on x [B, H, dx, dy]; returns the last layer's output
        (a view of an internal buffer, valid until the next call)."""
        if self.graph is not None:
            if x.data_ptr() != self._x.data_ptr():
                self._x.copy_(x)
            self.graph.replay()
            return self._out
        return self._run(x, stream)

    def capture(self, x_static):
        """Capture the chain on the static input buffer into a CUDA graph."""
        t = _device.torch()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            self._run(x_static)  # warm-up outside the graph (kernel attributes, twiddles)
        t.cuda.current_stream().wait_stream(s)
        from ._lib import lib
        g = t.cuda.CUDAGraph()
        n0 = lib().tfno_launch_count()
        with t.cuda.graph(g):
            self._out = self._run(x_static)
        self.kernels_per_forward = int(lib().tfno_launch_count() - n0)  # kernels inside the graph
        self.graph, self._x = g, x_static
        return self
