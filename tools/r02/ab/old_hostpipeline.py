# round-1 HostPipeline (per-stream H2D -> layer -> D2H), kept only for the e2e A/B in tools/r02/r2_e2e.sh
import ctypes
from paper_2504_11681_b200 import _device
from paper_2504_11681_b200.core import FnoLayerConfig
from paper_2504_11681_b200.pipeline import workspace_bytes, cfg_struct, MODE_CODES, PREC_CODES, lib, check

class HostPipeline:
    """End-to-end host-buffer execution: the batch is split into chunks that
    flow H2D -> layer -> D2H on ``nstreams`` CUDA streams, so PCIe copies in
    both directions overlap the sm_100a kernels of other chunks.  Inputs and
    outputs are pinned host tensors; device chunk buffers are allocated once
    and reused."""

    def __init__(self, cfg: FnoLayerConfig, mode: str = "fully_fused", precision: str = "fp32",
                 chunk: int | None = None, nstreams: int = 3, device=None):
        t = _device.torch()
        self.dev = _device.require_cuda(device)
        self.cfg, self.mode, self.precision = cfg, mode, precision
        per_b = 8 * cfg.dim_x * cfg.dim_y * (cfg.hidden_dim + cfg.output_dim)
        self.chunk = chunk or max(1, min(cfg.batch, (2 << 30) // max(per_b, 1)))
        self.nstreams = nstreams
        cc = self.chunk
        self.ccfg = FnoLayerConfig(cc, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                                   cfg.keep_x, cfg.keep_y, cfg.rank)
        self.streams = [t.cuda.Stream(self.dev) for _ in range(nstreams)]
        self.xb = [t.empty((cc, cfg.hidden_dim, cfg.dim_x, cfg.dim_y), dtype=t.complex64, device=self.dev)
                   for _ in range(nstreams)]
        self.yb = [t.empty((cc, cfg.output_dim, cfg.dim_x, cfg.dim_y), dtype=t.complex64, device=self.dev)
                   for _ in range(nstreams)]
        self.ws = []
        for _ in range(nstreams):
            nb = workspace_bytes(self.ccfg, mode, precision)
            self.ws.append(t.empty(max(nb, 1), dtype=t.uint8, device=self.dev))
        self.done = [None] * nstreams

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
        c = cfg_struct(self.ccfg)
        mcode, pcode = MODE_CODES[self.mode], PREC_CODES[self.precision]
        for i, b0 in enumerate(range(0, cfg.batch, self.chunk)):
            s = i % self.nstreams
            st = self.streams[s]
            nb = min(self.chunk, cfg.batch - b0)
            with t.cuda.stream(st):
                st.wait_event(ready)
                xb, yb = self.xb[s][:nb], self.yb[s][:nb]
                xb.copy_(x_host[b0:b0 + nb], non_blocking=True)
                if nb == self.chunk:
                    cc, ccfg = c, self.ccfg
                else:
                    ccfg = FnoLayerConfig(nb, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y,
                                          cfg.keep_x, cfg.keep_y, cfg.rank)
                    cc = cfg_struct(ccfg)
                ws = self.ws[s]
                rc = lib().tfno_layer_forward(ctypes.byref(cc), mcode, pcode, xb.data_ptr(), w_dev.data_ptr(),
                                              yb.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)
                check(rc, "tfno_layer_forward")
                out_host[b0:b0 + nb].copy_(yb, non_blocking=True)
        for st in self.streams:
            cur.wait_stream(st)
        cur.synchronize()
        return out_host


