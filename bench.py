#!/usr/bin/env python
"""Benchmark of the B200-native TurboFNO Fourier layer (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A "step" is one Fourier-layer forward (BASELINE.json's metric: fused-layer
GFLOP/s and us/layer vs cuFFT+cuBLAS, % of roofline) over one batch of
synthetic N(0,1) complex64 input already resident in HBM.  Default workload
is C4 (2D b128 512x512 H128->128 modes 64x64), the largest single-GPU config
of BASELINE.json; each rank processes its own batch of 128 (batch-sharded,
no collective on the data path, weak scaling; ``--scaling strong`` splits a
global batch of 128 instead).  Inputs are 32 GiB per GPU (> 126 MB L2), so
no L2 flush is needed between steps.

--impl reference times the reference algorithm on the host CPU (the numpy
oracle port of fnofuse, all host cores, batch-sharded process pool) on a
bounded sample of the same workload; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused Fourier-layer GFLOP/s and µs/layer vs cuFFT+cuBLAS, % of roofline"
WORKLOADS = {
    # name: (batch, hidden, out, dim_x, dim_y, keep_x, keep_y, rank, description)
    "C1": (16, 64, 64, 1, 128, 1, 32, 1, "C1: 1D FNO layer b16 N128 H64->64 modes 32"),
    "C3": (32, 64, 64, 256, 256, 32, 32, 2, "C3: 2D FNO layer b32 256x256 H64->64 modes 32x32"),
    "C4": (128, 128, 128, 512, 512, 64, 64, 2, "C4: 2D FNO layer b128 512x512 H128->128 modes 64x64"),
    "C5L": (256, 64, 64, 256, 256, 16, 16, 2, "C5 single layer: 2D b256 256x256 W64 modes 16x16"),
    "C5": (256, 64, 64, 256, 256, 16, 16, 2, "C5: 4-layer 2D FNO forward b256 256x256 W64 modes 16x16 "
                                             "(one CUDA graph, 12 kernels)"),
}
LAYERS = {"C5": 4}
for _n in (256, 1024, 4096):
    for _h in (64, 128, 256):
        for _b in (64, 256, 1024):
            WORKLOADS[f"C2-N{_n}-H{_h}-B{_b}"] = (_b, _h, _h, 1, _n, 1, _n // 8, 1,
                                                  f"C2 point: 1D b{_b} N{_n} H{_h}->{_h} modes {_n // 8}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured", p
    except Exception:
        return 6650.0, "fallback", {}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        self.th.join(1)
        sm, smax, pw, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "sm_mhz_min": min(sm) if sm else None, "power_w_max": max(pw) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def stage_algorithmic_bytes(cfg, desc):
    """Bytes each stage of the schedule must move (read + write, complex64)."""
    B, H, N = cfg.batch, cfg.hidden_dim, cfg.output_dim
    dx, dy, kx, ky = cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y
    E = 8
    t = {
        "x-fft": B * H * dx * dy + B * H * kx * dy,
        "y-fft": B * H * kx * dy + B * H * kx * ky,
        "fused-fft-cgemm-ifft": B * H * kx * dy + B * N * kx * dy + H * N,
        "fused1d-fft-cgemm-ifft": B * H * kx * dy + B * N * kx * dy + H * N,
        "tiny1d-fft-cgemm-ifft": B * H * kx * dy + B * N * kx * dy + H * N,
        "fused-fft-cgemm": B * H * kx * dy + B * N * kx * ky + H * N,
        "fused-cgemm-ifft": B * H * kx * ky + B * N * kx * dy + H * N,
        "cgemm": B * H * kx * ky + B * N * kx * ky + H * N,
        "cgemm-modes": B * H * kx * ky + B * N * kx * ky + H * N,
        "y-ifft": B * N * kx * ky + B * N * kx * dy,
        "x-ifft": B * N * kx * dy + B * N * dx * dy,
        "plane-fft2d": B * H * dx * dy + B * H * kx * ky,
        "plane-ifft2d": B * N * kx * ky + B * N * dx * dy,
        # channel mix fused into the inverse: A in, W, y out (C stays in the L2 ring)
        "plane-mix-ifft2d": B * H * kx * ky + H * N + B * N * dx * dy,
    }
    return [(name, E * t.get(name, 0)) for name in desc.split("|")]


def load_traffic(workload, kernel):
    """ncu dram bytes per launch (profiles/traffic.json, from `ncu --set full`)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


def load_n3(workload):
    """N3 evidence: ncu launch counts and DRAM bytes of our fully_fused layer and of the
    staged cuFFT+cuBLAS pipeline, captured in one process (tools/n3_traffic.py; the newest
    profiles/rNN/n3_traffic.json).  A committed capture, labelled as such."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "n3_traffic.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as f:
            d = json.load(f).get(workload)
    except Exception:
        return None
    if d:
        d = dict(d, source=os.path.relpath(files[-1], ROOT) + " (ncu, committed capture, not this run)")
    return d


REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # pip --target install of the unmodified reference


def workload_config(args, B, ws):
    """The `config` object of the JSON line: identical in both arms (no product import)."""
    _, H, N, dx, dy, kx, ky, rk, desc = WORKLOADS[args.workload]
    io = 8 * B * H * dx * dy
    return {"workload": desc, "batch_per_gpu": B, "global_batch": B * ws, "hidden": H, "out": N,
            "dims": [dx, dy], "keep": [kx, ky], "rank": rk, "mode": args.mode, "precision": args.precision,
            "parallelism": f"batch-sharded dp{ws}, no data-path collective",
            "l2": (f"inputs larger than L2 ({io / 2**30:.1f} GiB per GPU); no flush" if io > (126 << 20) else
                   f"inputs ({io / 2**20:.1f} MiB) fit in L2: L2-warm timing")}


def reference_layer_flops(F, cfg):
    """Canonical flops of one layer from the REFERENCE's own op statistics
    (fnofuse.pipeline.layer_op_stats, pipeline.py:369-416) + the CGEMM term
    (SURVEY.md §8d): 2*op_budget + 6*twiddle_muls + 8*B*kx*ky*H*N."""
    st = F.layer_op_stats(cfg, "fully_fused")
    return (2 * st["fft_op_budget"] + 6 * st["fft_twiddle_muls"]
            + 8 * cfg.batch * cfg.keep_x * cfg.keep_y * cfg.hidden_dim * cfg.output_dim)


# ---- CPU reference workers (one process per host core, single-threaded BLAS) ----
_RW = None


def _ref_import(kind):
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import fnofuse
        return fnofuse
    from oracle import fnofuse_port
    return fnofuse_port


def _ref_init(kind, cfg1, seed):
    """Worker initializer: import the CPU implementation, draw this worker's
    batch element (random_spectral / ComplexMatrix.random, core.py:239-244)."""
    global _RW
    F = _ref_import(kind)
    import numpy as np_
    if kind == "reference":
        cfg = F.FnoLayerConfig(**cfg1)
        rng = np_.random.default_rng(seed + os.getpid())
        x = F.random_spectral(cfg, rng) if seed >= 0 else None
        w = F.ComplexMatrix.random(cfg.hidden_dim, cfg.output_dim, rng) if seed >= 0 else None
    else:
        from types import SimpleNamespace
        cfg = SimpleNamespace(**cfg1)
        x, w = F.random_inputs(cfg, seed + os.getpid()) if seed >= 0 else (None, None)
    _RW = (kind, F, cfg, x, w)


def _ref_step(_i):
    """One batch element of the workload through the CPU implementation's public API."""
    kind, F, cfg, x, w = _RW
    if kind == "reference":
        y, _led = F.run_layer(cfg, x, w, mode="fully_fused")
        return float(np.abs(y.data[0, 0, 0, 0]))
    return float(np.abs(F.run_layer_values(cfg, x, w)[0, 0, 0, 0]))


def _ref_run(args):
    """Run given inputs (parity leg): returns the CPU output values."""
    x, w = args
    kind, F, cfg, _, _ = _RW
    if kind == "reference":
        y, _led = F.run_layer(cfg, F.SpectralTensor(x), F.ComplexMatrix(w), mode="fully_fused")
        return np.asarray(y.data)
    return F.run_layer_values(cfg, x, w)


class RefPool:
    """Batch-sharded CPU execution of the reference's fused layer: `workers`
    processes (spawned; OPENBLAS_NUM_THREADS=1), one batch element each per
    step.  kind "reference" = the unmodified fnofuse from baseline/_ref through
    its public run_layer (pipeline.py:129); "port" = the numpy oracle port
    (bitwise equal, used only when the install is absent)."""

    def __init__(self, cfg_t, workers, seed=-1):
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        self.kind = "reference" if os.path.isdir(os.path.join(REF_DIR, "fnofuse")) else "port"
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = "1"
        self.workers = workers
        cfg1 = dict(cfg_t, batch=1)
        self.ex = ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn"), initializer=_ref_init,
                                      initargs=(self.kind, cfg1, seed))
        self.F = _ref_import(self.kind)
        self.cfg1 = cfg1

    def step(self):
        return list(self.ex.map(_ref_step, range(self.workers)))

    def run(self, xs, w):
        return np.concatenate([y for y in self.ex.map(_ref_run, [(xs[i:i + 1], w) for i in range(len(xs))])],
                              axis=0)

    def flops(self, batch):
        if self.kind == "reference":
            cfg = self.F.FnoLayerConfig(**dict(self.cfg1, batch=batch))
            return reference_layer_flops(self.F, cfg)
        from types import SimpleNamespace

        from oracle import fnofuse_port as O
        return O.layer_flops(SimpleNamespace(**dict(self.cfg1, batch=batch)))

    def close(self):
        self.ex.shutdown()


def run_reference_arm(args):
    """--impl reference: the reference's own CPU path (fnofuse.run_layer from
    baseline/_ref, all host cores, one batch element per process per step) on
    the same workload/config as our arm.  Never imports the product package."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    B, H, N, dx, dy, kx, ky, rk, desc = WORKLOADS[args.workload]
    Bl = B // ws if args.scaling == "strong" else B
    workers = max(1, min(Bl, len(os.sched_getaffinity(0))))
    cfg_t = dict(batch=1, hidden_dim=H, output_dim=N, dim_x=dx, dim_y=dy, keep_x=kx, keep_y=ky, rank=rk)
    pool = RefPool(cfg_t, workers, seed=1234)
    nl = LAYERS.get(args.workload, 1)
    flops = pool.flops(workers) * nl
    for _ in range(args.warmup):
        for _l in range(nl):
            pool.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _l in range(nl):
            pool.step()
    dt = (time.perf_counter() - t0) / args.steps
    kind = pool.kind
    pool.close()
    val = flops / dt / 1e9
    src = ("unmodified fnofuse 0.1.0 (baseline/_ref) fnofuse.run_layer(mode='fully_fused')" if kind == "reference"
           else "numpy oracle port of fnofuse (baseline/_ref absent; bitwise equal to the reference)")
    sample = (f"{workers} of the {Bl} batch elements of {args.workload} per step x {nl} layer(s), all {H}->{N} "
              f"channels, 1 batch element per worker process ({workers} processes, OPENBLAS_NUM_THREADS=1): {src}")
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak" if args.scaling == "weak" else "strong",
            "vs_baseline": None, "dtype": "fp32 (complex64 in/out, fp32 arithmetic)",
            "data": "synthetic (seeded N(0,1) re/im, reference random_spectral)",
            "config": workload_config(args, Bl, ws),
            "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": workers, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def time_steps(fn, steps, warmup, stream, barrier):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    barrier()
    return s.elapsed_time(e) / steps


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_11681_b200 as T
    from paper_2504_11681_b200 import _lib
    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.device(f"cuda:{torch.cuda.current_device()}")

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(v):
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    B, H, N, dx, dy, kx, ky, rk, desc = WORKLOADS[args.workload]
    if args.scaling == "strong":
        if B % ws:
            raise SystemExit(f"global batch {B} not divisible by {ws} ranks")
        B = B // ws
    cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rk)
    mode, prec = args.mode, args.precision
    nlaunch, sched = T.layer_schedule(cfg, mode, prec)
    g = torch.Generator(device=dev)
    g.manual_seed(4000 + rank)
    xr = torch.randn((B, H, dx, dy, 2), generator=g, device=dev, dtype=torch.float32)
    x = torch.view_as_complex(xr)
    del xr
    wr = torch.randn((H, N, 2), generator=g, device=dev, dtype=torch.float32)
    w = torch.view_as_complex(wr).contiguous()
    y = torch.empty((B, N, dx, dy), dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream()
    lib = _lib.lib()

    def step():
        T.run_layer_device(cfg, x, w, out=y, mode=mode, precision=prec, validate=False)

    nlayers = LAYERS.get(args.workload, 1)
    chain = None
    io_bytes = 8 * B * (H + N) * dx * dy
    # auto: chains, and layers whose step is short enough (<= 4 GiB of I/O, < ~1 ms) that the
    # eager launch + stage-event gaps show (C3 0.443 -> 0.425 ms, profiles/r02/c3_graph_pdl.txt)
    use_graph = nlayers > 1 or args.graph == "on" or (args.graph == "auto" and io_bytes <= (4 << 30))
    if use_graph:  # launch-latency-bound workloads (and chains) replay one CUDA graph per step
        from paper_2504_11681_b200.chain import FnoChain
        ws_ = [w] + [torch.view_as_complex(torch.randn((H, N, 2), generator=g, device=dev,
                                                        dtype=torch.float32)).contiguous()
                     for _ in range(nlayers - 1)]
        chain = FnoChain(cfg, ws_, mode=mode, precision=prec).capture(x)

    # ---- stage events inside the timed region (dominant-kernel roofline) ----
    nst = len(sched.split("|")) + 1
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst)] for _ in range(args.steps)]
    for row in ev:  # torch creates the cudaEvent_t lazily: force creation before handing it over
        for e_ in row:
            e_.record(stream)
    handles = [(ctypes_arr(e)) for e in ev]
    cur = [0]

    def step_timed():
        h = handles[cur[0]]
        lib.tfno_set_stage_events(h, nst)
        step()
        cur[0] += 1

    if chain is not None:
        # per-kernel events of one layer (graph replays carry no events), then the
        # graph-launched chain is the timed step
        for _ in range(args.warmup):
            step()
        for i in range(args.steps):
            step_timed()
        torch.cuda.synchronize()
        lib.tfno_set_stage_events(None, 0)
        layer_stage_ms = [statistics.mean(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(args.steps))
                          for j in range(nst - 1)]

        def step_timed():  # noqa: F811
            chain.forward(x)

    for _ in range(args.warmup):
        step() if chain is None else chain.forward(x)
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local])
                          if os.environ.get("CUDA_VISIBLE_DEVICES") else local)
    clocks.start()
    time.sleep(0.3)
    n0 = lib.tfno_launch_count()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        step_timed()
    e0.record(stream)
    torch.cuda.synchronize()
    launches = lib.tfno_launch_count() - n0
    if chain is not None:  # graph replays: the kernels were recorded once at capture
        launches = args.steps * chain.kernels_per_forward
    lib.tfno_set_stage_events(None, 0)
    clk = clocks.stop()
    barrier()
    ms_local = s0.elapsed_time(e0) / args.steps
    ms = max_over_ranks(ms_local)
    # per-stage average durations
    names = sched.split("|")
    if chain is None:
        stage_ms = [statistics.mean(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(args.steps))
                    for j in range(len(names))]
    else:
        stage_ms = layer_stage_ms
    fl = T.layer_flops(cfg, mode)
    fl = {k: v * nlayers for k, v in fl.items()} if nlayers > 1 else fl
    total_flops = fl["flops"] * ws
    value = total_flops / (ms * 1e-3) / 1e9
    hbm_peak, peak_kind, pk = peaks()
    sbytes = stage_algorithmic_bytes(cfg, sched)
    dom = max(range(len(names)), key=lambda j: stage_ms[j])
    achieved = sbytes[dom][1] / (stage_ms[dom] * 1e-3) / 1e9
    traffic = load_traffic(args.workload, names[dom])
    layer_bytes = fl["bytes"]
    t_mem_8 = layer_bytes / 8.0e12
    t_cmp = fl["flops"] / 74.4e12
    t_roof = max(t_mem_8, t_cmp)

    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "us_per_layer": round(ms * 1e3, 2),
        "layers_per_s": round(ws * nlayers * 1e3 / ms, 2), "higher_is_better": True,
        "scaling": "weak" if args.scaling == "weak" else "strong", "vs_baseline": None,
        "dtype": ("fp32 (complex64 in/out, fp32 arithmetic)" if prec == "fp32" else
                  f"fp32 FFTs + {prec} tcgen05 channel contraction (complex64 in/out)"),
        "data": "synthetic (device-generated N(0,1) re/im, seeded per rank)",
        "config": workload_config(args, B, ws),
        "schedule": sched, "launch": "one CUDA graph replay per step" if chain is not None else "eager launches",
        "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                     "traffic_source": ("committed ncu --set full capture (profiles/traffic.json), not measured in this run"
                                        if traffic is not None else None),
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": sbytes[dom][1],
                     "launch_ms": round(stage_ms[dom], 4),
                     "share_of_step": round(stage_ms[dom] / sum(stage_ms), 4) if sum(stage_ms) else None},
        "stages": [{"kernel": n, "ms": round(t, 4), "algorithmic_bytes": b,
                    "GBps": round(b / (t * 1e-3) / 1e9, 1) if t > 0 else None}
                   for n, t, (_, b) in zip(names, stage_ms, sbytes)],
        "layer_roofline": {"bytes": layer_bytes, "fft_flops": fl["fft_flops"], "cgemm_flops": fl["cgemm_flops"],
                           "T_roof_us": round(t_roof * 1e6, 1),
                           "frac_of_roof_8TBps_74TF": round(t_roof / (ms * 1e-3), 4),
                           "frac_of_measured_hbm": round(layer_bytes / (ms * 1e-3) / 1e9 / hbm_peak, 4),
                           "achieved_GBps": round(layer_bytes / (ms * 1e-3) / 1e9, 1)},
        "gpu_launches": int(launches), "launches_per_layer": nlaunch, "layers_per_step": nlayers, "clocks": clk,
    }

    # ---- unfused baselines measured in the same run (rank-local, max over ranks) ----
    if not args.no_baselines:
        base = {}
        y2 = torch.empty_like(y)

        def staged():
            for _ in range(nlayers):  # same depth as the timed step
                T.run_layer_device(cfg, x, w, out=y2, mode="staged", validate=False)

        def graphed(fn):  # baselines replayed as CUDA graphs too when our step is a graph
            if chain is None:
                return fn
            fn()
            torch.cuda.synchronize()
            gs = torch.cuda.Stream()
            gs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(gs):
                fn()
            torch.cuda.current_stream().wait_stream(gs)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            return gr.replay
        base["launch"] = "CUDA-graph replays" if chain is not None else "eager"
        try:
            ms_st = max_over_ranks(time_steps(graphed(staged), max(3, args.steps // 2), 2, stream, barrier))
            base["cufft_cublas_staged"] = {"ms": round(ms_st, 4),
                                           "GFLOPps": round(fl["flops"] * ws / (ms_st * 1e-3) / 1e9, 2)}
        except Exception as ex:  # noqa: BLE001
            base["cufft_cublas_staged"] = {"error": str(ex)[:200]}
        T._device.release_workspace()
        try:
            ms_tf = max_over_ranks(time_steps(graphed(lambda: [torch_fft_layer(cfg, x, w, y2) for _ in range(nlayers)]),
                                              max(3, args.steps // 2), 2, stream, barrier))
            base["torch_fft_matmul"] = {"ms": round(ms_tf, 4),
                                        "GFLOPps": round(fl["flops"] * ws / (ms_tf * 1e-3) / 1e9, 2)}
        except Exception as ex:  # noqa: BLE001
            base["torch_fft_matmul"] = {"error": str(ex)[:200]}
        best = min((v["ms"] for v in base.values() if isinstance(v, dict) and "ms" in v), default=None)
        if best:
            base["speedup_vs_best_unfused"] = round(best / ms, 3)
        n3 = load_n3(args.workload if args.workload != "C5" else "C5L")
        if n3:
            base["ncu_launch_and_dram_reduction"] = n3
        result["baselines"] = base
        del y2
        torch.cuda.empty_cache()

    # ---- tensor-core contraction variants of the same layer (reported, not the headline) ----
    if not args.no_baselines and prec == "fp32" and args.mode == "fully_fused":
        var = {}
        for vp in ("tf32x3", "tf32", "bf16"):
            try:
                ms_v = max_over_ranks(time_steps(
                    lambda vp=vp: [T.run_layer_device(cfg, x, w, out=y, mode=mode, precision=vp, validate=False)
                                   for _ in range(nlayers)],
                    max(3, args.steps // 2), 2, stream, barrier))
                var[vp] = {"ms": round(ms_v, 4), "GFLOPps": round(fl["flops"] * ws / (ms_v * 1e-3) / 1e9, 2),
                           "tolerance": {"tf32x3": 1e-5, "tf32": 1e-3, "bf16": 5e-3}[vp]}
            except Exception as ex:  # noqa: BLE001
                var[vp] = {"error": str(ex)[:200]}
        T.run_layer_device(cfg, x, w, out=y, mode=mode, precision=prec, validate=False)  # restore FP32 output
        if chain is not None:
            for v in var.values():
                v["note"] = f"{nlayers} layers launched eagerly (no graph)"
        result["precision_variants"] = var

    # ---- end to end through the public host-buffer API ----
    if not args.no_e2e and chain is not None:
        try:
            xh = torch.empty(x.shape, dtype=torch.complex64, pin_memory=True)
            xh.copy_(x)
            yh = torch.empty(y.shape, dtype=torch.complex64, pin_memory=True)
            xs_dev = torch.empty_like(x)
            for _ in range(1):
                xs_dev.copy_(xh, non_blocking=True)
                yh.copy_(chain.forward(xs_dev), non_blocking=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(max(1, args.e2e_steps)):
                xs_dev.copy_(xh, non_blocking=True)
                yh.copy_(chain.forward(xs_dev), non_blocking=True)
            torch.cuda.synchronize()
            ms_e = max_over_ranks((time.perf_counter() - t0) * 1e3 / max(1, args.e2e_steps))
            result["e2e"] = {"value": round(fl["flops"] * ws / (ms_e * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                             "h2d_bytes_per_step": int(xh.numel() * 8), "d2h_bytes_per_step": int(yh.numel() * 8),
                             "steps": max(1, args.e2e_steps), "ms_per_step": round(ms_e, 2),
                             "api": "pinned H2D -> FnoChain.forward (CUDA graph) -> pinned D2H"}
            del xh, yh, xs_dev
        except Exception as ex:  # noqa: BLE001
            result["e2e"] = {"error": str(ex)[:300]}
    elif not args.no_e2e:
        try:
            e2e = run_e2e(T, cfg, x, w, mode, prec, args, barrier, max_over_ranks, stream)
            fe = T.layer_flops(T.FnoLayerConfig(e2e["batch_per_rank"], H, N, dx, dy, kx, ky, rk), mode)["flops"]
            e2e["value"] = round(fe * ws / (e2e.pop("ms") * 1e-3) / 1e9, 2)
            result["e2e"] = e2e
        except Exception as ex:  # noqa: BLE001
            result["e2e"] = {"error": str(ex)[:300]}

    # ---- parity + CPU baseline (rank 0, N=1 only) ----
    if rank == 0 and ws == 1 and not args.no_cpu:
        workers = len(os.sched_getaffinity(0))
        sb = max(1, min(B, workers))
        xs = x[:sb].cpu().numpy()
        cfg_t = dict(batch=1, hidden_dim=H, output_dim=N, dim_x=dx, dim_y=dy, keep_x=kx, keep_y=ky, rank=rk)
        pool = RefPool(cfg_t, sb)
        if chain is None:
            wh = w.cpu().numpy()
            ys = y[:sb].cpu().numpy()
            t0 = time.perf_counter()
            ref = pool.run(xs, wh)
            dt = time.perf_counter() - t0
        else:
            ys = chain.forward(x)[:sb].cpu().numpy()
            dt, ref = 0.0, xs
            for wl in chain.weights:
                t0 = time.perf_counter()
                ref = pool.run(ref, wl.cpu().numpy())
                dt += time.perf_counter() - t0
        sflops = pool.flops(sb) * nlayers
        kind = pool.kind
        pool.close()
        src = ("unmodified fnofuse.run_layer from baseline/_ref" if kind == "reference"
               else "numpy oracle port of fnofuse run_layer")
        result["cpu_baseline"] = {"value": round(sflops / dt / 1e9, 4), "unit": "GFLOP/s", "cores": sb,
                                  "kind": kind,
                                  "sample": f"first {sb} batch elements of the timed input, 1 per worker process "
                                            f"({dt:.1f} s wall incl. input pickling), {src}"}
        result["max_rel_error"] = float(T.max_rel_error(ys, ref))
        result["parity_sample"] = f"batch[0:{sb}] vs the CPU {kind} ({src}); FP32 tolerance 1e-5"

    if rank == 0:
        print(json.dumps(result), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def ctypes_arr(events):
    import ctypes
    arr = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
    return arr


def torch_fft_layer(cfg, x, w, out, chunk=16):
    """B2 baseline: torch.fft (cuFFT) + slicing + matmul (cuBLAS) + padded inverse, chunked over batch."""
    import torch
    kx, ky = cfg.keep_x, cfg.keep_y
    for b0 in range(0, cfg.batch, chunk):
        xb = x[b0:b0 + chunk]
        if cfg.rank == 2:
            s = torch.fft.fft2(xb)[:, :, :kx, :ky]
        else:
            s = torch.fft.fft(xb, dim=-1)[..., :ky]
        c = torch.einsum("bhxy,hn->bnxy", s, w)
        if cfg.rank == 2:
            out[b0:b0 + chunk] = torch.fft.ifft2(c, s=(cfg.dim_x, cfg.dim_y))
        else:
            out[b0:b0 + chunk] = torch.fft.ifft(c, n=cfg.dim_y, dim=-1)


def e2e_batch(cfg, ws):
    """Per-rank batch for the pinned-host e2e leg: all of it unless the ranks
    of this host would pin more than ~60% of host RAM (8 x 64 GiB for C4)."""
    per_b = 8 * cfg.dim_x * cfg.dim_y * (cfg.hidden_dim + cfg.output_dim)
    try:
        import psutil
        total = psutil.virtual_memory().total
    except Exception:  # noqa: BLE001
        total = 256 << 30
    cap = int(0.6 * total / max(1, ws) / per_b)
    return max(1, min(cfg.batch, cap))


def run_e2e(T, cfg, x, w, mode, prec, args, barrier, max_over_ranks, stream):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    eb = e2e_batch(cfg, ws)
    if eb < cfg.batch:
        cfg = T.FnoLayerConfig(eb, cfg.hidden_dim, cfg.output_dim, cfg.dim_x, cfg.dim_y, cfg.keep_x, cfg.keep_y,
                               cfg.rank)
        x = x[:eb]
    xh = torch.empty(x.shape, dtype=torch.complex64, pin_memory=True)
    xh.copy_(x)
    yh = torch.empty((cfg.batch, cfg.output_dim, cfg.dim_x, cfg.dim_y), dtype=torch.complex64, pin_memory=True)
    wh = w.cpu()
    pipe = T.pipeline.HostPipeline(cfg, mode, prec)
    steps = max(1, args.e2e_steps)
    for _ in range(1):
        pipe(xh, wh, yh)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        pipe(xh, wh, yh)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    ms = max_over_ranks(ms)
    barrier()
    bi = xh.numel() * 8 + wh.numel() * 8
    bo = yh.numel() * 8
    del xh, yh, pipe
    torch.cuda.empty_cache()
    return {"ms": ms, "unit": "GFLOP/s", "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(bo),
            "batch_per_rank": cfg.batch,
            "steps": steps, "api": "paper_2504_11681_b200.pipeline.HostPipeline (pinned host in/out, "
                                   f"chunk {pipe_chunk(cfg)} batch elems; 2 H2D + 2 D2H copy streams, 1 kernel stream, 4 buffers)",
            "ms_per_step": round(ms, 2)}


def pipe_chunk(cfg):
    from paper_2504_11681_b200.pipeline import default_pipe_chunk
    return default_pipe_chunk(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="fully_fused")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "tf32x3", "bf16"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="time CUDA-graph replays of the layer (auto: chains and workloads <= 4 GiB of I/O)")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
