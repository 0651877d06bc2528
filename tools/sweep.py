"""Sweep BASELINE configs (C1, C2 grid, C3, C4, C5 layer) x modes on one GPU:
our sm_100a layer in every mode vs the unfused cuFFT+cuBLAS pipeline (staged
mode) and torch.fft+einsum, CUDA-event timed on the current stream.

    python tools/sweep.py [--out profiles/r01/sweep.json] [--quick]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2504_11681_b200 as T  # noqa: E402
from oracle import fnofuse_port as O  # noqa: E402  (checker only: parity per sweep point)


def timeit(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def graphed(fn):
    """Capture fn (already warmed up: plans / workspaces exist) into a CUDA
    graph and return its replay: removes host launch overhead from small
    layers, for our kernels and the cuFFT/cuBLAS baselines alike."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "sweep.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--workloads", default="")
    args = ap.parse_args()
    names = [n for n in bench.WORKLOADS if n != "C5"]
    if args.workloads:
        names = args.workloads.split(",")
    dev = torch.device("cuda:0")
    rows = []
    for name in names:
        B, H, N, dx, dy, kx, ky, rk, desc = bench.WORKLOADS[name]
        cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, rk)
        fl = T.layer_flops(cfg)
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        x = torch.view_as_complex(torch.randn((B, H, dx, dy, 2), generator=g, device=dev))
        w = torch.view_as_complex(torch.randn((H, N, 2), generator=g, device=dev)).contiguous()
        y = torch.empty((B, N, dx, dy), dtype=torch.complex64, device=dev)
        reps = 5 if args.quick else max(5, min(50, int(2e10 / max(fl["bytes"], 1))))
        small = fl["bytes"] < (256 << 20)
        wrap = graphed if small else (lambda f: f)
        row = {"workload": name, "desc": desc, "bytes": fl["bytes"], "flops": fl["flops"],
               "timing": "CUDA-graph replays" if small else "eager launches"}
        for mode in T.MODES:
            ms = timeit(wrap(lambda: T.run_layer_device(cfg, x, w, out=y, mode=mode, validate=False)), reps)
            row[mode] = round(ms, 4)
            row[mode + "_schedule"] = T.layer_schedule(cfg, mode)[1]
        for prec in ("tf32x3", "tf32"):
            try:
                mode = "fully_fused" if rk == 2 else "fft_optimized"
                row[prec] = round(timeit(wrap(lambda: T.run_layer_device(cfg, x, w, out=y, mode=mode, precision=prec,
                                                                           validate=False)), reps), 4)
            except Exception as ex:  # noqa: BLE001
                row[prec] = str(ex)[:80]
        T._device.release_workspace()
        row["torch_fft"] = round(timeit(wrap(lambda: bench.torch_fft_layer(cfg, x, w, y)), reps), 4)
        ours = min(row[m] for m in T.MODES if m != "staged")
        best_base = min(row["staged"], row["torch_fft"])
        row["best_ours_fp32"] = ours
        row["speedup_vs_best_unfused"] = round(best_base / ours, 3)
        row["speedup_vs_staged"] = {m: round(row["staged"] / row[m], 3) for m in T.MODES if m != "staged"}
        row["frac_measured_hbm"] = round(fl["bytes"] / (ours * 1e-3) / 6543.4e9, 4)
        t_roof = max(fl["bytes"] / 8.0e12, fl["flops"] / 74.4e12)  # SURVEY.md §8d layer roofline
        row["frac_layer_roofline"] = round(t_roof / (ours * 1e-3), 4)
        # parity per point (north_star: max relative error reported per config): every mode on a
        # batch slice against the CPU oracle (bitwise equal to fnofuse.run_layer)
        nb = min(B, 2 if rk == 2 else 4)
        cs = T.FnoLayerConfig(nb, H, N, dx, dy, kx, ky, rk)
        xs = x[:nb].cpu().numpy()
        ref = O.run_layer_values(cs, xs, w.cpu().numpy())
        errs = {}
        for mode in T.MODES:
            ys = T.run_layer_device(cs, x[:nb].contiguous(), w, mode=mode)
            errs[mode] = float(T.max_rel_error(ys.cpu().numpy(), ref))
        row["max_rel_error"] = errs
        row["parity_sample"] = f"batch[0:{nb}] vs oracle port (fnofuse.run_layer semantics)"
        rows.append(row)
        print(json.dumps({k: row[k] for k in ("workload", "fully_fused", "fully_fused_schedule", "best_ours_fp32",
                                              "staged", "speedup_vs_staged", "frac_layer_roofline",
                                              "frac_measured_hbm", "max_rel_error")}), flush=True)
        del x, w, y
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
