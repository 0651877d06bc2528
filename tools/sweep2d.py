"""2D plane-path sweep: rank-2 shapes beyond the BASELINE configs (the reference
acceptance grid's 128^2 / 256^2 planes with keep 64 / 128, every row length
64..1024, non-square planes, ragged keeps) -- our fully_fused layer vs the
paper schedule (fft_optimized), the unfused cuFFT+cuBLAS pipeline (staged) and
torch.fft, CUDA-event timed, with the layer roofline fraction (SURVEY.md §8d:
T_roof = max(bytes / 8 TB/s, flops / 74.4 TF)) and max_rel_error of batch
element 0 against the float64 oracle composition.

    python tools/sweep2d.py [--out profiles/r02/sweep2d.json] [--shapes "B,H,N,dx,dy,kx,ky;..."]
    TFNO_PLANE_GENERIC=1 python tools/sweep2d.py ...   # generic kernels on the tuned shapes too
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import paper_2504_11681_b200 as T  # noqa: E402
from sweep import timeit  # noqa: E402

DEFAULT = [
    (128, 64, 64, 128, 128, 64, 64), (128, 64, 64, 128, 128, 128, 128),
    (32, 64, 64, 256, 256, 64, 64), (32, 64, 64, 256, 256, 128, 128),
    (512, 64, 64, 64, 64, 8, 8), (512, 64, 64, 64, 64, 32, 32),
    (32, 64, 64, 512, 512, 32, 32), (16, 64, 64, 512, 512, 128, 128),
    (8, 64, 64, 1024, 1024, 64, 64), (8, 64, 64, 1024, 1024, 128, 128),
    (32, 64, 64, 128, 1024, 64, 64), (32, 64, 64, 1024, 128, 32, 32),
    (32, 64, 64, 256, 256, 20, 12),
    (32, 64, 64, 256, 256, 32, 32), (256, 64, 64, 256, 256, 16, 16), (32, 128, 128, 512, 512, 64, 64),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "sweep2d.json"))
    ap.add_argument("--shapes", default="")
    ap.add_argument("--modes", default="fully_fused,fft_optimized,staged")
    ap.add_argument("--no-torch", action="store_true")
    args = ap.parse_args()
    shapes = DEFAULT if not args.shapes else [tuple(int(v) for v in s.split(",")) for s in args.shapes.split(";")]
    from oracle import fnofuse_port as O
    dev = torch.device("cuda:0")
    rows = []
    for s in shapes:
        B, H, N, dx, dy, kx, ky = s
        cfg = T.FnoLayerConfig(B, H, N, dx, dy, kx, ky, 2)
        fl = T.layer_flops(cfg)
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        x = torch.view_as_complex(torch.randn((B, H, dx, dy, 2), generator=g, device=dev))
        w = torch.view_as_complex(torch.randn((H, N, 2), generator=g, device=dev)).contiguous()
        y = torch.empty((B, N, dx, dy), dtype=torch.complex64, device=dev)
        reps = max(5, min(50, int(2e10 / max(fl["bytes"], 1))))
        row = {"shape": s, "bytes": fl["bytes"], "flops": fl["flops"],
               "generic_env": os.environ.get("TFNO_PLANE_GENERIC", "0")}
        for mode in args.modes.split(","):
            ms = timeit(lambda: T.run_layer_device(cfg, x, w, out=y, mode=mode, validate=False), reps)
            row[mode] = round(ms, 4)
            row[mode + "_schedule"] = T.layer_schedule(cfg, mode)[1]
        T.run_layer_device(cfg, x, w, out=y, mode="fully_fused", validate=False)
        torch.cuda.synchronize()
        c1 = T.FnoLayerConfig(1, H, N, dx, dy, kx, ky, 2)
        x0 = x[0:1].cpu().numpy()
        row["max_rel_error"] = float(T.max_rel_error(y[0:1].cpu().numpy(), O.reference_layer(c1, x0, w.cpu().numpy())))
        T._device.release_workspace()
        if not args.no_torch:
            row["torch_fft"] = round(timeit(lambda: bench.torch_fft_layer(cfg, x, w, y), reps), 4)
        ours = row["fully_fused"]
        base = [row[k] for k in ("staged", "torch_fft") if k in row]
        if base:
            row["speedup_vs_best_unfused"] = round(min(base) / ours, 3)
        if "fft_optimized" in row:
            row["speedup_vs_paper_schedule"] = round(row["fft_optimized"] / ours, 3)
        t_roof = max(fl["bytes"] / 8.0e12, fl["flops"] / 74.4e12)
        row["frac_layer_roofline"] = round(t_roof / (ours * 1e-3), 4)
        row["frac_measured_hbm"] = round(fl["bytes"] / (ours * 1e-3) / 6543.4e9, 4)
        rows.append(row)
        print(json.dumps({k: row[k] for k in row if not k.endswith("_schedule")}), flush=True)
        del x, w, y
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
