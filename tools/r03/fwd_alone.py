"""Is the C4 forward slower inside the layer loop than alone?  Times the plane forward
(tfno_spectrum_forward) repeated back to back, then alternating with the padded inverse
(tfno_spectrum_inverse), with CUDA events per launch, and samples SM clocks / power."""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2504_11681_b200 as T  # noqa: E402
from paper_2504_11681_b200 import multigpu as MG  # noqa: E402

cfg = T.FnoLayerConfig(128, 128, 128, 512, 512, 64, 64, rank=2)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.view_as_complex(torch.randn((128, 128, 512, 512, 2), generator=g, device=dev))
st = torch.cuda.current_stream()


def smi():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,temperature.memory",
                          "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
    return out


def run(label, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    samples = []
    stop = [False]

    def sampler():
        while not stop[0]:
            samples.append(smi())
            time.sleep(0.05)
    th = threading.Thread(target=sampler)
    th.start()
    evs = []
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(st)
        fn(e)
        evs.append(e)
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    f = sorted(a[0].elapsed_time(a[1]) for a in evs)
    print(label, "forward ms median %.3f min %.3f" % (f[len(f) // 2], f[0]), "| smi", samples[len(samples) // 2] if samples else None)


modes = MG.spectrum_forward(cfg, x)


def fwd_only(e=None):
    MG.spectrum_forward(cfg, x)
    if e:
        e[1].record(st)
        e[2].record(st)


def fwd_inv(e=None):
    MG.spectrum_forward(cfg, x)
    if e:
        e[1].record(st)
    MG.spectrum_inverse(cfg, modes, (128, 128))
    if e:
        e[2].record(st)


run("alone  ", fwd_only)
run("w/ inv ", fwd_inv)
run("alone  ", fwd_only)
run("w/ inv ", fwd_inv)
