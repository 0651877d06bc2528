"""bench.py contract on the CPU container: the reference arm (the oracle port
of fnofuse timed on host cores) prints one JSON line with the driver's keys,
and our arm refuses to run without a GPU (no CPU fallback)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--workload", "C1", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "GFLOP/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "C1" in d["config"]["workload"]


def test_our_arm_needs_a_gpu():
    import torch
    if torch.cuda.is_available():
        return
    r = _run(["--workload", "C1", "--steps", "1", "--warmup", "3", "--no-baselines", "--no-e2e", "--no-cpu"])
    assert r.returncode != 0


def test_reference_arm_under_torchrun_world2():
    """Driver launch for N > 1: rank 0 alone times the CPU reference and prints one line; rank 1 exits 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--workload", "C1", "--gpus", "2", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_reference_arm_never_loads_the_product():
    """The reference arm times the unmodified reference (or the port) and must not
    import the product package or map libturbofno.so (void ratio)."""
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--workload','C1','--steps','1',"
            "'--warmup','3']; import bench; bench.main(); "
            "assert not [m for m in sys.modules if m.startswith('paper_2504_11681_b200')]; "
            "maps=open('/proc/self/maps').read(); assert 'libturbofno' not in maps; print('CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "CLEAN" in r.stdout
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "fnofuse")):
        assert d["cpu_baseline"]["kind"] == "reference"
    assert d["config"]["hidden"] == 64 and d["config"]["out"] == 64
