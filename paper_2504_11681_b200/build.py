"""Build libturbofno.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2504_11681_b200.build [--force]

The shared library lands next to this file (``paper_2504_11681_b200/libturbofno.so``)
so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OUT = os.path.join(HERE, "libturbofno.so")
BUILD_DIR = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--cudart", "shared",
              "-Xptxas", "-v"] + ARCH
# (source, extra nvcc flags, object name): plane_g.cu is built once per row length
PLANE_G = [("plane_g.cu", ["-DPLANE_G_DY=%d" % d], "plane_g_%d.cu.o" % d) for d in (64, 128, 256, 512, 1024)]
SOURCES = ["kernels.cu", "plane2d.cu", "rows1d.cu", "cgemm_tc.cu", "warpfft.cu", "warpfft_fwd.cu", "fused1d.cu", "tiny1d.cu", "permode.cu", "realfield.cu", "api.cu", "plan.cpp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


DIGEST = OUT + ".sha256"  # content digest of everything the library is built from


def source_digest() -> str:
    """sha256 over every source / header, this build script, the nvcc version and
    the A/B build hooks: the library is rebuilt whenever any of them changes
    (content, not modification times, so a copied tree or a clock skew cannot
    make build() reuse a stale binary)."""
    import hashlib
    h = hashlib.sha256()
    paths = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC))
    paths += sorted(os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE))
    paths.append(os.path.abspath(__file__))
    for p in paths:
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    try:
        h.update(subprocess.run([_nvcc(), "--version"], capture_output=True, text=True).stdout.encode())
    except Exception:  # noqa: BLE001
        pass
    for k in ("TFNO_SCALAR_FILES", "TFNO_NVCC_DEFS"):
        h.update(f"{k}={os.environ.get(k, '')}".encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    digest = source_digest()
    if not force and os.path.exists(OUT) and os.path.exists(DIGEST):
        with open(DIGEST) as f:
            if f.read().strip() == digest:
                return OUT
    os.makedirs(BUILD_DIR, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(item):
        src, extra, oname = item if isinstance(item, tuple) else (item, [], item + ".o")
        obj = os.path.join(BUILD_DIR, oname)
        path = os.path.join(CSRC, src)
        if src.endswith(".cpp"):
            cmd = [nvcc, "-O3", "-std=c++17", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-fPIC", "-c", path, "-o", obj]
        else:
            cmd = [nvcc] + NVCC_FLAGS + extra + ["-I", INCLUDE, "-c", path, "-o", obj]
            # A/B hook: TFNO_SCALAR_FILES=a.cu,b.cu builds those files with the scalar complex primitives
            if src in os.environ.get("TFNO_SCALAR_FILES", "").split(","):
                cmd.insert(1, "-DTFNO_SCALAR_COMPLEX")
            # A/B hook: TFNO_NVCC_DEFS=A,B adds -DA -DB to every CUDA translation unit
            for d in filter(None, os.environ.get("TFNO_NVCC_DEFS", "").split(",")):
                cmd.insert(1, "-D" + d)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        with open(os.path.join(BUILD_DIR, oname[:-2] + ".ptxas.txt"), "w") as f:
            f.write(res.stderr)
        return obj

    # translation units are independent: compile them in parallel
    from concurrent.futures import ThreadPoolExecutor
    items = PLANE_G + SOURCES
    with ThreadPoolExecutor(max_workers=min(len(items), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, items))
    tmp = OUT + ".tmp"
    cmd = [nvcc, "-shared", "--cudart", "shared"] + ARCH + ["-o", tmp] + objs + [
        "-L/usr/local/cuda/lib64", "-lcufft", "-lcublas", "-lcudart",
        "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, OUT)
    with open(DIGEST, "w") as f:
        f.write(digest + "\n")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
