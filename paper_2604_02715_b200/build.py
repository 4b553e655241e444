"""Build libxpgb.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2604_02715_b200.build [--force]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libxpgb.so")
OBJ = os.path.join(ROOT, "build", "obj")
SOURCES = ["moe_kernels.cu", "moe_gemm_pair.cu", "moe_gemm_dec.cu", "codec.cu", "fx4.cu", "ep_p2p.cu", "runtime.cu"]
HEADERS = ["moe_kernels.cuh", "ptx_sm100.cuh", "launch_count.h", "codec.cuh", "codec_dev.cuh", "fx4.cuh", "ep_p2p.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libxpgb.so")


def _mtime(path: str) -> float:
    return os.path.getmtime(path) if os.path.exists(path) else -1.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "xpgb.h")]
    dep_time = max(_mtime(d) for d in deps)
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), dep_time):
            cmd = [nvcc(), *ARCH, *FLAGS, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            jobs.append(subprocess.Popen(cmd))
    failed = [j.args for j in jobs if j.wait() != 0]  # sources compile in parallel
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _mtime(OUT) < max(_mtime(o) for o in objs):
        tmp = OUT + ".tmp"
        cmd = [nvcc(), "-shared", "-cudart", "static", *ARCH, "-o", tmp, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
