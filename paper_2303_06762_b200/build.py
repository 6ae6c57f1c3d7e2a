"""Builds the in-tree shared library paper_2303_06762_b200/lib/libhpmg.so.

nvcc compiles every CUDA source for sm_100a only (no multi-arch fallback);
the host bookkeeping headers are compiled into the same library.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libhpmg.so")

SOURCES = [os.path.join(CSRC, "kernels", "kernels.cu"), os.path.join(CSRC, "kernels", "small_levels.cu"), os.path.join(CSRC, "kernels", "dense_level.cu"),
           os.path.join(CSRC, "kernels", "sweep_rec.cu"), os.path.join(CSRC, "kernels", "post.cu"),
           os.path.join(CSRC, "context.cu"), os.path.join(CSRC, "ns.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, d, f) for d in ("kernels", "host") for f in os.listdir(os.path.join(CSRC, d))] + [
    os.path.join(ROOT, "include", "hpmg", "capi.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-O3",
]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: the hpmg library needs the CUDA toolkit")
    return path


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in DEPS if os.path.exists(p))


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:  # translation units compile in parallel
        obj = os.path.join(LIB_DIR, os.path.basename(src) + ".o")
        cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(obj)
    for src, p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB] + objs + ["-lcudart"]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
