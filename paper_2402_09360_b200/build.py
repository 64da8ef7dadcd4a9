"""Builds libhire_cuda.so in-tree for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhire_cuda.so")
SOURCES = [os.path.join(CSRC, "hire_cuda.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + [
    os.path.join(ROOT, "include", "hire_cuda.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared",
]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def _src_hash() -> str:
    import hashlib
    h = hashlib.sha256(" ".join(NVCC_FLAGS + os.environ.get("HIRE_NVCC_EXTRA", "").split()).encode())
    for p in sorted(DEPS):
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def stale() -> bool:
    """The library is stale unless it was built from exactly these sources
    (a hash beside the .so; mtimes lie when sources change mid-build)."""
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".srchash"):
        return True
    with open(LIB + ".srchash") as f:
        return f.read().strip() != _src_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    extra = os.environ.get("HIRE_NVCC_EXTRA", "").split()  # experiments only
    h = _src_hash()  # of the sources as they are when the compile starts
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", LIB, *SOURCES, "-lnccl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stderr[-4000:]}")
    with open(LIB + ".srchash", "w") as f:
        f.write(h + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
