"""Build libpif.so in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libpif.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "pif.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    if out is None and not force and up_to_date():
        return LIB
    target = out or LIB
    cmd = [NVCC, "-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC,-O3", "-shared",
           "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
           "-Xptxas", "-v" if verbose else "-O3",
           *[f"-D{d}" for d in defines], *sources(), "-o", target + ".tmp", "-lcufft", "-lnccl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libpif.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
