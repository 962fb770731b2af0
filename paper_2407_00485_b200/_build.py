"""Build libpif.so in-tree with nvcc for sm_100a (B200): one object per .cu
(compiled in parallel), then one shared-library link."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

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
    objdir = os.path.join(os.path.dirname(target), "build", os.path.basename(target) + ".objs")
    os.makedirs(objdir, exist_ok=True)
    flags = ["-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC,-O3",
             "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
             "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines]]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        r = subprocess.run([NVCC, *flags, "-c", src, "-o", obj], capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(src)}")
        if verbose:
            sys.stderr.write(r.stderr)
    r = subprocess.run([NVCC, *ARCH, "-shared", *[o for _, o, _ in results], "-o", target + ".tmp",
                        "-lcufft", "-lnccl"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libpif.so")
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
