"""C ABI checks that need no GPU: the library builds, loads, exports every
symbol include/pif.h declares, the ctypes structs match the C layout, and
host-side argument validation rejects bad input before touching CUDA."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pif.h")


@pytest.fixture(scope="module")
def L():
    import __graft_entry__

    __graft_entry__._build_module().build()
    from paper_2407_00485_b200 import _lib

    return _lib


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pif_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert "pif_init" in names and "pif_parareal" in names and "pif_step" in names
    out = subprocess.run(["nm", "-D", "--defined-only", L._LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pif_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(L.lib, n)


def test_struct_layout_matches_c(L):
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "pif.h"
int main(void) {
  printf("%zu %zu %zu %zu\n", sizeof(pif_physics), sizeof(pif_propagator), sizeof(pif_dist),
         sizeof(pif_parareal_report));
  printf("%zu %zu %zu %zu %zu %zu\n", offsetof(pif_propagator, tol), offsetof(pif_propagator, flags),
         offsetof(pif_dist, nccl_id),
         offsetof(pif_parareal_report, retired_at), offsetof(pif_parareal_report, t_coarse0),
         offsetof(pif_physics, E_ext_c));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        open(src, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(v) for v in out]
    assert sizes[:4] == [ctypes.sizeof(L.PifPhysics), ctypes.sizeof(L.PifPropagator),
                         ctypes.sizeof(L.PifDist), ctypes.sizeof(L.PifPararealReport)]
    assert sizes[4:] == [L.PifPropagator.tol.offset, L.PifPropagator.flags.offset, L.PifDist.nccl_id.offset,
                         L.PifPararealReport.retired_at.offset,
                         L.PifPararealReport.t_coarse0.offset, L.PifPhysics.E_ext_c.offset]


@pytest.mark.parametrize("kw,status", [
    (dict(n=7), "PIF_ERR_ARG"),           # N odd
    (dict(n=0), "PIF_ERR_ARG"),
    (dict(tol=1e-16), "PIF_ERR_ARG"),     # tol outside [1e-15, 1e-1)
    (dict(tol=0.5), "PIF_ERR_ARG"),
    (dict(dt=0.0), "PIF_ERR_ARG"),
    (dict(kind=7), "PIF_ERR_ARG"),
])
def test_init_rejects_bad_propagator(L, kw, status):
    args = dict(kind=0, n=8, dt=0.05, tol=1e-12)
    args.update(kw)
    phys = L.physics(12.566, -1.0, -1984.4)
    with pytest.raises(L.PifError) as e:
        L.pif_init(phys, L.propagator(**args), None, 1000)
    assert L.STATUS[e.value.status] == status


def test_init_rejects_bad_layout_and_physics(L):
    phys = L.physics(12.566, -1.0, -1984.4)
    fine = L.propagator("pif", 8, 0.05, tol=1e-12)
    with pytest.raises(L.PifError) as e:
        L.pif_init(phys, fine, None, 1000, world=3, space_size=2, rank=0, nccl_id=b"\0" * 128)
    assert L.STATUS[e.value.status] == "PIF_ERR_CONFIG"
    with pytest.raises(L.PifError) as e:
        L.pif_init(L.physics(-1.0, -1.0, -1.0), fine, None, 1000)
    assert L.STATUS[e.value.status] == "PIF_ERR_ARG"
    coarse = L.propagator("pif", 8, 0.1, tol=1e-13)  # coarse tighter than fine
    with pytest.raises(L.PifError) as e:
        L.pif_init(phys, fine, coarse, 1000)
    assert L.STATUS[e.value.status] == "PIF_ERR_CONFIG"
    with pytest.raises(L.PifError) as e:
        L.pif_init(phys, L.propagator("pic", 32, 0.05, spline_order=2), None, 1000)
    assert L.STATUS[e.value.status] == "PIF_ERR_ARG"
