"""Multi-process host logic on CPU (gloo): the C++ pipelined-parareal protocol
of libpif.so (pif_debug_parareal_protocol -- the code pif_parareal runs with
NCCL on GPUs) driven by world_size 2 and 4 processes, with gloo send/recv for
the state hand-off and the CPU oracle as F and G.  The last rank's U_{Ns},
every slice's retirement iteration and the per-iteration errors must equal
the oracle's serial parareal.

Also the particle-decomposition arithmetic of the space group (PAPER.md:
139-141): per-rank partial type-1 sums all-reduced over gloo equal the
single-process sum, with the partition of pif_local_count's rule."""
import ctypes as C
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from pif_inputs import landau_physics, landau_state

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem():
    ph = O.PhysicsParams.from_inputs(landau_physics())
    x0, v0 = landau_state(96, 21)
    F = O.make_propagator_fn(O.Propagator("pif", 4, 0.05), ph, 4)
    G = O.make_propagator_fn(O.Propagator("pic", 4, 0.1), ph, 2)
    return ph, x0, v0, F, G


CB_STORE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)
CB_PROP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int)
CB_CORR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                      C.POINTER(C.c_double), C.POINTER(C.c_double))
CB_SEND = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_double)
CB_RECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_double))


class Ops(C.Structure):
    _fields_ = [("user", C.c_void_p), ("store_initial", CB_STORE), ("propagate", CB_PROP),
                ("correct", CB_CORR), ("send", CB_SEND), ("recv", CB_RECV)]


def _worker(rank, world, port, max_iter, tol, out):
    try:
        _worker_body(rank, world, port, max_iter, tol, out)
    except Exception:  # report instead of hanging the parent
        import traceback
        out.put(dict(rank=rank, error=traceback.format_exc()))


def _worker_body(rank, world, port, max_iter, tol, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__
    __graft_entry__._build_module().build()
    from paper_2407_00485_b200 import _lib as L
    ph, x0, v0, F, G = problem()
    n = x0.shape[1]
    bufs = [None] * 5

    def store(_, dst):
        bufs[dst] = (x0.copy(), v0.copy())
        return 0

    def prop(_, which, src, dst):
        bufs[dst] = (F if which == 0 else G)(bufs[src])
        return 0

    def corr(_, f, gn, go, u, ex, ev):
        Fk, Gn, Go = bufs[f], bufs[gn], bufs[go]
        bufs[u] = (O.wrap(Fk[0] + Gn[0] - Go[0], ph.L), Fk[1] + Gn[1] - Go[1])
        dx = O.min_image(Gn[0] - Go[0], ph.L)
        ex[0] = float(np.linalg.norm(dx) / np.linalg.norm(Gn[0]))
        ev[0] = float(np.linalg.norm(Gn[1] - Go[1]) / np.linalg.norm(Gn[1]))
        return 0

    def send(_, b, flag):
        x, v = bufs[b]
        dist.send(torch.from_numpy(np.concatenate([x.ravel(), v.ravel(), [flag]])), rank + 1)
        return 0

    def recv(_, b, flagp):
        t = torch.empty(6 * n + 1, dtype=torch.float64)
        dist.recv(t, rank - 1)
        a = t.numpy()
        bufs[b] = (a[:3 * n].reshape(3, n).copy(), a[3 * n:6 * n].reshape(3, n).copy())
        flagp[0] = a[-1]
        return 0

    cbs = (CB_STORE(store), CB_PROP(prop), CB_CORR(corr), CB_SEND(send), CB_RECV(recv))
    ops = Ops(None, *cbs)
    it, ret, fb = C.c_int32(), C.c_int32(), C.c_int32()
    ex = (C.c_double * max_iter)()
    ev = (C.c_double * max_iter)()
    st = L.lib.pif_debug_parareal_protocol(rank, world, max_iter, tol, C.addressof(ops),
                                           C.byref(it), C.byref(ret), ex, ev, C.byref(fb))
    assert st == 0
    res = dict(rank=rank, iterations=it.value, retired_at=ret.value, ex=list(ex), ev=list(ev))
    if rank == world - 1:
        res["x"], res["v"] = bufs[fb.value]
    out.put(res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,tol", [(2, 1e-6), (4, 1e-6), (4, 0.0)])
def test_pipelined_protocol_equals_serial_parareal(world, tol):
    import __graft_entry__
    __graft_entry__._build_module().build()
    max_iter = world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, max_iter, tol, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r["rank"])
    errs = [r["error"] for r in res if "error" in r]
    assert not errs, errs[0]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ph, x0, v0, F, G = problem()
    ref = O.parareal_serial((x0, v0), F, G, world, max_iter, tol, L=ph.L)
    assert [r["retired_at"] for r in res] == ref.retired_at
    assert max(r["iterations"] for r in res) == ref.iterations
    for r in res:
        for k in range(ref.iterations):
            a, b = r["ex"][k], ref.err_x[k][r["rank"]]
            assert (math.isnan(a) and math.isnan(b)) or abs(a - b) <= 1e-12 * max(1.0, abs(b))
    xs, vs = ref.U[world]
    assert np.abs(O.min_image(res[-1]["x"] - xs, ph.L)).max() <= 1e-12
    assert np.abs(res[-1]["v"] - vs).max() <= 1e-12


def _space_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, _ = landau_state(1001, 5)
    n = x.shape[1]
    from paper_2407_00485_b200 import _lib as L  # host-only partition rule of pif_init
    first, count = L.pif_partition(n, world, rank)
    part = O.nudft_type1(x[:, first:first + count], np.ones(count), 6, landau_physics().L)
    t = torch.from_numpy(np.stack([part.real, part.imag]))
    dist.all_reduce(t)
    cover = torch.zeros(n, dtype=torch.int64)
    cover[first:first + count] = 1
    dist.all_reduce(cover)
    out.put((rank, t.numpy(), cover.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_space_decomposition_allreduce_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_space_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, _ = landau_state(1001, 5)
    full = O.nudft_type1(x, np.ones(1001), 6, landau_physics().L)
    for _, t, cover in res:
        assert np.all(cover == 1)
        assert np.abs(t[0] + 1j * t[1] - full).max() <= 1e-11 * np.abs(full).max()
