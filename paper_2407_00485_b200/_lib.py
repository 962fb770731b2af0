"""ctypes binding of libpif.so (include/pif.h) -- argument marshalling only.

Every computation happens in the CUDA library; this module only converts
Python/numpy/torch arguments into the C ABI's plain pointers and sizes.  There
is no fallback: if libpif.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB_PATH = os.environ.get("PIF_LIBRARY") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libpif.so")  # override: kernel A/B experiments
if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a). There is no CPU fallback.")
lib = C.CDLL(_LIB_PATH)

PIF_PROP_PIF_NUFFT = 0
PIF_PROP_PIC_CIC = 1
PIF_FLAG_FP32_ALLREDUCE = 1
PIF_FLAG_FP32 = 2
STATUS = {0: "PIF_OK", 1: "PIF_ERR_ARG", 2: "PIF_ERR_CONFIG", 3: "PIF_ERR_NUMERIC",
          4: "PIF_ERR_CUDA", 5: "PIF_ERR_NCCL", 6: "PIF_ERR_OOM", 7: "PIF_ERR_STATE"}


class PifPhysics(C.Structure):
    _fields_ = [("L", C.c_double), ("q_over_m", C.c_double), ("total_charge", C.c_double),
                ("B_ext", C.c_double * 3), ("E_ext_A", C.c_double * 9), ("E_ext_c", C.c_double * 3)]


class PifPropagator(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("spline_order", C.c_int32),
                ("flags", C.c_int32), ("tol", C.c_double), ("dt", C.c_double)]


class PifDist(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("space_size", C.c_int32), ("nccl_id", C.c_void_p), ("stream", C.c_void_p)]


class PifPararealReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("retired_at", C.POINTER(C.c_int32)), ("err_x", C.POINTER(C.c_double)),
                ("err_v", C.POINTER(C.c_double)), ("t_coarse0", C.c_double),
                ("t_fine", C.c_double), ("t_coarse", C.c_double), ("t_comm", C.c_double),
                ("t_total", C.c_double)]


_ctx = C.c_void_p
_i64 = C.c_int64
_dp = C.c_void_p  # double* (host or device)
_sig = {
    "pif_init": [C.POINTER(PifPhysics), C.POINTER(PifPropagator), C.POINTER(PifPropagator), _i64,
                 C.POINTER(PifDist), C.POINTER(_ctx)],
    "pif_local_count": [_ctx, C.POINTER(_i64), C.POINTER(_i64)],
    "pif_partition": [_i64, C.c_int32, C.c_int32, C.POINTER(_i64), C.POINTER(_i64)],
    "pif_workspace_size": [_ctx, C.POINTER(C.c_size_t)],
    "pif_set_workspace": [_ctx, C.c_void_p, C.c_size_t],
    "pif_set_state": [_ctx, _dp, _dp, _i64, C.c_int],
    "pif_get_state": [_ctx, _dp, _dp, _i64, C.c_int],
    "pif_step": [_ctx, C.c_int, _i64],
    "pif_field_energy": [_ctx, C.POINTER(C.c_double), C.POINTER(C.c_double),
                         C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "pif_parareal": [_ctx, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                     C.POINTER(PifPararealReport)],
    "pif_finalize": [_ctx],
    "pif_nccl_unique_id": [C.c_void_p],
    "pif_plan_info": [_ctx, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                      C.POINTER(C.c_int32)],
    "pif_debug_type1": [_ctx, C.c_int, _dp, _i64, _dp, _dp],
    "pif_debug_type2": [_ctx, C.c_int, _dp, _dp, _i64, _dp],
    "pif_debug_push": [_ctx, C.c_int, _dp, _dp, _dp, _i64, C.c_int, C.c_int],
    "pif_profile": [_ctx, C.c_int],
    "pif_comm_info": [_ctx, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "pif_get_rho": [_ctx, _dp],
    "pif_debug_parareal_protocol": [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_void_p,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int32)],
    "pif_profile_read": [_ctx, C.POINTER(C.c_double), C.c_int32, C.POINTER(_i64), C.c_int],
}
for _name, _args in _sig.items():
    if os.environ.get("PIF_LIBRARY") and not hasattr(lib, _name):
        continue  # A/B runs against an older build may lack newer exports
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
lib.pif_last_error.argtypes = []
lib.pif_last_error.restype = C.c_char_p


class PifError(RuntimeError):
    def __init__(self, func, status):
        self.status = status
        msg = lib.pif_last_error().decode(errors="replace")
        super().__init__(f"{func}: {STATUS.get(status, status)}: {msg}")


def _check(func, status):
    if status != 0:
        raise PifError(func, status)


def _ptr(a):
    """(address, on_device) of a contiguous float64 torch tensor or numpy array."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError("numpy arrays must be C-contiguous float64")
        return a.ctypes.data, 0
    import torch
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("tensors must be contiguous float64")
        return a.data_ptr(), int(a.is_cuda)
    raise TypeError(type(a))


# ------------------------------------------------------------------ helpers --
def physics(L, q_over_m, total_charge, B=(0.0, 0.0, 0.0), A=(0.0,) * 9, c=(0.0, 0.0, 0.0)):
    p = PifPhysics()
    p.L, p.q_over_m, p.total_charge = L, q_over_m, total_charge
    p.B_ext[:] = list(B)
    p.E_ext_A[:] = list(A)
    p.E_ext_c[:] = list(c)
    return p


def propagator(kind, n, dt, tol=1e-12, spline_order=1, fp32_allreduce=False, fp32=False):
    if isinstance(kind, str):
        kind = {"pif": PIF_PROP_PIF_NUFFT, "pic": PIF_PROP_PIC_CIC}[kind]
    p = PifPropagator()
    p.kind, p.n, p.spline_order, p.tol, p.dt = kind, n, spline_order, tol, dt
    p.flags = (PIF_FLAG_FP32_ALLREDUCE if fp32_allreduce else 0) | (PIF_FLAG_FP32 if fp32 else 0)
    return p


# ------------------------------------------------------- ABI, same names ----
def pif_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check("pif_nccl_unique_id", lib.pif_nccl_unique_id(buf))
    return buf.raw


def pif_init(phys, fine, coarse, n_particles_global, device=0, rank=0, world=1, space_size=1,
             nccl_id=None, stream=0):
    d = PifDist()
    d.device, d.rank, d.world, d.space_size = device, rank, world, space_size
    idbuf = None
    if nccl_id is not None:
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        d.nccl_id = C.cast(idbuf, C.c_void_p)
    d.stream = stream
    ctx = _ctx()
    _check("pif_init", lib.pif_init(C.byref(phys), C.byref(fine),
                                    C.byref(coarse) if coarse is not None else None,
                                    n_particles_global, C.byref(d), C.byref(ctx)))
    return ctx


def pif_local_count(ctx):
    a, b = _i64(), _i64()
    _check("pif_local_count", lib.pif_local_count(ctx, C.byref(a), C.byref(b)))
    return a.value, b.value


def pif_partition(n_global, space_size, s_idx):
    a, b = _i64(), _i64()
    _check("pif_partition", lib.pif_partition(n_global, space_size, s_idx, C.byref(a), C.byref(b)))
    return a.value, b.value


def pif_workspace_size(ctx) -> int:
    s = C.c_size_t()
    _check("pif_workspace_size", lib.pif_workspace_size(ctx, C.byref(s)))
    return s.value


def pif_set_workspace(ctx, ptr, nbytes):
    _check("pif_set_workspace", lib.pif_set_workspace(ctx, ptr, nbytes))


def pif_set_state(ctx, x, v):
    px, dx = _ptr(x)
    pv, dv = _ptr(v)
    assert dx == dv and x.shape[0] == 3 and x.shape == v.shape
    _check("pif_set_state", lib.pif_set_state(ctx, px, pv, x.shape[1], dx))


def pif_get_state(ctx, x, v):
    px, dx = _ptr(x)
    pv, dv = _ptr(v)
    assert dx == dv and x.shape[0] == 3 and x.shape == v.shape
    _check("pif_get_state", lib.pif_get_state(ctx, px, pv, x.shape[1], dx))


def pif_step(ctx, which, n_steps):
    _check("pif_step", lib.pif_step(ctx, which, n_steps))


def pif_field_energy(ctx):
    W = (C.c_double * 3)()
    ke = C.c_double()
    P = (C.c_double * 3)()
    ce = C.c_double()
    _check("pif_field_energy", lib.pif_field_energy(ctx, W, C.byref(ke), P, C.byref(ce)))
    return np.array(W[:]), ke.value, np.array(P[:]), ce.value


def pif_parareal(ctx, t0, t1, n_slices, max_iter, stop_tol, n_blocks=1):
    ret = (C.c_int32 * n_slices)()
    ex = (C.c_double * max(1, max_iter * n_slices))()
    ev = (C.c_double * max(1, max_iter * n_slices))()
    r = PifPararealReport()
    r.retired_at = C.cast(ret, C.POINTER(C.c_int32))
    r.err_x = C.cast(ex, C.POINTER(C.c_double))
    r.err_v = C.cast(ev, C.POINTER(C.c_double))
    _check("pif_parareal", lib.pif_parareal(ctx, t0, t1, n_slices, max_iter, stop_tol, n_blocks,
                                            C.byref(r)))
    shape = (max_iter, n_slices)
    return dict(iterations=r.iterations, converged=bool(r.converged), retired_at=list(ret),
                err_x=np.array(ex[:max_iter * n_slices]).reshape(shape),
                err_v=np.array(ev[:max_iter * n_slices]).reshape(shape),
                t_coarse0=r.t_coarse0, t_fine=r.t_fine, t_coarse=r.t_coarse, t_comm=r.t_comm,
                t_total=r.t_total)


def pif_get_rho(ctx, N):
    """rho_tilde on the Hermitian half box, complex array [N+1, N+1, N/2+1] indexed
    [mx + N/2, my + N/2, mz]."""
    out = np.empty(2 * (N + 1) ** 2 * (N // 2 + 1))
    _check("pif_get_rho", lib.pif_get_rho(ctx, out.ctypes.data))
    return out.view(np.complex128).reshape(N + 1, N + 1, N // 2 + 1)


def pif_finalize(ctx):
    _check("pif_finalize", lib.pif_finalize(ctx))


def pif_plan_info(ctx, which=0):
    w, b, n = C.c_int32(), C.c_double(), C.c_int32()
    _check("pif_plan_info", lib.pif_plan_info(ctx, which, C.byref(w), C.byref(b), C.byref(n)))
    return w.value, b.value, n.value


def pif_debug_type1(ctx, which, x, s, N):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.empty(2 * N ** 3)
    _check("pif_debug_type1", lib.pif_debug_type1(ctx, which, x.ctypes.data, x.shape[1],
                                                  s.ctypes.data, out.ctypes.data))
    return out.view(np.complex128).reshape(N, N, N)


def pif_debug_type2(ctx, which, c, x):
    c = np.ascontiguousarray(c, dtype=np.complex128)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.shape[1])
    _check("pif_debug_type2", lib.pif_debug_type2(ctx, which, c.ctypes.data, x.ctypes.data,
                                                  x.shape[1], out.ctypes.data))
    return out


def pif_debug_push(ctx, which, x, v, E, kicks, drift):
    """In place on host float64 arrays of shape (3, n)."""
    for a in (x, v, E):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    _check("pif_debug_push", lib.pif_debug_push(ctx, which, x.ctypes.data, v.ctypes.data,
                                                E.ctypes.data, x.shape[1], kicks, drift))


def pif_comm_info(ctx):
    """-> {"world_nranks", "space_nranks", "time_nranks"} from ncclCommCount."""
    a, b, d = C.c_int32(), C.c_int32(), C.c_int32()
    _check("pif_comm_info", lib.pif_comm_info(ctx, C.byref(a), C.byref(b), C.byref(d)))
    return {"world_nranks": a.value, "space_nranks": b.value, "time_nranks": d.value}


PHASES = ("sort", "spread", "fft_fwd", "box", "allreduce", "poisson", "fft_inv", "interp_push",
          "pic_deposit", "pic_gather_push", "other")


def pif_profile(ctx, enable=True):
    _check("pif_profile", lib.pif_profile(ctx, int(bool(enable))))


def pif_profile_read(ctx, reset=True):
    """-> ({phase: ms}, launches) summed since the last reset."""
    ms = (C.c_double * len(PHASES))()
    n = _i64()
    _check("pif_profile_read", lib.pif_profile_read(ctx, ms, len(PHASES), C.byref(n), int(reset)))
    return dict(zip(PHASES, ms[:])), n.value
