"""Plain, slow, exact CPU oracle of the PIF timestep and parareal (fp64, numpy).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg and --impl reference).  The CUDA product path never
calls it.

What it computes is the *exact* finite-dimensional PIF scheme of the paper --
direct NUDFT instead of NUFFT (footnote "Exact here refers to the
use of NUDFT instead of NUFFT") -- plus the CIC-PIC coarse propagator, the
KDK/Boris push and the serial parareal iteration.  Readings of silent or
ambiguous points are the ones listed in DESIGN.md ("Readings", R1..R20) and
referenced below as [Rn].

Conventions (SOA, as the C ABI): x, v have shape (3, N_p), float64.
Mode arrays are indexed [ix, iy, iz] with integer mode m = i - N/2, i.e. the
row-major order over (mx, my, mz) each from -N/2 to N/2-1 [R1].

Chunking over particles below is memory management only: every sum is the
plain sum over j of the definition (rounding order differs, nothing else).
Library primitives used as steps: numpy einsum/tensordot (a contraction),
numpy.fft (the PIC grid DFT), np.add.at (a scatter-add).

Parity status: every function here is pinned by tests/test_oracle_pins.py;
see DESIGN.md "Oracle pins" for which pin covers which function.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

def _chunk(N: int) -> int:
    """Particles per chunk: keeps the (chunk, N, N) temporaries near 16 MB."""
    return max(1024, (1 << 20) // (N * N))


# --------------------------------------------------------------------------
# Mode set, shape factor
# --------------------------------------------------------------------------
def mode_indices(N: int) -> np.ndarray:
    """Integer modes m in [-N/2, N/2-1] (N even) -- the symmetric reading of
    K_N = {(2 pi/L)[0, N-1]}^3 [R1]."""
    if N < 2 or N % 2:
        raise ValueError("N must be even and >= 2")
    return np.arange(-N // 2, N // 2)


def wavenumbers(N: int, L: float) -> np.ndarray:
    """k = (2 pi / L) m."""
    return (2.0 * math.pi / L) * mode_indices(N)


def shape_factor_1d(N: int, L: float, order: int = 1) -> np.ndarray:
    """Per-dimension Fourier transform of the B-spline shape of order m (CIC:
    m=1): S(k) = sinc(k h / 2)^(m+1), h = L/N, sinc u = sin(u)/u
    ("analytic form", "linear B-spline ... and the
    analytical Fourier transform of it is used for the PIF scheme") [R3][R4]."""
    h = L / N
    u = wavenumbers(N, L) * h / 2.0
    s = np.ones_like(u)
    nz = u != 0
    s[nz] = np.sin(u[nz]) / u[nz]
    return s ** (order + 1)


def shape_factor(N: int, L: float, order: int = 1) -> np.ndarray:
    """S_k = S(kx) S(ky) S(kz) on K_N, shape (N,N,N) (tensor-product B-spline)."""
    s = shape_factor_1d(N, L, order)
    return s[:, None, None] * s[None, :, None] * s[None, None, :]


# --------------------------------------------------------------------------
# Direct NUDFT (the exact P and P^H of PAPER.md:180-184)
# --------------------------------------------------------------------------
def nudft_type1(x: np.ndarray, s: np.ndarray, N: int, L: float) -> np.ndarray:
    """out[mx,my,mz] = sum_j s_j exp(-i k . x_j),  k in K_N.

    The sum of eq. scatter_pif without the factor q S_k / L^3.
    Phases are the separable product exp(-i kx x) exp(-i ky y) exp(-i kz z) of
    directly evaluated complex exponentials (no recurrences).
    """
    k = wavenumbers(N, L)
    s = np.asarray(s)
    out = np.zeros((N, N, N), dtype=np.complex128)
    for a in range(0, x.shape[1], _chunk(N)):
        sl = slice(a, a + _chunk(N))
        ex = np.exp(-1j * np.outer(x[0, sl], k))
        ey = np.exp(-1j * np.outer(x[1, sl], k))
        ez = np.exp(-1j * np.outer(x[2, sl], k))
        # out[a,b,c] += sum_j (s_j ex[j,a] ey[j,b]) ez[j,c]  (a contraction over j)
        exy = ((s[sl, None] * ex)[:, :, None] * ey[:, None, :]).reshape(-1, N * N)
        out += (exy.T @ ez).reshape(N, N, N)
    return out


def nudft_type2_complex(c: np.ndarray, x: np.ndarray, N: int, L: float) -> np.ndarray:
    """out_j = sum_{k in K_N} c_k exp(+i k . x_j)   (eq. gather_pif).

    c: (N,N,N) -> out (N_p,); or a stack (D,N,N,N) of D coefficient arrays
    evaluated at the same positions (the three field components) -> (D, N_p)."""
    k = wavenumbers(N, L)
    cs = c.reshape(-1, N, N, N)
    D = cs.shape[0]
    out = np.empty((D, x.shape[1]), dtype=np.complex128)
    for a in range(0, x.shape[1], _chunk(N)):
        sl = slice(a, a + _chunk(N))
        ex = np.exp(1j * np.outer(x[0, sl], k))
        ey = np.exp(1j * np.outer(x[1, sl], k))
        ez = np.exp(1j * np.outer(x[2, sl], k))
        # y[j,d,(a,b)] = sum_c c_d[a,b,c] ez[j,c]  (a contraction over c), then
        # out_dj = sum_{a,b} y[j,d,a,b] ex[j,a] ey[j,b]
        y = (ez @ cs.reshape(D * N * N, N).T).reshape(-1, D, N, N)
        exy = ex[:, :, None] * ey[:, None, :]
        out[:, sl] = np.sum(y * exy[:, None], axis=(2, 3)).T
    return out[0] if c.ndim == 3 else out


def nudft_type2(c: np.ndarray, x: np.ndarray, N: int, L: float) -> np.ndarray:
    """Re sum_{k in K_N} c_k exp(+i k . x_j): the field at a particle is real [R2]."""
    return nudft_type2_complex(c, x, N, L).real


# --------------------------------------------------------------------------
# Exact PIF field solve
# --------------------------------------------------------------------------
@dataclass
class FieldSolve:
    E: np.ndarray          # (3, N_p) self-consistent field at the particles
    rho_tilde: np.ndarray  # (N,N,N) (q/L^3) sum_j exp(-ik.x_j), before S_k
    E_k: np.ndarray        # (3,N,N,N) spectral field E_{d,k}


def poisson_spectral(rho_tilde: np.ndarray, N: int, L: float, order: int = 1) -> np.ndarray:
    """E_{d,k} = -i k_d rho_k / |k|^2 with rho_k = S_k rho_tilde_k and rho_0 := 0.

    PAPER.md:186 ("E_k = -ik/|k|^2 rho_k"), PAPER.md:85-89 (uniform neutralising
    ion background removes k = 0) [R5]; S_k inside rho_k per eq. scatter_pif.
    """
    k = wavenumbers(N, L)
    kx, ky, kz = np.meshgrid(k, k, k, indexing="ij")
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    rho = shape_factor(N, L, order) * rho_tilde
    inv = np.zeros_like(k2)
    nz = k2 > 0
    inv[nz] = 1.0 / k2[nz]
    rho = np.where(nz, rho, 0.0)
    return np.stack([-1j * kx * rho * inv, -1j * ky * rho * inv, -1j * kz * rho * inv])


def field_from_rho_tilde(rho_tilde: np.ndarray, x: np.ndarray, N: int, L: float,
                         order: int = 1):
    """E(x_j) = Re sum_k S_k E_k exp(i k x_j)  (eq. gather_pif) [R2]."""
    E_k = poisson_spectral(rho_tilde, N, L, order)
    S = shape_factor(N, L, order)
    E = nudft_type2(S[None] * E_k, x, N, L)  # the three components, shape (3, N_p)
    return E, E_k


def pif_field(x: np.ndarray, N: int, L: float, q: float, order: int = 1) -> FieldSolve:
    """Full exact PIF field solve at positions x (all particles carry charge q):
    rho_tilde_k = (q / L^3) sum_j exp(-i k.x_j)  (eq. scatter_pif without S_k)."""
    rho_tilde = (q / L ** 3) * nudft_type1(x, np.ones(x.shape[1]), N, L)
    E, E_k = field_from_rho_tilde(rho_tilde, x, N, L, order)
    return FieldSolve(E=E, rho_tilde=rho_tilde, E_k=E_k)


# --------------------------------------------------------------------------
# CIC particle-in-cell field solve
# --------------------------------------------------------------------------
def cic_weights(x: np.ndarray, Ng: int, L: float):
    """Linear B-spline (cloud-in-cell) weights; nodes at p*h, h = L/Ng [R14].

    Returns (i0, i1, w0, w1), each (3, N_p): node indices i, i+1 (mod Ng) and
    weights 1-f, f per dimension."""
    h = L / Ng
    s = x / h
    i = np.floor(s)
    f = s - i
    i0 = np.mod(i.astype(np.int64), Ng)
    i1 = np.mod(i0 + 1, Ng)
    return i0, i1, 1.0 - f, f


def cic_deposit(x: np.ndarray, Ng: int, L: float, q: float) -> np.ndarray:
    """rho_p = (q / h^3) sum_j W_pj ("scatter")."""
    h = L / Ng
    i0, i1, w0, w1 = cic_weights(x, Ng, L)
    rho = np.zeros((Ng, Ng, Ng))
    for cx in (0, 1):
        for cy in (0, 1):
            for cz in (0, 1):
                ix = i1[0] if cx else i0[0]
                iy = i1[1] if cy else i0[1]
                iz = i1[2] if cz else i0[2]
                wt = (w1[0] if cx else w0[0]) * (w1[1] if cy else w0[1]) * (w1[2] if cz else w0[2])
                np.add.at(rho, (ix, iy, iz), wt)
    return rho * (q / h ** 3)


def pic_grid_field(rho: np.ndarray, L: float) -> np.ndarray:
    """FFT Poisson solve on the grid [R15]:
    rho_hat = DFT(rho); E_hat_d = -i k_d rho_hat / |k|^2 with k = 2 pi m / L,
    E_hat = 0 at k = 0 and on every plane with some m_d = -Ng/2 (Nyquist);
    E = inverse DFT (normalised).  Returns E on nodes, shape (3, Ng, Ng, Ng)."""
    Ng = rho.shape[0]
    m = np.rint(np.fft.fftfreq(Ng) * Ng).astype(np.int64)
    k = 2.0 * math.pi * m / L
    kx, ky, kz = np.meshgrid(k, k, k, indexing="ij")
    mx, my, mz = np.meshgrid(m, m, m, indexing="ij")
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    keep = (k2 > 0) & (mx != -Ng // 2) & (my != -Ng // 2) & (mz != -Ng // 2)
    rho_hat = np.fft.fftn(rho)
    inv = np.zeros_like(k2)
    inv[keep] = 1.0 / k2[keep]
    E = np.empty((3, Ng, Ng, Ng))
    for d, kd in enumerate((kx, ky, kz)):
        E[d] = np.fft.ifftn(-1j * kd * rho_hat * inv).real
    return E


def cic_gather(Egrid: np.ndarray, x: np.ndarray, L: float) -> np.ndarray:
    """E(x_j) = sum_p W_pj E_p, same weights as the deposit ("gather")."""
    Ng = Egrid.shape[1]
    i0, i1, w0, w1 = cic_weights(x, Ng, L)
    E = np.zeros((3, x.shape[1]))
    for cx in (0, 1):
        for cy in (0, 1):
            for cz in (0, 1):
                ix = i1[0] if cx else i0[0]
                iy = i1[1] if cy else i0[1]
                iz = i1[2] if cz else i0[2]
                wt = (w1[0] if cx else w0[0]) * (w1[1] if cy else w0[1]) * (w1[2] if cz else w0[2])
                for d in range(3):
                    E[d] += wt * Egrid[d][ix, iy, iz]
    return E


def pic_field(x: np.ndarray, Ng: int, L: float, q: float) -> np.ndarray:
    return cic_gather(pic_grid_field(cic_deposit(x, Ng, L, q), L), x, L)


# --------------------------------------------------------------------------
# Push: KDK velocity Verlet / Boris [R7][R8]
# --------------------------------------------------------------------------
def wrap(x: np.ndarray, L: float) -> np.ndarray:
    """Periodic wrap into [0, L): x - L floor(x / L), with L itself mapped to 0."""
    y = x - L * np.floor(x / L)
    return np.where(y >= L, 0.0, y)


def external_field(x: np.ndarray, A, c) -> np.ndarray:
    """E_ext(x) = A x + c (Penning quadrupole, eq. penning_ext_efield)."""
    A = np.asarray(A, dtype=np.float64).reshape(3, 3)
    return A @ x + np.asarray(c, dtype=np.float64)[:, None]


def kick_half(v: np.ndarray, E: np.ndarray, dt: float, q_over_m: float, B) -> np.ndarray:
    """Boris step of size dt/2 (half-kick) with electric field E and constant B [R7]:
    v- = v + (dt/4) a E; t = (dt/4) a B; s = 2t/(1+|t|^2);
    v' = v- + v- x t; v+ = v- + v' x s; return v+ + (dt/4) a E   (a = q/m).
    With B = 0 this is the velocity-Verlet half kick v + (dt/2) a E."""
    h = 0.25 * dt * q_over_m
    vm = v + h * E
    t = h * np.asarray(B, dtype=np.float64)
    if not np.any(t):
        return vm + h * E
    s = 2.0 * t / (1.0 + t @ t)
    vp = vm + np.cross(vm, t, axis=0)
    vplus = vm + np.cross(vp, s, axis=0)
    return vplus + h * E


@dataclass
class Propagator:
    """One propagator: 'pif' (exact NUDFT PIF with N modes) or 'pic' (CIC, Ng=N)."""
    kind: str
    N: int
    dt: float
    order: int = 1


@dataclass
class PhysicsParams:
    L: float
    q_over_m: float
    total_charge: float
    B: tuple = (0.0, 0.0, 0.0)
    A: tuple = (0.0,) * 9
    c: tuple = (0.0, 0.0, 0.0)

    @classmethod
    def from_inputs(cls, p):
        return cls(L=p.L, q_over_m=p.q_over_m, total_charge=p.total_charge,
                   B=tuple(p.B), A=tuple(p.A), c=tuple(p.c))


def particle_charge_mass(phys: PhysicsParams, n_particles: int):
    """q = Q_e / N_p, m = |Q_e| / N_p  [R6] (so q/m = -1 in normalised units)."""
    return phys.total_charge / n_particles, abs(phys.total_charge) / n_particles


def total_field(x: np.ndarray, prop: Propagator, phys: PhysicsParams, n_global=None):
    """E_tot = E_sc + E_ext at x [R8]."""
    n = x.shape[1] if n_global is None else n_global
    q, _ = particle_charge_mass(phys, n)
    if prop.kind == "pif":
        Esc = pif_field(x, prop.N, phys.L, q, prop.order).E
    elif prop.kind == "pic":
        Esc = pic_field(x, prop.N, phys.L, q)
    else:
        raise ValueError(prop.kind)
    return Esc + external_field(x, phys.A, phys.c)


def run(x: np.ndarray, v: np.ndarray, n_steps: int, prop: Propagator, phys: PhysicsParams,
        trace=None):
    """n_steps of Strang KDK [R7]:
    v <- K_half(v, E(x_n)); x <- wrap(x + dt v); v <- K_half(v, E(x_{n+1})).
    E(x_{n+1}) of the closing kick is reused as E(x_n) of the next opening kick
    (same positions, same field -- velocity Verlet).  Returns new (x, v)."""
    x = x.copy()
    v = v.copy()
    if n_steps == 0:
        return x, v
    E = total_field(x, prop, phys)
    for s in range(n_steps):
        v = kick_half(v, E, prop.dt, phys.q_over_m, phys.B)
        x = wrap(x + prop.dt * v, phys.L)
        E = total_field(x, prop, phys)
        v = kick_half(v, E, prop.dt, phys.q_over_m, phys.B)
        if trace is not None:
            trace(s + 1, x, v)
    return x, v


# --------------------------------------------------------------------------
# Diagnostics [R9]
# --------------------------------------------------------------------------
def field_energy(E_k: np.ndarray, L: float) -> np.ndarray:
    """W_d = (L^3 / 2) sum_{k in K_N} |E_{d,k}|^2, d = x, y, z  [R9]."""
    return 0.5 * L ** 3 * np.sum(np.abs(E_k) ** 2, axis=(1, 2, 3))


def kinetic_energy(v: np.ndarray, m: float) -> float:
    return 0.5 * m * float(np.sum(v * v))


def momentum(v: np.ndarray, m: float) -> np.ndarray:
    return m * v.sum(axis=1)


def diagnostics(x, v, prop: Propagator, phys: PhysicsParams):
    """(W[3], kinetic, momentum[3], charge_err) of a PIF state.
    charge_err = |L^3 rho_tilde_0 - Q_e| / |Q_e|, which is 0 up to rounding for
    the exact NUDFT (the NUFFT's k = 0 mode carries its tolerance error)."""
    q, m = particle_charge_mass(phys, x.shape[1])
    fs = pif_field(x, prop.N, phys.L, q, prop.order)
    N = prop.N
    rho0 = fs.rho_tilde[N // 2, N // 2, N // 2]
    cerr = abs(phys.L ** 3 * rho0.real - phys.total_charge) / abs(phys.total_charge)
    return field_energy(fs.E_k, phys.L), kinetic_energy(v, m), momentum(v, m), cerr


# --------------------------------------------------------------------------
# Parareal, serial (eq. parareal_correction; PAPER.md:371-376,
# eq. stop_criteria; PAPER.md:692-693 local exit) [R16][R17][R18]
# --------------------------------------------------------------------------
def min_image(d: np.ndarray, L: float) -> np.ndarray:
    return d - L * np.rint(d / L)


@dataclass
class PararealResult:
    U: list            # U_0 .. U_Ns, each (x, v)
    iterations: int
    retired_at: list   # iteration (1-based) after which slice n retired, or -1
    err_x: list        # per iteration: list of e_x(n) (nan if slice frozen)
    err_v: list


def parareal_serial(u0, F, G, n_slices: int, max_iter: int, tol: float, L=None):
    """Parareal exactly as eq. parareal_correction applied to u = {x, v}:

      iteration 0 (coarse sweep): U_0 = u0, U_{n+1} = G(U_n)
      iteration k = 0, 1, ...:
        Fk_n = F(U_n^k) for every non-retired slice          ("in parallel")
        serially over n:  Gnew_n = G(U_n^{k+1})
                          U_{n+1}^{k+1} = Fk_n + Gnew_n - Gold_n   (x wrapped [R17])
                          e_x = |mi(Gnew.x - Gold.x)|_2 / |Gnew.x|_2, e_v likewise
                          retire n if e_x, e_v <= tol and (n == 0 or n-1 retired)
                          Gold_n <- Gnew_n
      stop when all slices retired or after max_iter iterations.
    Retired slices are frozen (their U_{n+1} no longer changes) [R18].
    F, G map (x, v) -> (x, v).  L = None disables wrap / minimum image (used to
    test the recursion on linear scalar propagators)."""
    def combine(f, gn, go):
        x = f[0] + gn[0] - go[0]
        v = f[1] + gn[1] - go[1]
        if L is not None:
            x = wrap(x, L)
        return (x, v)

    def rel(new, old, img):
        # eq. stop_criteria: |G(u^{k+1}) - G(u^k)|_2 / |G(u^{k+1})|_2
        d = new - old
        if img and L is not None:
            d = min_image(d, L)
        den = np.linalg.norm(new)
        return float(np.linalg.norm(d) / den) if den > 0 else float(np.linalg.norm(d))

    U = [None] * (n_slices + 1)
    U[0] = (u0[0].copy(), u0[1].copy())
    Gold = [None] * n_slices
    for n in range(n_slices):
        Gold[n] = G(U[n])
        U[n + 1] = Gold[n]
    retired = [False] * n_slices
    retired_at = [-1] * n_slices
    errx, errv = [], []
    it = 0
    for k in range(max_iter):
        if all(retired):
            break
        it = k + 1
        Fk = {n: F(U[n]) for n in range(n_slices) if not retired[n]}
        ex_row = [float("nan")] * n_slices
        ev_row = [float("nan")] * n_slices
        for n in range(n_slices):
            if retired[n]:
                continue
            Gnew = G(U[n])
            U[n + 1] = combine(Fk[n], Gnew, Gold[n])
            ex_row[n] = rel(Gnew[0], Gold[n][0], True)
            ev_row[n] = rel(Gnew[1], Gold[n][1], False)
            Gold[n] = Gnew
            if ex_row[n] <= tol and ev_row[n] <= tol and (n == 0 or retired[n - 1]):
                retired[n] = True
                retired_at[n] = it
        errx.append(ex_row)
        errv.append(ev_row)
    return PararealResult(U=U, iterations=it, retired_at=retired_at, err_x=errx, err_v=errv)


def parareal_blocks(u0, make_F, make_G, n_slices: int, n_blocks: int, max_iter: int, tol: float,
                    L=None):
    """Multi-block (windowed) parareal (reading R22): the time
    domain is cut into n_blocks equal windows solved one after the other, each by
    parareal_serial with n_slices slices; a window's U_{n_slices} seeds the next.
    make_F / make_G: window index -> propagator (the slice length is the same
    for every window).  Returns the list of per-window PararealResults."""
    out = []
    u = u0
    for b in range(n_blocks):
        res = parareal_serial(u, make_F(b), make_G(b), n_slices, max_iter, tol, L)
        out.append(res)
        u = res.U[n_slices]
    return out


def make_propagator_fn(prop: Propagator, phys: PhysicsParams, n_steps: int):
    """(x, v) -> run(x, v, n_steps) for parareal."""
    return lambda u: run(u[0], u[1], n_steps, prop, phys)
