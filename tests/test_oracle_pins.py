"""Pins of the CPU oracle to things other than itself (CPU only, -m "not gpu").

Each test names the oracle function(s) it pins and what fixes the expected
value: brute force on tiny inputs, a closed form, an invariant the paper
states, or a printed value (tests/golden/paper_constants.txt).
"""
import cmath
import math
import os

import numpy as np
import pytest

import oracle as O
from pif_inputs import landau_physics, landau_state, penning_physics

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_constants.txt")


def golden():
    vals = {}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        name, value, tol = line.split()[:3]
        vals[name] = (float(value), float(tol))
    return vals


L4PI = 4.0 * math.pi


# ---------------------------------------------------------------- NUDFT ----
def test_type1_brute_force():
    """nudft_type1 vs an explicit double loop with the dot-product phase
    exp(-i (kx x + ky y + kz z)) (not the separable product) -- catches index
    order / transposition / sign errors in the factorised contraction."""
    rng = np.random.default_rng(1)
    N, L, n = 4, L4PI, 7
    x = rng.random((3, n)) * L
    s = rng.standard_normal(n)
    got = O.nudft_type1(x, s, N, L)
    m = range(-N // 2, N // 2)
    for ia, a in enumerate(m):
        for ib, b in enumerate(m):
            for ic, c in enumerate(m):
                k = (2 * math.pi / L) * np.array([a, b, c])
                ref = sum(s[j] * cmath.exp(-1j * float(k @ x[:, j])) for j in range(n))
                assert abs(got[ia, ib, ic] - ref) <= 1e-13 * max(1.0, abs(ref))


def test_type2_brute_force():
    rng = np.random.default_rng(2)
    N, L, n = 4, 25.0, 5
    x = rng.random((3, n)) * L
    c = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    got = O.nudft_type2_complex(c, x, N, L)
    m = list(range(-N // 2, N // 2))
    for j in range(n):
        ref = 0j
        for ia, a in enumerate(m):
            for ib, b in enumerate(m):
                for ic, cc in enumerate(m):
                    k = (2 * math.pi / L) * np.array([a, b, cc])
                    ref += c[ia, ib, ic] * cmath.exp(1j * float(k @ x[:, j]))
        assert abs(got[j] - ref) <= 1e-12 * abs(ref)
    assert np.allclose(O.nudft_type2(c, x, N, L), got.real, rtol=0, atol=0)


def test_type2_stacked_coefficients_brute_force():
    """A stack of D coefficient arrays (the field components) at the same
    positions: row d is the brute-force sum for c_d."""
    rng = np.random.default_rng(3)
    N, L, n, D = 4, 7.0, 4, 3
    x = rng.random((3, n)) * L
    c = rng.standard_normal((D, N, N, N)) + 1j * rng.standard_normal((D, N, N, N))
    got = O.nudft_type2_complex(c, x, N, L)
    assert got.shape == (D, n)
    m = list(range(-N // 2, N // 2))
    for d in range(D):
        for j in range(n):
            ref = sum(c[d, ia, ib, ic] * cmath.exp(1j * (2 * math.pi / L) * (a * x[0, j] + b * x[1, j] + cc * x[2, j]))
                      for ia, a in enumerate(m) for ib, b in enumerate(m) for ic, cc in enumerate(m))
            assert abs(got[d, j] - ref) <= 1e-12 * abs(ref)


def test_type1_single_particle_at_origin():
    """A point at x = 0: every exponential is 1."""
    out = O.nudft_type1(np.zeros((3, 1)), np.array([2.5]), 6, L4PI)
    assert np.all(out == 2.5)


def test_type2_zero_mode_only():
    """Spectrum with only the k = 0 coefficient: constant output."""
    N = 6
    c = np.zeros((N, N, N), complex)
    c[N // 2, N // 2, N // 2] = 1.0 - 0.5j
    x = np.random.default_rng(3).random((3, 9)) * L4PI
    assert np.all(O.nudft_type2(c, x, N, L4PI) == 1.0)


def test_adjointness():
    """Re <P s, c> = <s, Re P^H c> for real s (P, P^H of PAPER.md:180-184)."""
    rng = np.random.default_rng(4)
    N, L, n = 6, L4PI, 300
    x = rng.random((3, n)) * L
    s = rng.standard_normal(n)
    c = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    lhs = np.real(np.vdot(c, O.nudft_type1(x, s, N, L)))
    rhs = float(s @ O.nudft_type2(c, x, N, L))
    assert abs(lhs - rhs) <= 1e-12 * np.abs(s).sum() * np.abs(c).sum()


def test_shape_factor_closed_form():
    """S(0) = 1; S at the Nyquist mode k h / 2 = -pi/2 is (2/pi)^(m+1)."""
    for order in (1, 3, 7):
        s = O.shape_factor_1d(8, L4PI, order)
        assert s[4] == 1.0
        assert abs(s[0] - (2 / math.pi) ** (order + 1)) < 1e-15
    s = O.shape_factor_1d(8, L4PI, 1)
    assert np.allclose(s[1:], s[1:][::-1], atol=1e-16)  # even in k


# ------------------------------------------------------------- Poisson -----
def test_single_mode_field_closed_form():
    """rho(z) = a cos(k1 z) (rho_tilde_{+-k1} = a/2): Gauss's law dE/dz = rho gives
    E_z = S_{k1}^2 a sin(k1 z) / k1, E_x = E_y = 0 (poisson_spectral +
    field_from_rho_tilde; pins the sign of -ik/|k|^2 and of exp(+ikx))."""
    N, L, a = 8, L4PI, 0.7
    k1 = 2 * math.pi / L
    rt = np.zeros((N, N, N), complex)
    rt[N // 2, N // 2, N // 2 + 1] = a / 2
    rt[N // 2, N // 2, N // 2 - 1] = a / 2
    z = np.linspace(0, L, 17)
    x = np.stack([np.full_like(z, 1.3), np.full_like(z, 2.9), z])
    E, E_k = O.field_from_rho_tilde(rt, x, N, L)
    S1 = math.sin(k1 * (L / N) / 2) / (k1 * (L / N) / 2)
    Sk = S1 ** 2  # CIC: sinc^2 in z, 1 in x, y
    assert np.allclose(E[2], Sk ** 2 * a * np.sin(k1 * z) / k1, atol=1e-14)
    assert np.allclose(E[:2], 0.0, atol=1e-14)


def test_momentum_invariant():
    """sum_j q E(x_j) = 0 to round-off: P^H L P is anti-Hermitian."""
    rng = np.random.default_rng(5)
    N, L, n = 8, L4PI, 500
    x = rng.random((3, n)) * L
    q = -(L ** 3) / n
    fs = O.pif_field(x, N, L, q)
    scale = np.abs(q) * np.abs(fs.E).sum()
    assert np.all(np.abs(q * fs.E.sum(axis=1)) <= 1e-14 * scale)


def test_two_particles_action_reaction():
    """Two particles: E at 1 due to 2 = -(E at 2 due to 1) (self-force is zero)."""
    N, L = 8, 25.0
    x = np.array([[3.1, 17.2], [8.8, 1.5], [12.0, 20.4]])
    fs = O.pif_field(x, N, L, q=-1.0)
    assert np.allclose(fs.E[:, 0], -fs.E[:, 1], atol=1e-15)
    self_ = O.pif_field(x[:, :1], N, L, q=-1.0).E
    assert np.all(np.abs(self_) < 1e-15)


# ----------------------------------------------------------------- push ----
def test_boris_rotation_closed_form():
    """E = 0, B = (0,0,5), q/m = -1: each Boris half-kick rotates v_perp by
    2 atan(|t|), |t| = (dt/4) B, counter-clockwise (u' = i B u, u = vx + i vy);
    |v| is preserved exactly and v_z is unchanged (kick_half, run)."""
    phys = O.PhysicsParams(L=25.0, q_over_m=-1.0, total_charge=-1e-30, B=(0.0, 0.0, 5.0))
    prop = O.Propagator("pif", 2, 0.05)
    x0 = np.array([[3.0], [4.0], [5.0]])
    v0 = np.array([[0.3], [-1.1], [0.25]])
    n = 40
    _, v = O.run(x0, v0, n, prop, phys)
    ang = n * 4.0 * math.atan(0.05 * 5.0 / 4.0)
    u = (v0[0, 0] + 1j * v0[1, 0]) * cmath.exp(1j * ang)
    assert abs(v[0, 0] - u.real) < 1e-13 and abs(v[1, 0] - u.imag) < 1e-13
    assert v[2, 0] == v0[2, 0]


def _fit_freqs(t, y, w0):
    """Least-squares fit of y(t) = sum_i a_i exp(i w_i t) (+ const) over w (nonlinear)."""
    from scipy.optimize import least_squares

    def resid(w):
        M = np.stack([np.exp(1j * wi * t) for wi in w] + [np.ones_like(t)], axis=1)
        coef, *_ = np.linalg.lstsq(M, y, rcond=None)
        r = M @ coef - y
        return np.concatenate([r.real, r.imag])

    return least_squares(resid, w0, x_scale=0.01).x


def test_penning_single_particle_frequencies():
    """One particle in the Penning external fields (self-force is exactly 0):
    axial omega_z = sqrt(30 |q/m| / L), radial omega_+- = (Omega +- sqrt(Omega^2 -
    2 omega_z^2))/2 with Omega = |q/m| B (u'' = 0.6 u + i B u').  Closed forms,
    also checked against the values printed at PAPER.md:451 (golden file)."""
    p = penning_physics()
    phys = O.PhysicsParams.from_inputs(p)
    dt = 0.005
    prop = O.Propagator("pif", 2, dt)
    x = np.array([[13.0], [12.1], [14.0]])
    v = np.array([[0.4], [0.3], [0.0]])
    ts, zs, us = [], [], []

    def trace(s, xx, vv):
        ts.append(s * dt)
        zs.append(xx[2, 0] - p.L / 2)
        us.append((xx[0, 0] - p.L / 2) + 1j * (xx[1, 0] - p.L / 2))

    O.run(x, v, 6000, prop, phys, trace=trace)
    t = np.array(ts)
    wz_exact = math.sqrt(30.0 / p.L)
    Om = 5.0
    wp = (Om + math.sqrt(Om ** 2 - 2 * wz_exact ** 2)) / 2
    wm = (Om - math.sqrt(Om ** 2 - 2 * wz_exact ** 2)) / 2
    wz = _fit_freqs(t, np.array(zs) + 0j, [1.1, -1.1])
    assert abs(abs(wz[0]) - wz_exact) < 2e-4 * wz_exact
    w = _fit_freqs(t, np.array(us), [4.875, 0.125])
    assert abs(w[0] - wp) < 2e-4 * wp
    assert abs(w[1] - wm) < 2e-3 * wm
    g = golden()
    for name, val in (("penning_omega_plus", wp), ("penning_omega_z", wz_exact),
                      ("penning_omega_minus", wm), ("penning_period_plus", 2 * math.pi / wp),
                      ("penning_period_z", 2 * math.pi / wz_exact)):
        ref, tol = g[name]
        assert abs(val - ref) <= tol * abs(ref), name


def test_energy_error_second_order():
    """Energy KE + sum_d W_d (R9) is conserved to O(dt^2) by KDK:
    halving dt divides the max relative energy error by about 4."""
    phys = O.PhysicsParams.from_inputs(landau_physics())
    x0, v0 = landau_state(400, 11)
    errs = []
    for dt in (0.2, 0.1, 0.05):
        prop = O.Propagator("pif", 4, dt)
        _, m = O.particle_charge_mass(phys, 400)
        energies = []

        def trace(s, xx, vv):
            W, ke, _, _ = O.diagnostics(xx, vv, prop, phys)
            energies.append(ke + W.sum())

        W0, ke0, _, _ = O.diagnostics(x0, v0, prop, phys)
        O.run(x0, v0, int(round(2.0 / dt)), prop, phys, trace=trace)
        e0 = ke0 + W0.sum()
        errs.append(max(abs(e - e0) for e in energies) / e0)
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.0 < r1 < 5.5 and 3.0 < r2 < 5.5, errs


def test_charge_and_momentum_diagnostics():
    """Q_e values printed in the paper (golden) and exact charge of the NUDFT k=0 mode."""
    g = golden()
    assert abs(landau_physics().total_charge - g["landau_total_charge"][0]) <= 1e-9 * 1985
    assert penning_physics().total_charge == g["penning_total_charge"][0]
    phys = O.PhysicsParams.from_inputs(landau_physics())
    x, v = landau_state(1000, 3)
    W, ke, P, cerr = O.diagnostics(x, v, O.Propagator("pif", 4, 0.1), phys)
    assert cerr < 1e-13
    m = abs(phys.total_charge) / 1000
    assert np.allclose(P, m * v.sum(axis=1)) and abs(ke - 0.5 * m * (v * v).sum()) < 1e-9 * ke


# ------------------------------------------------------------------ CIC ----
def test_cic_partition_of_unity_and_single_node():
    rng = np.random.default_rng(6)
    Ng, L, n, q = 8, L4PI, 333, -0.37
    x = rng.random((3, n)) * L
    rho = O.cic_deposit(x, Ng, L, q)
    h = L / Ng
    assert abs(rho.sum() * h ** 3 - q * n) < 1e-12 * abs(q * n)
    one = O.cic_deposit(np.array([[2 * h], [5 * h], [7 * h]]), Ng, L, 1.0)
    assert one[2, 5, 7] == 1.0 / h ** 3 and np.count_nonzero(one) == 1


def test_cic_deposit_gather_adjoint():
    """sum_p rho_p phi_p h^3 = q sum_j gather(phi)(x_j): same weights both ways."""
    rng = np.random.default_rng(7)
    Ng, L, n, q = 8, 25.0, 200, 0.9
    x = rng.random((3, n)) * L
    phi = rng.standard_normal((3, Ng, Ng, Ng))
    rho = O.cic_deposit(x, Ng, L, q)
    lhs = (rho * phi[1]).sum() * (L / Ng) ** 3
    rhs = q * O.cic_gather(phi, x, L)[1].sum()
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)


def test_pic_cosine_closed_form_and_lattice_neutrality():
    """Grid density a cos(2 pi x / L) -> E_x = a sin(2 pi x / L) / k exactly (a
    resolved mode); particles on every node -> uniform rho -> E = 0."""
    Ng, L, a = 16, L4PI, 0.3
    k = 2 * math.pi / L
    xs = np.arange(Ng) * L / Ng
    rho = a * np.cos(k * xs)[:, None, None] * np.ones((1, Ng, Ng))
    E = O.pic_grid_field(rho, L)
    assert np.allclose(E[0], (a * np.sin(k * xs) / k)[:, None, None], atol=1e-14)
    assert np.allclose(E[1:], 0.0, atol=1e-14)
    g = np.stack(np.meshgrid(xs, xs, xs, indexing="ij")).reshape(3, -1)
    Ep = O.pic_field(g, Ng, L, q=-1.0)
    assert np.abs(Ep).max() < 1e-13


# ------------------------------------------------------------- parareal ----
def test_parareal_linear_closed_form():
    """Scalar linear propagators F u = f u, G u = g u: with no retirement the
    parareal iterate is U_n^k = sum_{j<=k} binom(n, j) (f-g)^j g^(n-j) u0
    (truncated binomial expansion of f^n) -- pins eq. parareal_correction."""
    f, g, u0 = 0.9, 0.8, 1.3
    F = lambda u: (u[0] * f, u[1] * f)
    G = lambda u: (u[0] * g, u[1] * g)
    Ns = 6
    for K in range(0, 4):
        res = O.parareal_serial((np.array([u0]), np.array([u0])), F, G, Ns, K, tol=-1.0)
        for n in range(Ns + 1):
            ref = sum(math.comb(n, j) * (f - g) ** j * g ** (n - j) for j in range(min(K, n) + 1)) * u0
            assert abs(res.U[n][0][0] - ref) < 1e-14 and abs(res.U[n][1][0] - ref) < 1e-14


def test_parareal_G_equals_F_converges_in_one_iteration():
    phys = O.PhysicsParams.from_inputs(landau_physics())
    x, v = landau_state(64, 9)
    prop = O.Propagator("pif", 4, 0.1)
    F = O.make_propagator_fn(prop, phys, 2)
    res = O.parareal_serial((x, v), F, F, 4, 4, tol=1e-14, L=phys.L)
    assert res.iterations == 1 and res.retired_at == [1, 1, 1, 1]


def test_parareal_exact_after_Ns_iterations_pic_coarse():
    """tol = 0, max_iter = N_s: slice n retires at iteration n+1 and U_Ns equals the
    serial fine solution (recursion of PAPER.md:154-161)."""
    phys = O.PhysicsParams.from_inputs(landau_physics())
    x, v = landau_state(128, 10)
    Fp = O.Propagator("pif", 4, 0.05)
    Gp = O.Propagator("pic", 4, 0.1)
    Ns = 3
    F = O.make_propagator_fn(Fp, phys, 4)
    G = O.make_propagator_fn(Gp, phys, 2)
    res = O.parareal_serial((x, v), F, G, Ns, Ns, tol=0.0, L=phys.L)
    xs, vs = O.run(x, v, 4 * Ns, Fp, phys)
    assert res.retired_at == [1, 2, 3]
    dx = O.min_image(res.U[Ns][0] - xs, phys.L)
    assert np.abs(dx).max() < 1e-12 * phys.L and np.abs(res.U[Ns][1] - vs).max() < 1e-12


# --------------------------------------------------------------- physics ---
def test_cold_plasma_oscillation_closed_form():
    """Whole-step pin, deterministic: a cold (v = 0) lattice plasma with a small
    sinusoidal displacement z_j = z0_j + delta sin(k z0_j) oscillates at the
    shape-corrected plasma frequency omega = omega_p S(k) (omega_p = 1 for
    q = Q_e/N_p, m = |Q_e|/N_p, Q_e = -L^3: PAPER.md:335 units) -- and KDK turns
    omega into the discrete omega_d with cos(omega_d dt) = 1 - (omega dt)^2 / 2.
    Pins the charge/mass normalisation, S_k^2, the Poisson sign (a wrong sign
    grows exponentially) and the push together (pif_field + run)."""
    N, M, Mz, dt, nsteps = 4, 4, 32, 0.1, 120
    L = L4PI
    phys = O.PhysicsParams(L=L, q_over_m=-1.0, total_charge=-(L ** 3))
    k = 2 * math.pi / L
    g = (np.arange(M) + 0.5) * L / M
    gz = (np.arange(Mz) + 0.5) * L / Mz
    X, Y, Z = np.meshgrid(g, g, gz, indexing="ij")
    z0 = Z.ravel()
    delta = 1e-5 * L
    x = np.stack([X.ravel(), Y.ravel(), z0 + delta * np.sin(k * z0)])
    v = np.zeros_like(x)
    amp = []
    O.run(x, v, nsteps, O.Propagator("pif", N, dt), phys,
          trace=lambda s_, xx, vv: amp.append(
              np.mean(np.sin(k * z0) * O.min_image(xx[2] - z0, L)) * 2 / delta))
    S = O.shape_factor_1d(N, L)[N // 2 + 1]
    wd = math.acos(1 - (S * dt) ** 2 / 2) / dt
    t = dt * np.arange(1, nsteps + 1)
    assert np.max(np.abs(np.array(amp) - np.cos(wd * t))) < 2e-4


def test_parareal_blocks_exact_and_linear():
    """Multi-block parareal: (1) scalar linear propagators -- each window applies
    the truncated binomial expansion to its seed, so after B windows the result is
    (sum_{j<=K} C(Ns,j)(f-g)^j g^(Ns-j))^B u0; (2) tol = 0, K = N_s per window ->
    serial fine over all windows."""
    f, g, u0, Ns, B, K = 0.9, 0.8, 1.3, 3, 2, 1
    F = lambda u: (u[0] * f, u[1] * f)
    G = lambda u: (u[0] * g, u[1] * g)
    res = O.parareal_blocks((np.array([u0]), np.array([u0])), lambda b: F, lambda b: G, Ns, B, K, -1.0)
    per = sum(math.comb(Ns, j) * (f - g) ** j * g ** (Ns - j) for j in range(K + 1))
    assert abs(res[-1].U[Ns][0][0] - per ** B * u0) < 1e-14
    phys = O.PhysicsParams.from_inputs(landau_physics())
    x, v = landau_state(64, 12)
    Fp, Gp = O.Propagator("pif", 4, 0.05), O.Propagator("pic", 4, 0.1)
    res = O.parareal_blocks((x, v), lambda b: O.make_propagator_fn(Fp, phys, 2),
                            lambda b: O.make_propagator_fn(Gp, phys, 1), 2, 3, 2, 0.0, L=phys.L)
    xs, vs = O.run(x, v, 2 * 2 * 3, Fp, phys)
    assert np.abs(O.min_image(res[-1].U[2][0] - xs, phys.L)).max() < 1e-12 * phys.L
    assert np.abs(res[-1].U[2][1] - vs).max() < 1e-12
