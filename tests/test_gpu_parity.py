"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star):
* NUFFT type-1 / type-2 relative L2 error vs the direct NUDFT <= 10 eps;
* positions, velocities, field energy <= 1e-10 relative after 20 fine steps;
* CIC-PIC (an exact algorithm on both sides) <= 1e-12 after 20 steps;
* momentum drift <= 1e-13 sum m|v|.
"""
import math

import numpy as np
import pytest

import oracle as O
from dispersion import dispersion_root
from pif_inputs import landau_physics, landau_state, penning_physics, penning_state, tsi_physics, tsi_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2407_00485_b200 as P  # noqa: E402


def sim_for(phys, fine, coarse=None, n=1):
    return P.Simulation(P.physics(phys.L, phys.q_over_m, phys.total_charge, phys.B, phys.A, phys.c),
                        fine, coarse, n_particles=n)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ------------------------------------------------------------ transforms ---
@pytest.mark.parametrize("tol", [1e-12, 1e-7, 1e-4])
@pytest.mark.parametrize("signed", [False, True])
def test_type1_vs_nudft_C1(tol, signed):
    """C1 inputs (Landau, 8^3 modes, 16384 particles)."""
    phys = landau_physics()
    x, _ = landau_state(16384, 0)
    s = np.random.default_rng(1).standard_normal(16384) if signed else np.ones(16384)
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=tol), n=16384)
    got = P.pif_debug_type1(sim.ctx, 0, x, s, 8)
    ref = O.nudft_type1(x, s, 8, phys.L)
    assert rel_l2(got, ref) <= 10 * tol


@pytest.mark.parametrize("tol", [1e-12, 1e-7, 1e-4, 1e-3, 1e-2])  # w = 13, 8, 5, 4, 3
def test_type2_vs_nudft_C1(tol):
    phys = landau_physics()
    x, _ = landau_state(16384, 0)
    rng = np.random.default_rng(2)
    c = rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8))
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=tol), n=16384)
    got = P.pif_debug_type2(sim.ctx, 0, c, x)
    ref = O.nudft_type2(c, x, 8, phys.L)
    assert rel_l2(got, ref) <= 10 * tol


@pytest.mark.parametrize("tol", [1e-7, 1e-4])
def test_type1_type2_dense_tiles(tol):
    """>= 12 particles per upsampled cell (16^3 grid) selects the small dense tiles
    (interp 10x10x8 / 6x6x8); ragged count."""
    phys = landau_physics()
    npart = 16 * 16 ** 3 + 7
    x, _ = landau_state(npart, 5)
    rng = np.random.default_rng(5)
    s = rng.standard_normal(npart)
    c = rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8))
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=tol), n=npart)
    assert sim.plan_info(0)[2] == 16
    assert rel_l2(P.pif_debug_type1(sim.ctx, 0, x, s, 8), O.nudft_type1(x, s, 8, phys.L)) <= 10 * tol
    assert rel_l2(P.pif_debug_type2(sim.ctx, 0, c, x), O.nudft_type2(c, x, 8, phys.L)) <= 10 * tol


@pytest.mark.parametrize("N,npart", [(2, 1), (6, 37), (16, 5000), (32, 20000)])
def test_type1_type2_ragged_and_edge_sizes(N, npart):
    """Tiny / ragged particle counts, N = 2 (only Nyquist and k=0), larger N."""
    phys = penning_physics()
    rng = np.random.default_rng(N)
    x = rng.random((3, npart)) * phys.L
    x[:, 0] = [0.0, phys.L * (1 - 1e-16), phys.L / 2]  # edge positions
    s = rng.standard_normal(npart)
    c = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    sim = sim_for(phys, P.propagator("pif", N, 0.01, tol=1e-12), n=npart)
    assert rel_l2(P.pif_debug_type1(sim.ctx, 0, x, s, N), O.nudft_type1(x, s, N, phys.L)) <= 1e-11
    assert rel_l2(P.pif_debug_type2(sim.ctx, 0, c, x), O.nudft_type2(c, x, N, phys.L)) <= 1e-11


def test_type1_type2_adjoint_pair():
    """The GPU type-1/type-2 pair is adjoint to rounding (same kernel, w, n, psi^):
    the basis of momentum conservation at any eps."""
    phys = landau_physics()
    rng = np.random.default_rng(3)
    x = rng.random((3, 3000)) * phys.L
    s = rng.standard_normal(3000)
    c = rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8))
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=1e-4), n=3000)
    lhs = np.real(np.vdot(c, P.pif_debug_type1(sim.ctx, 0, x, s, 8)))
    rhs = float(s @ P.pif_debug_type2(sim.ctx, 0, c, x))
    assert abs(lhs - rhs) <= 1e-13 * np.abs(s).sum() * np.abs(c).sum()


# ------------------------------------------------------------------- push --
@pytest.mark.parametrize("case", ["landau", "penning"])
@pytest.mark.parametrize("kicks,drift", [(1, 1), (2, 1), (1, 0)])
def test_push_vs_oracle(case, kicks, drift):
    phys = penning_physics() if case == "penning" else landau_physics()
    x, v = (penning_state if case == "penning" else landau_state)(1000, 4)
    E = np.random.default_rng(5).standard_normal((3, 1000))
    sim = sim_for(phys, P.propagator("pif", 8, 0.003125, tol=1e-7), n=1000)
    xg, vg = x.copy(), v.copy()
    P.pif_debug_push(sim.ctx, 0, xg, vg, E, kicks, drift)
    ph = O.PhysicsParams.from_inputs(phys)
    Et = E + O.external_field(x, ph.A, ph.c)
    vr = v
    for _ in range(kicks):
        vr = O.kick_half(vr, Et, 0.003125, ph.q_over_m, ph.B)
    xr = O.wrap(x + 0.003125 * vr, ph.L) if drift else x
    assert np.abs(vg - vr).max() <= 1e-15 * np.abs(vr).max() * 4
    assert np.abs(O.min_image(xg - xr, ph.L)).max() <= 1e-15 * ph.L * 4


# ------------------------------------------------------------- full steps --
def run_gpu(phys, fine, x0, v0, steps, coarse=None, which=0):
    sim = sim_for(phys, fine, coarse, n=x0.shape[1])
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    sim.step(steps, which)
    x, v = sim.get_state()
    W, ke, mom, ce = sim.field_energy()
    return x.cpu().numpy(), v.cpu().numpy(), W, ke, mom, ce, sim


@pytest.mark.parametrize("case,N,npart,dt", [
    ("landau", 8, 16384, 0.05),    # C1
    ("tsi", 8, 4096, 0.05),
    ("penning", 8, 4096, 0.003125),
])
def test_fine_steps_vs_oracle(case, N, npart, dt):
    """20 fine PIF steps (tol 1e-12) vs the exact NUDFT PIF: x, v, W <= 1e-10 rel."""
    phys = {"landau": landau_physics, "tsi": tsi_physics, "penning": penning_physics}[case]()
    x0, v0 = {"landau": landau_state, "tsi": tsi_state, "penning": penning_state}[case](npart, 0)
    steps = 20
    x, v, W, ke, mom, ce, _ = run_gpu(phys, P.propagator("pif", N, dt, tol=1e-12), x0, v0, steps)
    ph = O.PhysicsParams.from_inputs(phys)
    prop = O.Propagator("pif", N, dt)
    xr, vr = O.run(x0, v0, steps, prop, ph)
    assert np.abs(O.min_image(x - xr, phys.L)).max() <= 1e-10 * phys.L
    assert np.abs(v - vr).max() <= 1e-10 * np.abs(vr).max()
    Wr, ker, momr, cer = O.diagnostics(xr, vr, prop, ph)
    assert np.all(np.abs(W - Wr) <= 1e-10 * Wr.sum())
    assert abs(ke - ker) <= 1e-10 * ker
    assert ce <= 1e-10


@pytest.mark.parametrize("tol", [1e-12, 1e-7])  # brick / dense warp-owned + 1-row slab tiles
def test_steps_interleaved_with_diagnostics_vs_oracle(tol):
    """Steps with a diagnostic after each one: the field-only solve of
    field_energy (no push: the gather sort) alternates with pushing steps (sort
    fused into spread and interp+push); the state after 8 steps and
    every W match the exact oracle (tolerance 10 eps on the field-driven
    change, as test_dense_tiles_steps_vs_oracle)."""
    phys = landau_physics()
    n, N, dt, K = 16 * 16 ** 3 + 5, 8, 0.05, 8
    x0, v0 = landau_state(n, 71)
    sim = sim_for(phys, P.propagator("pif", N, dt, tol=tol), n=n)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    ph = O.PhysicsParams.from_inputs(phys)
    prop = O.Propagator("pif", N, dt)
    xr, vr = x0, v0
    for _ in range(K):
        sim.step(1)
        W, ke, _, _ = sim.field_energy()
        xr, vr = O.run(xr, vr, 1, prop, ph)
        Wr, ker, _, _ = O.diagnostics(xr, vr, prop, ph)
        # (floor 1e-10: the bound of test_fine_steps_vs_oracle at eps = 1e-12)
        assert np.all(np.abs(W - Wr) <= max(10 * tol, 1e-10) * Wr.sum())
        assert abs(ke - ker) <= max(10 * tol, 1e-10) * ker
    x, v = sim.get_state()
    x, v = x.cpu().numpy(), v.cpu().numpy()
    assert np.linalg.norm(v - vr) <= 10 * tol * np.linalg.norm(vr - v0) + 1e-10 * np.linalg.norm(vr)
    disp_ref = O.min_image(xr - (x0 + K * dt * v0), phys.L)
    assert np.linalg.norm(O.min_image(x - xr, phys.L)) <= (10 * tol * np.linalg.norm(disp_ref)
                                                           + 1e-10 * phys.L * math.sqrt(n))


def test_momentum_conservation_any_tolerance():
    """Momentum drift <= 1e-13 sum m|v| for eps = 1e-4."""
    phys = landau_physics()
    x0, v0 = landau_state(20000, 6)
    for tol in (1e-4, 1e-12):
        x, v, W, ke, mom, ce, sim = run_gpu(phys, P.propagator("pif", 8, 0.05, tol=tol), x0, v0, 50)
        m = abs(phys.total_charge) / 20000
        mom0 = m * v0.sum(axis=1)
        scale = m * np.abs(v0).sum()
        assert np.abs(mom - mom0).max() <= 1e-13 * scale, (tol, mom - mom0)


@pytest.mark.parametrize("Ng", [16, 32, 64])
def test_pic_steps_vs_oracle(Ng):
    """20 CIC-PIC steps (exact algorithm on both sides) <= 1e-12: one z-chunk of
    the shared-memory deposit (16^3), two chunks (32^3, the C5 coarse grid) and
    the global-atomic deposit (64^3)."""
    phys = landau_physics()
    x0, v0 = landau_state(8192, 7)
    x, v, *_ = run_gpu(phys, P.propagator("pic", Ng, 0.05), x0, v0, 20)
    xr, vr = O.run(x0, v0, 20, O.Propagator("pic", Ng, 0.05), O.PhysicsParams.from_inputs(phys))
    assert np.abs(O.min_image(x - xr, phys.L)).max() <= 1e-12 * phys.L
    assert np.abs(v - vr).max() <= 1e-12 * np.abs(vr).max()


def test_fine_then_coarse_switch_and_lazy_kick():
    """Mixed fine/coarse stepping and repeated get_state equal the oracle sequence."""
    phys = landau_physics()
    ph = O.PhysicsParams.from_inputs(phys)
    x0, v0 = landau_state(4096, 8)
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=1e-12), P.propagator("pic", 16, 0.1), n=4096)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    sim.step(3, 0)
    sim.get_state()
    sim.step(2, 1)
    sim.step(2, 0)
    x, v = sim.get_state()
    xr, vr = O.run(x0, v0, 3, O.Propagator("pif", 8, 0.05), ph)
    xr, vr = O.run(xr, vr, 2, O.Propagator("pic", 16, 0.1), ph)
    xr, vr = O.run(xr, vr, 2, O.Propagator("pif", 8, 0.05), ph)
    assert np.abs(O.min_image(x.cpu().numpy() - xr, phys.L)).max() <= 1e-10 * phys.L
    assert np.abs(v.cpu().numpy() - vr).max() <= 1e-10 * np.abs(vr).max()


# --------------------------------------------------------------- parareal --
def test_parareal_matches_oracle_trace_pic_coarse():
    """Serial-schedule parareal on the GPU (F = PIF 1e-12, G = CIC-PIC) vs the
    oracle's parareal: same retirement pattern and per-iteration errors."""
    phys = landau_physics()
    ph = O.PhysicsParams.from_inputs(phys)
    x0, v0 = landau_state(2048, 9)
    Ns, nf, ng = 4, 4, 2
    fine = P.propagator("pif", 8, 0.05, tol=1e-12)
    coarse = P.propagator("pic", 8, 0.1)
    sim = sim_for(phys, fine, coarse, n=2048)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    rep = sim.parareal(0.0, Ns * nf * 0.05, Ns, Ns, 1e-6)
    x, v = sim.get_state()
    F = O.make_propagator_fn(O.Propagator("pif", 8, 0.05), ph, nf)
    G = O.make_propagator_fn(O.Propagator("pic", 8, 0.1), ph, ng)
    ref = O.parareal_serial((x0, v0), F, G, Ns, Ns, 1e-6, L=phys.L)
    assert rep["retired_at"] == ref.retired_at
    assert rep["iterations"] == ref.iterations
    ex_ref = np.array(ref.err_x)
    got = rep["err_x"][: ref.iterations]
    fin = np.isfinite(ex_ref)
    assert np.array_equal(fin, np.isfinite(got))
    assert np.allclose(got[fin], ex_ref[fin], rtol=1e-6, atol=1e-12)
    xs, vs = ref.U[Ns]
    assert np.abs(O.min_image(x.cpu().numpy() - xs, phys.L)).max() <= 1e-9 * phys.L


def test_parareal_tol0_equals_serial_fine():
    """max_iter = N_s, tol = 0: U_Ns equals the GPU serial fine run (<= 1e-12)."""
    phys = landau_physics()
    x0, v0 = landau_state(4096, 10)
    Ns, nf = 4, 3
    fine = P.propagator("pif", 8, 0.05, tol=1e-12)
    coarse = P.propagator("pif", 8, 0.15, tol=1e-4)
    sim = sim_for(phys, fine, coarse, n=4096)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    rep = sim.parareal(0.0, Ns * nf * 0.05, Ns, Ns, 0.0)
    x, v = sim.get_state()
    assert rep["retired_at"] == [1, 2, 3, 4] and rep["converged"]
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    sim.step(Ns * nf)
    xs, vs = sim.get_state()
    dx = O.min_image((x - xs).cpu().numpy(), phys.L)
    assert np.abs(dx).max() <= 1e-12 * phys.L
    assert (v - vs).abs().max().item() <= 1e-12 * vs.abs().max().item()


# ------------------------------------------------------- full-size checks --
def test_C2_full_size_sampled_modes_and_particles():
    """BASELINE configs[1] size (Landau 32^3 modes, 2^21 particles, tol 1e-12) in
    the bench's launch configuration: type-1 on 64 sampled modes against the
    per-mode direct sum, type-2 on 512 sampled particles."""
    phys = landau_physics()
    n = 1 << 21
    x, _ = landau_state(n, 1)
    N = 32
    sim = sim_for(phys, P.propagator("pif", N, 0.05, tol=1e-12), n=n)
    s = np.random.default_rng(11).standard_normal(n)
    got = P.pif_debug_type1(sim.ctx, 0, x, s, N)
    rng = np.random.default_rng(12)
    idx = rng.integers(0, N, size=(64, 3))
    k = 2 * math.pi / phys.L * (idx - N // 2)
    ref = np.array([np.sum(s * np.exp(-1j * (kk @ x))) for kk in k])
    g = got[idx[:, 0], idx[:, 1], idx[:, 2]]
    assert rel_l2(g, ref) <= 10 * 1e-12
    c = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    sel = rng.choice(n, 512, replace=False)
    out = P.pif_debug_type2(sim.ctx, 0, c, x)
    assert rel_l2(out[sel], O.nudft_type2(c, x[:, sel], N, phys.L)) <= 10 * 1e-12


# --------------------------------------------------- next rows --
def test_order7_bspline_fine_steps_vs_oracle():
    """f2: order-7 B-spline shape S_k = prod sinc^8(k h / 2)."""
    phys = landau_physics()
    x0, v0 = landau_state(4096, 13)
    x, v, W, ke, mom, ce, _ = run_gpu(phys, P.propagator("pif", 8, 0.05, tol=1e-12, spline_order=7),
                                      x0, v0, 20)
    xr, vr = O.run(x0, v0, 20, O.Propagator("pif", 8, 0.05, order=7), O.PhysicsParams.from_inputs(phys))
    assert np.abs(O.min_image(x - xr, phys.L)).max() <= 1e-10 * phys.L
    assert np.abs(v - vr).max() <= 1e-10 * np.abs(vr).max()


def test_multiblock_parareal_matches_oracle():
    """f1: 3 windows x 2 slices (serial schedule) vs oracle.parareal_blocks: last
    window's retirement / errors and the final state."""
    phys = landau_physics()
    ph = O.PhysicsParams.from_inputs(phys)
    x0, v0 = landau_state(2048, 14)
    Ns, B, nf, ng = 2, 3, 2, 1
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=1e-12), P.propagator("pic", 8, 0.1), n=2048)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    T = B * Ns * nf * 0.05
    rep = sim.parareal(0.0, T, Ns, Ns, 1e-6, n_blocks=B)
    x, v = sim.get_state()
    F = lambda b: O.make_propagator_fn(O.Propagator("pif", 8, 0.05), ph, nf)
    G = lambda b: O.make_propagator_fn(O.Propagator("pic", 8, 0.1), ph, ng)
    ref = O.parareal_blocks((x0, v0), F, G, Ns, B, Ns, 1e-6, L=phys.L)
    assert rep["retired_at"] == ref[-1].retired_at
    assert rep["iterations"] == sum(r.iterations for r in ref)
    xs, vs = ref[-1].U[Ns]
    assert np.abs(O.min_image(x.cpu().numpy() - xs, phys.L)).max() <= 1e-9 * phys.L
    assert np.abs(v.cpu().numpy() - vs).max() <= 1e-9 * np.abs(vs).max()


# ------------------------------------------------------------------ physics --
def _resonant_energy(sim, N, L, q):
    rho = P.pif_get_rho(sim.ctx, N)
    k1 = 2 * math.pi / L
    S = (math.sin(k1 * (L / N) / 2) / (k1 * (L / N) / 2)) ** 2
    r = rho[N // 2, N // 2, 1]  # mode (0, 0, +k1); its partner has the same modulus
    return L ** 3 * S ** 2 * abs(r) ** 2 / k1 ** 2  # (L^3/2)(|E_+|^2 + |E_-|^2), R9


def test_landau_damping_rate_C2():
    """Physics: C2 (Landau, 32^3 modes, 2^21 particles, eps 1e-12, dt 0.05): the
    resonant E_z energy ~ e^{2 gamma t} cos^2(omega t + phi) with (omega, gamma) the
    shape-corrected root (N = 32: 1.41322 - 0.15448 i; BASELINE.json 'about
    -0.1533' is the N -> inf limit).  gamma +-10 %, omega +-2 % (R11)."""
    from scipy.optimize import curve_fit
    phys = landau_physics()
    n, N, dt = 1 << 21, 32, 0.05
    x0, v0 = landau_state(n, 1)
    sim = sim_for(phys, P.propagator("pif", N, dt, tol=1e-12), n=n)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    ts, ws = [], []
    for s in range(241):
        if s:
            sim.step(1)
        ts.append(s * dt)
        ws.append(_resonant_energy(sim, N, phys.L, phys.total_charge / n))
    t, W = np.array(ts), np.array(ws)
    root = dispersion_root(N, phys.L, 0.5, 1.4 - 0.15j)
    assert abs(root.real - 1.41322) < 2e-4 and abs(root.imag + 0.15448) < 2e-4
    sel = t >= 1.0

    def model(t, lnA, g, w, ph, lnC):
        return np.log(np.exp(lnA + 2 * g * t) * np.cos(w * t + ph) ** 2 + np.exp(lnC))

    p0 = [math.log(W[0]), root.imag, root.real, 0.0, math.log(W[0]) - 8]
    p, _ = curve_fit(model, t[sel], np.log(W[sel]), p0=p0, maxfev=20000)
    assert abs(abs(p[2]) - root.real) < 0.02 * root.real, (p, root)
    assert abs(p[1] - root.imag) < 0.10 * abs(root.imag), (p, root)


def test_two_stream_growth_rate_C3():
    """Physics: C3 (TSI, 32^3 modes, 2^23 particles): resonant-mode energy grows as
    e^{2 gamma t}, gamma = shape-corrected root (N = 32: 0.31615).  The growing mode
    beats with stable modes excited by the cos(wz) perturbation (ln W oscillates by
    ~2), so the slope is the least-squares fit of ln W over t in [6, 17] (several
    beat periods, before saturation near t = 19), +-10 % (R11)."""
    phys = tsi_physics()
    n, N, dt = 1 << 23, 32, 0.05
    x0, v0 = tsi_state(n, 2)
    sim = sim_for(phys, P.propagator("pif", N, dt, tol=1e-12), n=n)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    ts, ws = [], []
    for s in range(341):
        if s:
            sim.step(1)
        if s * dt >= 6.0:
            ts.append(s * dt)
            ws.append(_resonant_energy(sim, N, phys.L, phys.total_charge / n))
    slope = np.polyfit(np.array(ts), np.log(np.array(ws)), 1)[0] / 2
    root = dispersion_root(N, phys.L, 0.5, 0.3j, sigma=0.1, vb=math.pi / 2)
    assert abs(root.imag - 0.31615) < 2e-3, root
    assert abs(slope - root.imag) < 0.10 * root.imag, (slope, root)


def test_error_paths():
    """pif_status behaviour on the GPU: non-finite input -> PIF_ERR_NUMERIC (state
    rejected); step before set_state -> PIF_ERR_STATE; n_local mismatch -> ARG;
    parareal interval not a multiple of dt -> CONFIG."""
    phys = landau_physics()
    x0, v0 = landau_state(1000, 15)
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=1e-7), P.propagator("pic", 8, 0.1), n=1000)
    with pytest.raises(P.PifError) as e:
        sim.step(1)
    assert e.value.status == 7
    bad = v0.copy()
    bad[1, 17] = np.nan
    with pytest.raises(P.PifError) as e:
        sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(bad).cuda())
    assert e.value.status == 3
    with pytest.raises(P.PifError) as e:
        sim.step(1)  # the rejected state was not installed
    assert e.value.status == 7
    with pytest.raises(P.PifError) as e:
        P.pif_set_state(sim.ctx, torch.from_numpy(x0[:, :999].copy()).cuda(),
                        torch.from_numpy(v0[:, :999].copy()).cuda())
    assert e.value.status == 1
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    with pytest.raises(P.PifError) as e:
        sim.parareal(0.0, 0.33, 2, 2, 1e-6)
    assert e.value.status == 2
    sim.step(2)
    x, v = sim.get_state()
    assert torch.isfinite(x).all() and torch.isfinite(v).all()


# ------------------------------------------ round-2 parity gaps --
def _cluster_state(n, L, center, sigma, frac, seed):
    """Penning-like crowded cloud: a fraction `frac` of the particles in a tight
    Gaussian (sigma in length units) around `center`, the rest uniform."""
    rng = np.random.default_rng(seed)
    m = int(frac * n)
    x = np.empty((3, n))
    x[:, :m] = np.mod(center + sigma * rng.standard_normal((3, m)), L)
    x[:, m:] = rng.random((3, n - m)) * L
    v = rng.standard_normal((3, n))
    return x, v


def test_crowded_bricks_item_splitting():
    """Work-item splitting of crowded bricks (Sched: > kSpreadItem = 4096 particles
    per spreading brick, > kInterpItem = 1024 per interpolation sub-brick, the C4
    Penning-core regime): 2^17 particles, 85 % of them in a cloud of sigma = 0.4
    (about half an upsampled cell, n = 32) -- type-1 / type-2 within 10 eps and 20
    Boris steps within 1e-10 of the exact NUDFT oracle."""
    phys = penning_physics()
    n, N, tol = 1 << 17, 8, 1e-12
    x, v = _cluster_state(n, phys.L, phys.L / 2, 0.4, 0.85, 21)
    h = phys.L / 32  # upsampled cell (w = 13 -> n = 32)
    cells = np.floor(x / h).astype(int)
    sub = cells // np.array([2, 2, 4])[:, None]   # interpolation sub-bricks (2x2x4 cells)
    brk = cells // 4                               # spreading bricks (4^3 cells)
    assert np.unique(sub, axis=1, return_counts=True)[1].max() > 2 * 1024
    assert np.unique(brk, axis=1, return_counts=True)[1].max() > 2 * 4096
    sim = sim_for(phys, P.propagator("pif", N, 0.003125, tol=tol), n=n)
    assert sim.plan_info(0)[2] == 32
    s = np.random.default_rng(22).standard_normal(n)
    assert rel_l2(P.pif_debug_type1(sim.ctx, 0, x, s, N), O.nudft_type1(x, s, N, phys.L)) <= 10 * tol
    c = np.random.default_rng(23).standard_normal((N, N, N)) + 1j * np.random.default_rng(24).standard_normal((N, N, N))
    assert rel_l2(P.pif_debug_type2(sim.ctx, 0, c, x), O.nudft_type2(c, x, N, phys.L)) <= 10 * tol
    sim.close()
    xg, vg, W, ke, mom, ce, _ = run_gpu(phys, P.propagator("pif", N, 0.003125, tol=tol), x, v, 20)
    xr, vr = O.run(x, v, 20, O.Propagator("pif", N, 0.003125), O.PhysicsParams.from_inputs(phys))
    assert np.abs(O.min_image(xg - xr, phys.L)).max() <= 1e-10 * phys.L
    assert np.abs(vg - vr).max() <= 1e-10 * np.abs(vr).max()


def test_C4_full_size_sampled_modes_and_particles():
    """BASELINE configs[3] size (Penning, 64^3 modes, upsampled n = 128, 2^24
    particles, tol 1e-12) in the bench's launch configuration (--config 3):
    type-1 on 16 sampled modes against per-mode direct sums, type-2 on 512
    sampled particles, both within 10 eps.  The C4 cloud core (~1300 particles
    per upsampled cell) also exercises the crowded-brick item splitting."""
    phys = penning_physics()
    n, N, tol = 1 << 24, 64, 1e-12
    x, _ = penning_state(n, 3)
    sim = sim_for(phys, P.propagator("pif", N, 0.003125, tol=tol), n=n)
    assert sim.plan_info(0)[2] == 128
    s = np.random.default_rng(31).standard_normal(n)
    got = P.pif_debug_type1(sim.ctx, 0, x, s, N)
    rng = np.random.default_rng(32)
    idx = rng.integers(0, N, size=(16, 3))
    k = 2 * math.pi / phys.L * (idx - N // 2)
    ref = np.array([np.sum(s * np.exp(-1j * (kk @ x))) for kk in k])
    assert rel_l2(got[idx[:, 0], idx[:, 1], idx[:, 2]], ref) <= 10 * tol
    del got
    c = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    sel = rng.choice(n, 512, replace=False)
    out = P.pif_debug_type2(sim.ctx, 0, c, x)
    assert rel_l2(out[sel], O.nudft_type2(c, x[:, sel], N, phys.L)) <= 10 * tol


@pytest.mark.parametrize("tol,w", [(1e-7, 8), (1e-4, 5)])
def test_dense_tiles_steps_vs_oracle(tol, w):
    """The dense slab tiles (w = 8: 10x10x8, w = 5: 6x6x8; chosen at >= 12 / 8
    particles per upsampled cell) through pif_step: 16 particles per cell on the
    16^3 grid (N = 8), 5 Landau steps of dt = 0.05 against the exact oracle.
    Tolerance from the NUFFT bound: each kick's field has relative L2 error
    <= 10 eps (R20), so the velocity change Dv = sum_k dt E_k has relative error
    <= 10 eps * sum_k |E_k| / |sum_k E_k| (~1: the field barely turns in 5 dt =
    0.25 << the plasma period 4.4), and the field-driven displacement
    x - (x0 + K dt v0) likewise; trajectory feedback is second order.  Written
    bound: 2 x 10 eps on both."""
    phys = landau_physics()
    n, N, dt, K = 16 * 16 ** 3, 8, 0.05, 5
    x0, v0 = landau_state(n, 41)
    sim = sim_for(phys, P.propagator("pif", N, dt, tol=tol), n=n)
    assert sim.plan_info(0)[0] == w and sim.plan_info(0)[2] == 16
    sim.close()
    x, v, *_ = run_gpu(phys, P.propagator("pif", N, dt, tol=tol), x0, v0, K)
    xr, vr = O.run(x0, v0, K, O.Propagator("pif", N, dt), O.PhysicsParams.from_inputs(phys))
    dv_ref = vr - v0
    assert np.linalg.norm(v - vr) <= 2 * 10 * tol * np.linalg.norm(dv_ref)
    disp_ref = O.min_image(xr - (x0 + K * dt * v0), phys.L)
    assert np.linalg.norm(O.min_image(x - xr, phys.L)) <= 2 * 10 * tol * np.linalg.norm(disp_ref)


def test_set_state_wraps_positions_outside_the_box():
    """Positions given outside [0, L) (here x + 2L and x - 2L, i.e. 2.5 L and
    -1.5 L for x = L/2) are wrapped periodically by pif_set_state: the state and
    the next steps equal those of the wrapped input."""
    phys = landau_physics()
    x0, v0 = landau_state(4096, 42)
    xs = x0.copy()
    xs[0, ::3] += 2 * phys.L
    xs[1, 1::3] -= 2 * phys.L
    xs[2, 2::5] += 7 * phys.L
    a = run_gpu(phys, P.propagator("pif", 8, 0.05, tol=1e-12), x0, v0, 3)
    b = run_gpu(phys, P.propagator("pif", 8, 0.05, tol=1e-12), xs, v0, 3)
    assert np.abs(O.min_image(a[0] - b[0], phys.L)).max() <= 1e-13 * phys.L
    assert np.abs(a[1] - b[1]).max() <= 1e-13 * np.abs(a[1]).max()
    assert np.all((b[0] >= 0) & (b[0] < phys.L))


# ------------------------------------------ f3: fp32 coarse propagator ------
@pytest.mark.parametrize("tol", [1e-2, 1e-3, 1e-4, 1e-5])  # w = 3, 4, 5, 6
@pytest.mark.parametrize("npart", [16384, 16 * 16 ** 3 + 3])  # sparse / dense tiles
def test_fp32_type2_vs_nudft(tol, npart):
    """PIF_FLAG_FP32: the fp32 interpolation is within 10 eps of the
    exact NUDFT (fp32 rounding ~1e-7 relative << 10 eps for eps >= 1e-5)."""
    phys = landau_physics()
    x, _ = landau_state(npart, 51)
    rng = np.random.default_rng(52)
    c = rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8))
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=tol, fp32=True), n=npart)
    got = P.pif_debug_type2(sim.ctx, 0, c, x)
    ref = O.nudft_type2(c, x, 8, phys.L)
    err = rel_l2(got, ref)
    assert err <= 10 * tol
    assert err > 1e-9  # it really ran in single precision


@pytest.mark.parametrize("tol", [1e-3, 1e-4, 1e-5])  # w = 4, 5, 6
@pytest.mark.parametrize("npart", [16384, 16 * 16 ** 3 + 3])  # sparse / dense tiles
def test_fp32_type1_vs_nudft(tol, npart):
    """PIF_FLAG_FP32 type-1 (the spread accumulates in fp64; on the dense
    warp-owned tiles its ES weights come from the fp32 Horner chains) within
    10 eps of the exact NUDFT, signed strengths, ragged count."""
    phys = landau_physics()
    x, _ = landau_state(npart, 54)
    s = np.random.default_rng(55).standard_normal(npart)
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=tol, fp32=True), n=npart)
    got = P.pif_debug_type1(sim.ctx, 0, x, s, 8)
    assert rel_l2(got, O.nudft_type1(x, s, 8, phys.L)) <= 10 * tol


def test_fp32_coarse_steps_vs_oracle():
    """5 steps of the fp32 coarse propagator (eps_g = 1e-4, dense w = 5 tile) vs
    the exact oracle, with the bound of test_dense_tiles_steps_vs_oracle
    (2 x 10 eps on the field-driven velocity change and displacement)."""
    phys = landau_physics()
    n, N, dt, K, tol = 16 * 16 ** 3, 8, 0.05, 5, 1e-4
    x0, v0 = landau_state(n, 53)
    x, v, *_ = run_gpu(phys, P.propagator("pif", N, dt, tol=tol, fp32=True), x0, v0, K)
    xr, vr = O.run(x0, v0, K, O.Propagator("pif", N, dt), O.PhysicsParams.from_inputs(phys))
    assert np.linalg.norm(v - vr) <= 2 * 10 * tol * np.linalg.norm(vr - v0)
    disp_ref = O.min_image(xr - (x0 + K * dt * v0), phys.L)
    assert np.linalg.norm(O.min_image(x - xr, phys.L)) <= 2 * 10 * tol * np.linalg.norm(disp_ref)


def test_fp32_flag_rejected_below_1e5():
    phys = landau_physics()
    with pytest.raises(P.PifError) as e:
        sim_for(phys, P.propagator("pif", 8, 0.05, tol=1e-7, fp32=True), n=100)
    assert e.value.status == 1


@pytest.mark.parametrize("tol", [1e-7, 1e-10])
def test_sparse_tiles_w8_w11(tol):
    """Below 4 particles per upsampled cell, w = 8 keeps the 12^3 tile on the
    per-item kernel; w = 11 (eps 1e-10) runs the 16^3 tile."""
    phys = landau_physics()
    npart = 3000
    x, _ = landau_state(npart, 61)
    rng = np.random.default_rng(62)
    s = rng.standard_normal(npart)
    c = rng.standard_normal((8, 8, 8)) + 1j * rng.standard_normal((8, 8, 8))
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=tol), n=npart)
    assert rel_l2(P.pif_debug_type1(sim.ctx, 0, x, s, 8), O.nudft_type1(x, s, 8, phys.L)) <= 10 * tol
    assert rel_l2(P.pif_debug_type2(sim.ctx, 0, c, x), O.nudft_type2(c, x, 8, phys.L)) <= 10 * tol


def test_repeatability_of_atomic_spread():
    """Reading c21: the spread flushes with fp64 atomics, so two runs
    differ only in summation order -- 20 identical Landau steps agree to ~1e-13
    relative (positions, velocities), not bitwise."""
    phys = landau_physics()
    x0, v0 = landau_state(16384, 71)
    a = run_gpu(phys, P.propagator("pif", 8, 0.05, tol=1e-12), x0, v0, 20)
    b = run_gpu(phys, P.propagator("pif", 8, 0.05, tol=1e-12), x0, v0, 20)
    assert np.abs(O.min_image(a[0] - b[0], phys.L)).max() <= 1e-13 * phys.L
    assert np.abs(a[1] - b[1]).max() <= 1e-13 * np.abs(a[1]).max()


def test_comm_info_single_process():
    """pif_comm_info: communicator sizes are 1 without NCCL (world == 1)."""
    phys = landau_physics()
    sim = sim_for(phys, P.propagator("pif", 8, 0.05, tol=1e-7), n=100)
    assert sim.comm_info() == {"world_nranks": 1, "space_nranks": 1, "time_nranks": 1}
