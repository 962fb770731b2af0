"""Seeded synthetic inputs for the PIF step (shared by oracle/ and the CUDA path).

This module holds NO arithmetic of the method (no transforms, no field solve,
no push).  It only draws the initial particle states of the paper's three
mini-apps and states their physical parameters:

* Landau damping      -- PAPER.md:331-335 (Sec. "Mini-apps", Landau damping)
* Two-stream (TSI)    -- PAPER.md:337-345 (Sec. "Mini-apps", two-stream)
* Penning trap        -- PAPER.md:347-358 (Sec. "Mini-apps", Penning trap,
                         eq. penning_ext_efield)

Sampling follows PAPER.md:361-362 ("randomly sampled ... by the inverse
transform sampling technique"): per axis, u ~ U[0,1) is pushed through the
inverse of the marginal CDF F(x) = (x + (alpha/w) sin(w x)) / L by Newton
iteration.  RNG: numpy PCG64(seed); draw order x-axis, y, z, v, beam sign
(SURVEY.md Sec. 8c "Initial data").

Layout returned: x, v as float64 arrays of shape (3, N_p) -- SoA, the layout
the C ABI takes (include/pif.h).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Physics",
    "landau_physics",
    "tsi_physics",
    "penning_physics",
    "landau_state",
    "tsi_state",
    "penning_state",
    "landau_state_quiet",
    "tsi_state_quiet",
    "make_case",
    "CONFIGS",
]


@dataclass
class Physics:
    """Physical parameters of a run (normalised units q_e=-1, m_e=1, eps0=1).

    E_ext(x) = A @ x + c ; B_ext constant.  total_charge = Q_e (< 0).
    """

    L: float
    q_over_m: float
    total_charge: float
    B: tuple = (0.0, 0.0, 0.0)
    A: tuple = (0.0,) * 9  # row-major 3x3
    c: tuple = (0.0, 0.0, 0.0)
    name: str = ""

    def as_dict(self):
        return dict(L=self.L, q_over_m=self.q_over_m, total_charge=self.total_charge,
                    B=tuple(self.B), A=tuple(self.A), c=tuple(self.c), name=self.name)


def landau_physics() -> Physics:
    # w = 0.5, L = 2 pi / w, Q_e = -L^3
    L = 2.0 * math.pi / 0.5
    return Physics(L=L, q_over_m=-1.0, total_charge=-(L ** 3), name="landau")


def tsi_physics() -> Physics:
    # same L and Q_e as Landau damping
    L = 2.0 * math.pi / 0.5
    return Physics(L=L, q_over_m=-1.0, total_charge=-(L ** 3), name="tsi")


def penning_physics() -> Physics:
    # B = (0,0,5); E_ext = (-15/L (x-L/2), -15/L (y-L/2), 30/L (z-L/2));
    # L = 25; Q_e = -1562.5
    L = 25.0
    a = (-15.0 / L, -15.0 / L, 30.0 / L)
    A = (a[0], 0.0, 0.0, 0.0, a[1], 0.0, 0.0, 0.0, a[2])
    c = tuple(-a[i] * L / 2.0 for i in range(3))
    return Physics(L=L, q_over_m=-1.0, total_charge=-1562.5, B=(0.0, 0.0, 5.0), A=A, c=c,
                   name="penning")


def _invert_cdf(u: np.ndarray, L: float, alpha: float, kw: float) -> np.ndarray:
    """Solve (x + (alpha/kw) sin(kw x)) / L = u for x in [0, L) by Newton (|F-u| <= 1e-14)."""
    x = u * L
    for _ in range(100):
        F = (x + (alpha / kw) * np.sin(kw * x)) / L - u
        dF = (1.0 + alpha * np.cos(kw * x)) / L
        x = x - F / dF
        if np.max(np.abs(F)) <= 1e-14:
            break
    return np.mod(x, L)


def landau_state(n_particles: int, seed: int, alpha: float = 0.05, kw: float = 0.5):
    """Landau damping initial state, x,v shape (3, N_p) float64."""
    L = 2.0 * math.pi / kw
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.empty((3, n_particles))
    for d in range(3):
        x[d] = _invert_cdf(rng.random(n_particles), L, alpha, kw)
    v = rng.standard_normal((3, n_particles))
    return x, v


def tsi_state(n_particles: int, seed: int, alpha: float = 0.01, kw: float = 0.5,
              sigma: float = 0.1, vb: float = math.pi / 2):
    """Two-stream instability initial state."""
    L = 2.0 * math.pi / kw
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.empty((3, n_particles))
    x[0] = rng.random(n_particles) * L
    x[1] = rng.random(n_particles) * L
    x[2] = _invert_cdf(rng.random(n_particles), L, alpha, kw)
    v = sigma * rng.standard_normal((3, n_particles))
    sign = np.where(rng.random(n_particles) < 0.5, -1.0, 1.0)
    v[2] += sign * vb
    return x, v


def penning_state(n_particles: int, seed: int, L: float = 25.0, sd=(2.0, 1.0, 3.0)):
    """Penning trap initial state: Gaussian, mean L/2, sd (2,1,3).

    Reading (R13): samples outside [0, L) are redrawn (truncation by
    resampling); with sd <= 3 and L/2 = 12.5 this is a > 4 sigma event.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.empty((3, n_particles))
    for d in range(3):
        xd = L / 2 + sd[d] * rng.standard_normal(n_particles)
        bad = (xd < 0) | (xd >= L)
        while np.any(bad):
            xd[bad] = L / 2 + sd[d] * rng.standard_normal(int(bad.sum()))
            bad = (xd < 0) | (xd >= L)
        x[d] = xd
    v = rng.standard_normal((3, n_particles))
    return x, v


def _halton(n: int, base: int) -> np.ndarray:
    """Radical inverse of 1..n in `base` (one coordinate of a Halton sequence)."""
    i = np.arange(1, n + 1)
    f = np.ones(n)
    r = np.zeros(n)
    while np.any(i > 0):
        f = f / base
        r = r + f * (i % base)
        i = i // base
    return r


def _ndtri(u: np.ndarray) -> np.ndarray:
    from scipy.special import ndtri
    return ndtri(u)


def landau_state_quiet(n_particles: int, alpha: float = 0.05, kw: float = 0.5):
    """Landau damping state with a low-discrepancy ("quiet") load: the recipe of
    landau_state with the uniform draws u replaced by the 6-D Halton sequence
    (bases 2, 3, 5 for x, y, z through the inverse CDF; 7, 11, 13 for v through
    the inverse normal CDF).  Used by the statistical rate pins of the oracle
    (R23): sampling noise in the resonant mode falls from ~1/sqrt(N_p)
    to ~log(N_p)/N_p, so 2^16 particles resolve the damping rate."""
    L = 2.0 * math.pi / kw
    x = np.stack([_invert_cdf(_halton(n_particles, b), L, alpha, kw) for b in (2, 3, 5)])
    v = np.stack([_ndtri(_halton(n_particles, b)) for b in (7, 11, 13)])
    return x, v


def tsi_state_quiet(n_particles: int, alpha: float = 0.01, kw: float = 0.5,
                    sigma: float = 0.1, vb: float = math.pi / 2):
    """Two-stream state with the Halton load (bases 2, 3 uniform x, y; 5 inverse
    CDF z; 7, 11, 13 thermal v; 17 the beam sign, u < 1/2 -> -vb)."""
    L = 2.0 * math.pi / kw
    x = np.stack([_halton(n_particles, 2) * L, _halton(n_particles, 3) * L,
                  _invert_cdf(_halton(n_particles, 5), L, alpha, kw)])
    v = sigma * np.stack([_ndtri(_halton(n_particles, b)) for b in (7, 11, 13)])
    v[2] += np.where(_halton(n_particles, 17) < 0.5, -1.0, 1.0) * vb
    return x, v


# BASELINE.json "configs" (index = config number; seed = config number)
CONFIGS = {
    0: dict(name="C1 landau 8^3 16384 dt0.05 x20", case="landau", N=8, n_particles=16384,
            tol=1e-12, dt=0.05, steps=20),
    1: dict(name="C2 landau 32^3 2^21 tol1e-12 T19.2", case="landau", N=32,
            n_particles=1 << 21, tol=1e-12, dt=0.05, steps=384),
    2: dict(name="C3 tsi 32^3 2^23", case="tsi", N=32, n_particles=1 << 23, tol=1e-12,
            dt=0.05, steps=100),
    3: dict(name="C4 penning 64^3 2^24 boris", case="penning", N=64, n_particles=1 << 24,
            tol=1e-12, dt=0.003125, steps=100),
    4: dict(name="C5 landau parareal 64^3 2^26", case="landau", N=64, n_particles=1 << 26,
            tol=1e-7, dt=0.003125, steps=768),
}


def make_case(case: str, n_particles: int, seed: int):
    """Return (Physics, x, v) for one of 'landau', 'tsi', 'penning'."""
    if case == "landau":
        return (landau_physics(),) + landau_state(n_particles, seed)
    if case == "tsi":
        return (tsi_physics(),) + tsi_state(n_particles, seed)
    if case == "penning":
        return (penning_physics(),) + penning_state(n_particles, seed)
    raise ValueError(f"unknown case {case!r}")
