"""Physics pins of the CPU oracle (north_star: "the oracle is checked ... Landau
damping rate ... two-stream growth rate"): the exact-NUDFT PIF oracle, run on
the paper's Landau and two-stream set-ups at N = 8 modes,
against the analytic linear modes of the scheme -- the shape-corrected roots of
1 + (S_k^2/k^2) chi(omega) = 0 (tests/dispersion.py; PAPER.md:617-618 compares
with "analytical rates from the dispersion relation").

Statistics (R23): random loading needs amplitude SNR (alpha/2)
sqrt(N_p) >~ 25, i.e. ~2^20 particles x 120-240 oracle steps (tens of CPU
minutes); the Halton ("quiet") load of pif_inputs.*_quiet brings the sampling
noise of the resonant mode to ~log(N_p)/N_p, so 2^16 particles suffice.

Estimators (reading R11): the complex amplitude r(t) = (1/N_p) sum_j exp(-i k1
z_j) of the resonant mode k = (0, 0, 2 pi/L) is fitted (variable projection:
the mode amplitudes by linear least squares, the frequencies by nonlinear
least squares) to the sum of the scheme's linear modes --
  Landau: c1 e^{(-i w + g) t} + c2 e^{(+i w + g) t}  over t in [2, 12]
          (after the ballistic free-streaming response has decayed);
  TSI:    c1 e^{g t} + c2 e^{-g t} + c3 e^{-i ws t} + c4 e^{+i ws t} over [0, 12]
          (the purely growing / damped pair of the symmetric beams plus the
          stable pair the density perturbation also excites).
"""
import math

import numpy as np
import pytest
from scipy.optimize import least_squares

import oracle as O
from dispersion import dispersion_root
from pif_inputs import landau_physics, landau_state_quiet, tsi_physics, tsi_state_quiet

pytestmark = pytest.mark.slow


def _mode_trace(x0, v0, phys, N, dt, t_end):
    ph = O.PhysicsParams.from_inputs(phys)
    k1 = 2 * math.pi / phys.L
    n = x0.shape[1]
    ts, rs = [0.0], [np.sum(np.exp(-1j * k1 * x0[2])) / n]

    def trace(s, x, v):
        ts.append(s * dt)
        rs.append(np.sum(np.exp(-1j * k1 * x[2])) / n)

    O.run(x0, v0, int(round(t_end / dt)), O.Propagator("pif", N, dt), ph, trace=trace)
    return np.array(ts), np.array(rs)


def _varpro(basis, p0, t, r):
    def resid(p):
        B = basis(p, t)
        c, *_ = np.linalg.lstsq(B, r, rcond=None)
        d = B @ c - r
        return np.concatenate([d.real, d.imag])

    sol = least_squares(resid, p0)
    return sol.x, sol.cost


def test_oracle_landau_damping_rate_N8():
    """Landau (alpha = 0.05, k = 0.5), N = 8, 2^16 quiet particles, dt = 0.1 to
    t = 12: (omega, gamma) of the resonant mode within 1 % / 5 % of the
    shape-corrected root 1.37725 - 0.17163 i (the N -> inf root 1.41566 -
    0.15336 i, BASELINE's "about -0.1533", is 2.8 % / 11 % away: the pin
    resolves the PIF shape factor)."""
    phys = landau_physics()
    root = dispersion_root(8, phys.L, 0.5, 1.4 - 0.15j)
    assert abs(root - (1.37725 - 0.17163j)) < 1e-5
    x0, v0 = landau_state_quiet(1 << 16)
    t, r = _mode_trace(x0, v0, phys, 8, 0.1, 12.0)
    sel = t >= 2.0
    (g, w), _ = _varpro(lambda p, tt: np.stack([np.exp((-1j * p[1] + p[0]) * tt),
                                                np.exp((1j * p[1] + p[0]) * tt)], 1),
                        [-0.15, 1.4], t[sel], r[sel])
    assert abs(abs(w) - root.real) <= 0.01 * root.real, (g, w, root)
    assert abs(g - root.imag) <= 0.05 * abs(root.imag), (g, w, root)


def test_oracle_two_stream_growth_rate_N8():
    """Two-stream (alpha = 0.01, sigma = 0.1, v_b = +-pi/2, k = 0.5), N = 8, 2^16
    quiet particles, dt = 0.1 to t = 12: growth rate within 3 % of the
    shape-corrected root 0.28265 i, and the stable pair's frequency within 1 %
    of its real root 1.49351."""
    phys = tsi_physics()
    root = dispersion_root(8, phys.L, 0.5, 0.3j, sigma=0.1, vb=math.pi / 2)
    stable = dispersion_root(8, phys.L, 0.5, 1.49, sigma=0.1, vb=math.pi / 2)
    assert abs(root.imag - 0.28265) < 1e-5 and abs(root.real) < 1e-9
    assert abs(stable.real - 1.49351) < 1e-5 and abs(stable.imag) < 1e-9
    x0, v0 = tsi_state_quiet(1 << 16)
    t, r = _mode_trace(x0, v0, phys, 8, 0.1, 12.0)

    def basis(p, tt):
        return np.stack([np.exp(p[0] * tt), np.exp(-p[0] * tt), np.exp(-1j * p[1] * tt),
                         np.exp(1j * p[1] * tt)], 1)

    fits = [_varpro(basis, [0.3, w0], t, r) for w0 in (0.5, 1.0, 1.5, 2.0)]
    (g, ws), _ = min(fits, key=lambda f: f[1])  # the best of the starting points
    assert abs(g - root.imag) <= 0.03 * root.imag, (g, ws, root)
    assert abs(abs(ws) - stable.real) <= 0.01 * stable.real, (g, ws, stable)
