"""Kinetic dispersion relation of the PIF scheme (test helper, no oracle code).

For a Maxwellian (or two drifting Maxwellian beams) the linear modes of mode k
satisfy 1 + (S_k^2 / k^2) chi(omega) = 0, chi the plasma susceptibility
(1 + zeta Z(zeta)) / sigma^2 per beam, Z the plasma dispersion function
(Z(zeta) = i sqrt(pi) w(zeta), Faddeeva w).  S_k^2 = sinc^4(k h / 2), h = L/N,
is the PIF shape factor entering twice (once in rho_k, once in E(x_j);
PAPER.md:121-131, readings R3/R4) -- the "shape-corrected" roots of
SURVEY.md Sec. 8c (Landau N = 8: 1.37725 - 0.17163 i; TSI N = 8: 0.28265 i).
"""
import math

from scipy.special import wofz


def dispersion_root(N, L, kk, guess, sigma=1.0, vb=0.0, order=1):
    """Newton root of 1 + (S^2/k^2) chi(omega) = 0 near `guess` (complex omega)."""
    h = L / N
    u = kk * h / 2
    S2 = (math.sin(u) / u) ** (2 * (order + 1))

    def chi(w):
        tot = 0.0
        beams = [(0.5, vb), (0.5, -vb)] if vb else [(1.0, 0.0)]
        for frac, ub in beams:
            z = (w - kk * ub) / (math.sqrt(2) * kk * sigma)
            tot += frac * (1 + z * 1j * math.sqrt(math.pi) * wofz(z)) / sigma ** 2
        return tot

    w = complex(guess)
    for _ in range(100):
        D = 1 + S2 / kk ** 2 * chi(w)
        dw = 1e-7 * (1 + abs(w))
        dD = (1 + S2 / kk ** 2 * chi(w + dw) - D) / dw
        w = w - D / dD
    return w
