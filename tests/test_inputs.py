"""Sanity of the seeded input generators (pif_inputs), CPU only."""
import math

import numpy as np

from pif_inputs import landau_state, penning_state, tsi_state


def test_landau_marginal_moments():
    # density (1 + a cos(w x)) / L  =>  E[cos(w x)] = a / 2 per axis
    x, v = landau_state(1 << 18, 1)
    m = np.mean(np.cos(0.5 * x), axis=1)
    assert np.all(np.abs(m - 0.025) < 5 / math.sqrt(1 << 18))
    assert np.all((x >= 0) & (x < 4 * math.pi))
    assert abs(v.std() - 1) < 0.01


def test_tsi_beams_and_penning_bounds():
    x, v = tsi_state(1 << 16, 2)
    assert abs(np.mean(np.abs(v[2])) - math.pi / 2) < 0.01
    assert abs(np.mean(np.cos(0.5 * x[2])) - 0.005) < 5 / math.sqrt(1 << 16)
    xp, vp = penning_state(1 << 16, 3)
    assert np.all((xp >= 0) & (xp < 25.0))
    assert np.allclose(xp.std(axis=1), [2, 1, 3], rtol=0.03)


def test_seeded_reproducible():
    a = landau_state(100, 5)
    b = landau_state(100, 5)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))
