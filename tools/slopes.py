#!/usr/bin/env python
"""Convergence-slope harness (PAPER.md Sec. "Verification of
theoretical estimates"; Theorem 5.4 / Fig. 4 bottom row and Fig. 5).

  python tools/slopes.py dtg   # error vs coarse time step (PIF coarse, eps_f = eps_g = 1e-6)
  python tools/slopes.py eps   # error vs coarse NUFFT tolerance (dt_g = dt_f)

Runs the serial-schedule parareal on one GPU with no early exit (tol < 0) for K
iterations and reports, per iteration k, the L-infinity over slices of the
stopping quantity of eq. stop_criteria (what the paper plots), then fits log-log
slopes across the swept parameter.  Theory (p = 2 integrator): Dt_g^{2k}
 and eps_g^k.  Output: one JSON line.
"""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00485_b200 as P  # noqa: E402
from pif_inputs import landau_physics, landau_state  # noqa: E402


def run(mode, N=16, n=1 << 20, T=4.8, slices=16, K=4, dtf=0.0125):
    p = landau_physics()
    phys = P.physics(p.L, p.q_over_m, p.total_charge)
    x0, v0 = landau_state(n, 7)
    xd, vd = torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda()
    if mode == "dtg":
        params = [0.3, 0.15, 0.075, 0.0375]
        props = [(P.propagator("pif", N, dtf, tol=1e-6), P.propagator("pif", N, d, tol=1e-6)) for d in params]
    else:
        params = [1e-2, 1e-3, 1e-4, 1e-5]
        props = [(P.propagator("pif", N, dtf, tol=1e-12), P.propagator("pif", N, dtf, tol=e)) for e in params]
    errs = []
    for fine, coarse in props:
        sim = P.Simulation(phys, fine, coarse, n_particles=n)
        sim.set_state(xd, vd)
        rep = sim.parareal(0.0, T, slices, K, -1.0)
        errs.append([float(np.nanmax(rep["err_x"][k])) for k in range(K)])
        sim.close()
    errs = np.array(errs)  # [param, k]
    slopes = [float(np.polyfit(np.log(params), np.log(errs[:, k]), 1)[0]) for k in range(K)]
    theory = [2.0 * (k + 1) if mode == "dtg" else float(k + 1) for k in range(K)]
    return dict(mode=mode, params=params, err_x_per_iter=errs.tolist(), fitted_slopes=slopes,
                theory_slopes=theory,
                config=dict(modes=N, n_particles=n, T=T, slices=slices, iterations=K, dt_f=dtf))


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "dtg"
    print(json.dumps(run(mode)), flush=True)
