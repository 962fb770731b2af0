#!/usr/bin/env python
"""Convergence-slope harness (PAPER.md Sec. "Verification of
theoretical estimates"; Theorems 5.3 / 5.4, Figs. 1, 2, 4, 5).

  python tools/slopes.py MODE [--quick]     MODE in pc | h | dtg | eps

Each point runs the serial-schedule parareal on one GPU with no early exit
(stop tol < 0) for K iterations and records, per iteration k, the maximum over
slices of the stopping quantity of eq. stop_criteria (the paper's "max local
error"); log-log slopes are fitted across the swept parameter, per k, using
only errors above FLOOR (the round-off floor of the stopping quantity is
~1e-15; points within 100x of it are dropped, as the paper's curves flatten
there too).  Theory (p = 2 integrators):
  pc  -- Landau, 32^3 modes, CIC-PIC coarse on 32^3, dt_f = dt_g = 0.05:
         err_k ~ P_c^(-k/2)         (Theorem 5.3, Fig. 1)
  h   -- Penning, P_c = 10, CIC-PIC coarse on N^3 with N^3 PIF modes, dt 0.05:
         err_k ~ h^(2k) = N^(-2k)   (Theorem 5.3, Fig. 2)
  dtg -- Landau, 16^3 modes, P_c = 640, PIF coarse, eps_f = eps_g = 1e-6:
         err_k ~ dt_g^(2k)          (Theorem 5.4, Fig. 4 bottom)
  eps -- Landau, 16^3 modes, P_c = 640, PIF coarse at eps_g, dt_f = dt_g:
         err_k ~ eps^k              (Theorem 5.4, Fig. 5); also fitted against
         the measured coarse NUFFT error delta(eps) (relative L2 of the coarse
         type-1 sum of the initial charges against the same sum at eps = 1e-14,
         both on the GPU): the theorem's C_nufft eps is that error, and the
         achieved error of width w = ceil(-log10(eps/10)) is not exactly eps.
Output: one JSON line.
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00485_b200 as P  # noqa: E402
from pif_inputs import landau_physics, landau_state, penning_physics, penning_state  # noqa: E402

FLOOR = 1e-13


def parareal_errors(phys, fine, coarse, x0, v0, T, slices, K):
    sim = P.Simulation(P.physics(phys.L, phys.q_over_m, phys.total_charge, phys.B, phys.A, phys.c),
                       fine, coarse, n_particles=x0.shape[1])
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    rep = sim.parareal(0.0, T, slices, K, -1.0)
    sim.close()
    return [float(np.nanmax(rep["err_x"][k])) for k in range(K)], [float(np.nanmax(rep["err_v"][k])) for k in range(K)]


def fit(params, errs, K):
    """Per k: slope of log err vs log param over the points above FLOOR (>= 2)."""
    out = []
    for k in range(K):
        pts = [(p, e[k]) for p, e in zip(params, errs) if e[k] > FLOOR]
        if len(pts) < 2:
            out.append(None)
            continue
        a = np.log([p for p, _ in pts])
        b = np.log([e for _, e in pts])
        out.append(dict(slope=float(np.polyfit(a, b, 1)[0]), points=len(pts)))
    return out


def nufft_error(phys, x, N, eps):
    """delta(eps): relative L2 of the type-1 sum of unit charges at eps vs eps = 1e-14."""
    def t1(tol):
        sim = P.Simulation(P.physics(phys.L, phys.q_over_m, phys.total_charge), P.propagator("pif", N, 0.05, tol=tol),
                           n_particles=x.shape[1])
        out = P.pif_debug_type1(sim.ctx, 0, x, np.ones(x.shape[1]), N)
        sim.close()
        return out
    ref = t1(1e-14)
    return float(np.linalg.norm(t1(eps) - ref) / np.linalg.norm(ref))


def run(mode, quick):
    K = 4
    slices = 16
    if mode == "pc":
        N, dt, T = 32, 0.05, (4.8 if quick else 19.2)
        params = [2, 8, 32, 128]
        phys = landau_physics()
        errs, errv = [], []
        for pc in params:
            x0, v0 = landau_state(pc * N ** 3, 11)
            ex, ev = parareal_errors(phys, P.propagator("pif", N, dt, tol=1e-12), P.propagator("pic", N, dt),
                                     x0, v0, T, slices, K)
            errs.append(ex)
            errv.append(ev)
        theory = [-0.5 * (k + 1) for k in range(K)]
        cfg = dict(case="landau", modes=N, pic_grid=N, dt_f=dt, dt_g=dt, T=T, tol_f=1e-12)
    elif mode == "h":
        dt, T, pc = 0.05, (4.8 if quick else 19.2), 10
        params = [16, 32, 64] if quick else [16, 32, 64, 128]
        phys = penning_physics()
        errs, errv = [], []
        for N in params:
            x0, v0 = penning_state(pc * N ** 3, 12)
            ex, ev = parareal_errors(phys, P.propagator("pif", N, dt, tol=1e-12), P.propagator("pic", N, dt),
                                     x0, v0, T, slices, K)
            errs.append(ex)
            errv.append(ev)
        params = [phys.L / N for N in params]  # mesh size h
        theory = [2.0 * (k + 1) for k in range(K)]
        cfg = dict(case="penning", particles_per_cell=pc, dt_f=dt, dt_g=dt, T=T, tol_f=1e-12)
    elif mode == "dtg":
        N, pc = 16, 640
        T, dtf = (4.8, 0.0125) if quick else (19.2, 0.003125)
        params = [0.3, 0.15, 0.075, 0.0375] if quick else [0.4, 0.2, 0.1, 0.05]
        phys = landau_physics()
        x0, v0 = landau_state(pc * N ** 3, 13)
        errs, errv = [], []
        for d in params:
            ex, ev = parareal_errors(phys, P.propagator("pif", N, dtf, tol=1e-6), P.propagator("pif", N, d, tol=1e-6),
                                     x0, v0, T, slices, K)
            errs.append(ex)
            errv.append(ev)
        theory = [2.0 * (k + 1) for k in range(K)]
        cfg = dict(case="landau", modes=N, particles_per_mode=pc, dt_f=dtf, tol_f=1e-6, tol_g=1e-6, T=T)
    elif mode == "eps":
        N, pc, dt = 16, 640, 0.05
        T = 4.8 if quick else 19.2
        params = [1e-2, 1e-3, 1e-4, 1e-5]
        phys = landau_physics()
        x0, v0 = landau_state(pc * N ** 3, 14)
        errs, errv = [], []
        for e in params:
            ex, ev = parareal_errors(phys, P.propagator("pif", N, dt, tol=1e-12), P.propagator("pif", N, dt, tol=e),
                                     x0, v0, T, slices, K)
            errs.append(ex)
            errv.append(ev)
        theory = [float(k + 1) for k in range(K)]
        delta = [nufft_error(phys, x0, N, e) for e in params]
        cfg = dict(case="landau", modes=N, particles_per_mode=pc, dt_f=dt, dt_g=dt, tol_f=1e-12, T=T,
                   measured_nufft_error=delta, slopes_vs_measured_nufft_error=fit(delta, errs, K))
    else:
        raise SystemExit(f"unknown mode {mode}")
    slopes = fit(params, errs, K)
    ok = [None if s is None else abs(s["slope"] - t) <= 0.15 * abs(t) for s, t in zip(slopes, theory)]
    return dict(mode=mode, params=params, err_x_per_iter=errs, err_v_per_iter=errv, floor=FLOOR,
                fitted_slopes=slopes, theory_slopes=theory, within_15pct=ok,
                config=dict(cfg, slices=slices, iterations=K, quick=quick))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["pc", "h", "dtg", "eps"])
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    print(json.dumps(run(a.mode, a.quick)), flush=True)
