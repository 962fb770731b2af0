#!/usr/bin/env python
"""Coarse-propagator parameter search (PAPER.md App. "Coarse propagator
parameter search", Figs. 11-12): Landau damping or Penning trap
with 64^3 modes and 10 particles per mode, parareal over T = 19.2 with 16
slices, the coarse propagator varied over {PIF at eps_g, CIC-PIC on 64^3} x
coarsening ratio dt_g / dt_f.

  python tools/heatmap.py [--case landau|penning] [--dtf 0.05|0.003125] [--max-iter 8]

The paper times the pipelined parareal on 16 time GPUs; this box offers at most
4, so each cell runs the serial-schedule parareal on one GPU (the same protocol:
tests/test_gpu_multi.py checks the pipelined runs against it) for the measured
iteration count K, and the measured per-slice fine and coarse costs c_F, c_G
give the modelled time on 16 time ranks:
    T_16 = N_s c_G + K (c_F + c_G),   speedup = N_s c_F / T_16
(communication, ~4 ms per iteration at C5 size, is neglected; a cell that does
not converge within --max-iter iterations is reported with K = None).  The
paper's parareal tolerances: 1e-5 at dt_f = 0.05 (eps_f = 1e-4) and 1e-8 at
dt_f = 0.003125 (eps_f = 1e-7).
Output: one JSON line.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00485_b200 as P  # noqa: E402
from pif_inputs import landau_physics, landau_state, penning_physics, penning_state  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="landau", choices=["landau", "penning"])
    ap.add_argument("--dtf", type=float, default=0.05)
    ap.add_argument("--max-iter", type=int, default=8)
    ap.add_argument("--modes", type=int, default=64)
    ap.add_argument("--pc", type=int, default=10)
    a = ap.parse_args()
    N, T, Ns = a.modes, 19.2, 16
    fine_tol, stop = (1e-4, 1e-5) if a.dtf >= 0.05 else (1e-7, 1e-8)
    coarse_tols = [1e-2, 1e-3] if a.dtf >= 0.05 else [1e-3, 1e-4, 1e-5]
    # coarse steps must divide the slice length T / N_s = 1.2
    ratios = [1, 2, 4, 8, 24] if a.dtf >= 0.05 else [4, 8, 16, 32]
    phys = landau_physics() if a.case == "landau" else penning_physics()
    n = a.pc * N ** 3
    x0, v0 = (landau_state if a.case == "landau" else penning_state)(n, 21)
    xd, vd = torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda()
    ph = P.physics(phys.L, phys.q_over_m, phys.total_charge, phys.B, phys.A, phys.c)
    fine = P.propagator("pif", N, a.dtf, tol=fine_tol)
    cells = []
    for coarse_kind in [("pif", e) for e in coarse_tols] + [("pic", None)]:
        for r in ratios:
            dtg = r * a.dtf
            m = (T / Ns) / dtg
            if m < 1 - 1e-9 or abs(m - round(m)) > 1e-9 * m:
                continue
            coarse = (P.propagator("pif", N, dtg, tol=coarse_kind[1]) if coarse_kind[0] == "pif"
                      else P.propagator("pic", N, dtg))
            sim = P.Simulation(ph, fine, coarse, n_particles=n)
            sim.set_state(xd, vd)
            sim.parareal(0.0, T / Ns, 1, 1, stop)  # warm-up (plans, first launches)
            sim.set_state(xd, vd)
            rep = sim.parareal(0.0, T, Ns, a.max_iter, stop)
            sim.close()
            K = rep["iterations"] if rep["converged"] else None
            # serial schedule: F runs on every non-retired slice per iteration,
            # G on the slices whose input changed
            nF = sum(1 for k in range(rep["iterations"]) for s in range(Ns)
                     if np.isfinite(rep["err_x"][k][s]))
            cF = rep["t_fine"] / max(nF, 1)
            cG = rep["t_coarse0"] / Ns
            T16 = Ns * cG + K * (cF + cG) if K else None
            cells.append(dict(coarse=coarse_kind[0], eps_g=coarse_kind[1], ratio=r, dt_g=dtg, K=K,
                              retired_at=rep["retired_at"], c_F_s=cF, c_G_s=cG,
                              model_time_16_time_ranks_s=T16,
                              model_speedup=(Ns * cF / T16) if T16 else None))
            print(json.dumps(cells[-1]), file=sys.stderr, flush=True)
    best = min((c for c in cells if c["K"]), key=lambda c: c["model_time_16_time_ranks_s"], default=None)
    print(json.dumps(dict(case=a.case, modes=N, particles_per_mode=a.pc, n_particles=n, T=T, slices=Ns,
                          dt_f=a.dtf, eps_f=fine_tol, stop_tol=stop, max_iter=a.max_iter, cells=cells,
                          best=best)), flush=True)


if __name__ == "__main__":
    main()
