#!/usr/bin/env python
"""Resonant-mode field energy traces (Landau C2 / TSI C3) on the GPU -> JSON,
for choosing fit windows of the physics checks (R11)."""
import json, math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00485_b200 as P
from pif_inputs import landau_physics, landau_state, tsi_physics, tsi_state

def trace(case, n, N=32, dt=0.05, T=20.0, seed=2):
    phys = tsi_physics() if case == "tsi" else landau_physics()
    x0, v0 = (tsi_state if case == "tsi" else landau_state)(n, seed)
    sim = P.Simulation(P.physics(phys.L, phys.q_over_m, phys.total_charge), P.propagator("pif", N, dt, tol=1e-12), None, n_particles=n)
    sim.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
    L = phys.L; k1 = 2 * math.pi / L; S = (math.sin(k1 * L / N / 2) / (k1 * L / N / 2)) ** 2
    out = []
    for s in range(int(round(T / dt)) + 1):
        if s: sim.step(1)
        rho = P.pif_get_rho(sim.ctx, N)
        out.append(L ** 3 * S ** 2 * abs(rho[N // 2, N // 2, 1]) ** 2 / k1 ** 2)
    return out

res = {"tsi": trace("tsi", 1 << 23), "landau": trace("landau", 1 << 21, seed=1)}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/physics_trace.json", "w"))
print("ok")
