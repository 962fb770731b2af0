#!/usr/bin/env python
"""Parareal speedup vs serial time stepping (BASELINE.json metric, second half;
configs[4] family: Landau damping, 64^3 modes, coarse = PIF eps 1e-4 or
CIC-PIC 32^3, both with temporal coarsening Delta t_g = 0.05).

  torchrun --nproc-per-node N bench_parareal.py [--coarse pif|pic] [--particles P]

One parareal slice per GPU (time_size = N, space_size = 1).  Rank 0 first runs
the serial fine propagator over [0, T] alone (the "serial time stepping"
reference of P:716-718), then all ranks run pif_parareal; speedup =
t_serial / t_parareal (t_parareal = max over ranks of the pif_parareal call,
from the start of the coarse sweep to the last slice's retirement).  Reading
R21 of DESIGN.md: T = 2.4, Delta t_f = 0.003125, eps_f = 1e-7, stop tol 1e-8.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coarse", default="pif", choices=["pif", "pic"])
    ap.add_argument("--particles", type=int, default=1 << 22)
    ap.add_argument("--modes", type=int, default=64)
    ap.add_argument("--T", type=float, default=2.4)
    ap.add_argument("--dtf", type=float, default=0.003125)
    ap.add_argument("--dtg", type=float, default=0.05)
    ap.add_argument("--tolf", type=float, default=1e-7)
    ap.add_argument("--tolg", type=float, default=1e-4)
    ap.add_argument("--stop", type=float, default=1e-8)
    ap.add_argument("--max-iter", type=int, default=0, help="0 = number of slices")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2407_00485_b200 as P
    from pif_inputs import landau_physics, landau_state

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nid = None
    if world > 1:
        obj = [P.pif_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    p = landau_physics()
    phys = P.physics(p.L, p.q_over_m, p.total_charge)
    fine = P.propagator("pif", args.modes, args.dtf, tol=args.tolf)
    coarse = (P.propagator("pif", args.modes, args.dtg, tol=args.tolg) if args.coarse == "pif"
              else P.propagator("pic", 32, args.dtg))
    n = args.particles
    x0, v0 = landau_state(n, 4)
    xd, vd = torch.from_numpy(x0).to(dev), torch.from_numpy(v0).to(dev)
    nsteps = int(round(args.T / args.dtf))
    slices = max(world, 1)
    max_iter = args.max_iter or slices

    t_serial = None
    xs = None
    if rank == 0:
        ser = P.Simulation(phys, fine, None, n_particles=n, device=local)
        ser.set_state(xd, vd)
        ser.step(3)  # warm-up (plans, caches)
        ser.set_state(xd, vd)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ser.step(nsteps)
        xs, vs = ser.get_state()
        torch.cuda.synchronize()
        t_serial = time.perf_counter() - t0
        ser.close()
    if world > 1:
        dist.barrier()

    sim = P.Simulation(phys, fine, coarse, n_particles=n, device=local, rank=rank, world=world,
                       space_size=1, nccl_id=nid)
    # untimed warm-up (lazy module loading, first cuFFT executions on every rank)
    sim.set_state(xd, vd)
    sim.parareal(0.0, slices * args.dtg, slices, 1, args.stop)
    sim.set_state(xd, vd)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = sim.parareal(0.0, args.T, slices, max_iter, args.stop)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    xp, vp = sim.get_state()
    tt = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        # final state of the last slice -> rank 0
        if rank == world - 1:
            dist.send(xp, 0)
            dist.send(vp, 0)
        if rank == 0:
            xp = torch.empty_like(xp)
            vp = torch.empty_like(vp)
            dist.recv(xp, world - 1)
            dist.recv(vp, world - 1)
    t_par = float(tt.item())
    if rank == 0:
        L = p.L
        dx = (xp - xs).cpu().numpy()
        dx -= L * np.rint(dx / L)
        line = {
            "metric": "parareal speedup vs serial (PIF fine)", "value": t_serial / t_par,
            "unit": "x", "n_gpus": world, "higher_is_better": True,
            "t_serial_s": t_serial, "t_parareal_s": t_par, "iterations": rep["iterations"],
            "converged": rep["converged"], "retired_at": rep["retired_at"],
            "max_rel_err_x_vs_serial": float(np.abs(dx).max() / L),
            "max_rel_err_v_vs_serial": float((vp - vs).abs().max().item() / vs.abs().max().item()),
            "phase_s_rank0": {k: rep[k] for k in ("t_coarse0", "t_fine", "t_coarse", "t_comm")},
            "push_rate_parareal": n * nsteps / t_par, "push_rate_serial": n * nsteps / t_serial,
            "config": {"workload": "landau_3d3v", "modes": args.modes, "n_particles": n, "T": args.T,
                       "dt_f": args.dtf, "eps_f": args.tolf, "coarse": args.coarse,
                       "dt_g": args.dtg, "eps_g": args.tolg if args.coarse == "pif" else None,
                       "pic_grid": 32 if args.coarse == "pic" else None, "stop_tol": args.stop,
                       "slices": slices, "fine_steps": nsteps},
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
