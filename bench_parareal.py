#!/usr/bin/env python
"""Parareal speedup (BASELINE.json metric, second half; configs[4] family:
Landau damping, 64^3 modes, coarse = PIF eps 1e-4 (fp64 or fp32) or CIC-PIC
32^3, both with temporal coarsening Delta t_g = 0.05).

  torchrun --nproc-per-node N bench_parareal.py [--coarse pif|pif32|pic]
           [--particles P] [--space S]

Rank layout: N = S x T ranks, T = N / S parareal slices, each slice particle-
decomposed over S GPUs (space x time, PAPER.md:139-141 with P:151-173).
Two references (reading c20 of SURVEY.md 8c; PAPER.md:534-535 compares with
"spatial parallelization alone", P:716-718 with serial time stepping):
  t_serial -- the fine propagator over [0, T] on 1 GPU (rank 0 alone);
  t_space  -- the fine propagator over [0, T] particle-decomposed over all N
              GPUs (max over ranks);
then all ranks run pif_parareal: t_parareal = max over ranks of the call, from
the start of the coarse sweep to the last slice's retirement.  Per-rank phase
times (coarse sweep, fine, coarse, communication wait, total) are all-gathered.
Reading R21 of DESIGN.md: T = 2.4, Delta t_f = 0.003125, eps_f = 1e-7, stop
tol 1e-8.
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
    ap.add_argument("--coarse", default="pif", choices=["pif", "pif32", "pic"])
    ap.add_argument("--space", type=int, default=1, help="GPUs per slice (space_size)")
    ap.add_argument("--no-space-ref", action="store_true")
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
    def new_id():
        """A fresh ncclUniqueId from rank 0 (one per communicator initialisation)."""
        if world == 1:
            return None
        obj = [P.pif_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    p = landau_physics()
    phys = P.physics(p.L, p.q_over_m, p.total_charge)
    fine = P.propagator("pif", args.modes, args.dtf, tol=args.tolf)
    coarse = (P.propagator("pic", 32, args.dtg) if args.coarse == "pic" else
              P.propagator("pif", args.modes, args.dtg, tol=args.tolg, fp32=args.coarse == "pif32"))
    S = args.space
    assert world % S == 0, "--space must divide the number of ranks"
    n = args.particles
    x0, v0 = landau_state(n, 4)
    xd, vd = torch.from_numpy(x0).to(dev), torch.from_numpy(v0).to(dev)
    nsteps = int(round(args.T / args.dtf))
    slices = max(world // S, 1)
    max_iter = args.max_iter or slices

    clk = None
    if rank == 0:  # clocks and throttle reasons of this GPU during the whole run
        from bench import ClockSampler
        clk = ClockSampler(local)
        clk.start()
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

    # spatial parallelization alone: the fine propagator particle-decomposed
    # over all ranks (one rho_hat all-reduce per step)
    t_space = None
    if world > 1 and not args.no_space_ref:
        sp = P.Simulation(phys, fine, None, n_particles=n, device=local, rank=rank, world=world,
                          space_size=world, nccl_id=new_id())
        a, c = sp.first, sp.n_local
        xa, va = xd[:, a:a + c].contiguous(), vd[:, a:a + c].contiguous()
        sp.set_state(xa, va)
        sp.step(3)
        sp.set_state(xa, va)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sp.step(nsteps)
        sp.get_state()
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_space = float(tt.item())
        sp.close()
        del xa, va

    sim = P.Simulation(phys, fine, coarse, n_particles=n, device=local, rank=rank, world=world,
                       space_size=S, nccl_id=new_id())
    a, c = sim.first, sim.n_local
    xd, vd = xd[:, a:a + c].contiguous(), vd[:, a:a + c].contiguous()
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
    phases = torch.tensor([rep[k] for k in ("t_coarse0", "t_fine", "t_coarse", "t_comm", "t_total")]
                          + [el], dtype=torch.float64, device=dev)
    per_rank = [phases]
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        per_rank = [torch.empty_like(phases) for _ in range(world)]
        dist.all_gather(per_rank, phases)
        # final state of the last slice (space ranks (T-1) S .. T S - 1) -> rank 0
        last = list(range((slices - 1) * S, slices * S))
        if rank in last and rank != 0:
            dist.send(xp, 0)
            dist.send(vp, 0)
        if rank == 0:
            parts_x, parts_v = [], []
            for r in last:
                cnt = P.pif_partition(n, S, r - (slices - 1) * S)[1]
                if r == 0:
                    bx, bv = xp, vp
                else:
                    bx = torch.empty((3, cnt), dtype=torch.float64, device=dev)
                    bv = torch.empty_like(bx)
                    dist.recv(bx, r)
                    dist.recv(bv, r)
                parts_x.append(bx)
                parts_v.append(bv)
            xp, vp = torch.cat(parts_x, dim=1), torch.cat(parts_v, dim=1)
    t_par = float(tt.item())
    if rank == 0:
        L = p.L
        dx = (xp - xs).cpu().numpy()
        dx -= L * np.rint(dx / L)
        line = {
            "metric": "parareal speedup vs serial (PIF fine)", "value": t_serial / t_par,
            "unit": "x", "n_gpus": world, "higher_is_better": True,
            "speedup_vs_space_only": (t_space / t_par) if t_space else None,
            "space_only_speedup_vs_serial": (t_serial / t_space) if t_space else None,
            "t_serial_s": t_serial, "t_space_only_s": t_space, "t_parareal_s": t_par,
            "layout": {"space": S, "time": slices}, "iterations": rep["iterations"],
            "converged": rep["converged"], "retired_at": rep["retired_at"],
            "max_rel_err_x_vs_serial": float(np.abs(dx).max() / L),
            "max_rel_err_v_vs_serial": float((vp - vs).abs().max().item() / vs.abs().max().item()),
            "phase_s_per_rank": [dict(zip(("t_coarse0", "t_fine", "t_coarse", "t_comm", "t_total",
                                           "t_call"), [round(float(v), 4) for v in t.tolist()]))
                                 for t in per_rank],
            "push_rate_parareal": n * nsteps / t_par, "push_rate_serial": n * nsteps / t_serial,
            "clocks_rank0": clk.stop() if clk else None,
            "config": {"workload": "landau_3d3v", "modes": args.modes, "n_particles": n, "T": args.T,
                       "dt_f": args.dtf, "eps_f": args.tolf, "coarse": args.coarse,
                       "dt_g": args.dtg, "eps_g": args.tolg if args.coarse != "pic" else None,
                       "pic_grid": 32 if args.coarse == "pic" else None, "stop_tol": args.stop,
                       "slices": slices, "fine_steps": nsteps},
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
