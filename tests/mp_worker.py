"""Multi-GPU worker (one process per GPU, launched by torchrun) for
tests/test_gpu_multi.py.  Every rank runs the distributed path through the C
ABI; rank 0 compares the gathered result with the CPU oracle (exact NUDFT PIF /
oracle parareal) and with the single-GPU run of the same problem.

  torchrun --nproc-per-node N tests/mp_worker.py {space|parareal|spacetime}
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2407_00485_b200 as P  # noqa: E402
from pif_inputs import landau_physics, landau_state  # noqa: E402


def setup():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [P.pif_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return rank, world, local, obj[0]


def phys():
    p = landau_physics()
    return P.physics(p.L, p.q_over_m, p.total_charge)


def gather_rows(t):
    """all_gather of variable-size (3, n) tensors along dim 1 (rank order)."""
    world = dist.get_world_size()
    n = torch.tensor([t.shape[1]], device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    mx = int(max(v.item() for v in ns))
    pad = torch.zeros((3, mx), dtype=t.dtype, device=t.device)
    pad[:, : t.shape[1]] = t
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    return torch.cat([o[:, : int(v.item())] for o, v in zip(outs, ns)], dim=1)


def run_space(rank, world, local, nid, fp32=False):
    """Particle decomposition over all ranks: 20 fine steps == single GPU (fp32:
    the rho_hat all-reduce in single precision)."""
    n, steps = 20000 + 3, 20  # ragged split
    x0, v0 = landau_state(n, 3)
    fine = P.propagator("pif", 8, 0.05, tol=1e-12, fp32_allreduce=fp32)
    sim = P.Simulation(phys(), fine, None, n_particles=n, device=local, rank=rank, world=world,
                       space_size=world, nccl_id=nid)
    a, c = sim.first, sim.n_local
    sim.set_state(torch.from_numpy(np.ascontiguousarray(x0[:, a:a + c])).cuda(),
                  torch.from_numpy(np.ascontiguousarray(v0[:, a:a + c])).cuda())
    sim.step(steps)
    x, v = sim.get_state()
    W, ke, mom, ce = sim.field_energy()
    xs, vs = gather_rows(x), gather_rows(v)
    sim.close()
    res = {}
    if rank == 0:
        ref = P.Simulation(phys(), P.propagator("pif", 8, 0.05, tol=1e-12), None, n_particles=n,
                           device=local)
        ref.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
        ref.step(steps)
        xr, vr = ref.get_state()
        Wr, ker, momr, cer = ref.field_energy()
        L = landau_physics().L
        dx = (xs - xr).cpu().numpy()
        dx -= L * np.rint(dx / L)
        res = dict(dx=float(np.abs(dx).max() / L),
                   dv=float((vs - vr).abs().max().item() / vr.abs().max().item()),
                   dW=float(np.abs(W - Wr).max() / Wr.sum()), dke=abs(ke - ker) / ker,
                   dmom=float(np.abs(mom - momr).max() / (abs(ker) ** 0.5)))
        ref.close()
        # the oracle: exact NUDFT PIF over all particles
        ph = O.PhysicsParams.from_inputs(landau_physics())
        prop = O.Propagator("pif", 8, 0.05)
        xo, vo = O.run(x0, v0, steps, prop, ph)
        Wo, keo, momo, ceo = O.diagnostics(xo, vo, prop, ph)
        res.update(dx_oracle=float(np.abs(O.min_image(xs.cpu().numpy() - xo, L)).max() / L),
                   dv_oracle=float(np.abs(vs.cpu().numpy() - vo).max() / np.abs(vo).max()),
                   dW_oracle=float(np.abs(W - Wo).max() / Wo.sum()),
                   dke_oracle=abs(ke - keo) / keo)
    return res


def run_parareal(rank, world, local, nid, space_size, blocks=1):
    """Pipelined parareal (time_size = world / space_size slices, one per time
    rank) == the serial-schedule parareal of the same problem on one GPU."""
    n = 4096 + 5
    x0, v0 = landau_state(n, 4)
    T = world // space_size
    nf, dtf, dtg = 4, 0.05, 0.1
    fine = P.propagator("pif", 8, dtf, tol=1e-12)
    coarse = P.propagator("pic", 8, dtg)
    t1 = blocks * T * nf * dtf
    sim = P.Simulation(phys(), fine, coarse, n_particles=n, device=local, rank=rank, world=world,
                       space_size=space_size, nccl_id=nid)
    a, c = sim.first, sim.n_local
    sim.set_state(torch.from_numpy(np.ascontiguousarray(x0[:, a:a + c])).cuda(),
                  torch.from_numpy(np.ascontiguousarray(v0[:, a:a + c])).cuda())
    rep = sim.parareal(0.0, t1, T, T, 1e-6, n_blocks=blocks)
    x, v = sim.get_state()
    # final state lives on the last time rank: gather its space group's rows
    t_idx = rank // space_size
    xs = gather_rows(x)  # all ranks' slices, rank order
    vs = gather_rows(v)
    sim.close()
    res = {}
    if rank == 0:
        last = slice((T - 1) * n, T * n)  # rows of the last time rank's space group
        xl, vl = xs[:, last], vs[:, last]
        ref = P.Simulation(phys(), fine, coarse, n_particles=n, device=local)
        ref.set_state(torch.from_numpy(x0).cuda(), torch.from_numpy(v0).cuda())
        rr = ref.parareal(0.0, t1, T, T, 1e-6, n_blocks=blocks)
        xr, vr = ref.get_state()
        L = landau_physics().L
        dx = (xl - xr).cpu().numpy()
        dx -= L * np.rint(dx / L)
        res = dict(retired=rep["retired_at"], retired_ref=rr["retired_at"],
                   iters=rep["iterations"], iters_ref=rr["iterations"],
                   ex=np.nan_to_num(rep["err_x"], nan=-1).tolist(),
                   ex_ref=np.nan_to_num(rr["err_x"], nan=-1).tolist(),
                   dx=float(np.abs(dx).max() / L),
                   dv=float((vl - vr).abs().max().item() / vr.abs().max().item()),
                   t_total=rep["t_total"], t_comm=rep["t_comm"])
        ref.close()
        # the oracle's parareal (eq. parareal_correction) with the
        # exact NUDFT PIF fine and CIC-PIC coarse propagators
        ph = O.PhysicsParams.from_inputs(landau_physics())
        F = O.make_propagator_fn(O.Propagator("pif", 8, dtf), ph, nf)
        G = O.make_propagator_fn(O.Propagator("pic", 8, dtg), ph, int(round(nf * dtf / dtg)))
        ores = O.parareal_blocks((x0, v0), lambda b: F, lambda b: G, T, blocks, T, 1e-6, L=L)
        xo, vo = ores[-1].U[T]
        res.update(retired_oracle=ores[-1].retired_at, iters_oracle=sum(r.iterations for r in ores),
                   dx_oracle=float(np.abs(O.min_image(xl.cpu().numpy() - xo, L)).max() / L),
                   dv_oracle=float(np.abs(vl.cpu().numpy() - vo).max() / np.abs(vo).max()))
    return res


def main():
    mode = sys.argv[1]
    rank, world, local, nid = setup()
    if mode == "space":
        res = run_space(rank, world, local, nid)
    elif mode == "space32":
        res = run_space(rank, world, local, nid, fp32=True)
    elif mode == "parareal":
        res = run_parareal(rank, world, local, nid, space_size=1)
    elif mode == "spacetime":
        res = run_parareal(rank, world, local, nid, space_size=2)
    elif mode == "blocks":
        res = run_parareal(rank, world, local, nid, space_size=1, blocks=3)
    else:
        raise SystemExit(mode)
    if rank == 0:
        print("RESULT " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
