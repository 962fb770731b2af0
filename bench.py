#!/usr/bin/env python
"""PIF-step throughput benchmark (BASELINE.json metric "particles pushed/s").

Workload (BASELINE.json configs[1]): Landau damping 3D-3V, 32^3 Fourier modes,
2^21 particles, fine PIF NUFFT tolerance 1e-12, dt = 0.05.  One "step" = one
PIF timestep of the whole hot path: bin/sort -> ES spread -> D2Z FFT ->
deconvolve/truncate -> [rho_hat allreduce] -> Poisson + pad -> Z2D FFT x3 ->
ES interpolation fused with the KDK push.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1: one process per GPU (launched by torchrun, or -- without torchrun --
bench.py re-executes itself under torch.distributed.run with N processes);
weak scaling, 2^21 particles per GPU, one particle-decomposed problem
(rho_hat allreduce over NCCL every step).  The line also carries "c3_strong":
BASELINE configs[2] (TSI, 32^3 modes, 2^23 particles in total) split over the
N GPUs (strong scaling of the particle decomposition).
Timing: CUDA events on the library's stream around each step, L2 flushed
(256 MB write) between steps outside the events, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = 1  # BASELINE.json configs[1] (the default workload); --config 2/3 for C3/C4 lines
N_MODES = 32
N_PER_GPU = 1 << 21
TOL = 1e-12
DT = 0.05
CASE = "landau"
CONFIGS = {1: ("landau", 32, 1 << 21, 1e-12, 0.05),     # C2
           2: ("tsi", 32, 1 << 23, 1e-12, 0.05),        # C3
           3: ("penning", 64, 1 << 24, 1e-12, 0.003125),  # C4 (Boris push)
           4: ("landau", 64, 1 << 26, 1e-7, 0.003125),    # C5 fine propagator (1 GPU)
           5: ("landau", 64, 1 << 22, 1e-7, 0.003125),    # C5-reduced parareal fine propagator
           6: ("landau", 64, 1 << 22, 1e-4, 0.05),        # C5-reduced parareal coarse (PIF) propagator
           7: ("landau", 64, 1 << 26, 1e-4, 0.05),        # C5 coarse (PIF, eps 1e-4) propagator (1 GPU)
           8: ("landau", 64, 1 << 26, 1e-4, 0.05),        # C5 coarse propagator in fp32 (PIF_FLAG_FP32)
           9: ("landau", 64, 1 << 22, 1e-4, 0.05),        # C5-reduced coarse propagator in fp32
           10: ("landau", 32, 1 << 26, 0.0, 0.05),        # C5 coarse G_B: CIC-PIC on a 32^3 grid
           11: ("landau", 64, 1 << 24, 1e-7, 0.003125)}   # C5 fine share of one GPU out of 4 (space-only)
FP32_CONFIGS = (8, 9)
PIC_CONFIGS = (10,)
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
SM_COUNT = 148
FP64_FMA_PER_SM_CLK = 64  # B200: 37 TFLOP/s FP64 at 1965 MHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3-strong", action="store_true")
    ap.add_argument("--nccl-log", action="store_true", help="NCCL INIT logging (N > 1)")
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS),
                    help="BASELINE.json configs index (default 1 = the headline workload)")
    args = ap.parse_args()
    global CFG, CASE, N_MODES, N_PER_GPU, TOL, DT
    CFG = args.config
    CASE, N_MODES, N_PER_GPU, TOL, DT = CONFIGS[CFG]
    return args


def env_dist():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms in the background."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------- cpu baseline --
def oracle_step_rate(n_sample, seed=CFG):
    """One steady-state KDK step of the exact-NUDFT oracle on n_sample particles
    of the configs[1] workload; returns (particles/s, seconds, threads)."""
    import numpy as np

    import oracle as O
    from pif_inputs import make_case

    p, x, v = make_case(CASE, n_sample, seed)
    ph = O.PhysicsParams.from_inputs(p)
    prop = O.Propagator("pif", N_MODES, DT)
    E = np.zeros_like(x)  # E(x_n) carried from the previous step
    t0 = time.perf_counter()
    v = O.kick_half(v, E, DT, ph.q_over_m, ph.B)
    x = O.wrap(x + DT * v, ph.L)
    E = O.total_field(x, prop, ph)
    v = O.kick_half(v, E, DT, ph.q_over_m, ph.B)
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:  # pragma: no cover
        threads = os.cpu_count()
    return n_sample / dt, dt, threads


def workload_name():
    if CFG in PIC_CONFIGS:
        return f"{CASE}_3d3v_cic-pic_{N_MODES}^3grid_{N_PER_GPU}particles_per_gpu_dt{DT}"
    return (f"{CASE}_3d3v_{N_MODES}^3modes_{N_PER_GPU}particles_per_gpu_tol{TOL:g}_dt{DT}"
            + ("_fp32" if CFG in FP32_CONFIGS else ""))


# ------------------------------------------------------------- reference --
def run_reference(args, rank, world):
    if rank != 0:
        return
    n_sample = (1 << 15) * 32 ** 3 // N_MODES ** 3  # ~3 s of NUDFT per step
    rates, secs = [], []
    for i in range(args.warmup + args.steps):
        r, s, threads = oracle_step_rate(n_sample, seed=CFG + i)
        if i >= args.warmup:
            rates.append(r)
            secs.append(s)
    total = sum(secs)
    value = n_sample * args.steps / total
    line = {
        "impl": "reference", "metric": "particles pushed/s (PIF step)", "value": value,
        "unit": "particles/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(), "sample_particles": n_sample},
        "cpu_baseline": {"value": value, "unit": "particles/s", "cores": threads, "kind": "oracle",
                         "sample": f"{n_sample} of the {N_PER_GPU} {CASE} particles per step, one "
                                   f"KDK step of the exact O(N_p N^3) NUDFT PIF at N={N_MODES}"},
        "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours --
def timed_steps(P, sim, stream, steps, flush, world, dist):
    """K steps bracketed by barrier + synchronize, CUDA events on the library's
    stream per step, L2 flushed outside the events; returns (max-over-ranks
    total ms, phases, launches)."""
    import torch

    P.pif_profile(sim.ctx, True)
    P.pif_profile_read(sim.ctx, reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        sim.step(1)
        e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    phases, launches = P.pif_profile_read(sim.ctx, reset=True)
    P.pif_profile(sim.ctx, False)
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([total_ms], dtype=torch.float64, device=flush.device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), phases, launches


def c3_strong(args, P, rank, world, local, new_id, flush, dist):
    """BASELINE configs[2]: TSI, 32^3 modes, 2^23 particles in total split over
    the world (particle decomposition, rho_hat allreduce), tol 1e-12, dt 0.05."""
    import torch
    from pif_inputs import make_case

    case, N, n_global, tol, dt = CONFIGS[2]
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    p, x0, v0 = make_case(case, n_global, 2)  # the same global problem on every N
    sim = P.Simulation(P.physics(p.L, p.q_over_m, p.total_charge, p.B, p.A, p.c),
                       P.propagator("pif", N, dt, tol=tol), None, n_particles=n_global,
                       device=local, rank=rank, world=world, space_size=world, nccl_id=new_id(),
                       stream=stream)
    a, c = sim.first, sim.n_local
    sim.set_state(torch.from_numpy(x0[:, a:a + c].copy()).to(dev), torch.from_numpy(v0[:, a:a + c].copy()).to(dev))
    sim.step(args.warmup)
    total_ms, phases, launches = timed_steps(P, sim, stream, args.steps, flush, world, dist)
    sim.close()
    return {"workload": f"{case}_3d3v_{N}^3modes_{n_global}particles_total_tol{tol:g}_dt{dt}",
            "metric": "particles pushed/s (PIF step)", "unit": "particles/s", "scaling": "strong",
            "n_particles_global": n_global, "n_gpus": world,
            "value": n_global * args.steps / (total_ms / 1000.0),
            "ms_per_step": total_ms / args.steps,
            "phase_ms_per_step_rank0": {k: v / args.steps for k, v in phases.items() if v > 0}}


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2407_00485_b200 as P
    from pif_inputs import make_case

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    def new_id():
        """A fresh ncclUniqueId from rank 0 (one per communicator initialisation)."""
        if world == 1:
            return None
        obj = [P.pif_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    nccl_id = new_id()
    p, x0, v0 = make_case(CASE, N_PER_GPU, CFG + 1000 * rank)
    n_global = N_PER_GPU * world
    stream = torch.cuda.current_stream(dev)
    sim = P.Simulation(P.physics(p.L, p.q_over_m, p.total_charge, p.B, p.A, p.c),
                       P.propagator("pic", N_MODES, DT) if CFG in PIC_CONFIGS else
                       P.propagator("pif", N_MODES, DT, tol=TOL, fp32=CFG in FP32_CONFIGS), None,
                       n_particles=n_global, device=local, rank=rank, world=world, space_size=world,
                       nccl_id=nccl_id, stream=stream)
    w, beta, n_up = sim.plan_info(0)
    try:
        comm = sim.comm_info()
    except AttributeError:  # PIF_LIBRARY A/B build without pif_comm_info
        comm = None
    xd = torch.from_numpy(x0).to(dev)
    vd = torch.from_numpy(v0).to(dev)
    sim.set_state(xd, vd)
    sim.step(args.warmup)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    total_ms, phases, launches = timed_steps(P, sim, stream, args.steps, flush, world, dist)
    clocks = clk.stop()
    value = n_global * args.steps / (total_ms / 1000.0)

    # roofline of the dominant kernel (per launch; one launch per step)
    dom = max(("spread", "interp_push", "pic_deposit", "pic_gather_push"), key=lambda k: phases[k])
    launch_s = phases[dom] / args.steps / 1000.0
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    if dom.startswith("pic"):
        # CIC-PIC kernels are HBM-bound: the deposit reads x (24 B/particle), the
        # gather + push reads and writes x, v (96 B/particle) -- SURVEY 8(d)
        bpp = 24 if dom == "pic_deposit" else 96
        achieved = sim.n_local * bpp / launch_s / 1e9
        peak = json.load(open(PEAKS_FILE)).get("hbm_gbs", 6542.7) if os.path.exists(PEAKS_FILE) else 6542.7
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None, "kernel": dom,
                    "algorithmic": f"{bpp} B/particle x {sim.n_local} particles per launch",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    else:
        # tensor-product work (spread 2w^3, interpolation 3 x 2w^3
        # flops) plus the kernel evaluation of one transform, 3 dims x w nodes x a
        # degree-(w+3) Horner polynomial = 6w(w+3) flops
        flops_per_particle = {"spread": 2 * w ** 3, "interp_push": 6 * w ** 3}[dom] + 6 * w * (w + 3)
        achieved = sim.n_local * flops_per_particle / launch_s / 1e12
        peak = SM_COUNT * FP64_FMA_PER_SM_CLK * 2 * sm_max * 1e6 / 1e12
        traffic = None  # the committed ncu capture is of the default (C2) step only
        if CFG == 1 and os.path.exists(TRAFFIC_FILE):
            try:
                traffic = json.load(open(TRAFFIC_FILE)).get(dom)
            except Exception:
                traffic = None
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                    "algorithmic": f"{flops_per_particle} FP64 flops/particle (w={w}: tensor product + ES kernel evaluation, SURVEY 8(d)) x {sim.n_local} particles per launch",
                    "peak_source": f"derived FP64: {SM_COUNT} SMs x {FP64_FMA_PER_SM_CLK} DFMA/clk x 2 x {sm_max:.0f} MHz"}
        if dom == "interp_push" and w <= 5:
            # the vector-pipe interpolation (w <= 5) is bound by shared-memory
            # bandwidth: w^3 field nodes per particle, 24 B (fp64) / 12 B (fp32)
            # each, against 128 B/clk/SM
            bpn = 12 if CFG in FP32_CONFIGS else 24
            smem_peak = SM_COUNT * 128 * sm_max * 1e6 / 1e12
            got = sim.n_local * w ** 3 * bpn / launch_s / 1e12
            roofline["smem"] = {"bound": "smem", "achieved": got, "peak": smem_peak, "unit": "TB/s",
                                "frac": got / smem_peak,
                                "algorithmic": f"{w ** 3} nodes x {bpn} B per particle (shared-memory loads)",
                                "peak_source": f"{SM_COUNT} SMs x 128 B/clk x {sm_max:.0f} MHz"}

    # end-to-end through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(x0).pin_memory()
        vh = torch.from_numpy(v0).pin_memory()
        xo = torch.empty_like(xh).pin_memory()
        vo = torch.empty_like(vh).pin_memory()
        ksteps = max(1, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            sim.set_state(xh, vh)     # H2D of the step's inputs
            sim.step(1)
            sim.get_state(xo, vo)     # D2H of the step's result (synchronises)
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        nb = 2 * 3 * sim.n_local * 8
        e2e = {"value": n_global * ksteps / float(el.item()), "unit": "particles/s",
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "steps": ksteps}
    n_local = sim.n_local
    sim.close()
    del xd, vd

    strong = None
    if CFG == 1 and not args.no_c3_strong:
        strong = c3_strong(args, P, rank, world, local, new_id, flush, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_sample = (3 << 17) * 32 ** 3 // N_MODES ** 3  # ~14 s of NUDFT work on 16 host cores (4.7 s per 2^17)
        rate, secs, threads = oracle_step_rate(n_sample, seed=CFG)
        cpu = {"value": rate, "unit": "particles/s", "cores": threads, "kind": "oracle",
               "sample": f"{n_sample} of the {N_PER_GPU} configs[{CFG}] {CASE} particles, one KDK "
                         f"step of the exact O(N_p N^3) NUDFT PIF at N={N_MODES} ({secs:.1f} s)"}
    if rank == 0:
        line = {
            "metric": "particles pushed/s (PIF step)", "value": value, "unit": "particles/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "data": "synthetic",
            "dtype": "f32 interpolation + f64" if CFG in FP32_CONFIGS else "f64",
            "config": {"workload": workload_name(), "n_particles_global": n_global,
                       "n_particles_per_gpu": n_local,
                       "modes": N_MODES, "nufft_tol": TOL, "es_width": w, "es_beta": beta,
                       "upsampled_grid": n_up, "dt": DT, "l2": "flushed (256 MB write) between steps",
                       "parallelism": f"particle-decomposition x{world} (rho_hat allreduce)"},
            "nccl": comm, "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "phase_ms_per_step": {k: v / args.steps for k, v in phases.items() if v > 0},
            "c3_strong": strong,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args):
    """--gpus N > 1 without torchrun: re-execute this script under
    torch.distributed.run with N processes (one per GPU) on 127.0.0.1; rank 0
    prints the JSON line."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = env_dist()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and world == 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if world > 1 and args.nccl_log:
        # NCCL INIT logging (every communicator's "... nranks N ... Init
        # COMPLETE" line, on NCCL's stdout); by default the JSON line's "nccl"
        # key carries the communicator sizes from ncclCommCount instead
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
