"""Multi-GPU paths on one box (skipped with fewer GPUs): particle decomposition
(rho_hat allreduce over NCCL) and the pipelined parareal (NCCL send/recv of the
particle state between time ranks), each against the CPU oracle (exact NUDFT
PIF / oracle parareal) and the single-GPU result."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def launch(nproc, mode, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mp_worker.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


@pytest.mark.skipif(ngpu() < 2, reason="needs 2 GPUs")
def test_space_decomposition_2gpu():
    r = launch(2, "space", 29611)
    assert r["dx_oracle"] <= 1e-10 and r["dv_oracle"] <= 1e-10, r
    assert r["dW_oracle"] <= 1e-10 and r["dke_oracle"] <= 1e-10, r
    assert r["dx"] <= 1e-12 and r["dv"] <= 1e-12, r
    assert r["dW"] <= 1e-12 and r["dke"] <= 1e-12, r


@pytest.mark.skipif(ngpu() < 2, reason="needs 2 GPUs")
def test_pipelined_parareal_2gpu():
    r = launch(2, "parareal", 29612)
    assert r["retired"] == r["retired_oracle"] and r["iters"] == r["iters_oracle"], r
    assert r["dx_oracle"] <= 1e-9 and r["dv_oracle"] <= 1e-9, r
    assert r["retired"] == r["retired_ref"] and r["iters"] == r["iters_ref"], r
    assert r["dx"] <= 1e-9 and r["dv"] <= 1e-9, r


@pytest.mark.skipif(ngpu() < 4, reason="needs 4 GPUs")
def test_spacetime_parareal_4gpu():
    r = launch(4, "spacetime", 29613)
    assert r["retired"] == r["retired_oracle"] and r["iters"] == r["iters_oracle"], r
    assert r["dx_oracle"] <= 1e-9 and r["dv_oracle"] <= 1e-9, r
    assert r["retired"] == r["retired_ref"] and r["iters"] == r["iters_ref"], r
    assert r["dx"] <= 1e-9 and r["dv"] <= 1e-9, r


@pytest.mark.skipif(ngpu() < 2, reason="needs 2 GPUs")
def test_space_decomposition_fp32_allreduce_2gpu():
    """f3: rho_hat all-reduced in fp32: same trajectories to single-precision level."""
    r = launch(2, "space32", 29614)
    assert 0 < r["dx"] <= 1e-6 and r["dv"] <= 1e-5, r
    assert r["dx_oracle"] <= 1e-6 and r["dv_oracle"] <= 1e-5, r


@pytest.mark.skipif(ngpu() < 2, reason="needs 2 GPUs")
def test_multiblock_pipelined_parareal_2gpu():
    """f1: 3 windows of pipelined parareal on 2 time ranks == serial schedule."""
    r = launch(2, "blocks", 29615)
    assert r["retired"] == r["retired_oracle"] and r["iters"] == r["iters_oracle"], r
    assert r["dx_oracle"] <= 1e-9 and r["dv_oracle"] <= 1e-9, r
    assert r["retired"] == r["retired_ref"] and r["iters"] == r["iters_ref"], r
    assert r["dx"] <= 1e-9 and r["dv"] <= 1e-9, r
