"""Multi-GPU parity (needs >= 2 GPUs in one box): 2 ranks x B images with
cross-replica BN and the NCCL gradient all-reduce equal the oracle on the 2B global
batch and the same 2B batch on one GPU; replicas stay bit-identical."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("compute,arch", [("f32", "biggan"), ("bf16", "biggan"), ("f32", "sndcgan")])
def test_two_gpu_step_parity(compute, arch):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, PARAGAN_COMPUTE=compute, PARAGAN_ARCH=arch, PARAGAN_SUBPIXEL="0" if compute == "bf16" else "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "dist_step_worker.py")]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [json.loads(l.split("DISTRESULT ", 1)[1]) for l in r.stdout.splitlines() if "DISTRESULT " in l]
    assert len(res) == 2
    assert all(x["replicas_identical"] for x in res)
    r0 = next(x for x in res if x["rank"] == 0)
    print(r0)
    assert r0["d_loss"] < r0["tol"] and r0["g_loss"] < r0["tol"]
    for k in ("d_grads", "g_grads", "d_state", "g_state"):
        assert not r0[k + "_bad"], (k, r0[k + "_bad"][:5])
    # 2 ranks x B == 1 rank x 2B (the data-parallel decomposition on the GPU itself)
    assert not r0["vs_single_bad"], r0["vs_single"]


def test_two_gpu_allreduce_sum_invariant():
    """paragan_allreduce_grads on integer-valued gradients (fp32 and bf16 wire formats): the exact mean on
    every rank, bit for bit; paragan_apply_update afterwards keeps the replicas bit-identical."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "dist_boundary_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [json.loads(l.split("DISTRESULT ", 1)[1]) for l in r.stdout.splitlines() if "DISTRESULT " in l]
    assert len(res) == 2
    for x in res:
        for k in ("f32", "bf16"):
            assert x[k]["exact_mean"] and x[k]["replicas_identical"], x


@pytest.mark.parametrize("g_batch,d_batch", [(4, 4), (4, 2)])
def test_two_gpu_async_scheme(g_batch, d_batch):
    """G on GPU 0, D on GPU 1 (the asynchronous scheme), staleness 1, equal and different G / D
    batch sizes ("Async G-512 D-256"): final G and D weights vs the oracle's schedule at 1e-4."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, ASYNC_G=str(g_batch), ASYNC_D=str(d_batch))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "dist_async_worker.py")]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [json.loads(l.split("DISTRESULT ", 1)[1]) for l in r.stdout.splitlines() if "DISTRESULT " in l]
    assert len(res) == 2
    print(res)
    for x in res:
        assert x["err"] < 1e-4, x
