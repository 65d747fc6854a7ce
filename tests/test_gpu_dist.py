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
    env = dict(os.environ, PARAGAN_COMPUTE=compute, PARAGAN_ARCH=arch)
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
