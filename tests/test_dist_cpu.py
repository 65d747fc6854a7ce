"""World-size-2 tests of the multi-rank host logic on CPU (gloo, 127.0.0.1):
NCCL-id bootstrap over torch.distributed, batch sharding (R15), the cross-replica
BN statistic exchange (A4) and the gradient mean all-reduce (A12) reproduce the
single-process global-batch oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

W = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        from oracle import biggan as bg
        from oracle import ops
        from paper_2411_03999_b200 import api, inputs
        from tests import parity as P
        res = {}
        # 1. NCCL unique-id bootstrap exactly as bench.py does it
        obj = [api.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        allids = [None] * W
        dist.all_gather_object(allids, obj[0])
        res["id_ok"] = len(obj[0]) == 128 and all(a == allids[0] for a in allids)
        # 2. cross-replica BN: local (sum, sum sq) -> all-reduce -> normalise == global oracle
        rng = np.random.default_rng(0)
        xg = rng.standard_normal((4 * W, 8, 4, 4)) * 1.7 + 0.3
        xl = inputs.shard(xg, rank, W)
        s = torch.tensor(np.concatenate([xl.sum(axis=(0, 2, 3)), (xl ** 2).sum(axis=(0, 2, 3))]))
        dist.all_reduce(s)
        cnt = xg.shape[0] * 16
        mu = s[:8].numpy() / cnt
        var = s[8:].numpy() / cnt - mu ** 2
        local_norm = (xl - mu[None, :, None, None]) / np.sqrt(var[None, :, None, None] + 1e-5)
        want = inputs.shard(ops.bn_normalise(torch.tensor(xg), 1e-5).numpy(), rank, W)
        res["bn_err"] = float(np.abs(local_norm - want).max())
        # 3. gradient mean all-reduce of D's local-mean loss == global-batch gradient
        ocfg = P.oracle_config(16, 2, 8, 5, 4, 3)
        gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, 2 * W, seed=9)
        G = bg.NetState.from_flat(gs, g0)
        D = bg.NetState.from_flat(ds, d0)
        real, ry, z, fy = dbs[0]
        glob = bg.d_step(ocfg, G, D, real, ry, z, fy, update=False)
        fake = inputs.shard(glob["fake"], rank, W)
        Dl = bg.NetState.from_flat(ds, d0)
        dp = {k: v.detach().clone().requires_grad_(True) for k, v in Dl.params.items()}
        sn = bg._SN(ds, dp, Dl.us, ocfg.sn_eps, False)
        x = torch.cat([torch.tensor(fake), bg.pack_real(ocfg, inputs.shard(real, rank, W))])
        yy = torch.cat([torch.tensor(inputs.shard(fy, rank, W), dtype=torch.long),
                        torch.tensor(inputs.shard(ry, rank, W), dtype=torch.long)])
        lg = bg.d_forward(ocfg, sn, x, yy)
        b = fake.shape[0]
        loss = ops.hinge_d(lg[b:], lg[:b])
        grads = torch.autograd.grad(loss, [dp[s_.name] for s_ in ds], allow_unused=True)
        flat = torch.cat([(g if g is not None else torch.zeros_like(dp[s_.name])).reshape(-1)
                          for g, s_ in zip(grads, ds)])
        dist.all_reduce(flat)
        flat /= W
        res["grad_err"] = P.rel(flat.numpy(), glob["grads"])
        # 4. max-over-ranks timing
        t = torch.tensor([10.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["tmax"] = float(t)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_host_logic_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=280) for _ in range(W))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(W):
        assert out[r]["id_ok"]
        assert out[r]["bn_err"] < 1e-10
        assert out[r]["grad_err"] < 1e-10
        assert out[r]["tmax"] == 11.0
