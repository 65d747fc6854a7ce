"""torchrun worker for tests/test_gpu_dist.py: W ranks x B images through the C-ABI
(cross-replica BN + NCCL gradient all-reduce) against the oracle on the W*B global batch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from paragan_b200 import api
    from tests import parity as P

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    compute = api.BF16 if os.environ.get("PARAGAN_COMPUTE", "f32") == "bf16" else api.F32
    tol = 2e-2 if compute == api.BF16 else 1e-4
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    obj = [api.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    B = 4
    ocfg = P.oracle_config(32, 4, 16, 10, 16, 4, bf16=(compute == api.BF16))
    cfg = api.make_config(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4, local_batch=B,
                          compute=compute, rank=rank, world_size=world, device=local)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, B * world, seed=31)
    got = P.run_gpu(cfg, g0, d0, dbs, gb, rank=rank, world=world, nccl_id=obj[0])
    # replicas bit-identical
    h = torch.tensor([float(np.frombuffer(got["d_state"].tobytes(), dtype=np.uint32).astype(np.uint64).sum() % 1000003),
                      float(np.frombuffer(got["g_state"].tobytes(), dtype=np.uint32).astype(np.uint64).sum() % 1000003)],
                     device="cuda")
    hs = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    same = all(torch.equal(hs[0], x) for x in hs)
    out = {"rank": rank, "replicas_identical": bool(same)}
    if rank == 0:
        want = P.run_oracle(ocfg, gs, ds, g0, d0, dbs, gb)
        out["d_loss"] = abs(got["d_loss"] - want["d_loss"]) / max(abs(want["d_loss"]), 1e-3)
        out["g_loss"] = abs(got["g_loss"] - want["g_loss"]) / max(abs(want["g_loss"]), 1e-3)
        # same bars as the single-GPU micro tests: fp32 per tensor 1e-4; bf16 global 2e-2, per tensor 6e-2
        ttol = tol if compute == api.F32 else 6e-2
        for key, specs in (("d_grads", ds), ("g_grads", gs)):
            bad, worst = P.compare_tensors(specs, got[key], want[key], ttol)
            out[key + "_bad"] = [b[0] for b in bad]
            out[key + "_worst"] = max(worst.values())
            out[key + "_global"] = P.rel(got[key], want[key])
            if out[key + "_global"] > tol:
                out[key + "_bad"].append("GLOBAL")
        g_rel = 1e-4 if compute == api.F32 else 2e-2
        from oracle import biggan as bg
        for key, gkey, specs in (("d_state", "d_grads", ds), ("g_state", "g_grads", gs)):
            nt = bg.n_trainable(specs)
            e = P.rel(got[key][:nt], want[key][:nt])
            out[key + "_bad"] = [] if e < tol else ["GLOBAL"]
            out[key + "_worst"] = e
        out["tol"] = tol
    print("DISTRESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
