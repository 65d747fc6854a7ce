"""torchrun worker for tests/test_gpu_dist.py::test_two_gpu_allreduce_sum_invariant: each rank sets an
integer-valued local gradient through paragan_set_grads, calls paragan_allreduce_grads, and checks the
result against the exact mean (integer sums are exact in fp32, and in bf16 below 256; /W is a power of
two), bit for bit, identical on every rank (north_star "allreduce-sum invariant"); then one
paragan_apply_update leaves the replicas bit-identical."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2411_03999_b200 import api

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    obj = [api.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out = {"rank": rank}
    for comm_bf16 in (False, True):
        cfg = api.make_config(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4, local_batch=2,
                              compute=api.BF16, rank=rank, world_size=world, device=local, grad_comm_bf16=comm_bf16)
        if comm_bf16:
            obj = [api.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
        ctx = api.Context(cfg, obj[0])
        ctx.init_params(0.1)
        ok = True
        for net in (api.NET_D, api.NET_G):
            n = ctx._n(net, False)
            idx = np.arange(n, dtype=np.int64)
            local_g = [((idx * 7 + 13 * r) % 61 - 30).astype(np.float32) for r in range(world)]
            ctx.set_grads(net, local_g[rank])
            ctx.allreduce_grads(net)
            got = ctx.get_grads(net)
            want = (np.sum(np.stack(local_g).astype(np.float64), 0) / world).astype(np.float32)
            ok &= bool(np.array_equal(got, want))
            ctx.apply_update(net)
        h = torch.tensor([float(np.frombuffer(ctx.get_params(net).tobytes(), np.uint32).astype(np.uint64).sum() % 1000003)
                          for net in (api.NET_D, api.NET_G)], device="cuda")
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        out["bf16" if comm_bf16 else "f32"] = {"exact_mean": ok, "replicas_identical": all(torch.equal(hs[0], x) for x in hs)}
        ctx.close()
    print("DISTRESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
