"""torchrun worker for tests/test_gpu_dist.py::test_two_gpu_async_scheme: G on rank 0, D on rank 1
(DistributedAsync, "run both generator and discriminator in parallel on different nodes") for three
ticks with staleness 1, against the oracle's schedule (oracle/async_scheme.py) on the same inputs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import async_scheme as OA
    from oracle import biggan as bg
    from paper_2411_03999_b200 import api, inputs
    from paper_2411_03999_b200.async_gan import DistributedAsync
    from tests import parity as P

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    dist.init_process_group("nccl", device_id=torch.device(dev))
    g_batch, d_batch, n_d = int(os.environ.get("ASYNC_G", 4)), int(os.environ.get("ASYNC_D", 4)), 1
    n_d = g_batch // d_batch
    from tests.test_gpu_async import SGD_D, SGD_G, sgd_configs
    ocfg, _, _ = sgd_configs(g_batch, d_batch, n_d)
    gs, ds = bg.g_param_specs(ocfg), bg.d_param_specs(ocfg)
    g0 = inputs.init_params(gs, 81, inputs.ROLE_PARAMS_G)
    d0 = inputs.init_params(ds, 81, inputs.ROLE_PARAMS_D)

    sgd = api.make_policy(rule=api.OPT_SGD)

    def make_cfg(b, r, w):
        return api.make_config(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4,
                               local_batch=b, d_steps_per_g=n_d, compute=api.F32, rank=r, world_size=w, device=local,
                               adam_d=SGD_D, adam_g=SGD_G, policy_d=sgd, policy_g=sgd)

    da = DistributedAsync(make_cfg, g_batch, d_batch, n_d)
    da.ctx.set_params(api.NET_G, g0)
    da.ctx.set_params(api.NET_D, d0)
    ticks = []
    for t in range(3):
        d = []
        for k in range(n_d):
            real, ry = inputs.real_batch(82, t * n_d + k, d_batch, 32, 10)
            zb, yb = inputs.latent_batch(82, inputs.ROLE_Z_D, t * n_d + k, d_batch, ocfg.dim_z, 10)
            d.append((real, ry, zb, yb))
        zg, yg = inputs.latent_batch(82, inputs.ROLE_Z_G, t, g_batch, ocfg.dim_z, 10)
        ticks.append({"d": d, "g": (zg, yg)})

    def tdev(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    # the boot batch (tick 0's img_buff entry) is g_batch images from the initial G: the oracle's cold start
    # generates d_batch at a time with the tick's (z_boot, y_boot); use those, concatenated
    boot_z = np.concatenate([d[2] for d in ticks[0]["d"]])
    boot_y = np.concatenate([d[3] for d in ticks[0]["d"]])
    for t, tk in enumerate(ticks):
        if da.is_g:
            da.tick(g_batch=(tdev(tk["g"][0]), tdev(tk["g"][1])), boot=(tdev(boot_z), tdev(boot_y)))
        else:
            packed = []
            for real, ry, _, _ in tk["d"]:
                rp = torch.empty((d_batch, 32, 32, 8), dtype=torch.float32, device=dev)
                api.layout_pack(tdev(real), rp, api.F32, 8)
                packed.append((rp, tdev(ry)))
            da.tick(d_batches=packed)
    torch.cuda.synchronize()
    G, D = bg.NetState.from_flat(gs, g0), bg.NetState.from_flat(ds, d0)
    # oracle schedule with the same cold start: tick 0's D steps consume one boot batch from the initial G
    want = OA.run(ocfg, G, D, ticks, max_staleness=1, d_batch=d_batch, boot_all_at_once=True)
    out = {"rank": rank, "role": "G" if da.is_g else "D"}
    if da.is_g:
        got = da.ctx.get_params(api.NET_G)
        nt = bg.n_trainable(gs)
        out["err"] = P.rel(got[:nt] - g0[:nt], G.flat()[:nt] - g0[:nt])
    else:
        got = da.ctx.get_params(api.NET_D)
        nt = bg.n_trainable(ds)
        out["err"] = P.rel(got[:nt] - d0[:nt], D.flat()[:nt] - d0[:nt])
        out["t_d"] = da.ctx.sync_stats(raise_nonfinite=False).t_d
    da.close()
    print("DISTRESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
