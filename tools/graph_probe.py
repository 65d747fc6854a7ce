"""Probe: how much of the 1-GPU iteration is launch overhead / inter-kernel gaps?  Captures one bench
iteration (D step + G step, pool entry 0) into a CUDA graph (relaxed capture) and times replays against
eager steps.  Diagnostic only (the replay re-applies the same Adam step count)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2411_03999_b200 import api, inputs
    B, R = 256, 128
    cfg = api.make_config(resolution=R, local_batch=B, compute=api.BF16, seed=1234)
    dev = "cuda:0"
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        ctx = api.Context(cfg, None, stream=stream)
        ctx.init_params(attn_gamma=0.1)
        dz = api.dim_z(cfg)
        packed = torch.zeros((B, R, R, cfg.c_pad_image), dtype=torch.bfloat16, device=dev)
        z, y = inputs.latent_batch(1000, inputs.ROLE_Z_D, 0, B, dz, 1000)
        zg, yg = inputs.latent_batch(1001, inputs.ROLE_Z_G, 0, B, dz, 1000)
        z, y, zg, yg = (torch.from_numpy(a).to(dev) for a in (z, y, zg, yg))
        real = torch.rand(B, 3, R, R, device=dev) * 2 - 1
        api.layout_pack(real, packed, api.BF16, cfg.c_pad_image, stream)

        def step():
            ctx.d_step(packed, y, z, y)
            ctx.g_step(zg, yg)

        for _ in range(4):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / 10
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
            step()
        torch.cuda.synchronize()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(10):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / 10
        print(f"eager {eager:.3f} ms/iter, graph replay {graph:.3f} ms/iter, nodes {g.__class__.__name__}")


if __name__ == "__main__":
    main()
