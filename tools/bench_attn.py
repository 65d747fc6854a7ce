"""Times the fused attention kernels through the op hooks at BigGAN-128's shapes (64x64 attention):
G (n = 256, C = 192: Cq = 32, C2 = 96) and D on [fake; real] (n = 512, C = 96: Cq = 16, C2 = 48).
Inputs ~ N(0, s^2) with s small enough that the single-pass forward applies.  python tools/bench_attn.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2411_03999_b200 import api
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    hw = 4096
    q = hw // 4
    for name, n, cq, c2, s in (("G", 256, 32, 96, 0.25), ("D", 512, 16, 48, 0.35)):
        ct = 2 * cq + c2
        g = torch.Generator(device="cuda").manual_seed(n)
        qkv = (torch.randn(n, hw, ct, device="cuda", generator=g) * s).to(torch.bfloat16)
        phi = (torch.randn(n, q, cq, device="cuda", generator=g) * s).to(torch.bfloat16)
        gp = (torch.randn(n, q, c2, device="cuda", generator=g)).to(torch.bfloat16)
        o = torch.empty(n, hw, c2, dtype=torch.bfloat16, device="cuda")
        o32 = torch.empty(n, hw, c2, device="cuda")
        lse = torch.empty(n, hw, device="cuda")
        dO = (torch.randn(n, hw, c2, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
        dqkv = torch.zeros(n, hw, ct, dtype=torch.bfloat16, device="cuda")
        dphi = torch.empty(n, q, cq, device="cuda")
        dgp = torch.empty(n, q, c2, device="cuda")
        for what, fn in (("fwd", lambda: api.op_attn_fwd(qkv, phi, gp, cq, c2, o, o32, lse)),
                         ("bwd", lambda: api.op_attn_bwd(qkv, phi, gp, dO, o32, lse, cq, c2, dqkv, dphi, dgp))):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            exps = n * hw * q
            print(f"attn {name} {what}: {ms:.3f} ms  ({exps / ms / 1e9:.2f} G exp/ms; SFU floor "
                  f"{exps / (16 * 148 * 1.85e9) * 1e3:.3f} ms)",
                  flush=True)


if __name__ == "__main__":
    main()
