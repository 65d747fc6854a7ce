"""Compare G's output layer on the tensor cores (op_out_conv_split, R36) with the fp32 SIMT kernels at
large batch (several 32-row strips per CTA).  python tools/check_outconv.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2411_03999_b200 import api
    for n in (8, 37, 148, 149, 256):
        h = w = 128
        c = 96
        g = torch.Generator(device="cuda").manual_seed(n)
        x = torch.relu(torch.randn(n, h, w, c, device="cuda", generator=g))
        wt = torch.randn(3, 9, c, device="cuda", generator=g) * 0.05
        b = torch.randn(3, device="cuda", generator=g)
        dy = torch.randn(n, h, w, 3, device="cuda", generator=g)
        y0 = torch.empty(n, h, w, 3, device="cuda")
        y1 = torch.full((n, h, w, 3), float("nan"), device="cuda")
        dw0 = torch.empty(3, 9, c, device="cuda")
        dw1 = torch.full((3, 9, c), float("nan"), device="cuda")
        dx0 = torch.empty(n, h, w, c, device="cuda")
        dx1 = torch.full((n, h, w, c), float("nan"), device="cuda")
        api.op_conv_fwd(api.F32, x, wt, b, 3, 3, y0)
        api.op_conv_wgrad(api.F32, x, dy, 3, 3, dw0)
        api.op_conv_dgrad(api.F32, dy, wt, c, 3, dx0)
        api.op_out_conv_split(x, wt, b, y1, dy, dw1, dx1)
        torch.cuda.synchronize()
        # fp64 weight gradient (shifted products): which of the two fp32 paths is closer
        xp = torch.nn.functional.pad(x.double(), (0, 0, 1, 1, 1, 1))
        dwx = torch.empty(3, 9, c, dtype=torch.float64, device="cuda")
        for t in range(9):
            r, s_ = divmod(t, 3)
            dwx[:, t] = torch.einsum("nhwo,nhwc->oc", dy.double(), xp[:, r:r + h, s_:s_ + w])
        rel = lambda a: float((a.double() - dwx).norm() / dwx.norm())
        print(f"n={n}: dw vs fp64: simt {rel(dw0):.3e} tensor-core {rel(dw1):.3e}", flush=True)
        d = (y1 - y0).abs()
        bad = (d > 1e-3 * (1 + y0.abs())) | torch.isnan(y1)
        print(f"n={n}: y rel {float((y1 - y0).norm() / y0.norm()):.3e} max {float(d.max()):.3e} bad {int(bad.sum())}"
              f" dw rel {float((dw1 - dw0).norm() / dw0.norm()):.3e} dx rel {float((dx1 - dx0).norm() / dx0.norm()):.3e}"
              f" dx nan {int(torch.isnan(dx1).sum())}", flush=True)
        if int(bad.sum()):
            idx = bad.nonzero()[:8].tolist()
            print("  first bad (n,h,w,o):", idx)
            rows = bad.any(dim=(2, 3))
            print("  bad rows per image (first 3 images):", [rows[i].nonzero().flatten().tolist()[:20] for i in range(min(3, n))])


if __name__ == "__main__":
    main()
