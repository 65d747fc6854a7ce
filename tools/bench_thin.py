"""Times G's fp32 output-layer kernels (k_thin_fwd / _dgrad / _wgrad) at the bench shape through the op
hooks: x [256,128,128,96] fp32, C_out = 3; also the tensor-core split path (R36).  python tools/bench_thin.py [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2411_03999_b200 import api
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    n, h, w, c = 256, 128, 128, 96
    x = torch.randn(n, h, w, c, device="cuda")
    wt = torch.randn(3, 9, c, device="cuda")
    b = torch.randn(3, device="cuda")
    y = torch.empty(n, h, w, 3, device="cuda")
    dy = torch.randn(n, h, w, 3, device="cuda")
    dx = torch.empty_like(x)
    dw = torch.empty(3, 9, c, device="cuda")
    db = torch.empty(3, device="cuda")
    fl = 2.0 * n * h * w * 27 * c
    for name, fn in (("fwd", lambda: api.op_conv_fwd(api.F32, x, wt, b, 3, 3, y)),
                     ("dgrad", lambda: api.op_conv_dgrad(api.F32, dy, wt, c, 3, dx)),
                     ("wgrad", lambda: api.op_conv_wgrad(api.F32, x, dy, 3, 3, dw, db=db)),
                     # R36 tensor-core path; the op also splits x (one fp32 read + bf16x2 write of x)
                     ("split fwd (+split)", lambda: api.op_out_conv_split(x, wt, b, y)),
                     ("split fwd+bwd (+split)", lambda: api.op_out_conv_split(x, wt, b, y, dy, dw, dx))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"thin {name}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  ({os.environ.get('PARAGAN_THIN_VARIANT', 'default')})")


if __name__ == "__main__":
    main()
