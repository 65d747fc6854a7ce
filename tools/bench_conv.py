"""Micro-benchmark of tcgen05 fprop launches (bias epilogue) at bench layer shapes; CUDA events, warm.

    python tools/bench_conv.py [filter]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03999_b200 import api  # noqa: E402

SHAPES = [  # n, h, w, cin, cout, k
    (512, 128, 128, 32, 96, 1),
    (256, 64, 64, 96, 192, 1),
    (512, 64, 64, 96, 192, 1),
    (512, 64, 64, 96, 48, 1),
    (512, 64, 64, 96, 64, 1),
    (512, 64, 64, 96, 96, 1),
    (512, 64, 64, 128, 48, 1),
    (512, 64, 64, 64, 48, 1),
    (512, 128, 128, 96, 96, 3),
    (512, 64, 64, 192, 192, 3),
]


def main():
    flt = sys.argv[1] if len(sys.argv) > 1 else ""
    dev = "cuda:0"
    for n, h, w, cin, cout, k in SHAPES:
        tag = f"{cin}->{cout}@{h}k{k}"
        if flt and flt not in tag:
            continue
        x = torch.randn(n, h, w, cin, device=dev).to(torch.bfloat16)
        wt = (torch.randn(cout, k * k, cin, device=dev) * 0.05).to(torch.bfloat16)
        b = torch.zeros(cout, device=dev)
        y = torch.empty(n, h, w, cout, device=dev, dtype=torch.bfloat16)
        for _ in range(3):
            api.op_conv_fwd(api.BF16, x, wt, b, cout, k, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 10
        e0.record()
        for _ in range(it):
            api.op_conv_fwd(api.BF16, x, wt, b, cout, k, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        fl = 2.0 * n * h * w * cin * cout * k * k
        by = (x.numel() + y.numel()) * 2
        print(f"fprop {tag} n{n}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s  {by / ms / 1e6:.0f} GB/s", flush=True)
        del x, y


if __name__ == "__main__":
    main()
