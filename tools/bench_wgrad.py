"""Micro-benchmark of the tcgen05 weight-gradient launches at the bench's layer shapes (CUDA events,
warm, one process per setting because the PARAGAN_* switches are read once).

    python tools/bench_wgrad.py [shape-filter]        # e.g. PARAGAN_WGRAD3=0 python tools/bench_wgrad.py 96
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_03999_b200 import api  # noqa: E402

SHAPES = [  # n, h, w, cin, cout (3x3)
    (512, 128, 128, 96, 96),
    (512, 64, 64, 96, 192),
    (512, 64, 64, 192, 192),
    (512, 32, 32, 192, 384),
    (512, 32, 32, 384, 384),
    (512, 16, 16, 384, 768),
    (512, 16, 16, 768, 768),
    (512, 8, 8, 1536, 1536),
]


def main():
    flt = sys.argv[1] if len(sys.argv) > 1 else ""
    dev = "cuda:0"
    for n, h, w, cin, cout in SHAPES:
        if flt and flt not in f"{cin}->{cout}@{h}":
            continue
        x = torch.randn(n, h, w, cin, device=dev).to(torch.bfloat16)
        dy = torch.randn(n, h, w, cout, device=dev).to(torch.bfloat16)
        dw = torch.empty(cout, 9, cin, device=dev)
        db = torch.empty(cout, device=dev)
        for _ in range(3):
            api.op_conv_wgrad(api.BF16, x, dy, cout, 3, dw, db=db)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 10
        e0.record()
        for _ in range(it):
            api.op_conv_wgrad(api.BF16, x, dy, cout, 3, dw, db=db)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        fl = 2.0 * n * h * w * cin * cout * 9
        print(f"wgrad {cin}->{cout}@{h} n{n}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s", flush=True)
        del x, dy


if __name__ == "__main__":
    main()
