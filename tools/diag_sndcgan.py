"""Diagnostic: SN-DCGAN (config 1) one iteration, CUDA path vs the fp64 oracle, per tensor."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2411_03999_b200 import api  # noqa: E402
from tests import parity as P  # noqa: E402

ch = int(sys.argv[1]) if len(sys.argv) > 1 else 32
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
nd = int(sys.argv[3]) if len(sys.argv) > 3 else 1
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 41
ocfg = P.sndcgan_oracle_config(ch=ch, n_d=nd)
cfg = api.make_sndcgan_config(ch=ch, local_batch=B, d_steps_per_g=nd)
gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, B, seed, nd)
want = P.run_oracle(ocfg, gs, ds, g0, d0, dbs, gb)
got = P.run_gpu(cfg, g0, d0, dbs, gb)
print("losses", got["d_loss"], want["d_loss"], got["g_loss"], want["g_loss"])
print("g logits oracle", np.round(want["g_logits"], 6))
print("fake rel", P.rel(got["fake"], want["fake"]))
for key, specs in (("d_grads", ds), ("g_grads", gs)):
    print(key, "global", P.rel(got[key], want[key]))
    if len(sys.argv) > 5:
        continue
    o = 0
    for s in specs:
        n = int(np.prod(s.shape))
        print(f"   {s.name:16s} {P.rel(got[key][o:o + n], want[key][o:o + n]):.2e}")
        o += n

if len(sys.argv) > 6:
    name = sys.argv[6]
    o = 0
    for s in gs:
        n = int(np.prod(s.shape))
        if s.name == name:
            print(name, "gpu ", np.array2string(got["g_grads"][o:o + n], precision=6, max_line_width=200))
            print(name, "want", np.array2string(want["g_grads"][o:o + n], precision=6, max_line_width=200))
        o += n
