import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2411_03999_b200 import api
from tests import parity as P
B = 8
ocfg = P.oracle_config(32, 4, 16, 10, 16, 4, bf16=True)
cfg = api.make_config(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4, local_batch=B, compute=api.BF16)
gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, B, seed=31)
got = P.run_gpu(cfg, g0, d0, dbs, gb)
want = P.run_oracle(ocfg, gs, ds, g0, d0, dbs, gb)
import dataclasses
pc = dataclasses.replace(ocfg, bf16=False)
plain = P.run_oracle(pc, *P.make_inputs(pc, B, seed=31))
for key, specs in (("d_grads", ds), ("g_grads", gs)):
    print(key, "global gpu-emu", P.rel(got[key], want[key]), "emu-plain", P.rel(want[key], plain[key]))
    o = 0
    for s in specs:
        n = int(np.prod(s.shape))
        e1 = P.rel(got[key][o:o+n], want[key][o:o+n]); e2 = P.rel(want[key][o:o+n], plain[key][o:o+n])
        if e1 > 0.05: print(f"   {s.name:20s} gpu-emu {e1:.3e} emu-plain {e2:.3e} |w|={np.linalg.norm(want[key][o:o+n]):.3e}")
        o += n
