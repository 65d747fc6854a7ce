"""Per-tensor parity report of one iteration: CUDA path vs the oracle (bf16-emulating
and plain fp64).  Diagnostic tool; tests/test_gpu_step.py holds the pass/fail bars.

    python tools/parity_report.py [--res 32 --ch 4 --attn 16 --classes 10 --shared 16 --zc 4 --batch 4 --bf16]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, default=32)
    ap.add_argument("--ch", type=int, default=4)
    ap.add_argument("--attn", type=int, default=16)
    ap.add_argument("--classes", type=int, default=10)
    ap.add_argument("--shared", type=int, default=16)
    ap.add_argument("--zc", type=int, default=4)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seed", type=int, default=23)
    ap.add_argument("--bf16", action="store_true")
    ap.add_argument("--summary", action="store_true")
    ap.add_argument("--d-only", action="store_true", help="D step alone, oracle fed the GPU's fake images")
    ap.add_argument("--g-isolated", action="store_true", help="G step alone, oracle fed the GPU's dL/dfake")
    a = ap.parse_args()
    import numpy as np
    from paper_2411_03999_b200 import api
    from tests import parity as P
    compute = api.BF16 if a.bf16 else api.F32
    cfg = api.make_config(resolution=a.res, ch=a.ch, attn_res=a.attn, n_classes=a.classes, shared_dim=a.shared,
                          z_chunk=a.zc, local_batch=a.batch, compute=compute)
    if a.g_isolated:
        import numpy as np
        from tests import test_gpu_step as T
        T._g_isolated(a.res, a.ch, a.attn, a.classes, a.shared, a.zc, a.batch, a.seed, compute, verbose=True)
        return
    if a.d_only:
        import torch
        from oracle import biggan as bg
        o = P.oracle_config(a.res, a.ch, a.attn, a.classes, a.shared, a.zc, bf16=a.bf16)
        gs, ds, g0, d0, dbs, gb = P.make_inputs(o, a.batch, a.seed)
        ctx = api.Context(cfg)
        ctx.set_params(api.NET_G, g0)
        ctx.set_params(api.NET_D, d0)
        real, ry, z, fy = dbs[0]
        tdt = torch.bfloat16 if a.bf16 else torch.float32
        rp = torch.empty((a.batch, a.res, a.res, 8), dtype=tdt, device="cuda:0")
        api.layout_pack(torch.from_numpy(real).cuda(), rp, compute, 8)
        ctx.d_step(rp, torch.from_numpy(ry).cuda(), torch.from_numpy(z).cuda(), torch.from_numpy(fy).cuda(),
                   flags=api.FLAG_NO_UPDATE)
        st = ctx.sync_stats(raise_nonfinite=False)
        fk = ctx.get_fakes()
        gd = ctx.get_grads(api.NET_D)
        G = bg.NetState.from_flat(gs, g0)
        D = bg.NetState.from_flat(ds, d0)
        want = bg.d_step(o, G, D, real, ry, z, fy, update=False, fake_override=fk)
        wfree = bg.d_step(o, bg.NetState.from_flat(gs, g0), bg.NetState.from_flat(ds, d0), real, ry, z, fy,
                          update=False)
        print(f"D-only: loss gpu {st.d_loss:.7f} oracle(gpu fakes) {want['loss']:.7f}; fake err {P.rel(fk, wfree['fake']):.2e}")
        print(f"D-only grads vs oracle on the GPU's fakes: {P.rel(gd, want['grads']):.2e}; "
              f"vs oracle's own fakes: {P.rel(gd, wfree['grads']):.2e}")
        return
    res = {}
    for emu in ([True, False] if a.bf16 else [False]):
        o = P.oracle_config(a.res, a.ch, a.attn, a.classes, a.shared, a.zc, bf16=emu)
        gs, ds, g0, d0, dbs, gb = P.make_inputs(o, a.batch, a.seed)
        res[emu] = P.run_oracle(o, gs, ds, g0, d0, dbs, gb)
    got = P.run_gpu(cfg, g0, d0, dbs, gb)
    first = next(iter(res.values()))
    print("oracle D logits", np.round(first["d_logits"], 4), "G logits", np.round(first["g_logits"], 4))
    print(f"losses gpu d={got['d_loss']:.6f} g={got['g_loss']:.6f}; oracle " +
          " ".join(f"[emu={k}] d={v['d_loss']:.6f} g={v['g_loss']:.6f}" for k, v in res.items()))
    print("fake rel err vs " + " ".join(f"emu={k}: {P.rel(got['fake'], v['fake']):.2e}" for k, v in res.items()))
    print("d_grads global " + " ".join(f"emu={k}: {P.rel(got['d_grads'], v['d_grads']):.2e}" for k, v in res.items()))
    print("g_grads global " + " ".join(f"emu={k}: {P.rel(got['g_grads'], v['g_grads']):.2e}" for k, v in res.items()))
    ref = res[False]
    for key, specs in (("d_grads", ds), ("g_grads", gs)):
        live = P.live_mask(specs, ref[key])
        print(f"{key} global over live tensors (exact gradient non-zero, {live.mean():.4f} of elements): " +
              " ".join(f"emu={k}: {P.rel(got[key][live], v[key][live]):.2e}" for k, v in res.items()) +
              f"; dead-tensor noise |gpu| / |g| = {np.linalg.norm(got[key][~live]) / np.linalg.norm(ref[key]):.2e}")
    if a.summary:
        return
    for key, specs in (("d_grads", ds), ("g_grads", gs)):
        print(f"\n{key}: tensor | rel err vs " + " | ".join(f"emu={k}" for k in res) + " | emu vs plain")
        o = 0
        for s in specs:
            n = int(np.prod(s.shape))
            row = []
            for k in res:
                row.append(P.rel(got[key][o:o + n], res[k][key][o:o + n]))
            extra = ""
            if len(res) == 2:
                extra = f" | {P.rel(res[True][key][o:o + n], res[False][key][o:o + n]):.2e}"
            nrm = np.linalg.norm(res[False][key][o:o + n]) / np.linalg.norm(res[False][key])
            print(f"  {s.name:22s} " + " ".join(f"{r:.2e}" for r in row) + extra + f" | norm share {nrm:.2e}")
            o += n


if __name__ == "__main__":
    main()
