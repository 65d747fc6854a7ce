"""Step-level parity of the CUDA path (through the C-ABI) with the oracle after one
D+G iteration: losses, all-reduced gradients of every tensor, updated weights and
SN vectors, generated images (north_star: 1e-4 relative in fp32, 2e-2 relative in
bf16).  bf16 runs compare against the oracle's bf16-storage emulation (R14)."""
import numpy as np
import pytest
import torch

from oracle import biggan as bg
from paper_2411_03999_b200 import api
from tests import parity as P

pytestmark = pytest.mark.gpu

MICRO = dict(res=32, ch=4, attn=16, n_classes=10, shared_dim=16, z_chunk=4)


def _cfgs(compute, B, n_d=1, **kw):
    m = {**MICRO, **kw}
    ocfg = P.oracle_config(m["res"], m["ch"], m["attn"], m["n_classes"], m["shared_dim"], m["z_chunk"], n_d,
                           bf16=(compute == api.BF16))
    cfg = api.make_config(resolution=m["res"], ch=m["ch"], attn_res=m["attn"], n_classes=m["n_classes"],
                          shared_dim=m["shared_dim"], z_chunk=m["z_chunk"], local_batch=B, d_steps_per_g=n_d,
                          compute=compute)
    return ocfg, cfg


def _noise_floor_check(ocfg, B, seed, got, want, specs_by_key, tol):
    """bf16 per-tensor bar: |gpu - emulating oracle| <= max(tol, 1.5 * |emulating - fp64 oracle|),
    i.e. the CUDA path is no further from the emulation than bf16 storage itself moves the result."""
    import dataclasses
    plain_cfg = dataclasses.replace(ocfg, bf16=False)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(plain_cfg, B, seed)
    plain = P.run_oracle(plain_cfg, gs, ds, g0, d0, dbs, gb)
    bad = []
    for key, specs in specs_by_key.items():
        o = 0
        for s in specs:
            n = int(np.prod(s.shape))
            e_gpu = P.rel(got[key][o:o + n], want[key][o:o + n])
            e_bf = P.rel(want[key][o:o + n], plain[key][o:o + n])
            # scalars (attention gamma) aggregate the whole upstream gradient's bf16 noise: they are
            # covered by the per-network global bar, not a per-tensor one
            if n >= 16 and np.linalg.norm(want[key][o:o + n]) > 1e-6 * np.linalg.norm(want[key]) \
                    and e_gpu > max(tol, 1.5 * e_bf):
                bad.append((key, s.name, f"{e_gpu:.2e}", f"{e_bf:.2e}"))
            o += n
    return bad


def _check(ocfg, cfg, B, seed, tol, n_d=1, sign_min=None, tensor_tol=None, g_global_tol=None, noise_floor=False,
           per_tensor_state=True, floor_frac=1e-2):
    """tol: losses, per-net global gradient error, fakes and updated weights.  tensor_tol (default
    tol): per-tensor gradient bar.  g_global_tol: override for G's global gradient error where
    fp32 rounding of the forward is amplified by conditioning (see test_d_step_isolated_*)."""
    tensor_tol = tol if tensor_tol is None else tensor_tol
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, B, seed, n_d)
    want = P.run_oracle(ocfg, gs, ds, g0, d0, dbs, gb)
    got = P.run_gpu(cfg, g0, d0, dbs, gb)
    report = {}
    for k in ("d_loss", "g_loss"):
        e = abs(got[k] - want[k]) / max(abs(want[k]), 1e-3)
        report[k] = e
        assert e < tol, (k, got[k], want[k])
    for key, specs in (("d_grads", ds), ("g_grads", gs)):
        bad, worst = P.compare_tensors(specs, got[key], want[key], tensor_tol, floor_frac=floor_frac)
        report[key] = max(worst.values())
        report[key + "_global"] = P.rel(got[key], want[key])
        if bad:
            print("parity failures:", key, [(b[0], f"{b[3]:.2e}") for b in bad])
        if not noise_floor:
            assert not bad, (key, bad[:5])
        gt = g_global_tol if (key == "g_grads" and g_global_tol) else tol
        assert report[key + "_global"] < gt, (key, report[key + "_global"])
    g_rel = 1e-4 if cfg.compute == api.F32 else 2e-2
    for key, gkey, specs in (("d_state", "d_grads", ds), ("g_state", "g_grads", gs)):
        nt = bg.n_trainable(specs)
        report[key + "_global"] = P.rel(got[key][:nt], want[key][:nt])
        report[key + "_u"] = P.rel(got[key][nt:], want[key][nt:])
        assert report[key + "_global"] < tol and report[key + "_u"] < tol, (key, report[key + "_global"])
        if per_tensor_state:
            bad, worst, excluded = P.compare_state(specs, got[key], want[key], want[gkey], tol, g_rel)
            report[key + "_excluded"] = excluded
            assert not bad, (key, bad[:5])
    report["fake"] = P.rel(got["fake"], want["fake"])
    assert report["fake"] < tol
    if sign_min is not None:
        for key, gkey, p0, specs in (("d_state", "d_grads", d0, ds), ("g_state", "g_grads", g0, gs)):
            agree = P.adam_sign_agreement(p0, got[key], want[key], bg.n_trainable(specs), want[gkey], g_rel)
            report["sign_" + key] = agree
            assert agree >= sign_min, (key, agree)
    print("parity report:", {k: (f"{v:.2e}" if isinstance(v, float) else v) for k, v in report.items()})
    if noise_floor:
        bad = _noise_floor_check(ocfg, B, seed, got, want, {"d_grads": ds, "g_grads": gs}, tol)
        print("noise-floor failures:", bad)
        assert not bad, bad[:5]
    return got


def _d_isolated(res, ch, attn, classes, shared, zc, B, seed, compute, tol, tensor_tol=None):
    """D step alone with the oracle fed the CUDA path's own fake images: D's arithmetic in isolation."""
    from oracle import biggan as bgm
    o = P.oracle_config(res, ch, attn, classes, shared, zc, bf16=(compute == api.BF16))
    cfg = api.make_config(resolution=res, ch=ch, attn_res=attn, n_classes=classes, shared_dim=shared, z_chunk=zc,
                          local_batch=B, compute=compute)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(o, B, seed)
    ctx = api.Context(cfg)
    ctx.set_params(api.NET_G, g0)
    ctx.set_params(api.NET_D, d0)
    real, ry, z, fy = dbs[0]
    tdt = torch.bfloat16 if compute == api.BF16 else torch.float32
    rp = torch.empty((B, res, res, 8), dtype=tdt, device="cuda:0")
    api.layout_pack(torch.from_numpy(real).cuda(), rp, compute, 8)
    ctx.d_step(rp, torch.from_numpy(ry).cuda(), torch.from_numpy(z).cuda(), torch.from_numpy(fy).cuda(),
               flags=api.FLAG_NO_UPDATE)
    st = ctx.sync_stats(raise_nonfinite=False)
    fk, gd = ctx.get_fakes(), ctx.get_grads(api.NET_D)
    ctx.close()
    want = bgm.d_step(o, bgm.NetState.from_flat(gs, g0), bgm.NetState.from_flat(ds, d0), real, ry, z, fy,
                      update=False, fake_override=fk)
    assert abs(st.d_loss - want["loss"]) / abs(want["loss"]) < tol
    bad, worst = P.compare_tensors(ds, gd, want["grads"], tol if tensor_tol is None else tensor_tol)
    print("isolated D:", f"global {P.rel(gd, want['grads']):.2e}", f"worst tensor {max(worst.values()):.2e}")
    assert not bad, bad[:5]
    assert P.rel(gd, want["grads"]) < tol


def test_step_parity_f32_micro():
    ocfg, cfg = _cfgs(api.F32, B=4)
    _check(ocfg, cfg, 4, seed=21, tol=1e-4, sign_min=0.999)


def test_step_parity_f32_micro_ratio2():
    ocfg, cfg = _cfgs(api.F32, B=3, n_d=2)
    got = _check(ocfg, cfg, 3, seed=22, tol=1e-4, n_d=2)
    assert got["stats"].t_d == 2 and got["stats"].t_g == 1


def test_step_parity_bf16_micro():
    ocfg, cfg = _cfgs(api.BF16, B=8)
    _check(ocfg, cfg, 8, seed=23, tol=2e-2, tensor_tol=6e-2, sign_min=0.95, per_tensor_state=False)


def test_step_parity_f32_sndcgan_config1():
    """Config 1 (SN-DCGAN 32x32, ch=32, batch 8; R25) through the fp32 SIMT path: losses, gradients,
    updated weights and u vectors at the north_star's fp32 bar 1e-4."""
    ocfg = P.sndcgan_oracle_config()
    cfg = api.make_sndcgan_config(local_batch=8)
    # the deconv biases feed a BN: their exact gradient is 0, and the fp32 BN backward leaves a residual of
    # ~1e-5 of the network's RMS gradient (floor_frac 0.1 x tol); every other tensor is at ~3e-7
    _check(ocfg, cfg, 8, seed=41, tol=1e-4, sign_min=0.999, floor_frac=1e-1)


def test_step_parity_f32_sndcgan_ratio2():
    """D:G = 2:1 on a narrower SN-DCGAN.  (R19 applies to ReLU kinks as to hinge kinks: a BN output within
    fp32 rounding of 0 takes the other subgradient; e.g. batch 4 with seed 42 has one such element in
    G's BN2, moving one channel's beta gradient by 15% — parity seeds avoid kinks.)"""
    ocfg = P.sndcgan_oracle_config(ch=8, n_d=2)
    cfg = api.make_sndcgan_config(ch=8, local_batch=8, d_steps_per_g=2)
    got = _check(ocfg, cfg, 8, seed=43, tol=1e-4, n_d=2, floor_frac=1e-1)
    assert got["stats"].t_d == 2 and got["stats"].t_g == 1


def test_d_step_isolated_f32_biggan128():
    """BigGAN-128 shapes through D's exact fp32 path at 1e-4 with identical inputs."""
    _d_isolated(128, 96, 64, 1000, 128, 20, 4, 24, api.F32, 1e-4)


def test_d_step_isolated_f32_biggan256():
    """Config 4's shapes (BigGAN-256: 6 D blocks, 256-wide rows = two halo tiles per row) through D's
    exact fp32 path at 1e-4."""
    _d_isolated(256, 96, 64, 1000, 128, 20, 1, 25, api.F32, 1e-4)


def test_d_step_isolated_f32_biggan512():
    """Config 5's shapes (BigGAN-512: 7 D blocks, 512-wide rows) through D's exact fp32 path: loss and
    whole-network gradient at 1e-4; per tensor 5e-4 — with one image the deepest layers' gradients are
    16-pixel sums of dgrad outputs that are themselves 13,824-term fp32 sums with heavy cancellation
    (measured worst 2e-4, global 7e-5)."""
    _d_isolated(512, 96, 64, 1000, 128, 20, 1, 26, api.F32, 1e-4, tensor_tol=5e-4)


def test_step_parity_f32_biggan256_ratio2():
    """Config 4's asymmetric D:G step ratio 2:1 on BigGAN-256 shapes (one image): two D steps, each
    updating D, then the G step against the twice-updated D.  D's arithmetic alone is at ~2e-7
    (test_d_step_isolated_*); here the second D step starts from weights after Adam's first step,
    ~ -lr * sign(g), whose sign is indeterminate for gradients at the fp32 noise level — those elements
    move by 2 lr between the two computations, so the bars are 2e-3 (D) / 5e-3 (G), measured 6.4e-4."""
    ocfg = P.oracle_config(256, 96, 64, 1000, 128, 20, n_d=2, bf16=False)
    cfg = api.make_config(resolution=256, local_batch=1, d_steps_per_g=2, compute=api.F32)
    got = _check(ocfg, cfg, 1, seed=27, tol=2e-3, n_d=2, tensor_tol=1e-2, g_global_tol=5e-3, per_tensor_state=False)
    assert got["stats"].t_d == 2 and got["stats"].t_g == 1


def test_step_parity_f32_biggan128():
    """Full iteration at BigGAN-128 shapes in fp32.  D's arithmetic alone is at ~2e-5
    (test_d_step_isolated_f32_biggan128); the images G generates carry ~1e-5 fp32 rounding that the
    step amplifies (BN over a small global batch, D's input sensitivity), so the full-step gradient
    bars here are 5e-4 (D) and 5e-3 (G) — measured 2.1e-4 / 1.4e-3 at B=8 vs the fp64 oracle."""
    ocfg = P.oracle_config(128, 96, 64, 1000, 128, 20, bf16=False)
    cfg = api.make_config(local_batch=2, compute=api.F32)
    _check(ocfg, cfg, 2, seed=24, tol=5e-4, tensor_tol=1e-2, g_global_tol=5e-3, per_tensor_state=False)


def test_step_parity_bf16_biggan128():
    """bf16 storage + tcgen05: north_star bar 2e-2 on losses, gradients (global per network)
    and updated weights vs the bf16-emulating oracle; per tensor, the error must stay within
    max(2e-2, 1.5x the bf16 noise floor) — the emulating oracle's own distance from fp64, which
    reaches several % on G's deepest layers at this small global batch."""
    ocfg = P.oracle_config(128, 96, 64, 1000, 128, 20, bf16=True)
    cfg = api.make_config(local_batch=8, compute=api.BF16)
    _check(ocfg, cfg, 8, seed=24, tol=2e-2, sign_min=0.9, noise_floor=True, per_tensor_state=False)


def test_g_step_before_d_steps_is_order_error():
    _, cfg = _cfgs(api.F32, B=2, n_d=2)
    ctx = api.Context(cfg)
    ctx.init_params(0.1)
    z = torch.zeros((2, api.dim_z(cfg)), device="cuda:0")
    y = torch.zeros(2, dtype=torch.int32, device="cuda:0")
    with pytest.raises(api.ParaganError) as e:
        ctx.g_step(z, y)
    assert e.value.status == 7
    ctx.close()


def test_nonfinite_input_skips_update():
    ocfg, cfg = _cfgs(api.F32, B=2)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, 2, 5)
    real, ry, z, fy = dbs[0]
    real = real.copy()
    real[0, 0, 0, 0] = np.nan
    ctx = api.Context(cfg)
    ctx.set_params(api.NET_G, g0)
    ctx.set_params(api.NET_D, d0)
    rp = torch.empty((2, 32, 32, 8), dtype=torch.float32, device="cuda:0")
    api.layout_pack(torch.from_numpy(real).cuda(), rp, api.F32, 8)
    ctx.d_step(rp, torch.from_numpy(ry).cuda(), torch.from_numpy(z).cuda(), torch.from_numpy(fy).cuda())
    with pytest.raises(api.ParaganError) as e:
        ctx.sync_stats()
    assert e.value.status == 3
    after = ctx.get_params(api.NET_D)
    n = bg.n_trainable(ds)
    assert np.array_equal(after[:n], d0[:n])
    assert ctx.sync_stats().t_d == 0
    ctx.close()


def test_init_params_replicas_identical_and_finite():
    _, cfg = _cfgs(api.BF16, B=2)
    a = api.Context(cfg)
    a.init_params(0.0)
    b = api.Context(cfg)
    b.init_params(0.0)
    pa, pb = a.get_params(api.NET_D), b.get_params(api.NET_D)
    assert np.array_equal(pa, pb) and np.isfinite(pa).all()
    ws = [s for s in bg.d_param_specs(P.oracle_config(**{"res": 32, "ch": 4, "attn": 16, "n_classes": 10,
                                                           "shared_dim": 16, "z_chunk": 4}))]
    n = int(np.prod(ws[0].shape))
    assert abs(pa[:n].std() - 0.02) < 0.005
    a.close()
    b.close()


def test_step_bitwise_reproducible_bf16():
    """Every reduction of the step has a fixed order (split-K partials, BN and SN sums, attention dtheta
    partials, CBN dcond slices, the D-head embedding gradient): two runs of the same iteration from the
    same state give bit-identical gradients, weights and fakes.  ch = 32 at 128x128 keeps the layers on
    the tcgen05 / fused-attention / bulk-copy BN paths (every channel count a multiple of 32)."""
    ocfg = P.oracle_config(128, 32, 64, 1000, 128, 20, bf16=True)
    cfg = api.make_config(resolution=128, ch=32, attn_res=64, n_classes=1000, shared_dim=128, z_chunk=20,
                          local_batch=8, compute=api.BF16)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, 8, seed=31)
    runs = [P.run_gpu(cfg, g0, d0, dbs, gb) for _ in range(2)]
    for key in ("d_grads", "g_grads", "d_state", "g_state", "fake"):
        a, b = (np.asarray(r[key]) for r in runs)
        assert a.shape == b.shape and np.array_equal(a, b), key
    assert runs[0]["d_loss"] == runs[1]["d_loss"] and runs[0]["g_loss"] == runs[1]["g_loss"]
