"""Step-level parity of the CUDA path (through the C-ABI) with the oracle after one
D+G iteration: losses, all-reduced gradients of every tensor, updated weights and
SN vectors, generated images (north_star: 1e-4 relative in fp32, 2e-2 relative in
bf16).  bf16 runs compare against the oracle's bf16-storage emulation (R14)."""
import numpy as np
import pytest
import torch

from oracle import biggan as bg
from paragan_b200 import api
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


def _check(ocfg, cfg, B, seed, tol, n_d=1, sign_min=None):
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, B, seed, n_d)
    want = P.run_oracle(ocfg, gs, ds, g0, d0, dbs, gb)
    got = P.run_gpu(cfg, g0, d0, dbs, gb)
    report = {}
    for k in ("d_loss", "g_loss"):
        e = abs(got[k] - want[k]) / max(abs(want[k]), 1e-3)
        report[k] = e
        assert e < tol, (k, got[k], want[k])
    for key, specs in (("d_grads", ds), ("g_grads", gs)):
        bad, worst = P.compare_tensors(specs, got[key], want[key], tol)
        report[key] = max(worst.values())
        report[key + "_global"] = P.rel(got[key], want[key])
        if bad:
            print("parity failures:", key, [(b[0], f"{b[3]:.2e}") for b in bad])
        assert not bad, (key, bad[:5])
    g_rel = 1e-4 if cfg.compute == api.F32 else 2e-2
    for key, gkey, specs in (("d_state", "d_grads", ds), ("g_state", "g_grads", gs)):
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
    return got


def test_step_parity_f32_micro():
    ocfg, cfg = _cfgs(api.F32, B=4)
    _check(ocfg, cfg, 4, seed=21, tol=1e-4, sign_min=0.999)


def test_step_parity_f32_micro_ratio2():
    ocfg, cfg = _cfgs(api.F32, B=3, n_d=2)
    got = _check(ocfg, cfg, 3, seed=22, tol=1e-4, n_d=2)
    assert got["stats"].t_d == 2 and got["stats"].t_g == 1


def test_step_parity_bf16_micro():
    ocfg, cfg = _cfgs(api.BF16, B=4)
    _check(ocfg, cfg, 4, seed=23, tol=2e-2, sign_min=0.95)


def test_step_parity_f32_biggan128_b2():
    """Every BigGAN-128 shape (channel padding, attention at 64^2 with C/8 = 12 -> 16, 4x4 head)
    through the exact fp32 path at 1e-4."""
    ocfg = P.oracle_config(128, 96, 64, 1000, 128, 20, bf16=False)
    cfg = api.make_config(local_batch=2, compute=api.F32)
    _check(ocfg, cfg, 2, seed=24, tol=1e-4, sign_min=0.999)


def test_step_parity_bf16_biggan128_b2():
    ocfg = P.oracle_config(128, 96, 64, 1000, 128, 20, bf16=True)
    cfg = api.make_config(local_batch=2, compute=api.BF16)
    _check(ocfg, cfg, 2, seed=24, tol=2e-2, sign_min=0.9)


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
