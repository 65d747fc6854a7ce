"""Pins for the oracle's model and training step: the paper's parameter count
(P:56), central finite differences of the full D and G losses on micro nets,
the data-parallel decomposition the multi-GPU path relies on, and step-level
invariants (non-finite skip, Adam bookkeeping, SN cadence)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import biggan as bg
from oracle import ops
from paper_2411_03999_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MICRO = dict(resolution=16, ch=2, n_classes=5, shared_dim=4, z_chunk=3, attn_res=8)
MICRO_DCGAN = dict(arch="sndcgan", resolution=32, ch=4, n_classes=5)   # config 1's topology at ch=4


def test_biggan128_parameter_count_matches_paper():
    with open(os.path.join(GOLDEN, "biggan128_params_p56.json")) as f:
        g = json.load(f)
    cfg = bg.Config(**g["config"])
    n = bg.n_trainable(bg.g_param_specs(cfg)) + bg.n_trainable(bg.d_param_specs(cfg))
    assert round(n / 1e6, 2) == g["params_millions_rounded_2dp"]
    assert n == 158_416_358
    # and the attention block is what makes it 158.42M rather than 158.36M
    cfg0 = bg.Config(**{**g["config"], "attn_res": 0})
    n0 = bg.n_trainable(bg.g_param_specs(cfg0)) + bg.n_trainable(bg.d_param_specs(cfg0))
    assert round(n0 / 1e6, 2) == 158.36


def test_sn_weight_counts_biggan128():
    cfg = bg.Config()
    assert sum(s.sn for s in bg.g_param_specs(cfg)) == 41
    assert sum(s.sn for s in bg.d_param_specs(cfg)) == 23


def _setup(cfg, B, seed=11, gamma=0.3):
    gs, ds = bg.g_param_specs(cfg), bg.d_param_specs(cfg)
    G = bg.NetState.from_flat(gs, inputs.init_params(gs, seed, inputs.ROLE_PARAMS_G, attn_gamma=gamma, std=0.2))
    D = bg.NetState.from_flat(ds, inputs.init_params(ds, seed, inputs.ROLE_PARAMS_D, attn_gamma=gamma, std=0.2))
    # non-zero biases so that every term is exercised
    rng = np.random.default_rng(seed)
    for st in (G, D):
        for s in st.specs:
            if s.init == "zero":
                st.params[s.name] = torch.tensor(rng.standard_normal(s.shape) * 0.1)
    real, ry = inputs.real_batch(seed, 0, B, cfg.resolution, cfg.n_classes)
    z, fy = inputs.latent_batch(seed, inputs.ROLE_Z_D, 0, B, cfg.dim_z, cfg.n_classes)
    return G, D, real, ry, z, fy


def _dir_check(loss_fn, params: dict, grads: dict, rng, h=1e-6):
    """Per tensor: central difference along a random direction vs <grad, d>."""
    worst = 0.0
    for name, p in params.items():
        d = torch.tensor(rng.standard_normal(tuple(p.shape)))
        scale = float(p.abs().mean()) or 1.0
        d = d * scale
        plus = {**params, name: p + h * d}
        minus = {**params, name: p - h * d}
        fd = (loss_fn(plus) - loss_fn(minus)) / (2 * h)
        an = float((grads[name] * d).sum())
        # FD noise floor ~ 1e-16 * |L| / h ~ 1e-10; BN makes some grads exactly 0
        assert abs(fd - an) <= 1e-5 * abs(an) + 1e-8, (name, fd, an)
        worst = max(worst, abs(fd - an) / max(abs(an), 1e-12))
    return worst


@pytest.mark.parametrize("micro", [MICRO, MICRO_DCGAN], ids=["biggan", "sndcgan"])
def test_d_step_gradients_match_finite_differences(micro):
    cfg = bg.Config(**micro)
    G, D, real, ry, z, fy = _setup(cfg, B=3)
    Dp0 = {k: v.clone() for k, v in D.params.items()}
    us_d0 = {k: v.clone() for k, v in D.us.items()}
    out = bg.d_step(cfg, G, D, real, ry, z, fy, update=False)
    assert np.all(np.abs(np.abs(out["logits"]) - 1.0) > 1e-4)     # away from hinge kinks (R19)
    # rebuild the exact frozen SN vectors of that forward
    fake = torch.tensor(out["fake"])
    snd = bg._SN(D.specs, dict(Dp0), dict(us_d0), cfg.sn_eps, False)
    x = torch.cat([fake, bg.pack_real(cfg, real)], 0)
    yy = torch.cat([torch.tensor(fy, dtype=torch.long), torch.tensor(ry, dtype=torch.long)])
    bg.d_forward(cfg, snd, x, yy)
    frozen = dict(snd.vectors)
    B = 3

    def loss(params):
        sn = bg._SN(D.specs, params, dict(us_d0), cfg.sn_eps, False, frozen=frozen)
        lg = bg.d_forward(cfg, sn, x, yy)
        return float(ops.hinge_d(lg[B:], lg[:B]))

    assert abs(loss(Dp0) - out["loss"]) < 1e-12
    grads, _ = bg.unflatten(D.specs, np.concatenate([out["grads"], np.zeros(sum(s.shape[0] for s in D.specs if s.sn))]))
    _dir_check(loss, Dp0, grads, np.random.default_rng(0))


@pytest.mark.parametrize("micro", [MICRO, MICRO_DCGAN], ids=["biggan", "sndcgan"])
def test_g_step_gradients_match_finite_differences(micro):
    cfg = bg.Config(**micro)
    G, D, real, ry, z, fy = _setup(cfg, B=3)
    Gp0 = {k: v.clone() for k, v in G.params.items()}
    us_g0 = {k: v.clone() for k, v in G.us.items()}
    us_d0 = {k: v.clone() for k, v in D.us.items()}
    out = bg.g_step(cfg, G, D, z, fy, update=False)
    zt = torch.tensor(z, dtype=torch.float64)
    yt = torch.tensor(fy, dtype=torch.long)
    sng = bg._SN(G.specs, dict(Gp0), dict(us_g0), cfg.sn_eps, False)
    fake = bg.g_forward(cfg, sng, zt, yt)
    snd = bg._SN(D.specs, D.params, dict(us_d0), cfg.sn_eps, False)
    bg.d_forward(cfg, snd, fake, yt)
    fg, fd_ = dict(sng.vectors), dict(snd.vectors)

    def loss(params):
        s1 = bg._SN(G.specs, params, dict(us_g0), cfg.sn_eps, False, frozen=fg)
        s2 = bg._SN(D.specs, D.params, dict(us_d0), cfg.sn_eps, False, frozen=fd_)
        return float(ops.hinge_g(bg.d_forward(cfg, s2, bg.g_forward(cfg, s1, zt, yt), yt)))

    assert abs(loss(Gp0) - out["loss"]) < 1e-12
    grads, _ = bg.unflatten(G.specs, np.concatenate([out["grads"], np.zeros(sum(s.shape[0] for s in G.specs if s.sn))]))
    _dir_check(loss, Gp0, grads, np.random.default_rng(1))


def test_iteration_bookkeeping_and_sn_cadence():
    cfg = bg.Config(**MICRO, d_steps_per_g=2)
    G, D, real, ry, z, fy = _setup(cfg, B=2)
    u_g0 = {k: v.clone() for k, v in G.us.items()}
    b2 = (real, ry, *inputs.latent_batch(11, inputs.ROLE_Z_D, 1, 2, cfg.dim_z, cfg.n_classes))
    zg, yg = inputs.latent_batch(11, inputs.ROLE_Z_G, 0, 2, cfg.dim_z, cfg.n_classes)
    out = bg.iteration(cfg, G, D, [(real, ry, z, fy), b2], (zg, yg))
    assert D.t == 2 and G.t == 1
    assert all(o["applied"] for o in out["d"]) and out["g"]["applied"]
    # G's u advanced n_d + 1 = 3 times: replay the power steps by hand
    name = "b0.conv1.w"
    w = bg.unflatten(G.specs, inputs.init_params(G.specs, 11, inputs.ROLE_PARAMS_G, attn_gamma=0.3, std=0.2))[0][name]
    u = u_g0[name]
    for _ in range(2):
        _, u, _ = ops.sn_power_step(w, u, cfg.sn_eps)   # G weights unchanged during D steps
    # the third step used the same W (G is updated after its forward)
    _, u, _ = ops.sn_power_step(w, u, cfg.sn_eps)
    assert torch.allclose(G.us[name], u, rtol=0, atol=1e-14)


def test_nonfinite_gradient_skips_update():
    cfg = bg.Config(**MICRO)
    G, D, real, ry, z, fy = _setup(cfg, B=2)
    before = D.flat().copy()
    real = real.copy()
    real[0, 0, 0, 0] = np.nan
    out = bg.d_step(cfg, G, D, real, ry, z, fy)
    assert not out["applied"] and D.t == 0
    after = D.flat()
    n = bg.n_trainable(D.specs)
    assert np.array_equal(before[:n], after[:n])


def test_data_parallel_decomposition_of_d_gradient():
    """D has no BN: the global-batch gradient equals the mean over W shards of each
    shard's mean-loss gradient — what the per-rank loss + all-reduce(mean) computes (R15)."""
    cfg = bg.Config(**MICRO)
    G, D, real, ry, z, fy = _setup(cfg, B=4)
    out = bg.d_step(cfg, G, D, real, ry, z, fy, update=False)
    fake = torch.tensor(out["fake"])
    xr = bg.pack_real(cfg, real)
    W = 2
    acc = None
    for r in range(W):
        sl = slice(2 * r, 2 * r + 2)
        dp = {k: v.detach().clone().requires_grad_(True) for k, v in D.params.items()}
        us = dict(bg.NetState.from_flat(D.specs, inputs.init_params(D.specs, 11, inputs.ROLE_PARAMS_D, 0.3, 0.2)).us)
        sn = bg._SN(D.specs, dp, us, cfg.sn_eps, False)
        lg = bg.d_forward(cfg, sn, torch.cat([fake[sl], xr[sl]]),
                          torch.cat([torch.tensor(fy[sl], dtype=torch.long), torch.tensor(ry[sl], dtype=torch.long)]))
        loss = ops.hinge_d(lg[2:], lg[:2])
        gl = torch.autograd.grad(loss, [dp[s.name] for s in D.specs], allow_unused=True)
        flat = torch.cat([(g if g is not None else torch.zeros_like(dp[s.name])).reshape(-1)
                          for g, s in zip(gl, D.specs)]).numpy()
        acc = flat / W if acc is None else acc + flat / W
    assert np.allclose(acc, out["grads"], rtol=1e-9, atol=1e-12)


def test_sndcgan_parameter_counts_and_deconv_adjoint():
    """Config 1 (R25): SURVEY Appendix B's counts follow from the layer listing (a reading — the
    paper prints none), and the deconv is the adjoint of the strided conv with the same weight."""
    cfg = bg.Config(arch="sndcgan", resolution=32, ch=32)
    assert bg.n_trainable(bg.g_param_specs(cfg)) == 1_226_243
    assert bg.n_trainable(bg.d_param_specs(cfg)) == 736_801
    assert sum(s.sn for s in bg.g_param_specs(cfg)) == 0 and sum(s.sn for s in bg.d_param_specs(cfg)) == 8
    rng = np.random.default_rng(3)
    x = torch.tensor(rng.standard_normal((2, 5, 4, 4)))
    y = torch.tensor(rng.standard_normal((2, 3, 8, 8)))
    w = torch.tensor(rng.standard_normal((5, 3, 4, 4)))
    lhs = (torch.nn.functional.conv_transpose2d(x, w, stride=2, padding=1) * y).sum()
    rhs = (x * torch.nn.functional.conv2d(y, w, stride=2, padding=1)).sum()
    assert abs(float(lhs - rhs)) < 1e-10 * abs(float(lhs))


def _bf16_exact(t: torch.Tensor) -> bool:
    t = t.detach()
    return bool(torch.equal(ops.bf16_round(t), t))


@pytest.mark.parametrize("bf16", [True, False])
def test_bf16_emulation_obeys_the_storage_rule(monkeypatch, bf16):
    """Pin of the oracle's bf16 mode (R14) by the rule itself, independent of any
    kernel: every tensor-core product of the step (each conv and each attention bmm) reads bf16
    operands in the forward, and the output gradient its backward reads (the dgrad/wgrad operand) is
    bf16 — except G's output conv, which is fp32 by P:202.  A dropped or misplaced q()/qv()/qg()
    breaks one of these.  The fp64 mode (bf16=False) must violate it (the check is not vacuous), and
    the emulation moves the losses by a bf16-sized amount, not zero and not more."""
    cfg = bg.Config(**MICRO, bf16=bf16)
    G, D, real, ry, z, fy = _setup(cfg, 3, seed=5)
    seen = {"fwd": 0, "bad_fwd": [], "bwd": 0, "bad_bwd": []}
    real_conv, real_bmm = ops.conv2d, torch.bmm

    def watch(name, out):
        def hook(g):
            seen["bwd"] += 1
            if not _bf16_exact(g):
                seen["bad_bwd"].append(name)
        if out.requires_grad:
            out.register_hook(hook)
        return out

    def conv(x, w, b):
        out = real_conv(x, w, b)
        if w.shape[0] == 3 and w.shape[-1] == 3 and x.shape[1] == cfg.ch * 1 * 1 * \
                bg._G_ARCH[cfg.resolution][1][-1]:
            return out                                  # G's output conv: fp32
        seen["fwd"] += 1
        if not (_bf16_exact(x) and _bf16_exact(w)):
            seen["bad_fwd"].append(("conv", tuple(w.shape)))
        if w.shape[-1] == 1 and 2 * w.shape[1] == w.shape[0] and x.shape[1] == w.shape[1] \
                and cfg.attn_res == x.shape[-1]:
            return out      # attention o conv: its epilogue scales by gamma, so its input gradient is gamma x bf16
        return watch(("conv", tuple(w.shape)), out)

    def bmm(a, b):
        out = real_bmm(a, b)
        seen["fwd"] += 1
        if not (_bf16_exact(a) and _bf16_exact(b)):
            seen["bad_fwd"].append(("bmm", tuple(a.shape)))
        return watch(("bmm", tuple(a.shape)), out)

    monkeypatch.setattr(ops, "conv2d", conv)
    monkeypatch.setattr(bg.torch, "bmm", bmm)
    out_d = bg.d_step(cfg, G, D, real, ry, z, fy)
    out_g = bg.g_step(cfg, G, D, z, fy)
    monkeypatch.undo()
    n_conv_d = sum(1 for s in bg.d_param_specs(cfg) if len(s.shape) == 4)
    assert seen["fwd"] >= n_conv_d + 2 and seen["bwd"] >= n_conv_d
    if bf16:
        assert not seen["bad_fwd"], seen["bad_fwd"][:5]
        assert not seen["bad_bwd"], seen["bad_bwd"][:5]
        # against the fp64 step from the same state: a bf16-sized, non-zero change of the losses
        cfg64 = bg.Config(**MICRO, bf16=False)
        G2, D2, real, ry, z, fy = _setup(cfg64, 3, seed=5)
        ref_d = bg.d_step(cfg64, G2, D2, real, ry, z, fy)
        ref_g = bg.g_step(cfg64, G2, D2, z, fy)
        for a, b in ((out_d["loss"], ref_d["loss"]), (out_g["loss"], ref_g["loss"])):
            assert 0 < abs(a - b) / abs(b) < 2e-2
    else:
        assert seen["bad_fwd"] and seen["bad_bwd"]


def test_async_schedule_staleness0_reduces_to_sync_iteration():
    """oracle/async_scheme.py with max_staleness = 0 is the synchronous iteration: same
    losses, G state and D weights after a tick; D's u vectors differ only by the G step's power step,
    which runs on the snapshot copy (R31) — and the snapshot copy equals the sync D exactly."""
    import copy
    from oracle import async_scheme as OA
    cfg = bg.Config(**MICRO)
    G, D, real, ry, z, fy = _setup(cfg, 2, seed=9)
    zg, yg = inputs.latent_batch(9, inputs.ROLE_Z_G, 0, 2, cfg.dim_z, cfg.n_classes)
    G2, D2 = copy.deepcopy(G), copy.deepcopy(D)
    sync = bg.iteration(cfg, G, D, [(real, ry, z, fy)], (zg, yg))
    rec = OA.run(cfg, G2, D2, [{"d": [(real, ry, z, fy)], "g": (zg, yg)}], max_staleness=0, d_batch=2)
    assert rec[0]["d_loss"][0] == sync["d"][0]["loss"] and rec[0]["g_loss"] == sync["g"]["loss"]
    assert rec[0]["d_staleness"] == [0] and rec[0]["g_snapshot_staleness"] == 0
    assert np.array_equal(G2.flat(), G.flat())
    nt = bg.n_trainable(D.specs)
    assert np.array_equal(D2.flat()[:nt], D.flat()[:nt])


def test_async_schedule_staleness1_uses_previous_tick():
    """With max_staleness = 1 the D step of tick t trains on the fakes G produced at tick t-1 (P:275
    "generator of the previous iteration") and the G step of tick t through D after tick t-1: the second
    tick's D loss equals a D step on tick 1's G-step fakes, computed directly."""
    import copy
    from oracle import async_scheme as OA
    cfg = bg.Config(**MICRO)
    G, D, real, ry, z, fy = _setup(cfg, 2, seed=10)
    ticks = []
    for t in range(2):
        r_, ry_ = inputs.real_batch(10, t, 2, cfg.resolution, cfg.n_classes)
        zb, yb = inputs.latent_batch(10, inputs.ROLE_Z_D, t, 2, cfg.dim_z, cfg.n_classes)
        zg, yg = inputs.latent_batch(10, inputs.ROLE_Z_G, t, 2, cfg.dim_z, cfg.n_classes)
        ticks.append({"d": [(r_, ry_, zb, yb)], "g": (zg, yg)})
    G0, D0 = copy.deepcopy(G), copy.deepcopy(D)
    rec = OA.run(cfg, G, D, ticks, max_staleness=1, d_batch=2)
    assert [r["d_staleness"] for r in rec] == [[0], [1]] and [r["g_snapshot_staleness"] for r in rec] == [1, 1]
    # by hand: tick 0 = D on G0's fresh fakes; G through the initial D; tick 1 = D on those G-step fakes
    r0 = bg.d_step(cfg, None, D0, *ticks[0]["d"][0][:2], None, ticks[0]["d"][0][3],
                   fakes=OA.generate(cfg, G0, ticks[0]["d"][0][2], ticks[0]["d"][0][3]))
    Dinit = bg.NetState.from_flat(D.specs, _setup(cfg, 2, seed=10)[1].flat())
    rg = bg.g_step(cfg, G0, Dinit, *ticks[0]["g"])
    r1 = bg.d_step(cfg, None, D0, *ticks[1]["d"][0][:2], None, ticks[0]["g"][1], fakes=rg["fake"])
    assert rec[0]["d_loss"][0] == r0["loss"] and rec[1]["d_loss"][0] == r1["loss"]
