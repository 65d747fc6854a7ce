"""Asynchronous update scheme on the GPU (paper_2411_03999_b200/async_gan.py):
max_staleness = 0 reproduces the synchronous iteration bit for bit, and staleness-1 runs —
equal and different G / D batch sizes ("Async G-512 D-256") — match the oracle's schedule
(oracle/async_scheme.py) at the fp32 bar."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import async_scheme as OA
from oracle import biggan as bg
from oracle import optim as O
from paper_2411_03999_b200 import api, inputs
from paper_2411_03999_b200.async_gan import LocalAsync
from tests import parity as P

pytestmark = pytest.mark.gpu
MICRO = dict(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4)
DEV = "cuda:0"


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _pack(real, compute):
    tdt = torch.bfloat16 if compute == api.BF16 else torch.float32
    rp = torch.empty((real.shape[0], 32, 32, 8), dtype=tdt, device=DEV)
    api.layout_pack(_dev(real), rp, compute, 8)
    return rp


def _ticks(ocfg, d_batch, g_batch, n_d, n_ticks, seed):
    out = []
    for t in range(n_ticks):
        d = []
        for k in range(n_d):
            real, ry = inputs.real_batch(seed, t * n_d + k, d_batch, 32, ocfg.n_classes)
            zb, yb = inputs.latent_batch(seed, inputs.ROLE_Z_D, t * n_d + k, d_batch, ocfg.dim_z, ocfg.n_classes)
            d.append((real, ry, zb, yb))
        zg, yg = inputs.latent_batch(seed, inputs.ROLE_Z_G, t, g_batch, ocfg.dim_z, ocfg.n_classes)
        out.append({"d": d, "g": (zg, yg)})
    return out


def test_staleness0_equals_sync_iteration_bitwise():
    compute = api.F32
    cfg = api.make_config(**MICRO, local_batch=4, compute=compute)
    ocfg = P.oracle_config(32, 4, 16, 10, 16, 4)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, 4, seed=71)
    sync_ctx = api.Context(cfg)
    sync = P.run_gpu(cfg, g0, d0, dbs, gb, ctx=sync_ctx)
    sync_ctx.close()
    la = LocalAsync(cfg, cfg, max_staleness=0)
    la.set_params(g0, d0)
    real, ry, z, fy = dbs[0]
    rec = la.tick([(_pack(real, compute), _dev(ry), _dev(z), _dev(fy))], (_dev(gb[0]), _dev(gb[1])))
    assert rec == {"d_staleness": [0], "g_snapshot_staleness": 0}
    g_async = la.ctx_g.get_params(api.NET_G)
    d_async = la.ctx_g.get_params(api.NET_D)    # the G side's D copy carries the G step's power step (R31)
    d_live = la.ctx_d.get_params(api.NET_D)
    nt = bg.n_trainable(ds)
    assert np.array_equal(g_async, sync["g_state"])
    assert np.array_equal(la.ctx_g.get_grads(api.NET_G), sync["g_grads"])
    assert np.array_equal(la.ctx_d.get_grads(api.NET_D), sync["d_grads"])
    assert np.array_equal(d_async, sync["d_state"])
    assert np.array_equal(d_live[:nt], sync["d_state"][:nt])
    la.close()


SGD_D, SGD_G = (0.1, 0.0, 0.999, None), (0.05, 0.0, 0.999, None)


def sgd_configs(g_batch, d_batch, n_d, **kw):
    """The schedule tests train with plain SGD at a large step (lr 0.1 / 0.05): every update is linear in its
    gradient, so the comparison measures the schedule (which fakes / which D snapshot each step used) with
    fp32 noise ~1e-6 — Adam's first steps ~ -lr sign(g) would turn rounding noise on near-zero gradients
    into full-size sign flips."""
    ocfg = dataclasses.replace(P.oracle_config(32, 4, 16, 10, 16, 4), adam_d=bg.AdamHP(0.1, 0.0, 0.999, 1e-8),
                               adam_g=bg.AdamHP(0.05, 0.0, 0.999, 1e-8), policy_d=O.Policy(rule="sgd"),
                               policy_g=O.Policy(rule="sgd"))
    sgd = api.make_policy(rule=api.OPT_SGD)
    cfg_g = api.make_config(**MICRO, local_batch=g_batch, compute=api.F32, adam_d=SGD_D, adam_g=SGD_G, policy_d=sgd,
                            policy_g=sgd, **kw)
    cfg_d = api.make_config(**MICRO, local_batch=d_batch, d_steps_per_g=n_d, compute=api.F32, adam_d=SGD_D,
                            adam_g=SGD_G, policy_d=sgd, policy_g=sgd, **kw)
    return ocfg, cfg_g, cfg_d


@pytest.mark.parametrize("d_batch,g_batch,n_d", [(4, 4, 1), (2, 4, 2)])
def test_staleness1_matches_oracle_schedule(d_batch, g_batch, n_d):
    """Three ticks with max_staleness = 1: D on the previous tick's fakes, G through the previous tick's D;
    the accumulated updates w_3 - w_0 of G and D vs the oracle's schedule at the fp32 bar 1e-4."""
    compute = api.F32
    ocfg, cfg_g, cfg_d = sgd_configs(g_batch, d_batch, n_d)
    gs, ds = bg.g_param_specs(ocfg), bg.d_param_specs(ocfg)
    g0 = inputs.init_params(gs, 72, inputs.ROLE_PARAMS_G)
    d0 = inputs.init_params(ds, 72, inputs.ROLE_PARAMS_D)
    ticks = _ticks(ocfg, d_batch, g_batch, n_d, 3, seed=73)
    G, D = bg.NetState.from_flat(gs, g0), bg.NetState.from_flat(ds, d0)
    want = OA.run(ocfg, G, D, ticks, max_staleness=1, d_batch=d_batch)
    la = LocalAsync(cfg_g, cfg_d, max_staleness=1)
    la.set_params(g0, d0)
    recs = []
    for tk in ticks:
        recs.append(la.tick([(_pack(r, compute), _dev(ry), _dev(zb), _dev(yb)) for r, ry, zb, yb in tk["d"]],
                            (_dev(tk["g"][0]), _dev(tk["g"][1]))))
    assert [r["d_staleness"] for r in recs] == [w["d_staleness"] for w in want]
    assert [r["g_snapshot_staleness"] for r in recs] == [w["g_snapshot_staleness"] for w in want]
    assert recs[1]["d_staleness"] == [1] * n_d and recs[1]["g_snapshot_staleness"] == 1
    got_g, got_d = la.ctx_g.get_params(api.NET_G), la.ctx_d.get_params(api.NET_D)
    st = la.ctx_d.sync_stats(raise_nonfinite=False)
    la.close()
    for got, st_, w0, specs in ((got_g, G, g0, gs), (got_d, D, d0, ds)):
        nt = bg.n_trainable(specs)
        e = P.rel(got[:nt] - w0[:nt], st_.flat()[:nt] - w0[:nt])
        print("async update rel err", f"{e:.2e}")
        assert e < 1e-4
    assert st.t_d == 3 * n_d
