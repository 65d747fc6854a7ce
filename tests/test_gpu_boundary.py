"""The C-ABI's split entry points on one GPU (include/paragan.h): paragan_allreduce_grads and
paragan_apply_update called directly reproduce the fused step bit for bit, and the gradient test hooks
round-trip exactly.  The multi-rank allreduce-sum invariant (north_star) is
tests/test_gpu_dist.py::test_two_gpu_allreduce_sum_invariant."""
import numpy as np
import pytest
import torch

from oracle import biggan as bg
from paper_2411_03999_b200 import api
from tests import parity as P

pytestmark = pytest.mark.gpu
MICRO = dict(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4)


def _iteration(cfg, g0, d0, dbs, gb, split):
    ctx = api.Context(cfg)
    ctx.set_params(api.NET_G, g0)
    ctx.set_params(api.NET_D, d0)
    tdt = torch.bfloat16 if cfg.compute == api.BF16 else torch.float32
    real, ry, z, fy = dbs[0]
    rp = torch.empty((cfg.local_batch, 32, 32, 8), dtype=tdt, device="cuda:0")
    api.layout_pack(torch.from_numpy(real).cuda(), rp, cfg.compute, 8)
    fl = api.FLAG_NO_ALLREDUCE | api.FLAG_NO_UPDATE if split else 0
    ctx.d_step(rp, torch.from_numpy(ry).cuda(), torch.from_numpy(z).cuda(), torch.from_numpy(fy).cuda(), flags=fl)
    if split:
        ctx.allreduce_grads(api.NET_D)
        ctx.apply_update(api.NET_D)
    zg, yg = gb
    ctx.g_step(torch.from_numpy(zg).cuda(), torch.from_numpy(yg).cuda(), flags=fl)
    if split:
        ctx.allreduce_grads(api.NET_G)
        ctx.apply_update(api.NET_G)
    st = ctx.sync_stats(raise_nonfinite=False)
    out = dict(d=ctx.get_params(api.NET_D), g=ctx.get_params(api.NET_G), gd=ctx.get_grads(api.NET_D),
               gg=ctx.get_grads(api.NET_G), t=(st.t_d, st.t_g))
    ctx.close()
    return out


@pytest.mark.parametrize("compute", [api.F32, api.BF16])
def test_split_calls_equal_fused_step(compute):
    cfg = api.make_config(**MICRO, local_batch=4, compute=compute)
    ocfg = P.oracle_config(32, 4, 16, 10, 16, 4, bf16=compute == api.BF16)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, 4, seed=61)
    a = _iteration(cfg, g0, d0, dbs, gb, split=False)
    b = _iteration(cfg, g0, d0, dbs, gb, split=True)
    for k in ("d", "g", "gd", "gg"):
        assert np.array_equal(a[k], b[k]), k
    assert a["t"] == b["t"] == (1, 1)


def test_set_get_grads_round_trip_and_single_rank_allreduce_is_identity():
    cfg = api.make_config(**MICRO, local_batch=2, compute=api.BF16)
    ctx = api.Context(cfg)
    ctx.init_params(0.1)
    for net in (api.NET_D, api.NET_G):
        n = ctx._n(net, False)
        g = np.random.default_rng(net).standard_normal(n).astype(np.float32)
        ctx.set_grads(net, g)
        assert np.array_equal(ctx.get_grads(net), g)
        ctx.allreduce_grads(net)
        assert np.array_equal(ctx.get_grads(net), g)
    ctx.close()


def test_apply_update_is_the_oracle_adam_step():
    """paragan_apply_update on a set gradient: one Adam step (R12) vs oracle/ops.adam_update in fp64."""
    cfg = api.make_config(**MICRO, local_batch=2, compute=api.F32)
    ocfg = P.oracle_config(32, 4, 16, 10, 16, 4)
    ctx = api.Context(cfg)
    ctx.init_params(0.1)
    ds = bg.d_param_specs(ocfg)
    w0 = ctx.get_params(api.NET_D)
    n = bg.n_trainable(ds)
    g = np.random.default_rng(5).standard_normal(n).astype(np.float32) * 1e-3
    ctx.set_grads(api.NET_D, g)
    ctx.apply_update(api.NET_D)
    w1 = ctx.get_params(api.NET_D)
    ctx.close()
    from oracle import ops
    hp = cfg.adam_d
    want, _, _ = ops.adam_update(torch.from_numpy(w0[:n]).double(), torch.from_numpy(g).double(),
                                 torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64), 1,
                                 hp.lr, hp.beta1, hp.beta2, hp.eps)
    d_got, d_want = w1[:n].astype(np.float64) - w0[:n], want.numpy() - w0[:n]
    assert np.linalg.norm(d_got - d_want) / np.linalg.norm(d_want) < 1e-5
    assert np.array_equal(w1[n:], w0[n:])


def _three_iterations(cfg, g0, d0, dbs, gb, graphs):
    """Three D+G iterations on the same device inputs (from the second on, the CUDA-graph step cache replays
    the captured steps); returns params, stats and the async stats of the last iteration."""
    import ctypes
    import os
    old = os.environ.get("PARAGAN_GRAPHS")
    os.environ["PARAGAN_GRAPHS"] = "1" if graphs else "0"
    try:
        ctx = api.Context(cfg)
    finally:
        if old is None:
            del os.environ["PARAGAN_GRAPHS"]
        else:
            os.environ["PARAGAN_GRAPHS"] = old
    ctx.set_params(api.NET_G, g0)
    ctx.set_params(api.NET_D, d0)
    tdt = torch.bfloat16 if cfg.compute == api.BF16 else torch.float32
    real, ry, z, fy = dbs[0]
    rp = torch.empty((cfg.local_batch, 32, 32, 8), dtype=tdt, device="cuda:0")
    api.layout_pack(torch.from_numpy(real).cuda(), rp, cfg.compute, 8)
    ry, z, fy = (torch.from_numpy(a).cuda() for a in (ry, z, fy))
    zg, yg = (torch.from_numpy(a).cuda() for a in gb)
    buf = torch.empty(ctypes.sizeof(api.Stats), dtype=torch.uint8).pin_memory()
    for _ in range(3):
        ctx.d_step(rp, ry, z, fy)
        ctx.g_step(zg, yg)
    ctx.stats_async(buf)
    torch.cuda.synchronize()
    sa = api.Context.read_stats(buf)
    st = ctx.sync_stats(raise_nonfinite=False)
    out = dict(d=ctx.get_params(api.NET_D), g=ctx.get_params(api.NET_G), launches=ctx.kernel_launches(),
               stats=(st.d_loss, st.g_loss, st.d_real_mean, st.d_fake_mean, st.t_d, st.t_g),
               async_stats=(sa.d_loss, sa.g_loss, sa.d_real_mean, sa.d_fake_mean, sa.t_d, sa.t_g))
    ctx.close()
    return out


def test_graph_step_cache_replays_the_eager_steps_and_async_stats_match():
    """The CUDA-graph step cache: three iterations with replayed steps are bit-identical to three
    eager ones (weights, losses, step counters, launch count); paragan_stats_async delivers what
    paragan_sync_stats reports."""
    cfg = api.make_config(**MICRO, local_batch=4, compute=api.BF16)
    ocfg = P.oracle_config(32, 4, 16, 10, 16, 4, bf16=True)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, 4, seed=67)
    a = _three_iterations(cfg, g0, d0, dbs, gb, graphs=True)
    b = _three_iterations(cfg, g0, d0, dbs, gb, graphs=False)
    assert np.array_equal(a["d"], b["d"]) and np.array_equal(a["g"], b["g"])
    assert a["stats"] == b["stats"] and a["stats"][4:] == (3, 3)
    assert a["launches"] == b["launches"]
    assert a["async_stats"] == a["stats"]
