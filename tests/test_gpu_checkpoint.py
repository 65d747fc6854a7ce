"""Asynchronous checkpoint writer (paragan_checkpoint_*): a checkpoint taken while
training continues restores the exact state — resuming from it reproduces the uninterrupted run bit for
bit (weights, SN vectors, optimiser moments and step counts, Lookahead slow weights) — and corrupt or
mismatched files are rejected."""
import numpy as np
import pytest
import torch

from paper_2411_03999_b200 import api
from tests import parity as P

pytestmark = pytest.mark.gpu
MICRO = dict(resolution=32, ch=4, attn_res=16, n_classes=10, shared_dim=16, z_chunk=4)


def _step(ctx, dbs, gb, compute):
    tdt = torch.bfloat16 if compute == api.BF16 else torch.float32
    real, ry, z, fy = dbs[0]
    rp = torch.empty((real.shape[0], 32, 32, 8), dtype=tdt, device="cuda:0")
    api.layout_pack(torch.from_numpy(real).cuda(), rp, compute, 8)
    ctx.d_step(rp, torch.from_numpy(ry).cuda(), torch.from_numpy(z).cuda(), torch.from_numpy(fy).cuda())
    ctx.g_step(torch.from_numpy(gb[0]).cuda(), torch.from_numpy(gb[1]).cuda())


@pytest.mark.parametrize("compute", [api.F32, api.BF16])
def test_checkpoint_resume_is_bit_exact(tmp_path, compute):
    pol = api.make_policy(rule=api.OPT_ADABELIEF, lookahead_k=2)
    cfg = api.make_config(**MICRO, local_batch=4, compute=compute, policy_g=pol)
    ocfg = P.oracle_config(32, 4, 16, 10, 16, 4)
    gs, ds, g0, d0, dbs1, gb1 = P.make_inputs(ocfg, 4, seed=91)
    _, _, _, _, dbs2, gb2 = P.make_inputs(ocfg, 4, seed=92)
    path = str(tmp_path / "ck.pgc")
    a = api.Context(cfg)
    a.set_params(api.NET_G, g0)
    a.set_params(api.NET_D, d0)
    _step(a, dbs1, gb1, compute)
    a.checkpoint_save_async(path)        # snapshot is stream-ordered: the next step cannot race it
    _step(a, dbs2, gb2, compute)         # training continues while the file is written
    _step(a, dbs1, gb2, compute)
    a.checkpoint_wait()
    ref = [a.get_params(api.NET_D), a.get_params(api.NET_G), a.sync_stats()]
    a.close()
    b = api.Context(cfg)
    b.init_params(0.3)                   # arbitrary state, overwritten by the load
    b.checkpoint_load(path)
    _step(b, dbs2, gb2, compute)
    _step(b, dbs1, gb2, compute)
    got = [b.get_params(api.NET_D), b.get_params(api.NET_G), b.sync_stats()]
    b.close()
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    assert (got[2].t_d, got[2].t_g) == (ref[2].t_d, ref[2].t_g) == (3, 3)


def test_checkpoint_rejects_corrupt_and_mismatched(tmp_path):
    cfg = api.make_config(**MICRO, local_batch=2, compute=api.F32)
    a = api.Context(cfg)
    a.init_params(0.1)
    path = str(tmp_path / "ck.pgc")
    a.checkpoint_save_async(path)
    a.checkpoint_wait()
    raw = bytearray(open(path, "rb").read())
    raw[-100] ^= 0xFF
    bad = str(tmp_path / "bad.pgc")
    open(bad, "wb").write(bytes(raw))
    with pytest.raises(api.ParaganError) as e:
        a.checkpoint_load(bad)
    assert e.value.status == 4
    other = api.Context(api.make_config(**{**MICRO, "ch": 8}, local_batch=2, compute=api.F32))
    with pytest.raises(api.ParaganError) as e:
        other.checkpoint_load(path)
    assert e.value.status == 2
    with pytest.raises(api.ParaganError) as e:
        a.checkpoint_load(str(tmp_path / "missing.pgc"))
    assert e.value.status == 4
    other.close()
    a.close()
