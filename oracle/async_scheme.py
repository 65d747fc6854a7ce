"""Asynchronous update scheme (PAPER.md:266-282 [Sec. 5.1], Fig. 5) — oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:277 "instead of waiting on the other component, the generator/discriminator can write their
intermediate output to the buffer and proceed to update using the current state of the network.  For
iteration t, discriminators D_t receive a batch of real and generated samples from the image buffer
(img_buff).  Similarly, the generators can use the snapshot of the current discriminator state ... to
calculate to gradient for backpropagation, breaking the data dependency."  P:275 "the discriminator can
still perform well even if its input comes from the generator of the previous iteration."

The schedule, written as a deterministic interleaving of ticks (readings R31-R33 in DESIGN.md):
  * img_buff holds (fakes, labels, tag) entries, tag = the tick of the G version that made them;
    the snapshot buffer holds (copy of D, tag), tag = the tick after whose D update it was taken
    (-1 = the initial D).
  * tick t, D side: n_d D steps; each drops img_buff entries with t - tag > max_staleness, pops the
    oldest remaining one, or — when none is left (cold start, or max_staleness = 0) — generates one
    from the current G (SN(G) power step + G forward, tag t); then a D step on it (no G forward).
    Afterwards the D state is snapshotted with tag t.
  * tick t, G side: the G step runs through the snapshot tagged t - max_staleness (the oldest one
    available at cold start), as a copy: the live D is not touched (its u vectors included, R31); the
    G step's fakes (tag t) are pushed, split into g_batch / d_batch entries ("possible to apply
    different batch sizes for both parties").
With max_staleness = 0 a tick is the synchronous iteration (D on fresh fakes of the current G, G through
the just-updated D); the only difference is R31 (the live D's u vectors do not advance in the G step).
"""
from __future__ import annotations

import copy

import numpy as np
import torch

from . import biggan as bg


def generate(cfg, G, z, y):
    """SN(G) power step + G forward without gradients: the images as stored for D (bf16 in bf16 mode)."""
    sng = bg._SN(G.specs, G.params, G.us, cfg.sn_eps, cfg.bf16)
    with torch.no_grad():
        f = bg.g_forward(cfg, sng, torch.as_tensor(np.asarray(z, np.float32)).double(),
                         torch.as_tensor(np.asarray(y)).long())
    return bg.q(f, cfg.bf16).numpy()


def run(cfg, G, D, ticks, max_staleness, d_batch, boot_all_at_once=False):
    """ticks: list of dicts with 'd' = [(real, real_y, z_boot, y_boot)] * n_d and 'g' = (z, y) (G batch).
    boot_all_at_once: the cold start generates tick 0's whole G-sized batch in one G forward (the
    distributed driver's G rank does this) instead of one d_batch per D step.
    Returns per-tick records (losses, staleness of what was consumed)."""
    img_buff, snaps = [], [(copy.deepcopy(D), -1)]
    out = []
    if boot_all_at_once:
        zb = np.concatenate([d[2] for d in ticks[0]["d"]])
        yb = np.concatenate([d[3] for d in ticks[0]["d"]])
        f = generate(cfg, G, zb, yb)
        for i in range(0, f.shape[0], d_batch):
            img_buff.append((f[i:i + d_batch], yb[i:i + d_batch], 0))
    for t, tk in enumerate(ticks):
        rec = {"d_loss": [], "d_staleness": []}
        for real, ry, zb, yb in tk["d"]:
            img_buff = [e for e in img_buff if t - e[2] <= max_staleness]
            if not img_buff:
                img_buff.append((generate(cfg, G, zb, yb), np.asarray(yb), t))
            fakes, fy, tag = img_buff.pop(0)
            r = bg.d_step(cfg, None, D, real, ry, None, fy, fakes=fakes)
            rec["d_loss"].append(r["loss"])
            rec["d_staleness"].append(t - tag)
        snaps.append((copy.deepcopy(D), t))
        want = t - max_staleness
        cand = [s for s in snaps if s[1] <= want]
        snap, stag = (cand[-1] if cand else snaps[0])
        snaps = [s for s in snaps if s[1] >= stag]
        Dsnap = copy.deepcopy(snap)
        z, y = tk["g"]
        rg = bg.g_step(cfg, G, Dsnap, z, y)
        rec["g_loss"] = rg["loss"]
        rec["g_snapshot_staleness"] = t - stag
        f, yy = rg["fake"], np.asarray(y)
        for i in range(0, f.shape[0], d_batch):
            img_buff.append((f[i:i + d_batch], yy[i:i + d_batch], t))
        out.append(rec)
    return out
