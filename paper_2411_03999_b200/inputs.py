"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds none of the method's arithmetic: it only draws random
numbers with the distributions of the paper's workload (ImageNet-shaped
images in [-1, 1], 1000 classes, Gaussian latents) and the
initial-weight distribution of BigGAN (N(0, 0.02), zero biases, unit BN
gains, unit-norm Gaussian SN vectors).  Every array is a pure function of
(seed, role, step), via ``numpy.random.SeedSequence``.
"""
from __future__ import annotations

import numpy as np

ROLE_REAL, ROLE_Z_D, ROLE_Z_G, ROLE_PARAMS_G, ROLE_PARAMS_D = range(5)


def _rng(seed: int, role: int, step: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), int(role), int(step)]))


def real_batch(seed: int, step: int, batch: int, res: int, n_classes: int):
    """Real images [B,3,R,R] fp32 ~ U(-1,1) and labels [B] int32 ~ U{0..n_classes-1}."""
    r = _rng(seed, ROLE_REAL, step)
    x = r.uniform(-1.0, 1.0, size=(batch, 3, res, res)).astype(np.float32)
    y = r.integers(0, n_classes, size=(batch,), dtype=np.int64).astype(np.int32)
    return x, y


def latent_batch(seed: int, role: int, step: int, batch: int, dim_z: int, n_classes: int):
    """z [B, dim_z] fp32 ~ N(0,1) and labels [B] int32."""
    r = _rng(seed, role, step)
    z = r.standard_normal(size=(batch, dim_z)).astype(np.float32)
    y = r.integers(0, n_classes, size=(batch,), dtype=np.int64).astype(np.int32)
    return z, y


def shard(a: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Rows [rB, (r+1)B) of a global batch (R15)."""
    b = a.shape[0] // world
    return a[rank * b:(rank + 1) * b]


def init_params(specs, seed: int, role: int, attn_gamma: float = 0.1, std: float = 0.02) -> np.ndarray:
    """Canonical flat fp32 state for a list of specs (objects with .shape, .init, .sn):
    trainables in order, then one unit-norm N(0,1) u-vector per SN weight."""
    r = _rng(seed, role)
    parts = []
    for s in specs:
        n = int(np.prod(s.shape))
        if s.init == "normal":
            parts.append(r.standard_normal(n) * std)
        elif s.init == "zero":
            parts.append(np.zeros(n))
        elif s.init == "one":
            parts.append(np.ones(n))
        elif s.init == "attn_gamma":
            parts.append(np.full(n, attn_gamma))
        else:
            raise ValueError(s.init)
    for s in specs:
        if s.sn:
            u = r.standard_normal(s.shape[0])
            parts.append(u / np.linalg.norm(u))
    return np.concatenate(parts).astype(np.float32)


# ---------------------------------------------------------------------------
# Counter-based integer generator: the value of element i is a pure function of
# (seed, i), so a test can fill a full-size tensor on the device and recompute
# any sampled element on the host without moving the tensor.  Written with torch
# integer ops so the SAME code runs on either device.
# ---------------------------------------------------------------------------
def counter_ints(idx, seed: int, lo: int, hi: int):
    """Integers in [lo, hi] for the int64 flat indices ``idx`` (< 2**31): a 32-bit multiply-xorshift
    hash of (seed, i).  Every product stays below 2**63."""
    import torch
    h = (idx * 0x9E3779B1 + (int(seed) * 0x7FEB352D + 0x165667B1)) & 0xFFFFFFFF
    h = h ^ (h >> 15)
    h = (h * 0x2C1B3C6D) & 0xFFFFFFFF
    h = h ^ (h >> 12)
    h = (h * 0x297A2D39) & 0xFFFFFFFF
    h = h ^ (h >> 15)
    return lo + torch.remainder(h, hi - lo + 1)


def counter_tensor(shape, seed: int, lo: int, hi: int, device, dtype, chunk: int = 1 << 26):
    """A tensor of ``shape`` whose flat element i is counter_ints(i, seed, lo, hi), filled in chunks."""
    import torch
    n = 1
    for s in shape:
        n *= int(s)
    assert n < 2 ** 31
    out = torch.empty(n, dtype=dtype, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b] = counter_ints(torch.arange(a, b, dtype=torch.int64, device=device), seed, lo, hi).to(dtype)
    return out.reshape(shape)
