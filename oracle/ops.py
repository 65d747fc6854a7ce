"""Primitive operations of the oracle (test infrastructure only; see oracle/__init__.py).

Each function is the plain definition of one step of the hot path, in float64
unless it *is* a storage rounding.  Citations: P:n = /root/reference/PAPER.md
line n; R<k> = the reading recorded in DESIGN.md §3.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

F64 = torch.float64


# ---------------------------------------------------------------------------
# bf16 storage rounding  ("mixed-precision training with bf16")
# ---------------------------------------------------------------------------
def bf16_round(x: torch.Tensor) -> torch.Tensor:
    """Round to the nearest bfloat16 (ties to even), returned as float64.

    The value is first taken to float32 (the GPU stores fp32 before rounding),
    then to bfloat16 by PyTorch's conversion (a library routine; pinned against
    an independent bit formula in tests/test_oracle_primitives.py)."""
    return x.to(torch.float32).to(torch.bfloat16).to(F64)


class _Q(torch.autograd.Function):
    """Identity in exact arithmetic; rounds the forward value and the incoming
    gradient to bf16 (see :func:`q`)."""

    @staticmethod
    def forward(ctx, x):
        return bf16_round(x)

    @staticmethod
    def backward(ctx, g):
        return bf16_round(g)


class _QV(torch.autograd.Function):
    """Rounds the value to bf16; the gradient passes unrounded (see :func:`qv`)."""

    @staticmethod
    def forward(ctx, x):
        return bf16_round(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _QG(torch.autograd.Function):
    """Identity value; rounds the gradient to bf16 (see :func:`qg`)."""

    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return bf16_round(g)


# The bf16 storage rule (precision policy R14, "mixed-precision training with bf16"),
# stated once as layer-by-layer semantics: every layer (linear, conv with its bias and fused residual add,
# CBN+ReLU, resampling, pool, the attention core) reads bf16 tensors and writes ONE bf16 output; its
# backward reads the bf16 output gradient and writes a bf16 gradient for each input (a tensor read by
# several layers receives one rounded contribution per layer, summed); inside a layer the arithmetic is
# fp32 or better; tensor-core operands are bf16 in the forward and the backward.  G's output layer and
# D's head are fp32 throughout.  Three primitives express it:

def q(x: torch.Tensor, on: bool) -> torch.Tensor:
    """A layer's output: value stored bf16, and its gradient (the next layers' backward output) bf16."""
    return _Q.apply(x) if on else x


def qv(x: torch.Tensor, on: bool) -> torch.Tensor:
    """A tensor-core operand internal to one layer (the attention probabilities): bf16 value; its
    gradient stays inside the layer in fp32."""
    return _QV.apply(x) if on else x


def qg(x: torch.Tensor, on: bool) -> torch.Tensor:
    """A layer's input as seen by that layer's backward: the input-gradient contribution it writes is
    bf16 (also a backward tensor-core operand internal to a layer, the attention score gradient)."""
    return _QG.apply(x) if on else x


# ---------------------------------------------------------------------------
# Hardware-aware layout transformation
# ---------------------------------------------------------------------------
def layout_pack(x_nchw: np.ndarray, c_pad: int, to_bf16: bool) -> np.ndarray:
    """NCHW float32 -> NHWC with the channel dim zero-padded to ``c_pad``.

    Returned as float32 values (bf16-representable when ``to_bf16``)."""
    n, c, h, w = x_nchw.shape
    assert c_pad >= c
    out = np.zeros((n, h, w, c_pad), dtype=np.float32)
    out[..., :c] = np.transpose(x_nchw.astype(np.float32), (0, 2, 3, 1))
    if to_bf16:
        out = bf16_round(torch.from_numpy(out)).to(torch.float32).numpy()
    return out


def layout_unpack(x_nhwc: np.ndarray, c: int) -> np.ndarray:
    """Exact inverse of :func:`layout_pack` on the first ``c`` channels."""
    return np.ascontiguousarray(np.transpose(x_nhwc[..., :c], (0, 3, 1, 2))).astype(np.float32)


def padding_waste(rows: int, cols: int, tile: int) -> tuple[int, float]:
    """Zeros needed to pad a [rows, cols] operand to multiples of ``tile`` and the
    wasted fraction of the padded unit ([100,100] on 128x128 -> 6384, 39%)."""
    pr = -(-rows // tile) * tile
    pc = -(-cols // tile) * tile
    zeros = pr * pc - rows * cols
    return zeros, zeros / (pr * pc)


# ---------------------------------------------------------------------------
# Spectral normalisation (SNGAN, cited P:495; reading R4)
# ---------------------------------------------------------------------------
def l2n(x: torch.Tensor, eps: float) -> torch.Tensor:
    """n(x) = x / max(||x||_2, eps)."""
    return x / torch.clamp(torch.linalg.vector_norm(x), min=eps)


def sn_power_step(w: torch.Tensor, u: torch.Tensor, eps: float):
    """One power-iteration step on W viewed as [C_out, K] (R4):
    v = n(W^T u); u' = n(W v); sigma = u'^T W v.

    Returns (sigma, u', v); u' and v are constants (detached), sigma carries the
    gradient u' v^T through W."""
    wm = w.reshape(w.shape[0], -1)
    with torch.no_grad():
        v = l2n(wm.t() @ u, eps)
        u_new = l2n(wm @ v, eps)
    sigma = u_new @ (wm @ v)
    return sigma, u_new.detach(), v.detach()


# ---------------------------------------------------------------------------
# Convolution, resampling (R7, R9)
# ---------------------------------------------------------------------------
def conv2d(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None) -> torch.Tensor:
    """Cross-correlation, stride 1, zero 'same' padding (3x3 -> pad 1, 1x1 -> pad 0)."""
    return F.conv2d(x, w, b, stride=1, padding=w.shape[-1] // 2)


def up2(x: torch.Tensor) -> torch.Tensor:
    """Nearest x2 upsample: out[2i+a, 2j+b] = in[i, j]."""
    return x.repeat_interleave(2, dim=2).repeat_interleave(2, dim=3)


def up2_conv3x3_phases(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor | None) -> torch.Tensor:
    """conv3x3(up2(x)) written as four 2x2 convs of the low-resolution x, one per output phase (a, b)
    (reading R24).  Output row 2i+a reads input rows i-1+a+p, p in {0, 1}, with the
    folded kernel Wf_ab[p][q] = sum_{r in R(a,p), s in R(b,q)} W[r][s], R(0,0)={0}, R(0,1)={1,2},
    R(1,0)={0,1}, R(1,1)={2}.  Identical to conv2d(up2(x), w, b) in exact arithmetic (pinned in
    tests/test_oracle_primitives.py).  Not used by the training-step oracle (which convolves the
    upsampled tensor as BigGAN defines it); kept as the written-out statement of the identity the
    CUDA path's G conv1 relies on."""
    rows = {(0, 0): (0,), (0, 1): (1, 2), (1, 0): (0, 1), (1, 1): (2,)}
    phases = []
    for a in (0, 1):
        row = []
        for bb in (0, 1):
            taps = []
            for p in (0, 1):
                for q_ in (0, 1):
                    taps.append(sum(w[:, :, r, sc] for r in rows[(a, p)] for sc in rows[(bb, q_)]))
            wf = torch.stack(taps, dim=-1).reshape(w.shape[0], w.shape[1], 2, 2)
            xp = F.pad(x, (1 - bb, bb, 1 - a, a))      # (left, right, top, bottom)
            row.append(F.conv2d(xp, wf, b))
        phases.append(torch.stack(row, dim=-1))          # [N, C, H, W, 2(b)]
    y = torch.stack(phases, dim=3)                       # [N, C, H, 2(a), W, 2(b)]
    n, c, h, _, w_, _ = y.shape
    return y.reshape(n, c, 2 * h, 2 * w_)


def avgpool2(x: torch.Tensor) -> torch.Tensor:
    """2x2 average pool, stride 2."""
    n, c, h, w = x.shape
    return x.reshape(n, c, h // 2, 2, w // 2, 2).mean(dim=(3, 5))


def maxpool2(x: torch.Tensor) -> torch.Tensor:
    """2x2 max pool, stride 2."""
    return F.max_pool2d(x, 2)


# ---------------------------------------------------------------------------
# Cross-replica (conditional) batch norm (BigGAN; reading R5, R6)
# ---------------------------------------------------------------------------
def bn_normalise(x: torch.Tensor, eps: float) -> torch.Tensor:
    """x_hat over the GLOBAL batch and H, W per channel; biased variance (two-pass)."""
    mu = x.mean(dim=(0, 2, 3), keepdim=True)
    var = ((x - mu) ** 2).mean(dim=(0, 2, 3), keepdim=True)
    return (x - mu) / torch.sqrt(var + eps)


def cbn(x, gain, bias, eps):
    """Conditional BN: x_hat * (1 + gain[n, c]) + bias[n, c]."""
    return bn_normalise(x, eps) * (1.0 + gain[:, :, None, None]) + bias[:, :, None, None]


def bn_affine(x, gamma, beta, eps):
    """Plain BN with learned per-channel gamma/beta (G output BN)."""
    return bn_normalise(x, eps) * gamma[None, :, None, None] + beta[None, :, None, None]


# ---------------------------------------------------------------------------
# Non-local attention block (BigGAN; reading R8)
# ---------------------------------------------------------------------------
def attention(x, w_theta, w_phi, w_g, w_o, gamma):
    """theta = 1x1(x); phi = maxpool2(1x1(x)); g = maxpool2(1x1(x));
    beta = softmax_rows(theta^T phi) (no 1/sqrt(d)); out = x + gamma * 1x1(g beta^T)."""
    n, c, h, w = x.shape
    theta = conv2d(x, w_theta, None).reshape(n, -1, h * w)
    phi = maxpool2(conv2d(x, w_phi, None)).reshape(n, -1, h * w // 4)
    g = maxpool2(conv2d(x, w_g, None)).reshape(n, -1, h * w // 4)
    beta = torch.softmax(torch.bmm(theta.transpose(1, 2), phi), dim=-1)
    o = torch.bmm(g, beta.transpose(1, 2)).reshape(n, -1, h, w)
    return x + gamma * conv2d(o, w_o, None)


# ---------------------------------------------------------------------------
# Hinge loss (north_star; reading R3 — the paper states the log form at P:90)
# ---------------------------------------------------------------------------
def hinge_d(l_real: torch.Tensor, l_fake: torch.Tensor) -> torch.Tensor:
    """L_D = mean relu(1 - l_real) + mean relu(1 + l_fake)."""
    return torch.relu(1.0 - l_real).mean() + torch.relu(1.0 + l_fake).mean()


def hinge_g(l_fake: torch.Tensor) -> torch.Tensor:
    """L_G = -mean l_fake."""
    return -l_fake.mean()


# ---------------------------------------------------------------------------
# Adam (asymmetric policy P:285-307; larger eps under bf16 P:252; reading R12)
# ---------------------------------------------------------------------------
def adam_update(w, g, m, v, t, lr, beta1, beta2, eps):
    """PyTorch-form Adam with bias correction, eps outside the sqrt.
    Returns (w', m', v'); t is the 1-based step count of this update."""
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    return w - lr * mhat / (torch.sqrt(vhat) + eps), m, v
