"""Convolution definitions evaluated at SAMPLED output elements (test infrastructure only; see
oracle/__init__.py).

At the benchmark's sizes (e.g. 512 images of 128x128x96) the full oracle convolution is too slow
on a CPU, so the full-size parity tests compare the CUDA path's outputs at sampled positions with
the plain definition evaluated at exactly those positions (task rule: "on sampled outputs the
oracle can compute one by one").  Each function is the textbook sum, written out:

  fprop (R9, cross-correlation, zero padding):
      y[n,i,j,o] = b[o] + sum_{r,s,c} x[n, i+r-p, j+s-p, c] * W[o, r*k+s, c],   p = k // 2
  with the step's fused epilogue terms in the order the layer defines them (mask, bias,
  residual, ReLU; dx = relu'(x) * dgrad + dskip);
  wgrad (A10):   dW[o, r*k+s, c] = sum_{n,i,j} dy[n,i,j,o] * x[n, i+r-p, j+s-p, c]
  G's conv1 on the nearest-x2-upsampled input (R7, A3): the same sums over up2(x)[I, J] =
  x[I // 2, J // 2]; its input gradient at low resolution is the up2 adjoint (sum over the 2x2
  block) of the full-resolution dgrad.

Values are supplied by callables ``x_at(n, i, j) -> [len(n), C]`` (in-bounds indices only) so
the caller decides how inputs are generated; everything is float64 (exact for the integer-valued
inputs the tests use)."""
from __future__ import annotations

import numpy as np


def _gather(x_at, n, i, j, H, W, C):
    """x at (n, i, j) with zero padding outside [0,H) x [0,W) -> [P, C] float64."""
    out = np.zeros((len(n), C), np.float64)
    ok = (i >= 0) & (i < H) & (j >= 0) & (j < W)
    if ok.any():
        out[ok] = x_at(n[ok], i[ok], j[ok])
    return out


def conv_fprop_at(x_at, H, W, cin, w_otc, k, n, i, j, bias=None, relu_ref_at=None, residual_at=None,
                  relu_out=False):
    """y[n,i,j,:] for the sampled output pixels (n, i, j) (int arrays) of a k x k, stride-1, 'same'
    conv; w_otc [cout, k*k, cin].  relu_ref_at(n,i,j) -> [P, cout] zeroes the conv sum where <= 0;
    residual_at(n,i,j) -> [P, cout] is added after the bias; relu_out applies ReLU last."""
    p = k // 2
    cout = w_otc.shape[0]
    acc = np.zeros((len(n), cout), np.float64)
    for r in range(k):
        for s in range(k):
            acc += _gather(x_at, n, i + r - p, j + s - p, H, W, cin) @ w_otc[:, r * k + s, :].T.astype(np.float64)
    if relu_ref_at is not None:
        acc = np.where(relu_ref_at(n, i, j) > 0, acc, 0.0)
    if bias is not None:
        acc = acc + bias[None, :]
    if residual_at is not None:
        acc = acc + residual_at(n, i, j)
    if relu_out:
        acc = np.maximum(acc, 0.0)
    return acc


def conv_wgrad_at(x_cols, dy_cols, H, W, k):
    """dW[o, r*k+s, c] for the sampled output channels o and input channels c, every tap:
    x_cols [N, H, W, Cs] = x[..., c in the sample], dy_cols [N, H, W, Os] = dy[..., o in the sample].
    Returns [Os, k*k, Cs] float64 (sum over every pixel of the batch)."""
    p = k // 2
    N = x_cols.shape[0]
    xp = np.zeros((N, H + 2 * p, W + 2 * p, x_cols.shape[-1]), np.float64)
    xp[:, p:p + H, p:p + W] = x_cols
    dy = dy_cols.reshape(-1, dy_cols.shape[-1]).astype(np.float64)
    out = np.zeros((dy_cols.shape[-1], k * k, x_cols.shape[-1]), np.float64)
    for r in range(k):
        for s in range(k):
            out[:, r * k + s, :] = dy.T @ xp[:, r:r + H, s:s + W].reshape(-1, x_cols.shape[-1])
    return out


def up2_conv3x3_fprop_at(x_at, h, w, cin, w_otc, n, I, J, bias=None):
    """conv3x3(up2(x)) + b at sampled full-resolution pixels (n, I, J); x is [N, h, w, cin]."""
    cout = w_otc.shape[0]
    acc = np.zeros((len(n), cout), np.float64)
    for r in range(3):
        for s in range(3):
            ii, jj = I + r - 1, J + s - 1
            ok = (ii >= 0) & (ii < 2 * h) & (jj >= 0) & (jj < 2 * w)
            v = np.zeros((len(n), cin), np.float64)
            if ok.any():
                v[ok] = x_at(n[ok], ii[ok] // 2, jj[ok] // 2)
            acc += v @ w_otc[:, r * 3 + s, :].T.astype(np.float64)
    if bias is not None:
        acc = acc + bias[None, :]
    return acc


def up2_conv3x3_dgrad_at(dy_at, h, w, cout, w_otc, n, i, j):
    """Low-resolution input gradient of conv3x3(up2(x)) at sampled pixels (n, i, j):
    dx[n,i,j,c] = sum_{a,b in {0,1}} sum_{r,s,o} dy[n, 2i+a-(r-1), 2j+b-(s-1), o] W[o, r*3+s, c]."""
    cin = w_otc.shape[2]
    acc = np.zeros((len(n), cin), np.float64)
    for a in range(2):
        for b in range(2):
            for r in range(3):
                for s in range(3):
                    acc += _gather(dy_at, n, 2 * i + a - (r - 1), 2 * j + b - (s - 1), 2 * h, 2 * w, cout) @ \
                        w_otc[:, r * 3 + s, :].astype(np.float64)
    return acc


def up2_conv3x3_wgrad_at(x_cols_lo, dy_cols, h, w):
    """dW of conv3x3(up2(x)) for sampled channels: x_cols_lo [N, h, w, Cs] (low resolution),
    dy_cols [N, 2h, 2w, Os] -> [Os, 9, Cs]."""
    up = np.repeat(np.repeat(x_cols_lo, 2, axis=1), 2, axis=2)
    return conv_wgrad_at(up, dy_cols, 2 * h, 2 * w, 3)
