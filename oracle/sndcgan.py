"""SN-DCGAN 32x32 (config 1) for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading R25 (the paper names SN-DCGAN as a workload — P:174 "SN-DCGAN ... BigGAN" — but gives no
layers): SNGAN's "standard CNN" with widths scaled by ch/64 (ch = 32 for config 1).

  G (no SN; BN cross-replica with learned gamma/beta, R5):
    z [B,128] -> Linear(128 -> 4*4*8ch, bias) -> BN per feature -> ReLU -> NHWC view [B,4,4,8ch] (R10)
    -> Deconv4x4 s2 p1 (8ch->4ch) -> BN -> ReLU -> Deconv (4ch->2ch) -> BN -> ReLU
    -> Deconv (2ch->ch) -> BN -> ReLU -> Conv3x3 s1 p1 (ch->3) -> tanh
  D (SN on every layer, biases, LeakyReLU 0.1 after every conv):
    Conv3x3 3->ch, Conv4x4 s2 p1 ch->ch, Conv3x3 ch->2ch, Conv4x4 s2 2ch->2ch, Conv3x3 2ch->4ch,
    Conv4x4 s2 4ch->4ch, Conv3x3 4ch->8ch, flatten NHWC [B, 4*4*8ch] -> SNLinear(-> 1)
  Unconditional (labels are ignored); hinge loss; fp32 throughout (no bf16 mode).

Deconv weights are PyTorch ConvTranspose2d's [C_in, C_out, 4, 4]; the deconv is the adjoint of the
strided conv with that weight read as [C_out_conv = C_in, C_in_conv = C_out] (pinned in
tests/test_oracle_model.py).
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from . import ops

LRELU = 0.1


def _widths(ch: int):
    return dict(g=[8 * ch, 4 * ch, 2 * ch, ch], d=[ch, ch, 2 * ch, 2 * ch, 4 * ch, 4 * ch, 8 * ch])


# D convs: (kernel, stride, C_in index)  — C_in of layer i is the previous layer's C_out (3 for the first)
_D_LAYERS = [(3, 1), (4, 2), (3, 1), (4, 2), (3, 1), (4, 2), (3, 1)]


def g_param_specs(cfg):
    from .biggan import PSpec
    w = _widths(cfg.ch)["g"]
    f0 = 16 * w[0]
    s = [PSpec("linear.w", (f0, cfg.dim_z), "normal"), PSpec("linear.b", (f0,), "zero"),
         PSpec("bn0.gamma", (f0,), "one"), PSpec("bn0.beta", (f0,), "zero")]
    for i in range(3):
        s += [PSpec(f"deconv{i + 1}.w", (w[i], w[i + 1], 4, 4), "normal"), PSpec(f"deconv{i + 1}.b", (w[i + 1],), "zero"),
              PSpec(f"bn{i + 1}.gamma", (w[i + 1],), "one"), PSpec(f"bn{i + 1}.beta", (w[i + 1],), "zero")]
    s += [PSpec("out_conv.w", (3, w[3], 3, 3), "normal"), PSpec("out_conv.b", (3,), "zero")]
    return s


def d_param_specs(cfg):
    from .biggan import PSpec
    w = _widths(cfg.ch)["d"]
    s, cin = [], 3
    for i, (k, _) in enumerate(_D_LAYERS):
        s += [PSpec(f"conv{i + 1}.w", (w[i], cin, k, k), "normal", True), PSpec(f"conv{i + 1}.b", (w[i],), "zero")]
        cin = w[i]
    s += [PSpec("linear.w", (1, 16 * w[-1]), "normal", True), PSpec("linear.b", (1,), "zero")]
    return s


def g_forward(cfg, sn, z: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Generator; ``y`` is ignored (unconditional).  Returns NCHW images in [-1, 1]."""
    p = sn.params
    w = _widths(cfg.ch)["g"]
    B = z.shape[0]
    h = z @ p["linear.w"].t() + p["linear.b"]                                   # [B, 16*8ch]
    # BN per feature over the global batch (the [B,1,1,F] view of the per-channel BN)
    h = ops.bn_affine(h[:, :, None, None], p["bn0.gamma"], p["bn0.beta"], cfg.bn_eps)[:, :, 0, 0]
    h = torch.relu(h).reshape(B, 4, 4, w[0]).permute(0, 3, 1, 2)               # R10: NHWC view
    for i in range(3):
        h = F.conv_transpose2d(h, p[f"deconv{i + 1}.w"], p[f"deconv{i + 1}.b"], stride=2, padding=1)
        h = torch.relu(ops.bn_affine(h, p[f"bn{i + 1}.gamma"], p[f"bn{i + 1}.beta"], cfg.bn_eps))
    return torch.tanh(ops.conv2d(h, p["out_conv.w"], p["out_conv.b"]))


def d_forward(cfg, sn, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Discriminator logits [N]; ``y`` is ignored (unconditional)."""
    h = x
    for i, (k, s) in enumerate(_D_LAYERS):
        h = F.conv2d(h, sn.w(f"conv{i + 1}.w"), sn.params[f"conv{i + 1}.b"], stride=s, padding=1)
        h = F.leaky_relu(h, LRELU)
    feat = h.permute(0, 2, 3, 1).reshape(h.shape[0], -1)                        # flatten NHWC
    return (feat @ sn.w("linear.w").t() + sn.params["linear.b"])[:, 0]
