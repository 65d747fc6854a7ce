"""BigGAN generator/discriminator and the ParaGAN training iteration (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What is computed, in the paper's order:
  * data parallelism with gradient synchronisation: the oracle
    runs the GLOBAL batch in one process, which is what W replicas with
    cross-replica BN and a gradient all-reduce(mean) compute (R15);
  * D step then G step, n_d D steps per G step ("update one after
    another"; asymmetric policy P:285-307; R13);
  * BigGAN backbone (topology reading R1, pinned by the parameter count
    158.42M of Table 1);
  * bf16 storage with fp32 last layers of G and D (R14) when
    ``cfg.bf16`` is set — one layer-by-layer rule (oracle/ops.py), written as
    explicit ``q()`` / ``qv()`` / ``qg()`` calls;
  * the D input is the concatenation [fake; real] ("concatenate the two
    input matrices before the matrix multiplication");
  * hinge loss (R3), spectral norm with one power step per forward (R4),
    cross-replica BN over the global batch (R5), Adam per network (R12).

Gradients are autograd's exact gradients of the written-out forward (u', v of
the power step are constants, R4).
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .ops import F64, q, qg, qv

# ---------------------------------------------------------------------------
# Architecture (reading R1; BigGAN-PyTorch G_arch / D_arch channel multipliers)
# ---------------------------------------------------------------------------
_G_ARCH = {  # resolution -> (in multipliers, out multipliers); bottom width 4
    16: ([4, 4], [4, 4]),
    32: ([4, 4, 4], [4, 4, 4]),
    64: ([16, 16, 8, 4], [16, 8, 4, 2]),
    128: ([16, 16, 8, 4, 2], [16, 8, 4, 2, 1]),
    256: ([16, 16, 8, 8, 4, 2], [16, 8, 8, 4, 2, 1]),
    512: ([16, 16, 8, 8, 4, 2, 1], [16, 8, 8, 4, 2, 1, 1]),
}
_D_ARCH = {  # resolution -> (in multipliers (first = RGB), out multipliers, downsample)
    16: ([None, 4, 4], [4, 4, 4], [1, 1, 0]),
    32: ([None, 4, 4, 4], [4, 4, 4, 4], [1, 1, 0, 0]),
    64: ([None, 1, 2, 4, 8], [1, 2, 4, 8, 16], [1, 1, 1, 1, 0]),
    128: ([None, 1, 2, 4, 8, 16], [1, 2, 4, 8, 16, 16], [1, 1, 1, 1, 1, 0]),
    256: ([None, 1, 2, 4, 8, 8, 16], [1, 2, 4, 8, 8, 16, 16], [1, 1, 1, 1, 1, 1, 0]),
    512: ([None, 1, 1, 2, 4, 8, 8, 16], [1, 1, 2, 4, 8, 8, 16, 16], [1, 1, 1, 1, 1, 1, 1, 0]),
}


@dataclass
class AdamHP:
    lr: float
    beta1: float
    beta2: float
    eps: float


@dataclass
class Config:
    resolution: int = 128
    ch: int = 96
    n_classes: int = 1000
    shared_dim: int = 128
    z_chunk: int = 20
    attn_res: int = 64          # 0 = no attention block
    bn_eps: float = 1e-5
    sn_eps: float = 1e-12
    d_steps_per_g: int = 1
    bf16: bool = False           # emulate the bf16 storage rule of R14 (oracle/ops.py q/qv/qg)
    arch: str = "biggan"          # "biggan" (R1) or "sndcgan" (config 1, R25; oracle/sndcgan.py)
    adam_d: AdamHP = field(default_factory=lambda: AdamHP(2e-4, 0.0, 0.999, 1e-8))
    adam_g: AdamHP = field(default_factory=lambda: AdamHP(5e-5, 0.0, 0.999, 1e-8))
    # asymmetric optimisation policy per network (NEXT-3; oracle/optim.py); None = Adam (R12)
    policy_d: object = None
    policy_g: object = None

    @property
    def n_blocks_g(self) -> int:
        return len(_G_ARCH[self.resolution][0])

    @property
    def dim_z(self) -> int:
        if self.arch == "sndcgan":
            return 128
        return (self.n_blocks_g + 1) * self.z_chunk

    @property
    def cond_dim(self) -> int:
        return self.shared_dim + self.z_chunk


def g_blocks(cfg: Config):
    """[(C_in, C_out, H_in, attention_after)] of the generator's up-blocks."""
    cin, cout = _G_ARCH[cfg.resolution]
    out, h = [], 4
    for a, b in zip(cin, cout):
        out.append((a * cfg.ch, b * cfg.ch, h, cfg.attn_res == 2 * h))
        h *= 2
    return out


def d_blocks(cfg: Config):
    """[(C_in, C_out, H_in, downsample, attention_after)] of the discriminator."""
    cin, cout, down = _D_ARCH[cfg.resolution]
    out, h, placed = [], cfg.resolution, False
    for a, b, dn in zip(cin, cout, down):
        c_in = 3 if a is None else a * cfg.ch
        h_out = h // 2 if dn else h
        att = (not placed) and cfg.attn_res == h_out     # once, after the first block ending at attn_res
        placed = placed or att
        out.append((c_in, b * cfg.ch, h, bool(dn), att))
        h = h_out
    return out


# ---------------------------------------------------------------------------
# Canonical parameter layout (SURVEY §8(b) "Ownership"): forward-layer order,
# weight then bias; conv weights OIHW; linears [out, in]; embeddings
# [classes, dim]; then the SN u-vectors in the same layer order.
# ---------------------------------------------------------------------------
@dataclass
class PSpec:
    name: str
    shape: tuple
    init: str          # 'normal' | 'zero' | 'one' | 'attn_gamma'
    sn: bool = False


def g_param_specs(cfg: Config) -> list[PSpec]:
    if cfg.arch == "sndcgan":
        from . import sndcgan
        return sndcgan.g_param_specs(cfg)
    c0 = g_blocks(cfg)[0][0]
    s = [PSpec("shared", (cfg.n_classes, cfg.shared_dim), "normal"),
         PSpec("linear.w", (16 * c0, cfg.z_chunk), "normal", True),
         PSpec("linear.b", (16 * c0,), "zero")]
    for i, (ci, co, _, att) in enumerate(g_blocks(cfg)):
        p = f"b{i}."
        s += [PSpec(p + "cbn1.gain", (ci, cfg.cond_dim), "normal", True),
              PSpec(p + "cbn1.bias", (ci, cfg.cond_dim), "normal", True),
              PSpec(p + "conv1.w", (co, ci, 3, 3), "normal", True),
              PSpec(p + "conv1.b", (co,), "zero"),
              PSpec(p + "cbn2.gain", (co, cfg.cond_dim), "normal", True),
              PSpec(p + "cbn2.bias", (co, cfg.cond_dim), "normal", True),
              PSpec(p + "conv2.w", (co, co, 3, 3), "normal", True),
              PSpec(p + "conv2.b", (co,), "zero"),
              PSpec(p + "sc.w", (co, ci, 1, 1), "normal", True),
              PSpec(p + "sc.b", (co,), "zero")]
        if att:
            s += _attn_specs("attn.", co)
    c_last = g_blocks(cfg)[-1][1]
    s += [PSpec("out_bn.gamma", (c_last,), "one"), PSpec("out_bn.beta", (c_last,), "zero"),
          PSpec("out_conv.w", (3, c_last, 3, 3), "normal", True), PSpec("out_conv.b", (3,), "zero")]
    return s


def d_param_specs(cfg: Config) -> list[PSpec]:
    if cfg.arch == "sndcgan":
        from . import sndcgan
        return sndcgan.d_param_specs(cfg)
    s = []
    for j, (ci, co, _, dn, att) in enumerate(d_blocks(cfg)):
        p = f"b{j}."
        s += [PSpec(p + "conv1.w", (co, ci, 3, 3), "normal", True), PSpec(p + "conv1.b", (co,), "zero"),
              PSpec(p + "conv2.w", (co, co, 3, 3), "normal", True), PSpec(p + "conv2.b", (co,), "zero")]
        if ci != co or dn:
            s += [PSpec(p + "sc.w", (co, ci, 1, 1), "normal", True), PSpec(p + "sc.b", (co,), "zero")]
        if att:
            s += _attn_specs("attn.", co)
    c = d_blocks(cfg)[-1][1]
    s += [PSpec("linear.w", (1, c), "normal", True), PSpec("linear.b", (1,), "zero"),
          PSpec("embed", (cfg.n_classes, c), "normal", True)]
    return s


def _attn_specs(p: str, c: int) -> list[PSpec]:
    return [PSpec(p + "theta", (c // 8, c, 1, 1), "normal", True),
            PSpec(p + "phi", (c // 8, c, 1, 1), "normal", True),
            PSpec(p + "g", (c // 2, c, 1, 1), "normal", True),
            PSpec(p + "o", (c, c // 2, 1, 1), "normal", True),
            PSpec(p + "gamma", (1,), "attn_gamma")]


def n_trainable(specs: list[PSpec]) -> int:
    return int(sum(np.prod(s.shape) for s in specs))


def n_state(specs: list[PSpec]) -> int:
    """Length of the canonical flat array: trainables then u-vectors."""
    return n_trainable(specs) + int(sum(s.shape[0] for s in specs if s.sn))


def unflatten(specs: list[PSpec], flat: np.ndarray):
    """Canonical flat fp32 array -> ({name: tensor}, {name: u})."""
    flat = torch.as_tensor(np.asarray(flat, dtype=np.float64))
    params, us, o = {}, {}, 0
    for s in specs:
        n = int(np.prod(s.shape))
        params[s.name] = flat[o:o + n].reshape(s.shape).clone()
        o += n
    for s in specs:
        if s.sn:
            us[s.name] = flat[o:o + s.shape[0]].clone()
            o += s.shape[0]
    assert o == flat.numel()
    return params, us


def flatten(specs: list[PSpec], params: dict, us: dict | None) -> np.ndarray:
    parts = [params[s.name].detach().reshape(-1) for s in specs]
    if us is not None:
        parts += [us[s.name].reshape(-1) for s in specs if s.sn]
    return torch.cat(parts).numpy()


# ---------------------------------------------------------------------------
# Forward passes
# ---------------------------------------------------------------------------
class _SN:
    """Applies one power step to every SN weight of a net (R4) and records sigma."""

    def __init__(self, specs, params, us, eps, bf16, frozen: dict | None = None):
        self.specs = {s.name: s for s in specs}
        self.params, self.us, self.eps, self.bf16 = params, us, eps, bf16
        self.sigma = {}
        self.vectors = {}            # name -> (u', v) of this forward's power step
        self.frozen = frozen         # finite-difference pins: reuse given (u', v)

    def w(self, name: str, mma: bool = False) -> torch.Tensor:
        """W / sigma(W); ``mma`` marks a tensor-core operand stored bf16 (R14)."""
        wt = self.params[name]
        if not self.specs[name].sn:
            return wt
        if self.frozen is not None:
            u_new, v = self.frozen[name]
            sigma = u_new @ (wt.reshape(wt.shape[0], -1) @ v)
        else:
            sigma, u_new, v = ops.sn_power_step(wt, self.us[name], self.eps)
        self.us[name] = u_new
        self.vectors[name] = (u_new, v)
        self.sigma[name] = sigma.detach().clone()
        w_hat = wt / sigma
        # straight-through: the value is the bf16 operand, the gradient is d/dW_hat (fp32)
        return ops.bf16_round(w_hat.detach()) + (w_hat - w_hat.detach()) if (mma and self.bf16) else w_hat


def _qw(sn: _SN, name: str) -> torch.Tensor:
    return sn.w(name, mma=True)


def g_forward(cfg: Config, sn: _SN, z: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Generator (Appendix A of SURVEY; R1, R10, R11).  Returns images NCHW in [-1, 1].

    bf16 mode: the layer-by-layer storage rule of R14 (oracle/ops.py): q() on every layer output,
    qg() on every layer input, bf16(W/sigma) for every tensor-core weight."""
    if cfg.arch == "sndcgan":
        from . import sndcgan
        return sndcgan.g_forward(cfg, sn, z, y)
    bf = cfg.bf16
    p = sn.params
    B = z.shape[0]
    e = p["shared"][y]                                   # shared class embedding (no SN)
    zs = torch.split(z, cfg.z_chunk, dim=1)              # R11: contiguous chunks
    blocks = g_blocks(cfg)
    c0 = blocks[0][0]
    h = zs[0] @ sn.w("linear.w").t() + p["linear.b"]     # fp32 linear
    h = q(h.reshape(B, 4, 4, c0).permute(0, 3, 1, 2), bf)  # R10: NHWC [4,4,C0] view
    for i, (ci, co, _, att) in enumerate(blocks):
        pre = f"b{i}."
        cond = torch.cat([e, zs[i + 1]], dim=1)
        g1 = cond @ sn.w(pre + "cbn1.gain").t()
        b1 = cond @ sn.w(pre + "cbn1.bias").t()
        x = h
        a = q(torch.relu(ops.cbn(qg(x, bf), g1, b1, cfg.bn_eps)), bf)       # CBN+ReLU layer
        a = q(ops.up2(a), bf)                                                # nearest x2 (resampling layer)
        a = q(ops.conv2d(a, _qw(sn, pre + "conv1.w"), p[pre + "conv1.b"]), bf)
        g2 = cond @ sn.w(pre + "cbn2.gain").t()
        b2 = cond @ sn.w(pre + "cbn2.bias").t()
        a = q(torch.relu(ops.cbn(a, g2, b2, cfg.bn_eps)), bf)
        # skip 1x1 conv before the upsample (it commutes with nearest x2), added in conv2's fp32 epilogue
        s = q(ops.conv2d(qg(x, bf), _qw(sn, pre + "sc.w"), p[pre + "sc.b"]), bf)
        h = q(ops.conv2d(a, _qw(sn, pre + "conv2.w"), p[pre + "conv2.b"]) + ops.up2(s), bf)
        if att:
            h = _attention(cfg, sn, "attn.", h)
    # last layer in fp32: BN -> ReLU -> conv 3x3 -> tanh
    h = torch.relu(ops.bn_affine(h, p["out_bn.gamma"], p["out_bn.beta"], cfg.bn_eps))
    return torch.tanh(ops.conv2d(h, sn.w("out_conv.w"), p["out_conv.b"]))


def _attention(cfg: Config, sn: _SN, pre: str, x: torch.Tensor) -> torch.Tensor:
    """Non-local block under the R14 rule: the theta/phi/g 1x1 convs and the o conv (with the
    gamma-scaled residual add fused) are layers; the attention core's tensor-core operands beta
    (forward) and the score gradient dS (backward) are bf16, the scores, softmax and dP fp32."""
    bf = cfg.bf16
    n, c, h, w = x.shape
    theta = q(ops.conv2d(qg(x, bf), _qw(sn, pre + "theta"), None), bf).reshape(n, -1, h * w)
    phi = q(ops.maxpool2(q(ops.conv2d(qg(x, bf), _qw(sn, pre + "phi"), None), bf)), bf).reshape(n, -1, h * w // 4)
    g = q(ops.maxpool2(q(ops.conv2d(qg(x, bf), _qw(sn, pre + "g"), None), bf)), bf).reshape(n, -1, h * w // 4)
    scores = qg(torch.bmm(theta.transpose(1, 2), phi), bf)
    beta = qv(torch.softmax(scores, dim=-1), bf)
    o = q(torch.bmm(g, beta.transpose(1, 2)).reshape(n, -1, h, w), bf)
    return q(x + sn.params[pre + "gamma"] * ops.conv2d(o, _qw(sn, pre + "o"), None), bf)


def d_forward(cfg: Config, sn: _SN, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Projection discriminator (Appendix A; R1, R7).  x NCHW; returns logits [N] (fp32 head).

    bf16 mode: the R14 rule as in g_forward (ReLU is exact on bf16 values and gradients)."""
    if cfg.arch == "sndcgan":
        from . import sndcgan
        return sndcgan.d_forward(cfg, sn, x, y)
    bf = cfg.bf16
    p = sn.params
    h = x
    blocks = d_blocks(cfg)
    for j, (ci, co, _, dn, att) in enumerate(blocks):
        pre = f"b{j}."
        a = h if j == 0 else torch.relu(h)
        a = q(ops.conv2d(qg(a, bf), _qw(sn, pre + "conv1.w"), p[pre + "conv1.b"]), bf)
        c2 = ops.conv2d(qg(torch.relu(a), bf), _qw(sn, pre + "conv2.w"), p[pre + "conv2.b"])
        learn = ci != co or dn
        if dn and j == 0:
            # block 0 (no pre-activation): pool the image, then the 1x1 skip conv (R7); the main branch's
            # conv2 output is a layer output, pooled and added to the skip in one layer
            s = q(ops.conv2d(qg(q(ops.avgpool2(h), bf), bf), _qw(sn, pre + "sc.w"), p[pre + "sc.b"]), bf)
            h = q(ops.avgpool2(q(c2, bf)) + s, bf)
        else:
            # later blocks: 1x1 skip conv, conv2 with the residual add fused, then pool (= pool of each
            # branch, R7)
            s = q(ops.conv2d(qg(h, bf), _qw(sn, pre + "sc.w"), p[pre + "sc.b"]), bf) if learn else h
            t = q(c2 + s, bf)
            h = q(ops.avgpool2(t), bf) if dn else t
        if att:
            h = _attention(cfg, sn, "attn.", h)
    feat = torch.relu(h).sum(dim=(2, 3))                       # fp32 head from here
    out = feat @ sn.w("linear.w").t() + p["linear.b"]
    return out[:, 0] + (sn.w("embed")[y] * feat).sum(dim=1)


# ---------------------------------------------------------------------------
# Training state and the iteration (north_star; R12, R13, R15, R16)
# ---------------------------------------------------------------------------
@dataclass
class NetState:
    specs: list
    params: dict
    us: dict
    m: dict
    v: dict
    t: int = 0

    @classmethod
    def from_flat(cls, specs, flat):
        params, us = unflatten(specs, flat)
        z = {k: torch.zeros_like(v) for k, v in params.items()}
        return cls(specs, params, us, z, {k: torch.zeros_like(v) for k, v in params.items()}, 0)

    def flat(self) -> np.ndarray:
        return flatten(self.specs, self.params, self.us)

    def grad_flat(self, grads: dict) -> np.ndarray:
        return torch.cat([grads[s.name].reshape(-1) for s in self.specs]).numpy()


def _adam(st: NetState, grads: dict, hp: AdamHP, policy=None) -> bool:
    """One Adam update (R12), or the net's optimisation policy (oracle/optim.py) when given; skipped
    entirely when any gradient is non-finite (R16)."""
    if not all(torch.isfinite(g).all() for g in grads.values()):
        return False
    st.t += 1
    if policy is not None:
        from . import optim
        p = dataclasses.replace(policy, lr=hp.lr, beta1=hp.beta1, beta2=hp.beta2, eps=hp.eps)
        if not hasattr(st, "opt_states"):
            st.opt_states = {k: optim.State(v) for k, v in st.params.items()}
        optim.step(p, st.params, grads, st.opt_states, st.t)
        return True
    for name, g in grads.items():
        st.params[name], st.m[name], st.v[name] = ops.adam_update(
            st.params[name], g, st.m[name], st.v[name], st.t, hp.lr, hp.beta1, hp.beta2, hp.eps)
    return True


def pack_real(cfg: Config, real_nchw: np.ndarray) -> torch.Tensor:
    """The real batch as D sees it after the layout pack (bf16 storage in bf16 mode)."""
    x = torch.as_tensor(np.asarray(real_nchw, dtype=np.float32)).to(F64)
    return ops.bf16_round(x) if cfg.bf16 else x


def d_step(cfg: Config, G: NetState, D: NetState, real, real_y, z, fake_y, update: bool = True,
           fake_override=None, fakes=None) -> dict:
    """One D step: SN(G), G forward (no grad), SN(D), D([fake; real]),
    hinge L_D, backward through D, Adam on D.  ``fake_override`` (test hook) replaces the
    generated images so D's own arithmetic can be compared in isolation.  ``fakes`` (the
    asynchronous scheme: D reads its generated batch from img_buff) skips SN(G) and
    the G forward entirely (G may be None)."""
    real = pack_real(cfg, real)
    real_y = torch.as_tensor(np.asarray(real_y), dtype=torch.long)
    fake_y = torch.as_tensor(np.asarray(fake_y), dtype=torch.long)
    if fakes is not None:
        fake = torch.as_tensor(np.asarray(fakes, dtype=np.float64))
        sng = None
    else:
        z = torch.as_tensor(np.asarray(z, dtype=np.float32)).to(F64)
        sng = _SN(G.specs, G.params, G.us, cfg.sn_eps, cfg.bf16)
        with torch.no_grad():
            fake = g_forward(cfg, sng, z, fake_y)
    if fake_override is not None:
        fake = torch.as_tensor(np.asarray(fake_override, dtype=np.float64))
    fake = q(fake, cfg.bf16)
    dparams = {k: v.detach().requires_grad_(True) for k, v in D.params.items()}
    snd = _SN(D.specs, dparams, D.us, cfg.sn_eps, cfg.bf16)
    logits = d_forward(cfg, snd, torch.cat([fake, real], 0), torch.cat([fake_y, real_y], 0))
    B = fake.shape[0]
    l_fake, l_real = logits[:B], logits[B:]
    loss = ops.hinge_d(l_real, l_fake)
    names = [s.name for s in D.specs]
    gl = torch.autograd.grad(loss, [dparams[n] for n in names], allow_unused=True)
    grads = {n: (g if g is not None else torch.zeros_like(dparams[n])).detach() for n, g in zip(names, gl)}
    D.params = {k: v.detach() for k, v in dparams.items()}
    ok = _adam(D, grads, cfg.adam_d, cfg.policy_d) if update else True
    return dict(loss=float(loss.detach()), logits=logits.detach().numpy(), fake=fake.detach().numpy(),
                grads=D.grad_flat(grads), applied=ok,
                sigma_g=dict(sng.sigma) if sng is not None else {}, sigma_d=dict(snd.sigma),
                d_real_mean=float(l_real.detach().mean()), d_fake_mean=float(l_fake.detach().mean()))


def g_step(cfg: Config, G: NetState, D: NetState, z, y, update: bool = True) -> dict:
    """One G step: SN(G), G forward, SN(D), D(fake), L_G, backward through D
    (inputs only) and G, Adam on G.  D parameters are not updated."""
    y = torch.as_tensor(np.asarray(y), dtype=torch.long)
    z = torch.as_tensor(np.asarray(z, dtype=np.float32)).to(F64)
    gparams = {k: v.detach().requires_grad_(True) for k, v in G.params.items()}
    sng = _SN(G.specs, gparams, G.us, cfg.sn_eps, cfg.bf16)
    fake = q(g_forward(cfg, sng, z, y), cfg.bf16)
    snd = _SN(D.specs, D.params, D.us, cfg.sn_eps, cfg.bf16)
    logits = d_forward(cfg, snd, fake, y)
    loss = ops.hinge_g(logits)
    names = [s.name for s in G.specs]
    gl = torch.autograd.grad(loss, [gparams[n] for n in names], allow_unused=True)
    grads = {n: (g if g is not None else torch.zeros_like(gparams[n])).detach() for n, g in zip(names, gl)}
    G.params = {k: v.detach() for k, v in gparams.items()}
    ok = _adam(G, grads, cfg.adam_g, cfg.policy_g) if update else True
    return dict(loss=float(loss.detach()), logits=logits.detach().numpy(), fake=fake.detach().numpy(),
                grads=G.grad_flat(grads), applied=ok, sigma_g=dict(sng.sigma), sigma_d=dict(snd.sigma))


def iteration(cfg: Config, G: NetState, D: NetState, d_batches, g_batch) -> dict:
    """n_d D steps (each with a fresh real batch and z), then one G step (R13)."""
    outs = [d_step(cfg, G, D, *b) for b in d_batches]
    assert len(outs) == cfg.d_steps_per_g
    og = g_step(cfg, G, D, *g_batch)
    return dict(d=outs, g=og)
