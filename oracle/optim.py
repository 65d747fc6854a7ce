"""Asymmetric optimisation policy (PAPER.md:285-307 [Sec. 5.2]) — oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:293 "ParaGAN firstly implements some of the latest work on optimizers including Adabelief, rectified
Adam (RAdam), Lookahead, and LARS"; "users can set the optimization policy for the generator and
discriminator respectively, which currently includes optimizers, learning rate schedulers, warmup
epochs, and gradient norms".  The paper gives no formulas; each rule below is written out from the
paper it cites, in that paper's notation (readings R26-R30 in DESIGN.md):

  adam       Kingma & Ba, Alg. 1 (PyTorch form: eps outside the sqrt; R12)
  adabelief  Zhuang et al. 2020, Alg. 2: s_t = b2 s + (1-b2)(g - m_t)^2 + eps, step m_hat/(sqrt(s_hat)+eps)
  radam      Liu et al. 2020, Alg. 2, with the authors' / PyTorch's rectification threshold rho_t > 5 and
             eps in the adaptive term (R27)
  sgd        w - lr * m, m = b1 m + g (heavy-ball momentum; b1 = 0 is plain SGD)
  lars       You et al. 2017: per layer (tensor) the step is scaled by the trust ratio
             trust * ||w|| / ||u||, u the inner rule's step direction (R28)
  lookahead  Zhang et al. 2019, Alg. 1: every k inner steps phi <- phi + alpha (theta - phi), theta <- phi
  clip_norm  global-norm clipping of the net's gradient before the rule: g <- g * min(1, c / ||g||)
  lr(t)      lr * warmup(t) * schedule(t): warmup(t) = min(1, t / W) (linear from 0, W = warmup steps);
             schedule: constant | cosine 0.5 (1 + cos(pi min(t,T)/T)) | linear max(0, 1 - t/T)  (R29)

t is the 1-based count of applied updates of the network (a skipped, non-finite step does not count).
Everything is float64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

RULES = ("adam", "adabelief", "radam", "sgd")
SCHEDULES = ("constant", "cosine", "linear")


@dataclass
class Policy:
    rule: str = "adam"
    lr: float = 2e-4
    beta1: float = 0.0
    beta2: float = 0.999
    eps: float = 1e-8
    lars: bool = False
    lars_trust: float = 1.0
    lookahead_k: int = 0          # 0 = off
    lookahead_alpha: float = 0.5
    warmup_steps: int = 0
    schedule: str = "constant"
    total_steps: int = 0          # T of the cosine / linear schedules
    clip_norm: float = 0.0        # 0 = off


def lr_at(p: Policy, t: int) -> float:
    """Learning rate of the t-th update (t >= 1)."""
    warm = min(1.0, t / p.warmup_steps) if p.warmup_steps > 0 else 1.0
    if p.schedule == "cosine" and p.total_steps > 0:
        sched = 0.5 * (1.0 + math.cos(math.pi * min(t, p.total_steps) / p.total_steps))
    elif p.schedule == "linear" and p.total_steps > 0:
        sched = max(0.0, 1.0 - t / p.total_steps)
    else:
        sched = 1.0
    return p.lr * warm * sched


def clip_scale(grads: list, c: float) -> float:
    """min(1, c / ||g||) over the whole network's gradient (global norm)."""
    if c <= 0:
        return 1.0
    norm = math.sqrt(sum(float((g.double() ** 2).sum()) for g in grads))
    return min(1.0, c / norm) if norm > 0 else 1.0


class State:
    """Optimizer state of one tensor: m, v (AdaBelief: s), lookahead slow weights phi."""

    def __init__(self, w: torch.Tensor):
        self.m = torch.zeros_like(w, dtype=torch.float64)
        self.v = torch.zeros_like(w, dtype=torch.float64)
        self.phi = w.detach().clone().double()


def direction(p: Policy, st: State, g: torch.Tensor, t: int) -> torch.Tensor:
    """The inner rule's step u (the update is w - lr(t) * u); updates st.m / st.v."""
    b1, b2, eps = p.beta1, p.beta2, p.eps
    if p.rule == "sgd":
        st.m = b1 * st.m + g
        return st.m.clone()
    st.m = b1 * st.m + (1.0 - b1) * g
    mhat = st.m / (1.0 - b1 ** t)
    if p.rule == "adam":
        st.v = b2 * st.v + (1.0 - b2) * g * g
        return mhat / (torch.sqrt(st.v / (1.0 - b2 ** t)) + eps)
    if p.rule == "adabelief":
        st.v = b2 * st.v + (1.0 - b2) * (g - st.m) ** 2 + eps
        return mhat / (torch.sqrt(st.v / (1.0 - b2 ** t)) + eps)
    if p.rule == "radam":
        st.v = b2 * st.v + (1.0 - b2) * g * g
        rho_inf = 2.0 / (1.0 - b2) - 1.0
        rho_t = rho_inf - 2.0 * t * b2 ** t / (1.0 - b2 ** t)
        if rho_t > 5.0:
            r = math.sqrt((rho_t - 4.0) * (rho_t - 2.0) * rho_inf / ((rho_inf - 4.0) * (rho_inf - 2.0) * rho_t))
            return r * mhat * math.sqrt(1.0 - b2 ** t) / (torch.sqrt(st.v) + eps)
        return mhat
    raise ValueError(p.rule)


def step(p: Policy, params: dict, grads: dict, states: dict, t: int) -> None:
    """Apply the t-th update (t >= 1) of one network in place: clipping, rule, LARS, lookahead."""
    cs = clip_scale(list(grads.values()), p.clip_norm)
    lr = lr_at(p, t)
    for name, w in params.items():
        g = grads[name].double() * cs
        u = direction(p, states[name], g, t)
        if p.lars:
            wn, un = float(torch.linalg.vector_norm(w)), float(torch.linalg.vector_norm(u))
            u = u * (p.lars_trust * wn / un if wn > 0 and un > 0 else 1.0)
        params[name] = w - lr * u
    if p.lookahead_k > 0 and t % p.lookahead_k == 0:
        for name in params:
            st = states[name]
            st.phi = st.phi + p.lookahead_alpha * (params[name] - st.phi)
            params[name] = st.phi.clone()
