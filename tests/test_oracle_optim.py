"""Pins of the asymmetric-policy oracle (oracle/optim.py): each rule against
a library implementation where one exists (torch.optim Adam / RAdam / SGD in fp64), closed forms where
not (AdaBelief on a constant gradient, Lookahead's slow-weight recursion, LARS's trust-ratio norm,
global-norm clipping, the warmup/schedule ramps), and the invariants SPEC lists (lr -> 0 leaves the
weights unchanged; Lookahead with k=1, alpha=1 is the inner rule)."""
import math

import numpy as np
import pytest
import torch

from oracle import optim as O


def _run(p, w0, grads):
    params = {"w": w0.clone()}
    st = {"w": O.State(w0)}
    for t, g in enumerate(grads, 1):
        O.step(p, params, {"w": g}, st, t)
    return params["w"]


def _grads(n=40, size=7, seed=0):
    r = np.random.default_rng(seed)
    return [torch.tensor(r.standard_normal(size)) for _ in range(n)]


@pytest.mark.parametrize("rule,lib", [("adam", "Adam"), ("radam", "RAdam"), ("sgd", "SGD")])
def test_rules_match_torch_optim_fp64(rule, lib):
    w0 = torch.tensor(np.random.default_rng(1).standard_normal(7))
    grads = _grads()
    p = O.Policy(rule=rule, lr=1e-2, beta1=0.5, beta2=0.99, eps=1e-8)
    got = _run(p, w0, grads)
    w = w0.clone().requires_grad_(True)
    if lib == "SGD":
        opt = torch.optim.SGD([w], lr=p.lr, momentum=p.beta1)
    else:
        opt = getattr(torch.optim, lib)([w], lr=p.lr, betas=(p.beta1, p.beta2), eps=p.eps)
    for g in grads:
        w.grad = g.clone()
        opt.step()
    assert torch.allclose(got, w.detach(), rtol=1e-12, atol=1e-14)


def test_radam_unrectified_then_rectified():
    """rho_1 = 1 for any beta2 (closed form): the first steps are the un-adapted momentum step lr * m_hat;
    rectification switches on once rho_t > 5 and its factor tends to 1."""
    b2 = 0.999
    rho_inf = 2 / (1 - b2) - 1
    assert abs(rho_inf - 2 * 1 * b2 / (1 - b2) - 1.0) < 1e-9
    p = O.Policy(rule="radam", lr=0.1, beta1=0.0, beta2=b2)
    w0 = torch.zeros(3, dtype=torch.float64)
    g = torch.tensor([1.0, -2.0, 0.5], dtype=torch.float64)
    assert torch.allclose(_run(p, w0, [g]), -0.1 * g)


def test_adabelief_constant_gradient_closed_form():
    """AdaBelief on a constant gradient g: m_t = g (1 - b1^t), g - m_t = g b1^t, so
    s_t = (1-b2) g^2 sum_{i=1..t} b2^(t-i) b1^(2i) + eps (1 - b2^t)/(1 - b2); the t-th step is
    lr * (m_t / (1-b1^t)) / (sqrt(s_t / (1-b2^t)) + eps) = lr * g / (sqrt(s_t/(1-b2^t)) + eps)."""
    b1, b2, eps, lr = 0.6, 0.95, 1e-6, 1e-2
    g = torch.tensor([0.3, -1.7], dtype=torch.float64)
    p = O.Policy(rule="adabelief", lr=lr, beta1=b1, beta2=b2, eps=eps)
    params, st = {"w": torch.zeros(2, dtype=torch.float64)}, {"w": O.State(torch.zeros(2, dtype=torch.float64))}
    for t in range(1, 31):
        before = params["w"].clone()
        O.step(p, params, {"w": g}, st, t)
        s_t = (1 - b2) * g * g * sum(b2 ** (t - i) * b1 ** (2 * i) for i in range(1, t + 1)) + eps * (1 - b2 ** t) / (1 - b2)
        want = -lr * g / (torch.sqrt(s_t / (1 - b2 ** t)) + eps)
        assert torch.allclose(params["w"] - before, want, rtol=1e-10, atol=0)


def test_lookahead_reductions_and_closed_form():
    w0 = torch.tensor([1.0, -2.0, 3.0], dtype=torch.float64)
    grads = _grads(12, 3, 2)
    inner = _run(O.Policy(rule="adam", lr=1e-2), w0, grads)
    same = _run(O.Policy(rule="adam", lr=1e-2, lookahead_k=1, lookahead_alpha=1.0), w0, grads)
    assert torch.equal(inner, same)
    # plain SGD on a constant gradient: every k steps the slow weights move by alpha * k * lr * g
    g = torch.tensor([0.5, -1.0, 2.0], dtype=torch.float64)
    k, alpha, lr = 3, 0.5, 0.1
    w = _run(O.Policy(rule="sgd", lr=lr, beta1=0.0, lookahead_k=k, lookahead_alpha=alpha), w0, [g] * (4 * k))
    assert torch.allclose(w, w0 - 4 * alpha * k * lr * g, rtol=1e-13)


def test_lars_update_norm_is_trust_times_weight_norm():
    """Per tensor the LARS-scaled step has norm lr * trust * ||w|| and the inner rule's direction."""
    r = np.random.default_rng(3)
    params = {"a": torch.tensor(r.standard_normal(5)), "b": torch.tensor(r.standard_normal(9)) * 10}
    grads = {k: torch.tensor(r.standard_normal(v.numel())) for k, v in params.items()}
    st = {k: O.State(v) for k, v in params.items()}
    p = O.Policy(rule="sgd", lr=0.1, beta1=0.0, lars=True, lars_trust=0.02)
    before = {k: v.clone() for k, v in params.items()}
    O.step(p, params, grads, st, 1)
    for k in params:
        d = params[k] - before[k]
        assert abs(float(d.norm()) - 0.1 * 0.02 * float(before[k].norm())) < 1e-12
        assert torch.allclose(d / d.norm(), -grads[k] / grads[k].norm(), atol=1e-12)


def test_global_norm_clipping():
    g = {"a": torch.tensor([3.0, 4.0], dtype=torch.float64), "b": torch.tensor([0.0, 0.0, 12.0], dtype=torch.float64)}
    assert abs(O.clip_scale(list(g.values()), 1.0) - 1.0 / 13.0) < 1e-15     # ||g|| = 13
    assert O.clip_scale(list(g.values()), 100.0) == 1.0
    # SGD step with clip 1: the applied gradient has norm 1 and the same direction
    params = {k: torch.zeros_like(v) for k, v in g.items()}
    st = {k: O.State(v) for k, v in params.items()}
    O.step(O.Policy(rule="sgd", lr=1.0, beta1=0.0, clip_norm=1.0), params, g, st, 1)
    applied = torch.cat([-params["a"], -params["b"]])
    assert abs(float(applied.norm()) - 1.0) < 1e-15
    assert torch.allclose(applied, torch.cat([g["a"], g["b"]]) / 13.0)


def test_warmup_and_schedules():
    p = O.Policy(lr=1.0, warmup_steps=4)
    assert [O.lr_at(p, t) for t in (1, 2, 4, 9)] == [0.25, 0.5, 1.0, 1.0]
    c = O.Policy(lr=2.0, schedule="cosine", total_steps=10)
    assert abs(O.lr_at(c, 5) - 1.0) < 1e-15 and O.lr_at(c, 10) < 1e-15 and O.lr_at(c, 20) < 1e-15
    lin = O.Policy(lr=2.0, schedule="linear", total_steps=10, warmup_steps=2)
    assert abs(O.lr_at(lin, 1) - 0.5 * 2.0 * 0.9) < 1e-15 and O.lr_at(lin, 10) == 0.0


@pytest.mark.parametrize("rule", O.RULES)
def test_zero_lr_leaves_weights_unchanged(rule):
    w0 = torch.tensor(np.random.default_rng(4).standard_normal(6))
    for lars, la in ((False, 0), (True, 2)):
        p = O.Policy(rule=rule, lr=0.0, lars=lars, lookahead_k=la)
        assert torch.equal(_run(p, w0, _grads(6, 6, 5)), w0)
