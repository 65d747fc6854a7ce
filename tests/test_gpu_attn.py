"""Fused tcgen05 attention core (reading R8) through the C-ABI
(`paragan_op_attn_fwd` / `paragan_op_attn_bwd`), element by element against the plain
definition in float64 with the bf16 storage points of R14 / R21 (the unnormalised
exp(S - m) and dS stored bf16; the kernel's offset m is the exact row max or, in the single-pass
forward, chunk 0's max — a rounding-level difference):

    S = theta phi^T,  m = rowmax(S),  l = rowsum(exp(S - m)),  beta = exp(S - m) / l
    o = bf16(exp(S - m)) g / l
    dP = dO g^T,  dS = beta * (dP - rowsum(dP * beta))
    dtheta = bf16(dS) phi,  dphi = bf16(dS)^T theta,  dg = bf16(beta)^T dO
"""
import pytest
import torch

from paper_2411_03999_b200 import api

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _bf(x):
    return x.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def _rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def _inputs(n, hw, cq, c2, ct, scale, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    q = hw // 4
    qkv = (torch.randn(n, hw, ct, generator=g) * scale).to(torch.bfloat16)
    phi = (torch.randn(n, q, cq, generator=g) * scale).to(torch.bfloat16)
    gp = torch.randn(n, q, c2, generator=g).to(torch.bfloat16)
    dO = torch.randn(n, hw, c2, generator=g).to(torch.bfloat16)
    return qkv, phi, gp, dO


def _reference(qkv, phi, gp, dO, cq):
    th = qkv[..., :cq].double()
    ph, g, do = phi.double(), gp.double(), dO.double()
    S = th @ ph.transpose(1, 2)
    P = torch.softmax(S, dim=-1)
    Pb = _bf(P)
    E = torch.exp(S - S.amax(-1, keepdim=True))
    o = (_bf(E) @ g) / E.sum(-1, keepdim=True)
    lse = torch.logsumexp(S, dim=-1)
    dP = do @ g.transpose(1, 2)
    dS = P * (dP - (dP * P).sum(-1, keepdim=True))
    dSb = _bf(dS)
    return dict(o=o, lse=lse, dth=dSb @ ph, dph=dSb.transpose(1, 2) @ th, dg=Pb.transpose(1, 2) @ do)


# (n, hw, cq, c2, ct): D's block at 64x64 (ch=96: C=96 -> C/8=12 -> cq 16, c2 48), G's (C=192 -> cq 32,
# c2 96), the smallest fused shape (one key block), c2 = 16 / 128 and a padded ct
CASES = [(2, 4096, 16, 48, 80), (1, 4096, 32, 96, 160), (3, 512, 16, 16, 48), (2, 1024, 32, 128, 200),
         (1, 2048, 16, 64, 104)]


@pytest.mark.parametrize("n,hw,cq,c2,ct", CASES)
@pytest.mark.parametrize("scale,flat", [(0.5, 1), (0.5, 0), (1.5, 1), (1.5, 0), (6.0, 1)])
def test_attn_fwd_bwd_vs_definition(n, hw, cq, c2, ct, scale, flat, monkeypatch):
    """scale 0.5: the image-wide score bound max|theta| max|phi| is below 40 and (flat = 1) every tile takes
    the flat forward with that bound as its softmax offset, or (flat = 0, PARAGAN_ATTN_FLAT=0) the per-tile
    single-pass decision; scale 1.5: every tile takes the single-pass forward (the score bound is within e^16
    of chunk 0's max, R21); scale 6: the scores spread over hundreds, the bound check fails and the tiles take
    the exact two-pass forward."""
    monkeypatch.setenv("PARAGAN_ATTN_FLAT", str(flat))
    qkv, phi, gp, dO = _inputs(n, hw, cq, c2, ct, scale, seed=hw + cq + c2)
    want = _reference(qkv, phi, gp, dO, cq)
    q = hw // 4
    qkv_d, phi_d, gp_d, dO_d = (t.to(DEV) for t in (qkv, phi, gp, dO))
    o = torch.empty(n, hw, c2, dtype=torch.bfloat16, device=DEV)
    o32 = torch.empty(n, hw, c2, dtype=torch.float32, device=DEV)
    lse = torch.empty(n, hw, dtype=torch.float32, device=DEV)
    api.op_attn_fwd(qkv_d, phi_d, gp_d, cq, c2, o, o32, lse)
    sentinel = 3.0
    dqkv = torch.full((n, hw, ct), sentinel, dtype=torch.bfloat16, device=DEV)
    dphi = torch.empty(n, q, cq, dtype=torch.float32, device=DEV)
    dgp = torch.empty(n, q, c2, dtype=torch.float32, device=DEV)
    api.op_attn_bwd(qkv_d, phi_d, gp_d, dO_d, o32, lse, cq, c2, dqkv, dphi, dgp)
    torch.cuda.synchronize()
    # forward: o32 and the reference each carry one bf16 rounding of every P~ = exp(S - m) (<= 2^-9
    # relative each), taken at different offsets m in the single-pass schedule: bar 2 * 2^-9; o adds one
    # bf16 rounding of the output
    assert _rel(o32.double().cpu(), want["o"]) < 2 * 2 ** -9
    assert _rel(o.double().cpu(), want["o"]) < 6e-3
    assert float((lse.double().cpu() - want["lse"]).abs().max()) < 1e-4 * max(1.0, float(want["lse"].abs().max()))
    # backward
    assert _rel(dgp.double().cpu(), want["dg"]) < 2e-3
    assert _rel(dphi.double().cpu(), want["dph"]) < 1e-2
    dth = dqkv[..., :cq].double().cpu()
    assert _rel(dth, want["dth"]) < 1e-2
    # channels beyond cq untouched
    assert bool((dqkv[..., cq:] == sentinel).all())


def test_attn_bwd_deterministic():
    n, hw, cq, c2, ct = 2, 2048, 32, 96, 160
    qkv, phi, gp, dO = (t.to(DEV) for t in _inputs(n, hw, cq, c2, ct, 1.0, seed=5))
    o = torch.empty(n, hw, c2, dtype=torch.bfloat16, device=DEV)
    o32 = torch.empty(n, hw, c2, dtype=torch.float32, device=DEV)
    lse = torch.empty(n, hw, dtype=torch.float32, device=DEV)
    api.op_attn_fwd(qkv, phi, gp, cq, c2, o, o32, lse)
    outs = []
    for _ in range(2):
        dqkv = torch.zeros(n, hw, ct, dtype=torch.bfloat16, device=DEV)
        dphi = torch.empty(n, hw // 4, cq, dtype=torch.float32, device=DEV)
        dgp = torch.empty(n, hw // 4, c2, dtype=torch.float32, device=DEV)
        api.op_attn_bwd(qkv, phi, gp, dO, o32, lse, cq, c2, dqkv, dphi, dgp)
        outs.append((dqkv, dphi, dgp))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_attn_rejects_unsupported_shapes():
    n, hw, cq, c2, ct = 1, 256, 16, 48, 80   # q = 64: not a multiple of 128
    qkv = torch.zeros(n, hw, ct, dtype=torch.bfloat16, device=DEV)
    phi = torch.zeros(n, hw // 4, cq, dtype=torch.bfloat16, device=DEV)
    gp = torch.zeros(n, hw // 4, c2, dtype=torch.bfloat16, device=DEV)
    o = torch.empty(n, hw, c2, dtype=torch.bfloat16, device=DEV)
    lse = torch.empty(n, hw, dtype=torch.float32, device=DEV)
    with pytest.raises(api.ParaganError):
        api.op_attn_fwd(qkv, phi, gp, cq, c2, o, None, lse)
    with pytest.raises(api.ParaganError):
        api.op_attn_fwd(qkv[:, :, :64].contiguous(), phi, gp, 24, c2, o, None, lse)
