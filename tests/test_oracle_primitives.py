"""Pins for the oracle's primitive ops against things other than the oracle itself:
independent bit formulas, brute-force loops, closed forms, library SVD, the paper's
printed padding example."""
import itertools
import json
import os

import numpy as np
import pytest
import torch

from oracle import ops

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- bf16 RNE
def _bf16_bits_formula(b: np.ndarray) -> np.ndarray:
    """Independent round-to-nearest-even on the bit pattern."""
    b = b.astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint32) & 0xFFFF


def test_bf16_rne_against_bit_formula_all_high_halves():
    # every sign/exponent/high-mantissa pattern x low halves that exercise the
    # tie, just-below, just-above, zero and all-ones cases
    hi = np.arange(1 << 16, dtype=np.uint32) << 16
    lows = np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0xFFFF, 0x1234, 0xC000], dtype=np.uint32)
    bits = (hi[:, None] | lows[None, :]).reshape(-1)
    x = bits.view(np.float32)
    got = ops.bf16_round(torch.from_numpy(x.copy())).to(torch.float32).numpy().view(np.uint32) >> 16
    nan = np.isnan(x)
    want = _bf16_bits_formula(bits)
    assert np.array_equal(got[~nan], want[~nan])
    # NaN stays NaN (the payload/sign is not part of the contract)
    gv = got[nan].astype(np.uint32)
    assert np.all((gv & 0x7F80) == 0x7F80) and np.all((gv & 0x7F) != 0)


def test_bf16_rne_random_full_patterns_and_idempotent():
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 1 << 32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    ok = ~np.isnan(x)
    r = ops.bf16_round(torch.from_numpy(x.copy())).to(torch.float32).numpy()
    assert np.array_equal(r.view(np.uint32)[ok] >> 16, _bf16_bits_formula(bits[ok]))
    r2 = ops.bf16_round(torch.from_numpy(r.copy())).to(torch.float32).numpy()
    assert np.array_equal(r2.view(np.uint32)[ok], r.view(np.uint32)[ok])


# ---------------------------------------------------------------- layout pack (A1)
def test_padding_example_from_paper():
    with open(os.path.join(GOLDEN, "padding_p239.json")) as f:
        g = json.load(f)
    zeros, frac = ops.padding_waste(*g["shape"], g["tile"])
    assert zeros == g["zeros"]
    assert round(frac * 100) == g["waste_percent_rounded"]


@pytest.mark.parametrize("to_bf16", [False, True])
def test_layout_pack_brute_force_and_round_trip(to_bf16):
    rng = np.random.default_rng(1)
    n, c, h, w, cp = 2, 3, 5, 4, 8
    x = rng.uniform(-1, 1, size=(n, c, h, w)).astype(np.float32)
    y = ops.layout_pack(x, cp, to_bf16)
    assert y.shape == (n, h, w, cp)
    for i, j, k, l in itertools.product(range(n), range(h), range(w), range(cp)):
        if l < c:
            want = x[i, l, j, k]
            if to_bf16:
                want = float(torch.tensor(want).to(torch.bfloat16).to(torch.float32))
            assert y[i, j, k, l] == want
        else:
            assert y[i, j, k, l] == 0.0 and not np.signbit(y[i, j, k, l])
    back = ops.layout_unpack(y, c)
    assert np.array_equal(ops.layout_pack(back, cp, to_bf16), y)
    if not to_bf16:
        assert np.array_equal(back, x)


# ---------------------------------------------------------------- spectral norm (A2)
def _spectral_gap_matrix(rng, m, k, s=(3.0, 1.0)):
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((k, k)))
    sv = np.linspace(s[1], 0.1, min(m, k))
    sv[0] = s[0]
    return (u[:, :len(sv)] * sv) @ v[:len(sv)]


def test_sn_converges_to_svd_sigma_max():
    rng = np.random.default_rng(3)
    for m, k in [(12, 96), (40, 27), (64, 64)]:
        w = torch.tensor(_spectral_gap_matrix(rng, m, k))
        u = torch.tensor(rng.standard_normal(m))
        u = u / u.norm()
        for _ in range(500):
            sigma, u, _ = ops.sn_power_step(w, u, 1e-12)
        smax = np.linalg.svd(w.numpy(), compute_uv=False)[0]
        assert abs(float(sigma) - smax) < 1e-6 * smax


def test_sn_one_step_bounded_and_rank1_exact():
    rng = np.random.default_rng(4)
    w = torch.tensor(rng.standard_normal((30, 50)))
    smax = np.linalg.svd(w.numpy(), compute_uv=False)[0]
    for _ in range(20):
        u = torch.tensor(rng.standard_normal(30))
        sigma, _, _ = ops.sn_power_step(w, u / u.norm(), 1e-12)
        assert float(sigma) <= smax * (1 + 1e-12)
    a, b = rng.standard_normal(7), rng.standard_normal(11)
    w1 = torch.tensor(np.outer(a, b))
    u = torch.tensor(rng.standard_normal(7))
    sigma, _, _ = ops.sn_power_step(w1, u, 1e-12)
    assert abs(float(sigma) - np.linalg.norm(a) * np.linalg.norm(b)) < 1e-12 * np.linalg.norm(a) * np.linalg.norm(b)


def test_sn_invariant_under_k_permutation_and_conv_view():
    rng = np.random.default_rng(5)
    w = torch.tensor(rng.standard_normal((6, 4, 3, 3)))
    u = torch.tensor(rng.standard_normal(6))
    s1, _, _ = ops.sn_power_step(w, u, 1e-12)
    perm = torch.tensor(rng.permutation(36))
    s2, _, _ = ops.sn_power_step(w.reshape(6, 36)[:, perm], u, 1e-12)
    s3, _, _ = ops.sn_power_step(w.permute(0, 2, 3, 1).contiguous(), u, 1e-12)  # OHWI storage
    assert abs(float(s1 - s2)) < 1e-12 and abs(float(s1 - s3)) < 1e-12


def test_sn_backward_is_rank1_correction_by_fd():
    """d/dW of sum(G * W/sigma) with u', v frozen, against central differences."""
    rng = np.random.default_rng(6)
    w = torch.tensor(rng.standard_normal((5, 8)), requires_grad=True)
    gmat = torch.tensor(rng.standard_normal((5, 8)))
    u = torch.tensor(rng.standard_normal(5))
    _, u1, v1 = ops.sn_power_step(w, u, 1e-12)

    def f(wt):
        return ((wt / (u1 @ (wt @ v1))) * gmat).sum()

    (gw,) = torch.autograd.grad(f(w), w)
    h = 1e-6
    fd = np.zeros((5, 8))
    for i in range(5):
        for j in range(8):
            e = torch.zeros(5, 8, dtype=torch.float64)
            e[i, j] = h
            fd[i, j] = float(f(w.detach() + e) - f(w.detach() - e)) / (2 * h)
    assert np.allclose(gw.numpy(), fd, rtol=1e-6, atol=1e-8)
    # closed form: (G - <G, W_hat> u' v^T) / sigma
    sigma = float(u1 @ (w.detach() @ v1))
    what = w.detach() / sigma
    cf = (gmat - (gmat * what).sum() * torch.outer(u1, v1)) / sigma
    assert np.allclose(gw.numpy(), cf.numpy(), rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- conv / resampling (A5, A9-A11)
def _conv_loops(x, w, b):
    n, c, h, wd = x.shape
    o, _, r, s = w.shape
    p = r // 2
    y = np.zeros((n, o, h, wd))
    for i in range(n):
        for oo in range(o):
            for yy in range(h):
                for xx in range(wd):
                    acc = b[oo] if b is not None else 0.0
                    for cc in range(c):
                        for rr in range(r):
                            for ss in range(s):
                                iy, ix = yy + rr - p, xx + ss - p
                                if 0 <= iy < h and 0 <= ix < wd:
                                    acc += x[i, cc, iy, ix] * w[oo, cc, rr, ss]
                    y[i, oo, yy, xx] = acc
    return y


@pytest.mark.parametrize("k", [1, 3])
def test_conv_matches_brute_force(k):
    rng = np.random.default_rng(10 + k)
    x = rng.standard_normal((2, 3, 5, 4))
    w = rng.standard_normal((4, 3, k, k))
    b = rng.standard_normal(4)
    got = ops.conv2d(torch.tensor(x), torch.tensor(w), torch.tensor(b)).numpy()
    assert np.allclose(got, _conv_loops(x, w, b), rtol=1e-12, atol=1e-12)


def test_conv_delta_kernel_shifts_and_adjoint_identity():
    rng = np.random.default_rng(12)
    x = torch.tensor(rng.standard_normal((1, 1, 6, 6)))
    for r, s in itertools.product(range(3), range(3)):
        w = torch.zeros(1, 1, 3, 3, dtype=torch.float64)
        w[0, 0, r, s] = 1.0
        y = ops.conv2d(x, w, None)[0, 0].numpy()
        xp = np.pad(x[0, 0].numpy(), 1)
        assert np.array_equal(y, xp[r:r + 6, s:s + 6])
    # <conv(x,W), dy> = <x, dgrad(dy,W)> = <W, wgrad(x,dy)>
    x = torch.tensor(rng.standard_normal((2, 3, 5, 5)), requires_grad=True)
    w = torch.tensor(rng.standard_normal((4, 3, 3, 3)), requires_grad=True)
    dy = torch.tensor(rng.standard_normal((2, 4, 5, 5)))
    y = ops.conv2d(x, w, None)
    gx, gw = torch.autograd.grad((y * dy).sum(), [x, w])
    lhs = float((y * dy).sum().detach())
    assert abs(lhs - float((x * gx).sum().detach())) < 1e-10 * abs(lhs)
    assert abs(lhs - float((w * gw).sum())) < 1e-10 * abs(lhs)


def test_resampling_brute_force():
    rng = np.random.default_rng(13)
    x = rng.standard_normal((2, 3, 4, 6))
    u = ops.up2(torch.tensor(x)).numpy()
    for i, j in itertools.product(range(8), range(12)):
        assert np.array_equal(u[:, :, i, j], x[:, :, i // 2, j // 2])
    a = ops.avgpool2(torch.tensor(x)).numpy()
    m = ops.maxpool2(torch.tensor(x)).numpy()
    for i, j in itertools.product(range(2), range(3)):
        blk = x[:, :, 2 * i:2 * i + 2, 2 * j:2 * j + 2]
        assert np.allclose(a[:, :, i, j], blk.sum(axis=(2, 3)) * 0.25, rtol=1e-15)
        assert np.array_equal(m[:, :, i, j], blk.max(axis=(2, 3)))


# ---------------------------------------------------------------- BN (A4, A11)
def test_bn_moments_and_backward_invariants():
    rng = np.random.default_rng(14)
    x = torch.tensor(rng.standard_normal((4, 5, 3, 3)) * 3 + 1, requires_grad=True)
    y = ops.cbn(x, torch.zeros(4, 5, dtype=torch.float64), torch.zeros(4, 5, dtype=torch.float64), 0.0)
    assert np.allclose(y.mean(dim=(0, 2, 3)).detach().numpy(), 0, atol=1e-12)
    assert np.allclose(y.var(dim=(0, 2, 3), unbiased=False).detach().numpy(), 1, atol=1e-12)
    dy = torch.tensor(rng.standard_normal((4, 5, 3, 3)))
    (dx,) = torch.autograd.grad((y * dy).sum(), x)
    assert np.allclose(dx.sum(dim=(0, 2, 3)).numpy(), 0, atol=1e-10)
    assert np.allclose((dx * y).sum(dim=(0, 2, 3)).detach().numpy(), 0, atol=1e-10)


def test_bn_split_batch_statistics_equal_global():
    """What W replicas exchange (per-channel sum, sum of squares, count) reproduces
    the single-process global statistics (R5, R15)."""
    rng = np.random.default_rng(15)
    x = rng.standard_normal((8, 6, 4, 4)) * 2 + 0.5
    shards = np.split(x, 4, axis=0)
    s1 = sum(s.sum(axis=(0, 2, 3)) for s in shards)
    s2 = sum((s ** 2).sum(axis=(0, 2, 3)) for s in shards)
    cnt = x.shape[0] * 16
    mu, var = s1 / cnt, s2 / cnt - (s1 / cnt) ** 2
    xt = torch.tensor(x)
    want = ops.bn_normalise(xt, 1e-5).numpy()
    got = (x - mu[None, :, None, None]) / np.sqrt(var[None, :, None, None] + 1e-5)
    assert np.allclose(got, want, rtol=1e-10, atol=1e-10)


# ---------------------------------------------------------------- attention (A6)
def test_attention_gamma0_identity_and_loop_form():
    rng = np.random.default_rng(16)
    c = 8
    x = rng.standard_normal((2, c, 4, 4))
    wt, wp = rng.standard_normal((c // 8, c, 1, 1)), rng.standard_normal((c // 8, c, 1, 1))
    wg, wo = rng.standard_normal((c // 2, c, 1, 1)), rng.standard_normal((c, c // 2, 1, 1))
    T = torch.tensor
    out0 = ops.attention(T(x), T(wt), T(wp), T(wg), T(wo), 0.0).numpy()
    assert np.array_equal(out0, x)
    gam = 0.7
    got = ops.attention(T(x), T(wt), T(wp), T(wg), T(wo), gam).numpy()
    # loop form
    for n in range(2):
        X = x[n].reshape(c, 16)
        th = wt[:, :, 0, 0] @ X
        ph = (wp[:, :, 0, 0] @ X).reshape(-1, 4, 4)
        gg = (wg[:, :, 0, 0] @ X).reshape(-1, 4, 4)
        php = np.stack([ph[:, 2 * i:2 * i + 2, 2 * j:2 * j + 2].max(axis=(1, 2)) for i in range(2) for j in range(2)], 1)
        ggp = np.stack([gg[:, 2 * i:2 * i + 2, 2 * j:2 * j + 2].max(axis=(1, 2)) for i in range(2) for j in range(2)], 1)
        out = np.zeros((c, 16))
        for p in range(16):
            s = np.array([th[:, p] @ php[:, k] for k in range(4)])
            e = np.exp(s - s.max())
            beta = e / e.sum()
            o = ggp @ beta
            out[:, p] = X[:, p] + gam * (wo[:, :, 0, 0] @ o)
        assert np.allclose(got[n].reshape(c, 16), out, rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- hinge (A8)
def test_hinge_closed_forms():
    B = 4
    lr_ = torch.zeros(B, dtype=torch.float64, requires_grad=True)
    lf = torch.zeros(B, dtype=torch.float64, requires_grad=True)
    ld = ops.hinge_d(lr_, lf)
    assert float(ld) == 2.0
    gr, gf = torch.autograd.grad(ld, [lr_, lf])
    assert np.allclose(gr.numpy(), -1.0 / B) and np.allclose(gf.numpy(), 1.0 / B)
    lg = ops.hinge_g(lf)
    assert float(lg) == 0.0
    (gg,) = torch.autograd.grad(lg, lf)
    assert np.allclose(gg.numpy(), -1.0 / B)
    # a perfect D: zero loss, zero gradient
    lr2 = torch.full((B,), 1.5, dtype=torch.float64, requires_grad=True)
    lf2 = torch.full((B,), -1.5, dtype=torch.float64, requires_grad=True)
    ld2 = ops.hinge_d(lr2, lf2)
    assert float(ld2) == 0.0
    g1, g2 = torch.autograd.grad(ld2, [lr2, lf2])
    assert float(g1.abs().sum() + g2.abs().sum()) == 0.0


# ---------------------------------------------------------------- Adam (A13)
def test_adam_first_step_closed_form():
    rng = np.random.default_rng(17)
    w = torch.tensor(rng.standard_normal(100))
    g = torch.tensor(rng.standard_normal(100))
    z = torch.zeros(100, dtype=torch.float64)
    for b1 in (0.0, 0.5, 0.9):
        w1, _, _ = ops.adam_update(w, g, z, z, 1, 1e-3, b1, 0.999, 1e-8)
        assert np.allclose((w1 - w).numpy(), (-1e-3 * g / (g.abs() + 1e-8)).numpy(), rtol=1e-9, atol=0)
    w1, _, _ = ops.adam_update(w, g, z, z, 1, 0.0, 0.0, 0.999, 1e-8)
    assert torch.equal(w1, w)


def test_adam_scalar_reference_1000_steps():
    """f(w) = w^2 against an independent scalar loop written with Python floats."""
    w = torch.tensor([1.5], dtype=torch.float64)
    m = torch.zeros(1, dtype=torch.float64)
    v = torch.zeros(1, dtype=torch.float64)
    ws, ms, vs = 1.5, 0.0, 0.0
    lr, b1, b2, eps = 1e-2, 0.5, 0.999, 1e-8
    for t in range(1, 1001):
        w, m, v = ops.adam_update(w, 2 * w, m, v, t, lr, b1, b2, eps)
        g = 2 * ws
        ms = b1 * ms + (1 - b1) * g
        vs = b2 * vs + (1 - b2) * g * g
        ws = ws - lr * (ms / (1 - b1 ** t)) / ((vs / (1 - b2 ** t)) ** 0.5 + eps)
    assert abs(float(w) - ws) < 1e-12
    assert abs(ws) < 0.05


def test_up2_conv_phase_decomposition_is_conv_of_upsampled():
    """R24: the four 2x2 phase convs of the low-resolution input equal conv3x3(up2(x)) — values and
    both gradients, in fp64 (the bf16 variant only moves the rounding point of the weights)."""
    rng = np.random.default_rng(11)
    x = torch.from_numpy(rng.standard_normal((2, 3, 5, 4))).requires_grad_(True)
    w = torch.from_numpy(rng.standard_normal((4, 3, 3, 3))).requires_grad_(True)
    b = torch.from_numpy(rng.standard_normal(4))
    dy = torch.from_numpy(rng.standard_normal((2, 4, 10, 8)))
    y1 = ops.up2_conv3x3_phases(x, w, b)
    y2 = ops.conv2d(ops.up2(x), w, b)
    assert torch.allclose(y1, y2, rtol=1e-12, atol=1e-12)
    g1 = torch.autograd.grad((y1 * dy).sum(), (x, w))
    g2 = torch.autograd.grad((y2 * dy).sum(), (x, w))
    for a, c in zip(g1, g2):
        assert torch.allclose(a, c, rtol=1e-12, atol=1e-12)
    # each output pixel of phase (a, b) reads exactly a 2x2 low-resolution window: a delta input
    # lights the 4x4 high-resolution block the 3x3 kernel over the 2x2 replicated pixel covers
    xd = torch.zeros(1, 1, 4, 4, dtype=torch.float64)
    xd[0, 0, 1, 2] = 1.0
    yd = ops.up2_conv3x3_phases(xd, torch.ones(1, 1, 3, 3, dtype=torch.float64), None)
    nz = torch.nonzero(yd[0, 0]).tolist()
    assert sorted({r for r, _ in nz}) == [1, 2, 3, 4] and sorted({c for _, c in nz}) == [3, 4, 5, 6]


def test_pooled_block_input_gradient_is_phase_conv_of_pooled_gradient():
    """R37: behind a 2x2 average pool the conv's output gradient is up2(g)/4, so its input gradient equals the
    sub-pixel phase conv of the pooled gradient g with the flipped, transposed kernel K[c][o][r][s] =
    W[o][c][2-r][2-s], divided by 4 — checked in fp64 against autograd through avgpool2(conv2d(x, W)).  The 1x1
    shortcut's input gradient commutes with the pool's adjoint the same way (up2(sc^T g)/4)."""
    rng = np.random.default_rng(13)
    x = torch.from_numpy(rng.standard_normal((2, 5, 8, 6))).requires_grad_(True)
    w = torch.from_numpy(rng.standard_normal((4, 5, 3, 3)))
    g = torch.from_numpy(rng.standard_normal((2, 4, 4, 3)))
    pooled = torch.nn.functional.avg_pool2d(ops.conv2d(x, w, None), 2)
    (want,) = torch.autograd.grad((pooled * g).sum(), x)
    k = w.flip(2, 3).transpose(0, 1).contiguous()
    got = ops.up2_conv3x3_phases(g, k, None) / 4.0
    assert torch.allclose(got, want, rtol=1e-12, atol=1e-12)
    # the 1x1 shortcut
    x1 = torch.from_numpy(rng.standard_normal((2, 5, 8, 6))).requires_grad_(True)
    w1 = torch.from_numpy(rng.standard_normal((4, 5, 1, 1)))
    (want1,) = torch.autograd.grad((torch.nn.functional.avg_pool2d(ops.conv2d(x1, w1, None), 2) * g).sum(), x1)
    got1 = ops.up2(ops.conv2d(g, w1.transpose(0, 1).contiguous(), None)) / 4.0
    assert torch.allclose(got1, want1, rtol=1e-12, atol=1e-12)


def test_pooled_block_forward_is_adjoint_of_phase_conv():
    """R38: avgpool2(conv3x3_W(x)) equals a quarter of the adjoint (up2^T conv^T) of the sub-pixel phase conv
    with the flipped, transposed kernel K = W[o][c][2-r][2-s]^T — the 16-tap stride-2 form the pooled forward
    runs through the phase input-gradient kernel — in fp64, the adjoint taken by autograd."""
    rng = np.random.default_rng(17)
    x = torch.from_numpy(rng.standard_normal((2, 5, 8, 6)))
    w = torch.from_numpy(rng.standard_normal((4, 5, 3, 3)))
    want = torch.nn.functional.avg_pool2d(ops.conv2d(x, w, None), 2)
    k = w.flip(2, 3).transpose(0, 1).contiguous()   # [5][4][3][3]: maps 4 channels -> 5
    g = torch.zeros((2, 4, 4, 3), dtype=torch.float64, requires_grad=True)
    (got,) = torch.autograd.grad((ops.up2_conv3x3_phases(g, k, None) * x).sum(), g)
    assert torch.allclose(got / 4.0, want, rtol=1e-12, atol=1e-12)
    # the 1x1 shortcut's weight gradient behind the pool on the pooled input: sum_full (up2(g)/4) x = sum_half g
    # avgpool(x)
    gp = torch.from_numpy(rng.standard_normal((2, 4, 4, 3)))
    w1 = torch.zeros((4, 5, 1, 1), dtype=torch.float64, requires_grad=True)
    (want1,) = torch.autograd.grad((torch.nn.functional.avg_pool2d(ops.conv2d(x, w1, None), 2) * gp).sum(), w1)
    got1 = torch.einsum("nohw,nchw->oc", gp, torch.nn.functional.avg_pool2d(x, 2))[:, :, None, None]
    assert torch.allclose(got1, want1, rtol=1e-12, atol=1e-12)


# ------------------------------------------------- sampled conv definitions (oracle/sampled.py)
def test_sampled_conv_definitions_match_full_oracle():
    """oracle/sampled.py (used by the full-size GPU tests) against the full fp64 conv of ops.conv2d and
    its autograd at every output element of small ragged shapes, epilogue terms included."""
    from oracle import sampled as S
    rng = np.random.default_rng(0)
    for (n, H, W, cin, cout, k) in [(2, 5, 7, 3, 4, 3), (1, 4, 4, 6, 5, 1), (3, 6, 3, 2, 3, 3)]:
        x = rng.integers(-2, 3, size=(n, H, W, cin)).astype(np.float64)
        w = rng.integers(-1, 2, size=(cout, k * k, cin)).astype(np.float64)
        b = rng.integers(-3, 4, size=cout).astype(np.float64)
        ref = rng.integers(-1, 2, size=(n, H, W, cout)).astype(np.float64)
        res = rng.integers(-2, 3, size=(n, H, W, cout)).astype(np.float64)
        wt = torch.from_numpy(w).reshape(cout, k, k, cin).permute(0, 3, 1, 2)
        xt = torch.from_numpy(x).permute(0, 3, 1, 2)
        conv = ops.conv2d(xt, wt, None).permute(0, 2, 3, 1).numpy()
        want = np.maximum(np.where(ref > 0, conv, 0.0) + b + res, 0.0)
        nn, ii, jj = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(H), np.arange(W), indexing="ij"))
        got = S.conv_fprop_at(lambda a, i, j: x[a, i, j], H, W, cin, w, k, nn, ii, jj, bias=b,
                              relu_ref_at=lambda a, i, j: ref[a, i, j], residual_at=lambda a, i, j: res[a, i, j],
                              relu_out=True)
        assert np.array_equal(got.reshape(n, H, W, cout), want)
        dy = rng.integers(-2, 3, size=(n, H, W, cout)).astype(np.float64)
        wv = torch.zeros(cout, cin, k, k, dtype=torch.float64, requires_grad=True)
        (gw,) = torch.autograd.grad((ops.conv2d(xt, wv, None) * torch.from_numpy(dy).permute(0, 3, 1, 2)).sum(), wv)
        gw = gw.permute(0, 2, 3, 1).reshape(cout, k * k, cin).numpy()
        cs, os_ = [0, cin - 1], [cout - 1, 0]
        assert np.array_equal(S.conv_wgrad_at(x[..., cs], dy[..., os_], H, W, k), gw[os_][:, :, cs])
    # G's conv1 on the upsampled input: forward, low-resolution input gradient, weight gradient
    n, h, w_, cin, cout = 2, 3, 4, 3, 5
    x = rng.integers(-2, 3, size=(n, h, w_, cin)).astype(np.float64)
    w = rng.integers(-1, 2, size=(cout, 9, cin)).astype(np.float64)
    b = rng.integers(-3, 4, size=cout).astype(np.float64)
    xt = torch.from_numpy(x).permute(0, 3, 1, 2).requires_grad_(True)
    wt = torch.from_numpy(w).reshape(cout, 3, 3, cin).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    y = ops.conv2d(ops.up2(xt), wt, torch.from_numpy(b))
    dy = rng.integers(-2, 3, size=tuple(y.shape)).astype(np.float64)
    gx, gw = torch.autograd.grad((y * torch.from_numpy(dy)).sum(), (xt, wt))
    nn, ii, jj = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(2 * h), np.arange(2 * w_), indexing="ij"))
    got = S.up2_conv3x3_fprop_at(lambda a, i, j: x[a, i, j], h, w_, cin, w, nn, ii, jj, bias=b)
    assert np.array_equal(got.reshape(n, 2 * h, 2 * w_, cout), y.detach().permute(0, 2, 3, 1).numpy())
    dyn = dy.transpose(0, 2, 3, 1)
    nn, ii, jj = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(h), np.arange(w_), indexing="ij"))
    got = S.up2_conv3x3_dgrad_at(lambda a, i, j: dyn[a, i, j], h, w_, cout, w, nn, ii, jj)
    assert np.array_equal(got.reshape(n, h, w_, cin), gx.permute(0, 2, 3, 1).numpy())
    gwn = gw.permute(0, 2, 3, 1).reshape(cout, 9, cin).numpy()
    assert np.array_equal(S.up2_conv3x3_wgrad_at(x, dyn, h, w_), gwn)


def test_counter_generator_same_on_any_slice():
    """The counter-based generator the full-size tests share: element i depends only on (seed, i)
    (chunked fill == direct evaluation), values cover [lo, hi] roughly uniformly."""
    from paper_2411_03999_b200.inputs import counter_ints, counter_tensor
    t = counter_tensor((3, 5, 7, 11), 9, -1, 1, "cpu", torch.float32, chunk=97)
    direct = counter_ints(torch.arange(t.numel(), dtype=torch.int64), 9, -1, 1).reshape(t.shape).float()
    assert torch.equal(t, direct)
    v = counter_ints(torch.arange(30000, dtype=torch.int64), 3, 0, 2)
    counts = torch.bincount(v, minlength=3).numpy()
    assert counts.min() > 9000 and v.min() == 0 and v.max() == 2
