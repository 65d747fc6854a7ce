"""Integer-exact parity of the tcgen05 convolutions at the EXACT layer shapes the benchmark runs
(BigGAN-128, ch=96, B=256 per GPU: G on 256 images, D on [fake; real] = 512 images in the D step and
on 256 fakes in the G step), so the launch configurations bench.py times (CTA-pair kernels, halo
tiles, persistent-grid tails, wave-aware split-K, sub-pixel phases) are the ones checked.

Inputs come from a counter-based generator (paper_2411_03999_b200/inputs.counter_tensor): the GPU
fills the full tensors, the host recomputes any element from its index, and the oracle
(oracle/sampled.py) evaluates the plain conv sums at sampled outputs.  Values are small integers
(x in {-1,0,1} or {0,1}, w in {-1,0,1}, dy in {-1,0,1}) so every partial sum is an exact fp32
integer (< 2^24 even for wgrad over 8.4M pixels): any summation or split-K order gives the same
result, and the comparison is bit-exact.  The bf16 outputs are compared with
the RNE bf16 rounding of the exact value."""
import numpy as np
import pytest
import torch

from oracle import biggan as bg
from oracle import ops
from oracle import sampled as S
from paper_2411_03999_b200 import api
from paper_2411_03999_b200.inputs import counter_ints, counter_tensor

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda:0"
B = 256


def _layers():
    """(kind, n, H, cin, cout, k, epilogue) of every conv launch of one bench iteration, deduplicated.
    kind: fprop (fprop and fprop-shaped dgrad), wgrad, up2f / up2d / up2w (G's conv1)."""
    cfg = bg.Config(resolution=128, ch=96)
    keys = []
    for ci, co, h, att in bg.g_blocks(cfg):
        keys += [("up2f", B, h, ci, co, 3, ""), ("up2d", B, h, ci, co, 3, ""), ("up2w", B, h, ci, co, 3, "")]
        keys += [("fprop", B, 2 * h, co, co, 3, "res2"), ("fprop", B, 2 * h, co, co, 3, "mask+res"),
                 ("wgrad", B, 2 * h, co, co, 3, "")]
        keys += [("fprop", B, h, ci, co, 1, ""), ("fprop", B, h, co, ci, 1, "mask+res"), ("wgrad", B, h, ci, co, 1, "")]
        if att:   # packed theta/phi/g 1x1 conv (cq padded to 32) and the o conv
            ct = 2 * 32 + co // 2
            keys += [("fprop", B, 2 * h, co, ct, 1, ""), ("wgrad", B, 2 * h, co, ct, 1, ""),
                     ("fprop", B, 2 * h, co // 2, co, 1, "res1"), ("wgrad", B, 2 * h, co // 2, co, 1, "")]
    for j, (ci, co, h, dn, att) in enumerate(bg.d_blocks(cfg)):
        cx = 8 if ci == 3 else ci
        for n in (2 * B, B):   # D step on [fake; real]; G step on the fakes (dgrad only)
            if j == 0:   # D's first conv: a 1x1 conv over the 27 (-> 32) channel im2col of the image
                keys += [("fprop", n, h, 32, co, 1, "relu_out")]
            else:
                keys += [("fprop", n, h, cx, co, 3, "relu_out"), ("fprop", n, h, co, ci, 3, "mask+res")]
            keys += [("fprop", n, h, co, co, 3, "res1" if not dn else ""), ("fprop", n, h, co, co, 3, "mask")]
            if ci != co or dn:
                hs = h // 2 if j == 0 else h
                keys += [("fprop", n, hs, cx, co, 1, ""), ("fprop", n, hs, co, cx, 1, "")]
        keys.append(("fprop", B, h, co, 32, 1, "") if j == 0 else ("fprop", B, h, co, ci, 3, "mask+res"))
        keys += [("wgrad", 2 * B, h, 32, co, 1, "") if j == 0 else ("wgrad", 2 * B, h, cx, co, 3, ""),
                 ("wgrad", 2 * B, h, co, co, 3, "")]
        if ci != co or dn:
            keys += [("wgrad", 2 * B, h // 2 if j == 0 else h, cx, co, 1, "")]
        if att:
            ct = 2 * 16 + co // 2
            for n in (2 * B, B):
                keys += [("fprop", n, h // 2, co, ct, 1, ""), ("fprop", n, h // 2, co // 2, co, 1, "res1")]
            keys += [("wgrad", 2 * B, h // 2, co, ct, 1, ""), ("wgrad", 2 * B, h // 2, co // 2, co, 1, "")]
    out = []
    for k_ in keys:
        if k_ not in out:
            out.append(k_)
    return out


LAYERS = _layers()


def _ids(k):
    return "-".join(str(v) for v in k if v != "")


class Gen:
    """Counter-generated NHWC tensor: full tensor on the GPU, any element on the host."""

    def __init__(self, shape, seed, lo, hi):
        self.shape, self.seed, self.lo, self.hi = shape, seed, lo, hi

    def device(self):
        return counter_tensor(self.shape, self.seed, self.lo, self.hi, DEV, torch.bfloat16)

    def at(self, n, i, j):
        _, H, W, C = self.shape
        base = ((n.astype(np.int64) * H + i) * W + j) * C
        idx = torch.from_numpy(base[:, None] + np.arange(C, dtype=np.int64)[None, :])
        return counter_ints(idx, self.seed, self.lo, self.hi).numpy().astype(np.float64)

    def cols(self, cs):
        """[N, H, W, len(cs)] for the channel sample cs."""
        N, H, W, C = self.shape
        p = torch.arange(N * H * W, dtype=torch.int64)[:, None] * C + torch.as_tensor(cs, dtype=torch.int64)[None, :]
        return counter_ints(p, self.seed, self.lo, self.hi).numpy().astype(np.float64).reshape(N, H, W, len(cs))


def _sample_pixels(n, H, W, rng, count=1536):
    """Output pixels covering the first and last 128-pixel tiles, one pixel in evenly spaced tiles across
    the whole M range, every image border of a few images, and random pixels."""
    M = n * H * W
    m = [np.arange(min(128, M)), np.arange(max(0, M - 128), M)]
    tiles = (M + 127) // 128
    t = np.linspace(0, tiles - 1, num=min(tiles, 512)).astype(np.int64)
    m.append(np.minimum(t * 128 + (t * 37) % 128, M - 1))
    m.append(rng.integers(0, M, size=count))
    for img in (0, n // 2, n - 1):
        e = np.concatenate([np.arange(W), (H - 1) * W + np.arange(W), np.arange(H) * W, np.arange(H) * W + W - 1])
        m.append(img * H * W + e[:256])
    m = np.unique(np.concatenate(m))
    nn = m // (H * W)
    r = m % (H * W)
    return m, nn, r // W, r % W


def _spread(c, count=8):
    """Sampled channel indices covering both ends and 32/64-channel block boundaries."""
    cand = [0, 1, 15, 16, 31, 32, 63, 64, 95, 96, 127, 128, c // 2, c - 33, c - 32, c - 2, c - 1]
    s = sorted({v for v in cand if 0 <= v < c})
    rng = np.random.default_rng(c)
    return np.array(sorted(set(s[:: max(1, len(s) // count)] + [c - 1] + list(rng.integers(0, c, 2)))))


def _weights(rng, cout, taps, cin):
    return rng.integers(-1, 2, size=(cout, taps, cin)).astype(np.float32)


@pytest.mark.parametrize("layer", LAYERS, ids=[_ids(k) for k in LAYERS])
def test_bench_shape_conv_integer_exact(layer):
    kind, n, H, cin, cout, k, epi = layer
    rng = np.random.default_rng(abs(hash(layer)) % 2 ** 32)
    seed = int(rng.integers(1, 2 ** 20))
    torch.cuda.synchronize()
    if kind == "fprop":
        xg = Gen((n, H, H, cin), seed, -1, 1)
        wt = _weights(rng, cout, k * k, cin)
        b = rng.integers(-3, 4, size=cout).astype(np.float32)
        res = relu = None
        kw = {}
        if "res1" in epi or "mask+res" in epi:
            res = Gen((n, H, H, cout), seed + 1, -2, 2)
            kw["residual_at"] = res.at
        if "res2" in epi:
            res = Gen((n, H // 2, H // 2, cout), seed + 1, -2, 2)
            kw["residual_at"] = lambda nn, i, j: res.at(nn, i // 2, j // 2)
        if "mask" in epi:
            relu = Gen((n, H, H, cout), seed + 2, -1, 1)
            kw["relu_ref_at"] = relu.at
        y = torch.full((n, H, H, cout), float("nan"), dtype=torch.bfloat16, device=DEV)
        api.op_conv_fwd_ex(xg.device(), torch.from_numpy(wt).to(DEV).to(torch.bfloat16), torch.from_numpy(b).to(DEV),
                           cout, k, y, residual=None if res is None else res.device(),
                           res_mode=2 if "res2" in epi else 1, relu_ref=None if relu is None else relu.device(),
                           relu_out="relu_out" in epi)
        m, nn, ii, jj = _sample_pixels(n, H, H, rng)
        got = y.reshape(-1, cout)[torch.from_numpy(m).to(DEV)].float().cpu().numpy()
        want = S.conv_fprop_at(xg.at, H, H, cin, wt, k, nn, ii, jj, bias=b.astype(np.float64),
                               relu_out="relu_out" in epi, **kw)
    elif kind == "up2f":
        xg = Gen((n, H, H, cin), seed, -1, 1)
        wt = _weights(rng, cout, 9, cin)
        b = rng.integers(-3, 4, size=cout).astype(np.float32)
        y = torch.full((n, 2 * H, 2 * H, cout), float("nan"), dtype=torch.bfloat16, device=DEV)
        api.op_conv_up2_fwd(xg.device(), torch.from_numpy(wt).to(DEV), torch.from_numpy(b).to(DEV), cout, y)
        m, nn, ii, jj = _sample_pixels(n, 2 * H, 2 * H, rng)
        got = y.reshape(-1, cout)[torch.from_numpy(m).to(DEV)].float().cpu().numpy()
        want = S.up2_conv3x3_fprop_at(xg.at, H, H, cin, wt, nn, ii, jj, bias=b.astype(np.float64))
    elif kind == "up2d":
        dyg = Gen((n, 2 * H, 2 * H, cout), seed, -1, 1)
        wt = _weights(rng, cout, 9, cin)
        dx = torch.full((n, H, H, cin), float("nan"), dtype=torch.bfloat16, device=DEV)
        api.op_conv_up2_dgrad(dyg.device(), torch.from_numpy(wt).to(DEV), cin, dx)
        m, nn, ii, jj = _sample_pixels(n, H, H, rng)
        got = dx.reshape(-1, cin)[torch.from_numpy(m).to(DEV)].float().cpu().numpy()
        want = S.up2_conv3x3_dgrad_at(dyg.at, H, H, cout, wt, nn, ii, jj)
    else:   # wgrad / up2w: x in {0,1}, dy in {-1,0,1}: |sum| <= pixels < 2^24
        up = kind == "up2w"
        Hy = 2 * H if up else H
        xg = Gen((n, H, H, cin), seed, 0, 1)
        dyg = Gen((n, Hy, Hy, cout), seed + 3, -1, 1)
        assert n * Hy * Hy < 2 ** 24
        kk = 3 if up else k
        dw = torch.full((cout, kk * kk, cin), float("nan"), dtype=torch.float32, device=DEV)
        db = torch.full((cout,), float("nan"), dtype=torch.float32, device=DEV)
        if up:
            api.op_conv_up2_wgrad(xg.device(), dyg.device(), cout, dw, db=db)
        else:
            api.op_conv_wgrad(api.BF16, xg.device(), dyg.device(), cout, k, dw, db=db)
        os_, cs = _spread(cout), _spread(cin)
        torch.cuda.synchronize()
        got = dw.cpu().numpy()[os_][:, :, cs]
        xc, dc = xg.cols(cs), dyg.cols(os_)
        want = S.up2_conv3x3_wgrad_at(xc, dc, H, H) if up else S.conv_wgrad_at(xc, dc, H, H, k)
        assert np.array_equal(got, want.astype(np.float32)), np.argwhere(got != want)[:5]
        got_b = db.cpu().numpy()[os_]
        assert np.array_equal(got_b, dc.reshape(-1, len(os_)).sum(0).astype(np.float32))
        return
    want_b = ops.bf16_round(torch.from_numpy(want)).numpy()
    bad = np.argwhere(got != want_b)
    assert bad.size == 0, (len(bad), bad[:5], got[tuple(bad[0])], want[tuple(bad[0])])
