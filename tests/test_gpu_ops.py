"""Kernel-level parity through the C-ABI: layout pack (bit-exact), tcgen05 conv
fprop/dgrad-shaped/wgrad on integer-valued inputs (bit-exact: every partial sum is
an exact fp32 integer) and on random inputs, SIMT fp32 conv."""
import numpy as np
import pytest
import torch

from oracle import ops
from paper_2411_03999_b200 import api

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _bf16_np(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("n,c,h,w,cp", [(2, 3, 5, 7, 8), (4, 3, 128, 128, 8), (1, 3, 1, 1, 8), (3, 5, 9, 4, 16)])
def test_layout_pack_bit_exact(n, c, h, w, cp):
    rng = np.random.default_rng(n * 100 + h)
    x = rng.uniform(-1, 1, size=(n, c, h, w)).astype(np.float32)
    x.flat[0] = 0.5 + 2 ** -9          # a bf16 tie (rounds to even)
    xs = torch.from_numpy(x).to(DEV)
    for dt, tdt in ((api.BF16, torch.bfloat16), (api.F32, torch.float32)):
        y = torch.full((n, h, w, cp), 7.0, dtype=tdt, device=DEV)   # pads must be overwritten with 0
        api.layout_pack(xs, y, dt, cp)
        torch.cuda.synchronize()
        want = ops.layout_pack(x, cp, dt == api.BF16)
        got = y.float().cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        back = torch.empty((n, c, h, w), dtype=torch.float32, device=DEV)
        api.layout_unpack(y, dt, back, cp)
        torch.cuda.synchronize()
        assert np.array_equal(back.cpu().numpy(), ops.layout_unpack(want, c))


def test_tc_conv_rejects_untileable_geometry():
    x = torch.zeros((1, 12, 12, 32), dtype=torch.bfloat16, device=DEV)
    w = torch.zeros((48, 9, 32), dtype=torch.bfloat16, device=DEV)
    y = torch.zeros((1, 12, 12, 48), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(api.ParaganError) as e:
        api.op_conv_fwd(api.BF16, x, w, None, 48, 3, y)
    assert e.value.status == 1


def test_layout_pack_rejects_bad_args():
    x = torch.zeros((1, 3, 4, 4), device=DEV)
    y = torch.zeros((1, 4, 4, 4), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(api.ParaganError) as e:
        api.layout_pack(x, y, api.BF16, 4)     # bf16 needs c_pad % 8 == 0
    assert e.value.status == 1


CONV_SHAPES = [  # n, h, w, cin, cout, k
    (2, 8, 8, 64, 128, 3),
    (3, 16, 16, 96, 96, 3),      # 96-channel tail chunk
    (1, 4, 4, 8, 32, 3),         # M < 128 (ragged single tile), tiny C
    (2, 128, 128, 8, 96, 3),     # RGB-padded first D layer geometry
    (1, 32, 256, 16, 16, 3),     # W > 128: row-segment tiles
    (5, 32, 32, 192, 384, 1),    # 1x1
    (2, 64, 64, 192, 24, 1),     # attention-sized N tail
    (3, 8, 8, 1536, 256, 3),     # deep layer, several K chunks
    (3, 8, 8, 32, 48, 3),        # M = 192: ragged last tile
    (1, 2, 2, 16, 16, 1),        # M = 4
    (2, 4, 128, 96, 96, 3),      # halo-tile kernel (W % 128 == 0): 96 = 64 + 32 channels
    (1, 3, 256, 64, 192, 3),     # halo-tile kernel, two tiles per row
    (2, 2, 128, 192, 96, 3),     # halo-tile kernel, top and bottom rows out of the image
    (2, 64, 64, 96, 192, 3),     # column-shifted halo units, W = 64 (2 rows per tile)
    (2, 32, 32, 192, 96, 3),     # column-shifted halo units, W = 32
    (1, 16, 16, 8, 32, 3),       # column-shifted halo units, W = 16, one K step
    (5, 8, 8, 64, 128, 3),       # odd number of M tiles (CTA-pair kernel: last pair half empty)
    (4, 8, 8, 1536, 1536, 3),    # CTA pairs with several N tiles
    (2, 16, 32, 384, 136, 3),    # wgrad, one filter row per CTA: 3 x 128-channel blocks, C_out tail
    (3, 4, 8, 512, 256, 1),      # wgrad on the CTA-pair kernel, 1x1, odd M tile count
    (2, 8, 8, 256, 768, 3),      # wgrad on the CTA-pair kernel, three pair tiles
]


def _int_inputs(rng, n, h, w, cin, cout, k):
    x = rng.integers(-2, 3, size=(n, h, w, cin)).astype(np.float32)
    wt = rng.integers(-1, 2, size=(cout, k * k, cin)).astype(np.float32)
    b = rng.integers(-3, 4, size=(cout,)).astype(np.float32)
    return x, wt, b


def _oracle_conv(x_nhwc, w_otc, b, k):
    x = torch.from_numpy(x_nhwc).double().permute(0, 3, 1, 2)
    cout, _, cin = w_otc.shape
    w = torch.from_numpy(w_otc).double().reshape(cout, k, k, cin).permute(0, 3, 1, 2)
    y = ops.conv2d(x, w, torch.from_numpy(b).double() if b is not None else None)
    return y.permute(0, 2, 3, 1).numpy()


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_tc_conv_fprop_integer_exact(shape):
    n, h, w, cin, cout, k = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    x, wt, b = _int_inputs(rng, n, h, w, cin, cout, k)
    want = ops.bf16_round(torch.from_numpy(_oracle_conv(x, wt, b, k))).float().numpy()
    xd, wd = _bf16_np(x).to(DEV), _bf16_np(wt).to(DEV)
    bd = torch.from_numpy(b).to(DEV)
    y = torch.full((n, h, w, cout), float("nan"), dtype=torch.bfloat16, device=DEV)
    api.op_conv_fwd(api.BF16, xd, wd, bd, cout, k, y)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_tc_conv_wgrad_integer_exact(shape):
    n, h, w, cin, cout, k = shape
    if cout % 8:
        pytest.skip("wgrad needs C_out % 8")
    rng = np.random.default_rng(hash(shape) % 2**31 + 1)
    x = rng.integers(-2, 3, size=(n, h, w, cin)).astype(np.float32)
    dy = rng.integers(-2, 3, size=(n, h, w, cout)).astype(np.float32)
    # oracle: dW = d/dW <conv(x, W), dy>  (autograd of the plain conv)
    xt = torch.from_numpy(x).double().permute(0, 3, 1, 2)
    wv = torch.zeros(cout, cin, k, k, dtype=torch.float64, requires_grad=True)
    (gw,) = torch.autograd.grad((ops.conv2d(xt, wv, None) * torch.from_numpy(dy).double().permute(0, 3, 1, 2)).sum(), wv)
    want = gw.permute(0, 2, 3, 1).reshape(cout, k * k, cin).numpy().astype(np.float32)
    assert np.abs(want).max() < 2 ** 24
    dw = torch.full((cout, k * k, cin), float("nan"), dtype=torch.float32, device=DEV)
    db = torch.full((cout,), float("nan"), dtype=torch.float32, device=DEV)
    api.op_conv_wgrad(api.BF16, _bf16_np(x).to(DEV), _bf16_np(dy).to(DEV), cout, k, dw, db=db)
    torch.cuda.synchronize()
    got = dw.cpu().numpy()
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]
    # the bias gradient from the same launch: sum of dy over every pixel (exact integers)
    assert np.array_equal(db.cpu().numpy(), dy.reshape(-1, cout).sum(0).astype(np.float32))


@pytest.mark.parametrize("shape", CONV_SHAPES[:4])
def test_tc_conv_random_within_bf16_accumulation_error(shape):
    n, h, w, cin, cout, k = shape
    rng = np.random.default_rng(7)
    x = ops.bf16_round(torch.from_numpy(rng.standard_normal((n, h, w, cin)).astype(np.float32))).float().numpy()
    wt = ops.bf16_round(torch.from_numpy(rng.standard_normal((cout, k * k, cin)).astype(np.float32) * 0.05)).float().numpy()
    want = _oracle_conv(x, wt, None, k)
    y = torch.empty((n, h, w, cout), dtype=torch.bfloat16, device=DEV)
    api.op_conv_fwd(api.BF16, _bf16_np(x).to(DEV), _bf16_np(wt).to(DEV), None, cout, k, y)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    # only the final bf16 rounding (2^-9 relative) plus fp32 accumulation
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 4e-3


@pytest.mark.parametrize("shape", [(2, 8, 8, 16, 24, 3), (1, 5, 7, 3, 8, 3), (2, 6, 6, 96, 3, 3), (3, 4, 4, 40, 70, 1)])
def test_simt_conv_f32(shape):
    n, h, w, cin, cout, k = shape
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    wt = rng.standard_normal((cout, k * k, cin)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    want = _oracle_conv(x, wt, b, k)
    y = torch.empty((n, h, w, cout), dtype=torch.float32, device=DEV)
    api.op_conv_fwd(api.F32, torch.from_numpy(x).to(DEV), torch.from_numpy(wt).to(DEV), torch.from_numpy(b).to(DEV),
                    cout, k, y)
    dy = rng.standard_normal((n, h, w, cout)).astype(np.float32)
    dw = torch.empty((cout, k * k, cin), dtype=torch.float32, device=DEV)
    api.op_conv_wgrad(api.F32, torch.from_numpy(x).to(DEV), torch.from_numpy(dy).to(DEV), cout, k, dw)
    torch.cuda.synchronize()
    assert np.linalg.norm(y.cpu().numpy() - want) <= 1e-5 * np.linalg.norm(want)
    xt = torch.from_numpy(x).double().permute(0, 3, 1, 2)
    wv = torch.zeros(cout, cin, k, k, dtype=torch.float64, requires_grad=True)
    (gw,) = torch.autograd.grad((ops.conv2d(xt, wv, None) * torch.from_numpy(dy).double().permute(0, 3, 1, 2)).sum(), wv)
    wantw = gw.permute(0, 2, 3, 1).reshape(cout, k * k, cin).numpy()
    assert np.linalg.norm(dw.cpu().numpy() - wantw) <= 1e-5 * np.linalg.norm(wantw)


@pytest.mark.parametrize("shape", [(2, 128, 128, 96), (3, 37, 70, 8), (1, 16, 16, 4), (2, 33, 65, 12), (1, 9, 130, 128)])
def test_thin_conv_f32_fwd_dgrad_wgrad(shape):
    """G's fp32 output layer (C_out = 3): the three thin kernels against fp64 autograd of
    the plain cross-correlation, ragged tiles at the image edges included."""
    n, h, w, cin = shape
    cout, k = 3, 3
    rng = np.random.default_rng(h * w + cin)
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    wt = rng.standard_normal((cout, k * k, cin)).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    dy = rng.standard_normal((n, h, w, cout)).astype(np.float32)
    xd, wd, bd, dyd = (torch.from_numpy(a).to(DEV) for a in (x, wt, b, dy))
    y = torch.empty((n, h, w, cout), dtype=torch.float32, device=DEV)
    dx = torch.empty((n, h, w, cin), dtype=torch.float32, device=DEV)
    dw = torch.empty((cout, k * k, cin), dtype=torch.float32, device=DEV)
    api.op_conv_fwd(api.F32, xd, wd, bd, cout, k, y)
    api.op_conv_dgrad(api.F32, dyd, wd, cin, k, dx)
    db = torch.empty((cout,), dtype=torch.float32, device=DEV)
    api.op_conv_wgrad(api.F32, xd, dyd, cout, k, dw, db=db)
    torch.cuda.synchronize()
    assert np.allclose(db.cpu().numpy(), dy.reshape(-1, cout).astype(np.float64).sum(0), rtol=1e-5, atol=1e-3)
    xt = torch.from_numpy(x).double().permute(0, 3, 1, 2).requires_grad_(True)
    wv = torch.from_numpy(wt).double().reshape(cout, k, k, cin).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    yt = ops.conv2d(xt, wv, torch.from_numpy(b).double())
    gx, gw = torch.autograd.grad((yt * torch.from_numpy(dy).double().permute(0, 3, 1, 2)).sum(), (xt, wv))
    want_y = yt.detach().permute(0, 2, 3, 1).numpy()
    want_dx = gx.permute(0, 2, 3, 1).numpy()
    want_dw = gw.permute(0, 2, 3, 1).reshape(cout, k * k, cin).numpy()
    for got, want in ((y, want_y), (dx, want_dx), (dw, want_dw)):
        assert np.linalg.norm(got.cpu().numpy() - want) <= 1e-5 * np.linalg.norm(want)


def _bf16_split(a, terms):
    """a (float64 holding fp32 values) -> [t1, t2, ...], t_k = bf16(a - t1 - ... - t_{k-1}) (R36)."""
    out, r = [], np.asarray(a, np.float64)
    for _ in range(terms):
        t = torch.from_numpy(r.astype(np.float32)).to(torch.bfloat16).double().numpy()
        out.append(t)
        r = r - t
    return out


@pytest.mark.parametrize("shape", [(2, 128, 128, 96), (1, 37, 128, 32), (3, 1, 128, 8), (2, 64, 128, 16), (1, 65, 128, 128)])
def test_out_conv_split_tensor_core_fwd_wgrad(shape):
    """G's fp32 output layer as the BF16 engine runs it (R36): the tensor-core conv of the bf16 splits.
    (i) Against the split's own definition, (x1 + x2)(w1 + w2) + x1 w3 in fp64: only the fp32 accumulation
    differs (4e-6: the tensor core's fp32 sums measured 1.4e-6 at the bench shape; leaving out the x1 w3
    term alone would add ~2^-17 = 7.6e-6, an x2 term ~2^-9).  (ii) Against the plain fp64 conv of the fp32 x and w: the split drops x2 w3 and
    leaves |x - x1 - x2| <= 2^-18 |x| per element, so the bar is the thin fp32 kernels' own 1e-5.  The
    backward kernel: dW from (dy1 + dy2)(x1 + x2) and dX from (dy1 + dy2) w1 + dy1 (w2 + w3), each against its
    split definition (4e-6) and the plain fp64 gradient (1e-5).  Shapes (W = 128, one image row per
    tile): the bench layer, a ragged last 32-row strip (H = 37, 65), a one-row image, C = 8 / 16 (one partial
    K chunk) and C = 128 (four chunks)."""
    n, h, w, cin = shape
    rng = np.random.default_rng(h * w + cin + n)
    x = np.maximum(rng.standard_normal((n, h, w, cin)), 0).astype(np.float32)   # a ReLU output, as in G
    wt = (rng.standard_normal((3, 9, cin)) * 0.05).astype(np.float32)
    b = rng.standard_normal(3).astype(np.float32)
    dy = rng.standard_normal((n, h, w, 3)).astype(np.float32)
    xd, wd, bd, dyd = (torch.from_numpy(a).to(DEV) for a in (x, wt, b, dy))
    y = torch.full((n, h, w, 3), float("nan"), dtype=torch.float32, device=DEV)
    dw = torch.full((3, 9, cin), float("nan"), dtype=torch.float32, device=DEV)
    dx = torch.full((n, h, w, cin), float("nan"), dtype=torch.float32, device=DEV)
    api.op_out_conv_split(xd, wd, bd, y, dyd, dw, dx)
    torch.cuda.synchronize()
    x1, x2 = _bf16_split(x, 2)
    w1, w2, w3 = _bf16_split(wt, 3)

    def conv(xa, wa, bias=None):
        xt = torch.from_numpy(xa).permute(0, 3, 1, 2)
        wv = torch.from_numpy(wa).reshape(3, 3, 3, cin).permute(0, 3, 1, 2)
        return ops.conv2d(xt, wv, bias).permute(0, 2, 3, 1).numpy()

    bt = torch.from_numpy(b).double()
    want_split = conv(x1 + x2, w1 + w2, bt) + conv(x1, w3)
    want = conv(x.astype(np.float64), wt.astype(np.float64), bt)
    got = y.cpu().numpy()
    assert np.linalg.norm(got - want_split) <= 4e-6 * np.linalg.norm(want_split)
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want)
    def grads(xa, wa, dya):
        xt = torch.from_numpy(np.asarray(xa, np.float64)).permute(0, 3, 1, 2).requires_grad_(True)
        wv = torch.from_numpy(np.asarray(wa, np.float64)).reshape(3, 3, 3, cin).permute(0, 3, 1, 2).contiguous()
        wv.requires_grad_(True)
        gx, gw = torch.autograd.grad((ops.conv2d(xt, wv, None) * torch.from_numpy(dya).permute(0, 3, 1, 2)).sum(),
                                     (xt, wv))
        return gx.permute(0, 2, 3, 1).numpy(), gw.permute(0, 2, 3, 1).reshape(3, 9, cin).numpy()

    dy1, dy2 = _bf16_split(dy, 2)
    _, want_split_w = grads(x1 + x2, wt, dy1 + dy2)
    want_split_x = grads(x, w1, dy1 + dy2)[0] + grads(x, w2 + w3, dy1)[0]
    want_x, want_w = grads(x, wt, dy.astype(np.float64))
    gw_, gx_ = dw.cpu().numpy(), dx.cpu().numpy()
    assert np.linalg.norm(gw_ - want_split_w) <= 4e-6 * np.linalg.norm(want_split_w)
    assert np.linalg.norm(gw_ - want_w) <= 1e-5 * np.linalg.norm(want_w)
    assert np.linalg.norm(gx_ - want_split_x) <= 4e-6 * np.linalg.norm(want_split_x)
    assert np.linalg.norm(gx_ - want_x) <= 1e-5 * np.linalg.norm(want_x)


UP2_SHAPES = [  # n, h, w, cin, cout  (low-resolution input; output 2h x 2w)
    (2, 4, 4, 64, 128),          # G block 0 geometry: 16-pixel images, 8 images per tile
    (1, 8, 8, 96, 96),
    (2, 16, 16, 192, 96),        # 96-channel tail chunk, odd N tiles
    (1, 64, 64, 192, 96),        # G's last conv1 at quarter batch
    (3, 8, 8, 32, 256),          # several N tiles, odd number of M tiles
    (2, 4, 4, 256, 512),         # wgrad on the CTA-pair kernel (C_in, C_out multiples of 256)
]


def _oracle_up2_conv(x_nhwc, w_otc, b):
    x = torch.from_numpy(x_nhwc).double().permute(0, 3, 1, 2)
    cout, _, cin = w_otc.shape
    w = torch.from_numpy(w_otc).double().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    y = ops.conv2d(ops.up2(x), w, torch.from_numpy(b).double())
    return y.permute(0, 2, 3, 1).numpy()


@pytest.mark.parametrize("shape", UP2_SHAPES)
def test_conv_up2_phase_decomposition_integer_exact(shape):
    """The sub-pixel (phase-decomposed) conv3x3(up2(x)) equals the plain conv on the upsampled
    tensor bit for bit on integer data (folded weights are small exact integers)."""
    n, h, w, cin, cout = shape
    rng = np.random.default_rng(h * 31 + cin)
    x = rng.integers(-2, 3, size=(n, h, w, cin)).astype(np.float32)
    wt = rng.integers(-1, 2, size=(cout, 9, cin)).astype(np.float32)
    b = rng.integers(-3, 4, size=(cout,)).astype(np.float32)
    want = _oracle_up2_conv(x, wt, b).astype(np.float32)
    y = torch.full((n, 2 * h, 2 * w, cout), float("nan"), dtype=torch.bfloat16, device=DEV)
    api.op_conv_up2_fwd(_bf16_np(x).to(DEV), torch.from_numpy(wt).to(DEV), torch.from_numpy(b).to(DEV), cout, y)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    assert np.abs(want).max() < 256   # exact in bf16
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]


def test_conv_up2_random_within_bf16_error():
    n, h, w, cin, cout = 2, 32, 32, 96, 192
    rng = np.random.default_rng(7)
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    wt = (rng.standard_normal((cout, 9, cin)) * 0.05).astype(np.float32)
    b = rng.standard_normal(cout).astype(np.float32)
    xb = _bf16_np(x)
    want = _oracle_up2_conv(xb.float().numpy(), wt, b)
    y = torch.empty((n, 2 * h, 2 * w, cout), dtype=torch.bfloat16, device=DEV)
    api.op_conv_up2_fwd(xb.to(DEV), torch.from_numpy(wt).to(DEV), torch.from_numpy(b).to(DEV), cout, y)
    torch.cuda.synchronize()
    err = np.linalg.norm(y.float().cpu().numpy() - want) / np.linalg.norm(want)
    assert err < 4e-3   # folded weights and the output rounded once each to bf16


@pytest.mark.parametrize("shape", UP2_SHAPES)
def test_conv_up2_dgrad_integer_exact(shape):
    """Input gradient of conv3x3(up2(x)) at low resolution through the phase decomposition (the 2x2
    up2 adjoint included) equals fp64 autograd of the plain definition bit for bit on integers."""
    n, h, w, cin, cout = shape
    rng = np.random.default_rng(h * 37 + cout)
    x = np.zeros((n, h, w, cin), np.float32)
    wt = rng.integers(-1, 2, size=(cout, 9, cin)).astype(np.float32)
    dy = rng.integers(-2, 3, size=(n, 2 * h, 2 * w, cout)).astype(np.float32)
    xt = torch.from_numpy(x).double().permute(0, 3, 1, 2).requires_grad_(True)
    wv = torch.from_numpy(wt).double().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    (gx,) = torch.autograd.grad((ops.conv2d(ops.up2(xt), wv, None) *
                                 torch.from_numpy(dy).double().permute(0, 3, 1, 2)).sum(), xt)
    want = gx.permute(0, 2, 3, 1).numpy().astype(np.float32)
    assert np.abs(want).max() < 2 ** 24
    dx = torch.full((n, h, w, cin), float("nan"), dtype=torch.float32, device=DEV).to(torch.bfloat16)
    api.op_conv_up2_dgrad(_bf16_np(dy).to(DEV), torch.from_numpy(wt).to(DEV), cin, dx)
    torch.cuda.synchronize()
    got = dx.float().cpu().numpy()
    # bf16 output: compare against the bf16 rounding of the exact integer result
    want_b = torch.from_numpy(want).to(torch.bfloat16).float().numpy()
    assert np.array_equal(got, want_b), np.argwhere(got != want_b)[:5]


# D's pooled blocks at small sizes: (n, full-resolution h, w, channels) — conv2 is square (C -> C)
POOL_FWD_SHAPES = [(2, 8, 8, 96), (1, 16, 16, 192), (3, 8, 8, 64), (1, 32, 32, 128)]


@pytest.mark.parametrize("shape", POOL_FWD_SHAPES)
def test_pooled_forward_through_phase_dgrad_kernel_integer_exact(shape):
    """R38: 4 * avgpool2(conv3x3_W(x)) is the phase input-gradient kernel applied to x with the
    flipped, transposed kernel W'[c][t][o] = W[o][8 - t][c] — the launch D's pooled forward makes (the engine
    then scales by 0.25 in the epilogue).  Against fp64 conv + 2x2 sum pooling of the oracle, bf16 rounding of
    the exact integer result, bit for bit."""
    n, H, W, C = shape
    rng = np.random.default_rng(H * 41 + C)
    x = rng.integers(-2, 3, size=(n, H, W, C)).astype(np.float32)
    wt = rng.integers(-1, 2, size=(C, 9, C)).astype(np.float32)   # [o][t][c]
    xt = torch.from_numpy(x).double().permute(0, 3, 1, 2)
    wv = torch.from_numpy(wt).double().reshape(C, 3, 3, C).permute(0, 3, 1, 2)
    want = (torch.nn.functional.avg_pool2d(ops.conv2d(xt, wv, None), 2) * 4.0).permute(0, 2, 3, 1).numpy()
    assert np.abs(want).max() < 2 ** 24
    wflip = np.ascontiguousarray(wt[:, ::-1, :].transpose(2, 1, 0))   # [c][t][o] = W[o][8 - t][c]
    y = torch.full((n, H // 2, W // 2, C), float("nan"), dtype=torch.float32, device=DEV).to(torch.bfloat16)
    api.op_conv_up2_dgrad(_bf16_np(x).to(DEV), torch.from_numpy(wflip).to(DEV), C, y)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    want_b = torch.from_numpy(want.astype(np.float32)).to(torch.bfloat16).float().numpy()
    assert np.array_equal(got, want_b), np.argwhere(got != want_b)[:5]


@pytest.mark.parametrize("shape", UP2_SHAPES)
def test_conv_up2_wgrad_integer_exact(shape):
    """Weight (and bias) gradient of conv3x3(up2(x)) from the low-resolution x through the 16 folded
    phase taps and the unfolding reduction equals fp64 autograd of the plain definition bit for bit."""
    n, h, w, cin, cout = shape
    rng = np.random.default_rng(h * 41 + cin + cout)
    x = rng.integers(-2, 3, size=(n, h, w, cin)).astype(np.float32)
    dy = rng.integers(-2, 3, size=(n, 2 * h, 2 * w, cout)).astype(np.float32)
    xt = torch.from_numpy(x).double().permute(0, 3, 1, 2)
    wv = torch.zeros(cout, cin, 3, 3, dtype=torch.float64, requires_grad=True)
    (gw,) = torch.autograd.grad((ops.conv2d(ops.up2(xt), wv, None) *
                                 torch.from_numpy(dy).double().permute(0, 3, 1, 2)).sum(), wv)
    want = gw.permute(0, 2, 3, 1).reshape(cout, 9, cin).numpy().astype(np.float32)
    assert np.abs(want).max() < 2 ** 24
    dw = torch.full((cout, 9, cin), float("nan"), dtype=torch.float32, device=DEV)
    db = torch.full((cout,), float("nan"), dtype=torch.float32, device=DEV)
    api.op_conv_up2_wgrad(_bf16_np(x).to(DEV), _bf16_np(dy).to(DEV), cout, dw, db=db)
    torch.cuda.synchronize()
    got = dw.cpu().numpy()
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]
    assert np.array_equal(db.cpu().numpy(), dy.reshape(-1, cout).sum(0).astype(np.float32))


POOL_SHAPES = [  # n, h, w, cin, cout, k: D's blocks 1-4 at B = 256 (W = 64 .. 8) and small ragged-batch cases
    (256, 64, 64, 192, 192, 3), (256, 32, 32, 384, 384, 3), (256, 16, 16, 768, 768, 3), (256, 8, 8, 1536, 1536, 3),
    (3, 16, 16, 32, 48, 3), (5, 8, 8, 64, 32, 1),
]


@pytest.mark.parametrize("shape", POOL_SHAPES)
def test_conv_fwd_pool_is_conv_then_avgpool(shape):
    """The fused pooling epilogue (D blocks with a downsample) equals the unfused path bit for bit: conv (+ bias
    + residual, rounded to bf16) through op_conv_fwd_ex, then the 2x2 average in fp32 in the order
    ((t00 + t01) + (t10 + t11)) * 0.25, rounded, and relu of it.  Integer-valued operands keep the conv exact."""
    n, h, w, cin, cout, k = shape
    g = torch.Generator(device=DEV).manual_seed(h * w + cin)
    x = torch.randint(-2, 3, (n, h, w, cin), device=DEV, generator=g).to(torch.bfloat16)
    wt = torch.randint(-1, 2, (cout, k * k, cin), device=DEV, generator=g).to(torch.bfloat16)
    b = torch.randint(-3, 4, (cout,), device=DEV, generator=g).float()
    res = torch.randint(-4, 5, (n, h, w, cout), device=DEV, generator=g).to(torch.bfloat16)
    t = torch.empty(n, h, w, cout, dtype=torch.bfloat16, device=DEV)
    api.op_conv_fwd_ex(x, wt, b, cout, k, t, residual=res, res_mode=1)
    yp = torch.full((n, h // 2, w // 2, cout), float("nan"), dtype=torch.bfloat16, device=DEV)
    yr = torch.full_like(yp, float("nan"))
    api.op_conv_fwd_pool(x, wt, b, cout, k, yp, residual=res, y_relu=yr)
    torch.cuda.synchronize()
    tf = t.float()
    want = (((tf[:, 0::2, 0::2] + tf[:, 0::2, 1::2]) + (tf[:, 1::2, 0::2] + tf[:, 1::2, 1::2])) * 0.25)
    want = want.to(torch.bfloat16)
    assert torch.equal(yp, want)
    assert torch.equal(yr, torch.relu(want.float()).to(torch.bfloat16))
