"""Out-of-bounds write checks of our own (compute-sanitizer is closed on this GPU pool): every output
buffer gets a guard band of sentinel values before and after the region the call may write, on shapes
with ragged tails (M not a multiple of the 128-pixel tile, C_out not a multiple of the N tile, partial
CTA pairs, halo tiles at image borders); the guard bands must come back untouched and the written region
must hold no sentinel."""
import numpy as np
import pytest
import torch

from paper_2411_03999_b200 import api

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GUARD = 4096


def _guarded(shape, dtype, fill):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), fill, dtype=dtype, device=DEV)
    return buf, buf[GUARD:GUARD + n].view(shape)


def _check(buf, fill, n):
    g = torch.cat([buf[:GUARD], buf[GUARD + n:]])
    assert bool((g == fill).all()), "guard band overwritten"


SHAPES = [  # n, h, w, cin, cout, k
    (1, 4, 4, 8, 32, 3), (3, 8, 8, 32, 48, 3), (5, 8, 8, 64, 128, 3), (2, 2, 128, 192, 96, 3),
    (1, 3, 256, 64, 192, 3), (2, 64, 64, 192, 24, 1), (2, 16, 32, 384, 136, 3), (3, 4, 8, 512, 256, 1),
]


@pytest.mark.parametrize("shape", SHAPES)
def test_conv_fprop_and_wgrad_write_only_their_outputs(shape):
    n, h, w, cin, cout, k = shape
    x = torch.randint(-2, 3, (n, h, w, cin), device=DEV).to(torch.bfloat16)
    wt = torch.randint(-1, 2, (cout, k * k, cin), device=DEV).to(torch.bfloat16)
    fill = -12345.0
    ybuf, y = _guarded((n, h, w, cout), torch.bfloat16, fill)
    api.op_conv_fwd(api.BF16, x, wt, None, cout, k, y)
    torch.cuda.synchronize()
    _check(ybuf, fill, y.numel())
    assert not bool((y == fill).any())
    if cout % 8 == 0:
        dy = torch.randint(-1, 2, (n, h, w, cout), device=DEV).to(torch.bfloat16)
        wbuf, dw = _guarded((cout, k * k, cin), torch.float32, fill)
        bbuf, db = _guarded((cout,), torch.float32, fill)
        api.op_conv_wgrad(api.BF16, x, dy, cout, k, dw, db=db)
        torch.cuda.synchronize()
        _check(wbuf, fill, dw.numel())
        _check(bbuf, fill, db.numel())
        assert not bool((dw == fill).any())


@pytest.mark.parametrize("shape", [(2, 4, 4, 64, 128), (3, 8, 8, 32, 256), (1, 64, 64, 192, 96)])
def test_up2_convs_write_only_their_outputs(shape):
    n, h, w, cin, cout = shape
    x = torch.randint(-2, 3, (n, h, w, cin), device=DEV).to(torch.bfloat16)
    wt = torch.randint(-1, 2, (cout, 9, cin), device=DEV).float()
    fill = -12345.0
    ybuf, y = _guarded((n, 2 * h, 2 * w, cout), torch.bfloat16, fill)
    api.op_conv_up2_fwd(x, wt, None, cout, y)
    dy = torch.randint(-1, 2, (n, 2 * h, 2 * w, cout), device=DEV).to(torch.bfloat16)
    dxbuf, dx = _guarded((n, h, w, cin), torch.bfloat16, fill)
    api.op_conv_up2_dgrad(dy, wt, cin, dx)
    wbuf, dw = _guarded((cout, 9, cin), torch.float32, fill)
    api.op_conv_up2_wgrad(x, dy, cout, dw)
    torch.cuda.synchronize()
    for b, t in ((ybuf, y), (dxbuf, dx), (wbuf, dw)):
        _check(b, fill, t.numel())
        assert not bool((t == fill).any())


def test_attention_writes_only_its_outputs():
    n, hw, cq, c2, ct = 2, 1024, 16, 48, 80
    q = hw // 4
    g = torch.Generator(device="cpu").manual_seed(3)
    qkv = torch.randn(n, hw, ct, generator=g).to(torch.bfloat16).to(DEV)
    phi = torch.randn(n, q, cq, generator=g).to(torch.bfloat16).to(DEV)
    gp = torch.randn(n, q, c2, generator=g).to(torch.bfloat16).to(DEV)
    dO = torch.randn(n, hw, c2, generator=g).to(torch.bfloat16).to(DEV)
    fill = -12345.0
    obuf, o = _guarded((n, hw, c2), torch.bfloat16, fill)
    o32buf, o32 = _guarded((n, hw, c2), torch.float32, fill)
    lbuf, lse = _guarded((n, hw), torch.float32, fill)
    api.op_attn_fwd(qkv, phi, gp, cq, c2, o, o32, lse)
    dqbuf, dqkv = _guarded((n, hw, ct), torch.bfloat16, fill)
    dpbuf, dphi = _guarded((n, q, cq), torch.float32, fill)
    dgbuf, dgp = _guarded((n, q, c2), torch.float32, fill)
    api.op_attn_bwd(qkv, phi, gp, dO, o32, lse, cq, c2, dqkv, dphi, dgp)
    torch.cuda.synchronize()
    for b, t in ((obuf, o), (o32buf, o32), (lbuf, lse), (dqbuf, dqkv), (dpbuf, dphi), (dgbuf, dgp)):
        _check(b, fill, t.numel())
    assert not bool((dqkv[..., :cq] == fill).any()) and bool((dqkv[..., cq:] == fill).all())


@pytest.mark.parametrize("shape", [(2, 128, 128, 96), (3, 37, 70, 8)])
def test_thin_fp32_layer_writes_only_its_outputs(shape):
    n, h, w, cin = shape
    x = torch.randn(n, h, w, cin, device=DEV)
    wt = torch.randn(3, 9, cin, device=DEV)
    dy = torch.randn(n, h, w, 3, device=DEV)
    fill = -12345.0
    ybuf, y = _guarded((n, h, w, 3), torch.float32, fill)
    dxbuf, dx = _guarded((n, h, w, cin), torch.float32, fill)
    wbuf, dw = _guarded((3, 9, cin), torch.float32, fill)
    api.op_conv_fwd(api.F32, x, wt, None, 3, 3, y)
    api.op_conv_dgrad(api.F32, dy, wt, cin, 3, dx)
    api.op_conv_wgrad(api.F32, x, dy, 3, 3, dw)
    torch.cuda.synchronize()
    for b, t in ((ybuf, y), (dxbuf, dx), (wbuf, dw)):
        _check(b, fill, t.numel())
        assert not bool((t == fill).any())


@pytest.mark.parametrize("shape", [(2, 128, 128, 96), (3, 5, 128, 16)])
def test_out_conv_split_writes_only_its_outputs(shape):
    """The tensor-core output layer (R36): y [M][3] fp32 written row by row from the 16-column accumulator."""
    n, h, w, cin = shape
    x = torch.randn(n, h, w, cin, device=DEV)
    wt = torch.randn(3, 9, cin, device=DEV)
    dy = torch.randn(n, h, w, 3, device=DEV)
    fill = -12345.0
    ybuf, y = _guarded((n, h, w, 3), torch.float32, fill)
    wbuf, dw = _guarded((3, 9, cin), torch.float32, fill)
    dxbuf, dx = _guarded((n, h, w, cin), torch.float32, fill)
    api.op_out_conv_split(x, wt, None, y, dy, dw, dx)
    torch.cuda.synchronize()
    for b, t in ((ybuf, y), (wbuf, dw), (dxbuf, dx)):
        _check(b, fill, t.numel())
        assert not bool((t == fill).any())
