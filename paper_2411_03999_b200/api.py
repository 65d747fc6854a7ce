"""Thin ctypes binding of libparagan (include/paragan.h) — argument marshalling only.

Every computation happens inside libparagan.so's CUDA kernels; this module only
converts Python/torch arguments to pointers.  There is no CPU fallback: loading
fails loudly when the library is missing, and paragan_init fails without an
sm_100 device.  PyTorch is used for device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libparagan.so")

PARAGAN_ABI_VERSION = 3
F32, BF16 = 0, 1
ARCH_BIGGAN, ARCH_SNDCGAN = 0, 1
NET_D, NET_G = 0, 1
FLAG_NO_ALLREDUCE, FLAG_NO_UPDATE, FLAG_KEEP_DFAKE, FLAG_ASYNC = 1, 2, 4, 8
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "CONFIG", 3: "NONFINITE", 4: "IO", 5: "CUDA", 6: "NCCL", 7: "ORDER", 8: "OOM"}


class Adam(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


OPT_ADAM, OPT_ADABELIEF, OPT_RADAM, OPT_SGD = 0, 1, 2, 3
SCHED_CONSTANT, SCHED_COSINE, SCHED_LINEAR = 0, 1, 2


class Policy(C.Structure):
    """paragan_policy: per-network optimisation policy."""
    _fields_ = [("rule", C.c_int32), ("lars", C.c_int32), ("lars_trust", C.c_float), ("lookahead_k", C.c_int32),
                ("lookahead_alpha", C.c_float), ("warmup_steps", C.c_int32), ("schedule", C.c_int32),
                ("total_steps", C.c_int32), ("clip_norm", C.c_float)]


def make_policy(rule=OPT_ADAM, lars=False, lars_trust=1.0, lookahead_k=0, lookahead_alpha=0.5, warmup_steps=0,
                schedule=SCHED_CONSTANT, total_steps=0, clip_norm=0.0) -> Policy:
    return Policy(rule, 1 if lars else 0, lars_trust, lookahead_k, lookahead_alpha, warmup_steps, schedule,
                  total_steps, clip_norm)


class PrefetchConfig(C.Structure):
    _fields_ = [("batch", C.c_int32), ("channels", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("min_workers", C.c_int32), ("max_workers", C.c_int32), ("min_depth", C.c_int32),
                ("max_depth", C.c_int32), ("window", C.c_int32), ("latency_threshold_ms", C.c_float),
                ("inject_latency_ms", C.c_float)]


class PrefetchStats(C.Structure):
    _fields_ = [("active_workers", C.c_int32), ("depth", C.c_int32), ("queued", C.c_int32),
                ("window_mean_ms", C.c_float), ("batches_read", C.c_int64), ("scale_ups", C.c_int64),
                ("scale_downs", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("resolution", C.c_int32), ("ch", C.c_int32),
                ("n_classes", C.c_int32), ("shared_dim", C.c_int32), ("z_chunk", C.c_int32),
                ("attn_res", C.c_int32), ("local_batch", C.c_int32), ("d_steps_per_g", C.c_int32),
                ("compute", C.c_int32), ("c_pad_image", C.c_int32), ("adam_d", Adam), ("adam_g", Adam),
                ("sn_eps", C.c_float), ("bn_eps", C.c_float), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("device", C.c_int32), ("seed", C.c_uint64), ("arch", C.c_int32), ("policy_d", Policy),
                ("policy_g", Policy), ("grad_comm_bf16", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("d_loss", C.c_float), ("g_loss", C.c_float), ("d_real_mean", C.c_float),
                ("d_fake_mean", C.c_float), ("nonfinite", C.c_int32), ("t_d", C.c_int64), ("t_g", C.c_int64)]


class ParaganError(RuntimeError):
    def __init__(self, fn, status, detail=""):
        super().__init__(f"{fn} -> PARAGAN_ERR_{STATUS.get(status, status)} {detail}".strip())
        self.status = status


_lib = None
SYMBOLS = {
    "paragan_get_unique_id": (C.c_int, [C.c_void_p]),
    "paragan_workspace_size": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_size_t)]),
    "paragan_param_count": (C.c_int, [C.POINTER(Config), C.c_int, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "paragan_init": (C.c_int, [C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                               C.POINTER(C.c_void_p)]),
    "paragan_init_params": (C.c_int, [C.c_void_p, C.c_float]),
    "paragan_set_params": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]),
    "paragan_get_params": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]),
    "paragan_get_grads": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]),
    "paragan_set_grads": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]),
    "paragan_layout_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_void_p]),
    "paragan_layout_unpack": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.c_void_p]),
    "paragan_d_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "paragan_g_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "paragan_d_step_fakes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]),
    "paragan_generate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "paragan_export_fakes": (C.c_int, [C.c_void_p, C.c_void_p]),
    "paragan_export_state": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "paragan_state_size": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_size_t)]),
    "paragan_import_state": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "paragan_allreduce_grads": (C.c_int, [C.c_void_p, C.c_int]),
    "paragan_apply_update": (C.c_int, [C.c_void_p, C.c_int]),
    "paragan_sync_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "paragan_stats_async": (C.c_int, [C.c_void_p, C.c_void_p]),
    "paragan_get_fakes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "paragan_get_dfake": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "paragan_kernel_launches": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "paragan_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "paragan_profile_read": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "paragan_checkpoint_save_async": (C.c_int, [C.c_void_p, C.c_char_p]),
    "paragan_checkpoint_wait": (C.c_int, [C.c_void_p]),
    "paragan_checkpoint_load": (C.c_int, [C.c_void_p, C.c_char_p]),
    "paragan_shard_write": (C.c_int, [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "paragan_prefetch_create": (C.c_int, [C.POINTER(PrefetchConfig), C.POINTER(C.c_char_p), C.c_int32,
                                          C.POINTER(C.c_void_p)]),
    "paragan_prefetch_next": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "paragan_prefetch_get_stats": (C.c_int, [C.c_void_p, C.POINTER(PrefetchStats)]),
    "paragan_prefetch_set_latency": (C.c_int, [C.c_void_p, C.c_float]),
    "paragan_prefetch_destroy": (C.c_int, [C.c_void_p]),
    "paragan_last_error": (C.c_char_p, [C.c_void_p]),
    "paragan_destroy": (C.c_int, [C.c_void_p]),
    "paragan_op_conv_fwd": (C.c_int, [C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                      C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "paragan_op_conv_fwd_ex": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                         C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                         C.c_int32, C.c_void_p, C.c_void_p]),
    "paragan_op_conv_wgrad": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "paragan_op_conv_fwd_pool": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                           C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p]),
    "paragan_op_out_conv_split": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
    "paragan_op_conv_up2_fwd": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                          C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "paragan_op_conv_up2_dgrad": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                            C.c_int32, C.c_void_p, C.c_void_p]),
    "paragan_op_conv_up2_wgrad": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "paragan_op_conv_dgrad": (C.c_int, [C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                        C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "paragan_op_attn_fwd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "paragan_op_attn_bwd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
}


def lib():
    """Load libparagan.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build
            build.build()
        import torch  # noqa: F401  (loads the CUDA runtime / NCCL torch ships, which the .so shares)
        # PARAGAN_LIB: load another build of the library (A/B measurements in one process tree)
        L = C.CDLL(os.environ.get("PARAGAN_LIB", LIB_PATH))
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(fn, status, ctx=None):
    if status != 0:
        detail = ""
        if ctx:
            detail = lib().paragan_last_error(ctx).decode(errors="replace")
        raise ParaganError(fn, status, detail)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_config(resolution=128, ch=96, n_classes=1000, shared_dim=128, z_chunk=20, attn_res=64, local_batch=256,
                d_steps_per_g=1, compute=BF16, c_pad_image=8, adam_d=(2e-4, 0.0, 0.999, None),
                adam_g=(5e-5, 0.0, 0.999, None), sn_eps=1e-12, bn_eps=1e-5, rank=0, world_size=1, device=0,
                seed=0, arch=0, policy_d=None, policy_g=None, grad_comm_bf16=False) -> Config:
    """BigGAN config; Adam eps defaults to 1e-6 under bf16 and 1e-8 in fp32.
    policy_d / policy_g: paragan_policy (make_policy); None = plain Adam."""
    eps = 1e-6 if compute == BF16 else 1e-8
    ad = Adam(adam_d[0], adam_d[1], adam_d[2], adam_d[3] if adam_d[3] is not None else eps)
    ag = Adam(adam_g[0], adam_g[1], adam_g[2], adam_g[3] if adam_g[3] is not None else eps)
    return Config(PARAGAN_ABI_VERSION, resolution, ch, n_classes, shared_dim, z_chunk, attn_res, local_batch,
                  d_steps_per_g, compute, c_pad_image, ad, ag, sn_eps, bn_eps, rank, world_size, device, seed, arch,
                  policy_d or make_policy(), policy_g or make_policy(), 1 if grad_comm_bf16 else 0)


def make_sndcgan_config(ch=32, n_classes=10, local_batch=8, d_steps_per_g=1, **kw) -> Config:
    """Config 1: SN-DCGAN 32x32 (R25), fp32."""
    return make_config(resolution=32, ch=ch, n_classes=n_classes, shared_dim=1, z_chunk=1, attn_res=0,
                       local_batch=local_batch, d_steps_per_g=d_steps_per_g, compute=F32, arch=ARCH_SNDCGAN, **kw)


def dim_z(cfg: Config) -> int:
    if cfg.arch == ARCH_SNDCGAN:
        return 128
    nb = {16: 2, 32: 3, 64: 4, 128: 5, 256: 6, 512: 7}[cfg.resolution]
    return (nb + 1) * cfg.z_chunk


def workspace_size(cfg: Config) -> int:
    n = C.c_size_t()
    _check("paragan_workspace_size", lib().paragan_workspace_size(C.byref(cfg), C.byref(n)))
    return n.value


def param_count(cfg: Config, net: int):
    ns, nt = C.c_size_t(), C.c_size_t()
    _check("paragan_param_count", lib().paragan_param_count(C.byref(cfg), net, C.byref(ns), C.byref(nt)))
    return ns.value, nt.value


def get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check("paragan_get_unique_id", lib().paragan_get_unique_id(buf))
    return bytes(buf)


def layout_pack(src_nchw, dst_nhwc, dtype: int, c_pad: int, stream=None):
    n, c, h, w = src_nchw.shape
    _check("paragan_layout_pack", lib().paragan_layout_pack(_ptr(src_nchw), _ptr(dst_nhwc), dtype, n, c, h, w, c_pad,
                                                            _stream(stream)))


def layout_unpack(src_nhwc, dtype: int, dst_nchw, c_pad: int, stream=None):
    n, c, h, w = dst_nchw.shape
    _check("paragan_layout_unpack", lib().paragan_layout_unpack(_ptr(src_nhwc), dtype, _ptr(dst_nchw), n, c, h, w,
                                                                c_pad, _stream(stream)))


def op_conv_fwd(dtype, x, wgt, bias, cout, ksz, y, stream=None):
    n, h, w, cin = x.shape
    _check("paragan_op_conv_fwd", lib().paragan_op_conv_fwd(dtype, _ptr(x), n, h, w, cin, _ptr(wgt), _ptr(bias), cout,
                                                            ksz, _ptr(y), _stream(stream)))


def op_conv_fwd_ex(x, wgt, bias, cout, ksz, y, residual=None, res_mode=0, relu_ref=None, relu_out=False,
                   stream=None):
    """BF16 tcgen05 conv with the step's fused epilogues (residual add, ReLU-backward mask, ReLU)."""
    n, h, w, cin = x.shape
    _check("paragan_op_conv_fwd_ex", lib().paragan_op_conv_fwd_ex(
        _ptr(x), n, h, w, cin, _ptr(wgt), _ptr(bias), cout, ksz, _ptr(residual), res_mode if residual is not None
        else 0, _ptr(relu_ref), 1 if relu_out else 0, _ptr(y), _stream(stream)))


def op_conv_wgrad(dtype, x, dy, cout, ksz, dw, stream=None, db=None):
    n, h, w, cin = x.shape
    _check("paragan_op_conv_wgrad", lib().paragan_op_conv_wgrad(dtype, _ptr(x), _ptr(dy), n, h, w, cin, cout, ksz,
                                                                _ptr(dw), _ptr(db), _stream(stream)))


def op_conv_fwd_pool(x, wgt, bias, cout, ksz, y_pool, residual=None, y_relu=None, stream=None):
    """y_pool = avgpool2(bf16(conv(x) + bias + residual)) (+ relu copy), the pooling fused in the epilogue."""
    n, h, w, cin = x.shape
    _check("paragan_op_conv_fwd_pool", lib().paragan_op_conv_fwd_pool(_ptr(x), n, h, w, cin, _ptr(wgt), _ptr(bias), cout,
                                                                      ksz, _ptr(residual), _ptr(y_pool), _ptr(y_relu),
                                                                      _stream(stream)))


def op_out_conv_split(x, wgt, bias, y, dy=None, dw=None, dx=None, stream=None):
    """G's output layer as the BF16 engine runs it (R36): x fp32 [n,h,w,cin], wgt fp32 [3,9,cin] -> y fp32
    [n,h,w,3] through the bf16 splits on the tensor cores; with dy/dw (and dx) also the backward."""
    n, h, w, cin = x.shape
    _check("paragan_op_out_conv_split", lib().paragan_op_out_conv_split(_ptr(x), n, h, w, cin, _ptr(wgt), _ptr(bias),
                                                                        _ptr(y), _ptr(dy), _ptr(dw), _ptr(dx),
                                                                        _stream(stream)))


def op_conv_up2_fwd(x, wgt, bias, cout, y, stream=None):
    """y [n,2h,2w,cout] = conv3x3(up2(x)) + bias; x bf16 [n,h,w,cin], wgt fp32 [cout,9,cin]."""
    n, h, w, cin = x.shape
    _check("paragan_op_conv_up2_fwd", lib().paragan_op_conv_up2_fwd(_ptr(x), n, h, w, cin, _ptr(wgt), _ptr(bias), cout,
                                                                    _ptr(y), _stream(stream)))


def op_conv_up2_dgrad(dy, wgt, cin, dx, stream=None):
    """dx [n,h,w,cin] (low resolution) = d/dx of conv3x3(up2(x)) given dy [n,2h,2w,cout]."""
    n, h2, w2, cout = dy.shape
    _check("paragan_op_conv_up2_dgrad", lib().paragan_op_conv_up2_dgrad(_ptr(dy), n, h2 // 2, w2 // 2, cout, _ptr(wgt),
                                                                        cin, _ptr(dx), _stream(stream)))


def op_conv_up2_wgrad(x, dy, cout, dw, db=None, stream=None):
    """dw [cout,9,cin] (+ db) of conv3x3(up2(x)); x bf16 [n,h,w,cin] low resolution, dy [n,2h,2w,cout]."""
    n, h, w, cin = x.shape
    _check("paragan_op_conv_up2_wgrad", lib().paragan_op_conv_up2_wgrad(_ptr(x), _ptr(dy), n, h, w, cin, cout,
                                                                        _ptr(dw), _ptr(db), _stream(stream)))


def op_conv_dgrad(dtype, dy, wgt, cin, ksz, dx, stream=None):
    n, h, w, cout = dy.shape
    _check("paragan_op_conv_dgrad", lib().paragan_op_conv_dgrad(dtype, _ptr(dy), n, h, w, cout, _ptr(wgt), cin, ksz,
                                                                _ptr(dx), _stream(stream)))


def op_attn_fwd(qkv, phi, gp, cq, c2, o, o32, lse, stream=None):
    """qkv [n][hw][ct], phi [n][hw/4][cq], gp [n][hw/4][c2] (bf16) -> o, o32 (or None), lse."""
    n, hw, ct = qkv.shape
    _check("paragan_op_attn_fwd", lib().paragan_op_attn_fwd(_ptr(qkv), _ptr(phi), _ptr(gp), n, hw, cq, c2, ct, _ptr(o),
                                                            _ptr(o32), _ptr(lse), _stream(stream)))


def op_attn_bwd(qkv, phi, gp, dO, o32, lse, cq, c2, dqkv, dphi, dgp, stream=None):
    n, hw, ct = qkv.shape
    _check("paragan_op_attn_bwd", lib().paragan_op_attn_bwd(_ptr(qkv), _ptr(phi), _ptr(gp), _ptr(dO), _ptr(o32),
                                                            _ptr(lse), n, hw, cq, c2, ct, _ptr(dqkv), _ptr(dphi),
                                                            _ptr(dgp), _stream(stream)))


def shard_write(path: str, images, labels):
    """images: float32 numpy [n, c, h, w]; labels: int32 [n]."""
    import numpy as np
    im = np.ascontiguousarray(images, dtype=np.float32)
    lb = np.ascontiguousarray(labels, dtype=np.int32)
    n, c, h, w = im.shape
    _check("paragan_shard_write", lib().paragan_shard_write(path.encode(), im.ctypes.data, lb.ctypes.data, n, c, h, w))


class Prefetcher:
    """Congestion-aware prefetcher (paragan_prefetch_*)."""

    def __init__(self, shards, batch, c, h, w, min_workers=1, max_workers=4, min_depth=2, max_depth=16, window=4,
                 latency_threshold_ms=20.0, inject_latency_ms=0.0):
        self.cfg = PrefetchConfig(batch, c, h, w, min_workers, max_workers, min_depth, max_depth, window,
                                  latency_threshold_ms, inject_latency_ms)
        arr = (C.c_char_p * len(shards))(*[s.encode() for s in shards])
        self.p = C.c_void_p()
        _check("paragan_prefetch_create", lib().paragan_prefetch_create(C.byref(self.cfg), arr, len(shards),
                                                                        C.byref(self.p)))
        self.shape = (batch, c, h, w)

    def next(self, images=None, labels=None):
        """Fills (or allocates) numpy / pinned-torch host buffers with the next batch."""
        import numpy as np
        if images is None:
            images = np.empty(self.shape, np.float32)
            labels = np.empty(self.shape[0], np.int32)
        ip = images.data_ptr() if hasattr(images, "data_ptr") else images.ctypes.data
        lp = labels.data_ptr() if hasattr(labels, "data_ptr") else labels.ctypes.data
        _check("paragan_prefetch_next", lib().paragan_prefetch_next(self.p, C.c_void_p(ip), C.c_void_p(lp)))
        return images, labels

    def set_latency(self, ms):
        _check("paragan_prefetch_set_latency", lib().paragan_prefetch_set_latency(self.p, ms))

    def stats(self) -> PrefetchStats:
        s = PrefetchStats()
        _check("paragan_prefetch_get_stats", lib().paragan_prefetch_get_stats(self.p, C.byref(s)))
        return s

    def close(self):
        if self.p:
            lib().paragan_prefetch_destroy(self.p)
            self.p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One rank's ParaGAN training context (paragan_init .. paragan_destroy)."""

    def __init__(self, cfg: Config, nccl_id: bytes | None = None, stream=None):
        import torch
        self.cfg = cfg
        self.stream = stream if stream is not None else torch.cuda.current_stream(cfg.device)
        nbytes = workspace_size(cfg)
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{cfg.device}")
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self.ctx = C.c_void_p()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        st = lib().paragan_init(C.byref(cfg), idbuf, C.c_void_p(base + off), nbytes, C.c_void_p(self.stream.cuda_stream),
                                C.byref(self.ctx))
        if st != 0:
            msg = lib().paragan_last_error(self.ctx).decode() if self.ctx else ""
            if self.ctx:
                lib().paragan_destroy(self.ctx)
            self.ctx = None
            raise ParaganError("paragan_init", st, msg)
        self.n_state_d, self.n_train_d = param_count(cfg, NET_D)
        self.n_state_g, self.n_train_g = param_count(cfg, NET_G)

    def _n(self, net, state=True):
        if net == NET_D:
            return self.n_state_d if state else self.n_train_d
        return self.n_state_g if state else self.n_train_g

    def init_params(self, attn_gamma=0.0):
        _check("paragan_init_params", lib().paragan_init_params(self.ctx, attn_gamma), self.ctx)

    def set_params(self, net, flat):
        import numpy as np
        a = np.ascontiguousarray(flat, dtype=np.float32)
        _check("paragan_set_params", lib().paragan_set_params(self.ctx, net, a.ctypes.data, a.size), self.ctx)

    def get_params(self, net):
        import numpy as np
        a = np.empty(self._n(net), dtype=np.float32)
        _check("paragan_get_params", lib().paragan_get_params(self.ctx, net, a.ctypes.data, a.size), self.ctx)
        return a

    def get_grads(self, net):
        import numpy as np
        a = np.empty(self._n(net, False), dtype=np.float32)
        _check("paragan_get_grads", lib().paragan_get_grads(self.ctx, net, a.ctypes.data, a.size), self.ctx)
        return a

    def set_grads(self, net, flat):
        """Test hook: this rank's local gradient (canonical layout, n_trainable floats)."""
        import numpy as np
        a = np.ascontiguousarray(flat, dtype=np.float32)
        _check("paragan_set_grads", lib().paragan_set_grads(self.ctx, net, a.ctypes.data, a.size), self.ctx)

    def get_fakes(self):
        import numpy as np
        r = self.cfg.resolution
        a = np.empty((self.cfg.local_batch, 3, r, r), dtype=np.float32)
        _check("paragan_get_fakes", lib().paragan_get_fakes(self.ctx, a.ctypes.data, a.size), self.ctx)
        return a

    def get_dfake(self):
        """dL_G/d(fake images) of the last g_step run with FLAG_KEEP_DFAKE (test hook), NCHW fp32."""
        import numpy as np
        r = self.cfg.resolution
        a = np.empty((self.cfg.local_batch, 3, r, r), dtype=np.float32)
        _check("paragan_get_dfake", lib().paragan_get_dfake(self.ctx, a.ctypes.data, a.size), self.ctx)
        return a

    def d_step(self, real_nhwc, real_y, z, fake_y, flags=0):
        _check("paragan_d_step", lib().paragan_d_step(self.ctx, _ptr(real_nhwc), _ptr(real_y), _ptr(z), _ptr(fake_y),
                                                      flags), self.ctx)

    def g_step(self, z, y, flags=0):
        _check("paragan_g_step", lib().paragan_g_step(self.ctx, _ptr(z), _ptr(y), flags), self.ctx)

    def d_step_fakes(self, real_nhwc, real_y, fakes_nhwc, fake_y, flags=0):
        _check("paragan_d_step_fakes", lib().paragan_d_step_fakes(self.ctx, _ptr(real_nhwc), _ptr(real_y),
                                                                  _ptr(fakes_nhwc), _ptr(fake_y), flags), self.ctx)

    def generate(self, z, y, dst_nhwc):
        _check("paragan_generate", lib().paragan_generate(self.ctx, _ptr(z), _ptr(y), _ptr(dst_nhwc)), self.ctx)

    def export_fakes(self, dst_nhwc):
        _check("paragan_export_fakes", lib().paragan_export_fakes(self.ctx, _ptr(dst_nhwc)), self.ctx)

    def checkpoint_save_async(self, path: str):
        _check("paragan_checkpoint_save_async", lib().paragan_checkpoint_save_async(self.ctx, path.encode()), self.ctx)

    def checkpoint_wait(self):
        _check("paragan_checkpoint_wait", lib().paragan_checkpoint_wait(self.ctx), self.ctx)

    def checkpoint_load(self, path: str):
        _check("paragan_checkpoint_load", lib().paragan_checkpoint_load(self.ctx, path.encode()), self.ctx)

    def state_size(self, net) -> int:
        n = C.c_size_t()
        _check("paragan_state_size", lib().paragan_state_size(self.ctx, net, C.byref(n)), self.ctx)
        return n.value

    def export_state(self, net, dst):
        _check("paragan_export_state", lib().paragan_export_state(self.ctx, net, _ptr(dst)), self.ctx)

    def import_state(self, net, src):
        _check("paragan_import_state", lib().paragan_import_state(self.ctx, net, _ptr(src)), self.ctx)

    def allreduce_grads(self, net):
        _check("paragan_allreduce_grads", lib().paragan_allreduce_grads(self.ctx, net), self.ctx)

    def apply_update(self, net):
        _check("paragan_apply_update", lib().paragan_apply_update(self.ctx, net), self.ctx)

    def sync_stats(self, raise_nonfinite=True):
        s = Stats()
        st = lib().paragan_sync_stats(self.ctx, C.byref(s))
        if st == 3 and not raise_nonfinite:
            return s
        _check("paragan_sync_stats", st, self.ctx)
        return s

    def stats_async(self, buf):
        """Enqueue the stats' device-to-host copy into `buf` (a page-locked uint8 torch tensor of at least
        ctypes.sizeof(Stats) bytes) on the context's stream, without synchronising; read_stats(buf) once the
        stream has passed this point."""
        _check("paragan_stats_async", lib().paragan_stats_async(self.ctx, C.c_void_p(buf.data_ptr())), self.ctx)

    @staticmethod
    def read_stats(buf) -> Stats:
        return Stats.from_buffer_copy(C.string_at(buf.data_ptr(), C.sizeof(Stats)))

    def kernel_launches(self) -> int:
        n = C.c_uint64()
        _check("paragan_kernel_launches", lib().paragan_kernel_launches(self.ctx, C.byref(n)), self.ctx)
        return n.value

    def profile(self, enable: bool):
        _check("paragan_profile", lib().paragan_profile(self.ctx, 1 if enable else 0), self.ctx)

    def profile_read(self, kind: int):
        n, ms, fl = C.c_uint64(), C.c_double(), C.c_double()
        _check("paragan_profile_read", lib().paragan_profile_read(self.ctx, kind, C.byref(n), C.byref(ms),
                                                                  C.byref(fl)), self.ctx)
        return n.value, ms.value, fl.value

    def close(self):
        if self.ctx:
            lib().paragan_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
