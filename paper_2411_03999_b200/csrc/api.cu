// C-ABI entry points of libparagan (include/paragan.h).  Argument checks
// happen here, synchronously, before anything is enqueued.
#include <nccl.h>

#include <cstring>
#include <new>

#include "../../include/paragan.h"
#include "common.cuh"
#include "engine.h"
#include "kernels.h"
#include "tc_attn.h"
#include "tc_conv.h"
#include "tc_outconv.h"

struct paragan_ctx {
  pg::EngineBase* eng = nullptr;
};

using namespace pg;

namespace {
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
paragan_status cuda_status(cudaError_t e) { return e == cudaSuccess ? PARAGAN_OK : PARAGAN_ERR_CUDA; }
bool device_ok(int dev) {
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return false;
  return p.major == 10;   // sm_100 family (B200)
}
}  // namespace

extern "C" {

paragan_status paragan_get_unique_id(uint8_t id[128]) {
  if (!id) return PARAGAN_ERR_INVALID_ARG;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return PARAGAN_ERR_NCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return PARAGAN_OK;
}

paragan_status paragan_workspace_size(const paragan_config* cfg, size_t* bytes) {
  if (!cfg || !bytes) return PARAGAN_ERR_INVALID_ARG;
  paragan_status st;
  EngineBase* e = make_engine(cfg, nullptr, &st);
  if (!e) return st;
  *bytes = e->workspace_bytes();
  delete e;
  return PARAGAN_OK;
}

paragan_status paragan_param_count(const paragan_config* cfg, paragan_net net, size_t* n_state, size_t* n_trainable) {
  if (!cfg || (net != PARAGAN_NET_D && net != PARAGAN_NET_G)) return PARAGAN_ERR_INVALID_ARG;
  paragan_status st;
  EngineBase* e = make_engine(cfg, nullptr, &st);
  if (!e) return st;
  e->counts(net, n_state, n_trainable);
  delete e;
  return PARAGAN_OK;
}

paragan_status paragan_init(const paragan_config* cfg, const uint8_t id[128], void* workspace, size_t ws_bytes,
                            void* stream, paragan_ctx** out) {
  if (!cfg || !workspace || !out) return PARAGAN_ERR_INVALID_ARG;
  if (cfg->world_size > 1 && !id) return PARAGAN_ERR_INVALID_ARG;
  *out = nullptr;
  if (cudaSetDevice(cfg->device) != cudaSuccess || !device_ok(cfg->device)) return PARAGAN_ERR_CUDA;
  paragan_status st;
  EngineBase* e = make_engine(cfg, stream, &st);
  if (!e) return st;
  auto* ctx = new (std::nothrow) paragan_ctx;
  if (!ctx) {
    delete e;
    return PARAGAN_ERR_OOM;
  }
  ctx->eng = e;
  st = e->init(id, workspace, ws_bytes);
  *out = ctx;   // returned even on failure so last_error can explain; caller destroys
  return st;
}

paragan_status paragan_init_params(paragan_ctx* ctx, float attn_gamma) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->init_params(attn_gamma);
}
paragan_status paragan_set_params(paragan_ctx* ctx, paragan_net net, const float* host, size_t n) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->set_params(net, host, n);
}
paragan_status paragan_get_params(paragan_ctx* ctx, paragan_net net, float* host, size_t n) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->get_params(net, host, n);
}
paragan_status paragan_get_grads(paragan_ctx* ctx, paragan_net net, float* host, size_t n) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->get_grads(net, host, n);
}

paragan_status paragan_set_grads(paragan_ctx* ctx, paragan_net net, const float* host, size_t n) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->set_grads(net, host, n);
}

paragan_status paragan_layout_pack(const float* src, void* dst, paragan_dtype dt, int32_t n, int32_t c, int32_t h,
                                   int32_t w, int32_t c_pad, void* stream) {
  if (!src || !dst || n < 0 || c < 1 || h < 1 || w < 1 || c_pad < c) return PARAGAN_ERR_INVALID_ARG;
  if (dt == PARAGAN_BF16 && (c_pad % 8 || !aligned16(dst))) return PARAGAN_ERR_INVALID_ARG;
  if (n == 0) return PARAGAN_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dt == PARAGAN_BF16) return cuda_status(layout_pack<bf16>(src, static_cast<bf16*>(dst), n, c, h, w, c_pad, 0, st));
  if (dt == PARAGAN_F32) return cuda_status(layout_pack<float>(src, static_cast<float*>(dst), n, c, h, w, c_pad, 0, st));
  return PARAGAN_ERR_INVALID_ARG;
}
paragan_status paragan_layout_unpack(const void* src, paragan_dtype dt, float* dst, int32_t n, int32_t c, int32_t h,
                                     int32_t w, int32_t c_pad, void* stream) {
  if (!src || !dst || n < 0 || c < 1 || h < 1 || w < 1 || c_pad < c) return PARAGAN_ERR_INVALID_ARG;
  if (n == 0) return PARAGAN_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dt == PARAGAN_BF16)
    return cuda_status(layout_unpack<bf16>(static_cast<const bf16*>(src), dst, n, c, h, w, c_pad, st));
  if (dt == PARAGAN_F32)
    return cuda_status(layout_unpack<float>(static_cast<const float*>(src), dst, n, c, h, w, c_pad, st));
  return PARAGAN_ERR_INVALID_ARG;
}

paragan_status paragan_d_step(paragan_ctx* ctx, const void* real, const int32_t* real_y, const float* z,
                              const int32_t* fake_y, uint32_t flags) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->d_step(real, real_y, z, fake_y, flags);
}
paragan_status paragan_g_step(paragan_ctx* ctx, const float* z, const int32_t* y, uint32_t flags) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->g_step(z, y, flags);
}
paragan_status paragan_d_step_fakes(paragan_ctx* ctx, const void* real, const int32_t* real_y, const void* fakes,
                                    const int32_t* fake_y, uint32_t flags) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->d_step_fakes(real, real_y, fakes, fake_y, flags);
}
paragan_status paragan_generate(paragan_ctx* ctx, const float* z, const int32_t* y, void* dst) {
  if (!ctx || !ctx->eng || !dst || !aligned16(dst)) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->generate(z, y, dst);
}
paragan_status paragan_export_fakes(paragan_ctx* ctx, void* dst) {
  if (!ctx || !ctx->eng || !dst) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->export_fakes(dst);
}
paragan_status paragan_state_size(paragan_ctx* ctx, paragan_net net, size_t* n_floats) {
  if (!ctx || !ctx->eng || !n_floats || (net != PARAGAN_NET_D && net != PARAGAN_NET_G)) return PARAGAN_ERR_INVALID_ARG;
  *n_floats = ctx->eng->state_floats(net);
  return PARAGAN_OK;
}
paragan_status paragan_export_state(paragan_ctx* ctx, paragan_net net, float* dst) {
  if (!ctx || !ctx->eng || !dst || (net != PARAGAN_NET_D && net != PARAGAN_NET_G)) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->export_state(net, dst);
}
paragan_status paragan_import_state(paragan_ctx* ctx, paragan_net net, const float* src) {
  if (!ctx || !ctx->eng || !src || (net != PARAGAN_NET_D && net != PARAGAN_NET_G)) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->import_state(net, src);
}
paragan_status paragan_allreduce_grads(paragan_ctx* ctx, paragan_net net) {
  if (!ctx || !ctx->eng || (net != PARAGAN_NET_D && net != PARAGAN_NET_G)) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->allreduce(net);
}
paragan_status paragan_apply_update(paragan_ctx* ctx, paragan_net net) {
  if (!ctx || !ctx->eng || (net != PARAGAN_NET_D && net != PARAGAN_NET_G)) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->update(net);
}
paragan_status paragan_sync_stats(paragan_ctx* ctx, paragan_stats* out) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->sync_stats(out);
}
paragan_status paragan_stats_async(paragan_ctx* ctx, paragan_stats* out) {
  if (!ctx || !ctx->eng || !out) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->stats_async(out);
}
paragan_status paragan_get_fakes(paragan_ctx* ctx, float* host, size_t n) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->get_fakes(host, n);
}
paragan_status paragan_get_dfake(paragan_ctx* ctx, float* host, size_t n) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->get_dfake(host, n);
}
paragan_status paragan_kernel_launches(const paragan_ctx* ctx, uint64_t* n) {
  if (!ctx || !ctx->eng || !n) return PARAGAN_ERR_INVALID_ARG;
  *n = ctx->eng->launches();
  return PARAGAN_OK;
}
paragan_status paragan_profile(paragan_ctx* ctx, int32_t enable) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->profile(enable);
}
paragan_status paragan_profile_read(paragan_ctx* ctx, int32_t kind, uint64_t* launches, double* ms, double* flops) {
  if (!ctx || !ctx->eng || kind < 0 || kind > 6) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->profile_read(kind, launches, ms, flops);
}
paragan_status paragan_checkpoint_save_async(paragan_ctx* ctx, const char* path) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->checkpoint_save_async(path);
}
paragan_status paragan_checkpoint_wait(paragan_ctx* ctx) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->checkpoint_wait();
}
paragan_status paragan_checkpoint_load(paragan_ctx* ctx, const char* path) {
  if (!ctx || !ctx->eng) return PARAGAN_ERR_INVALID_ARG;
  return ctx->eng->checkpoint_load(path);
}
const char* paragan_last_error(const paragan_ctx* ctx) {
  if (!ctx || !ctx->eng) return "null context";
  return ctx->eng->last_error();
}
paragan_status paragan_destroy(paragan_ctx* ctx) {
  if (!ctx) return PARAGAN_ERR_INVALID_ARG;
  delete ctx->eng;
  delete ctx;
  return PARAGAN_OK;
}

paragan_status paragan_op_conv_fwd(paragan_dtype dt, const void* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                                   const void* wgt, const float* bias, int32_t cout, int32_t ksz, void* y,
                                   void* stream) {
  if (!x || !wgt || !y || n < 1 || h < 1 || w < 1 || cin < 1 || cout < 1 || (ksz != 1 && ksz != 3))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dt == PARAGAN_BF16) {
    if (cin % 8 || !aligned16(x) || !aligned16(wgt) || !aligned16(y) || !tc_geometry_ok(h, w))
      return PARAGAN_ERR_INVALID_ARG;
    TcEpilogue e;
    e.bias = bias;
    e.out = y;
    return cuda_status(tc_conv_fprop(x, n, h, w, cin, wgt, cout, ksz, e, st));
  }
  if (dt == PARAGAN_F32 && cout == 3 && ksz == 3 && cin % 4 == 0 && aligned16(x))   // G's output layer kernel
    return cuda_status(thin_conv_fwd(static_cast<const float*>(x), n, h, w, cin, static_cast<const float*>(wgt), 3,
                                     bias, static_cast<float*>(y), st));
  if (dt == PARAGAN_F32)
    return cuda_status(simt_conv_fwd<float, float, float>(static_cast<const float*>(x), n, h, w, cin,
                                                          static_cast<const float*>(wgt), cout, ksz, bias, nullptr,
                                                          nullptr, 0, static_cast<float*>(y), st));
  return PARAGAN_ERR_INVALID_ARG;
}

paragan_status paragan_op_conv_fwd_ex(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const void* wgt,
                                      const float* bias, int32_t cout, int32_t ksz, const void* residual,
                                      int32_t res_mode, const void* relu_ref, int32_t relu_out, void* y,
                                      void* stream) {
  if (!x || !wgt || !y || n < 1 || h < 1 || w < 1 || cin < 8 || cout < 1 || (ksz != 1 && ksz != 3) || cin % 8 ||
      !aligned16(x) || !aligned16(wgt) || !aligned16(y) || !tc_geometry_ok(h, w) ||
      (residual && (res_mode != 1 && res_mode != 2)) || (residual && !aligned16(residual)) ||
      (res_mode == 2 && (h % 2 || w % 2)) || (relu_ref && !aligned16(relu_ref)))
    return PARAGAN_ERR_INVALID_ARG;
  TcEpilogue e;
  e.bias = bias;
  e.residual = residual;
  e.res_mode = residual ? res_mode : 0;
  e.relu_ref = relu_ref;
  e.relu_out = relu_out ? 1 : 0;
  e.out = y;
  return cuda_status(tc_conv_fprop(x, n, h, w, cin, wgt, cout, ksz, e, static_cast<cudaStream_t>(stream)));
}

paragan_status paragan_op_conv_fwd_pool(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const void* wgt,
                                        const float* bias, int32_t cout, int32_t ksz, const void* residual,
                                        void* y_pool, void* y_relu, void* stream) {
  if (!x || !wgt || !y_pool || n < 1 || h < 2 || w < 2 || cin < 8 || cin % 8 || cout % 16 || (ksz != 1 && ksz != 3) ||
      !aligned16(x) || !aligned16(wgt) || !aligned16(y_pool) || (y_relu && !aligned16(y_relu)) ||
      (residual && !aligned16(residual)) || !tc_geometry_ok(h, w))
    return PARAGAN_ERR_INVALID_ARG;
  TcEpilogue e;
  e.bias = bias;
  e.residual = residual;
  e.res_mode = residual ? 1 : 0;
  e.pool_out = y_pool;
  e.pool_relu = y_relu;
  return cuda_status(tc_conv_fprop(x, n, h, w, cin, wgt, cout, ksz, e, static_cast<cudaStream_t>(stream)));
}

paragan_status paragan_op_out_conv_split(const float* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                                         const float* wgt, const float* bias, float* y, const float* dy, float* dw,
                                         float* dx, void* stream) {
  if (!x || !wgt || !y || n < 1 || h < 1 || w < 1 || !out_conv_tc_ok(h, w, cin) || !aligned16(x) ||
      !aligned16(wgt) || (dw && !dy) || (dx && (!dw || !aligned16(dx))))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long P = (long long)n * h * w;
  const size_t plane_bytes = (size_t)P * 2 * cin * sizeof(uint16_t), ws_bytes = (size_t)96 * 2 * cin * 2;
  const int c16 = (cin + 15) / 16 * 16;
  const size_t wd_bytes = (size_t)c16 * 128 * 2, dx_bytes = dx ? 0 : (size_t)P * cin * 4;
  const size_t scratch_n = out_conv_bwd_scratch_floats(cin);
  char* tmp = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&tmp), plane_bytes + ws_bytes + wd_bytes + dx_bytes + scratch_n * 4,
                      st) != cudaSuccess)
    return PARAGAN_ERR_CUDA;
  bf16* xs = reinterpret_cast<bf16*>(tmp);
  bf16* ws = reinterpret_cast<bf16*>(tmp + plane_bytes);
  bf16* wd = reinterpret_cast<bf16*>(tmp + plane_bytes + ws_bytes);
  float* dxb = dx ? dx : reinterpret_cast<float*>(tmp + plane_bytes + ws_bytes + wd_bytes);
  float* scratch = reinterpret_cast<float*>(tmp + plane_bytes + ws_bytes + wd_bytes + dx_bytes);
  cudaError_t e = split_planes(x, P, cin, xs, st);
  if (e == cudaSuccess) e = split_out_weights(wgt, cin, ws, st);
  if (e == cudaSuccess) e = out_conv_fwd_tc(xs, n, h, w, cin, ws, bias, y, st);
  if (e == cudaSuccess && dw) e = split_out_weights_dgrad(wgt, cin, c16, wd, st);
  if (e == cudaSuccess && dw)
    e = out_conv_bwd_tc(xs, dy, n, h, w, cin, wd, dxb, dw, scratch, scratch_n, st);
  cudaFreeAsync(tmp, st);
  return cuda_status(e);
}

paragan_status paragan_op_conv_wgrad(paragan_dtype dt, const void* x, const void* dy, int32_t n, int32_t h, int32_t w,
                                     int32_t cin, int32_t cout, int32_t ksz, float* dw, float* db, void* stream) {
  if (!x || !dy || !dw || n < 1 || h < 1 || w < 1 || cin < 1 || cout < 1 || (ksz != 1 && ksz != 3))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dt == PARAGAN_BF16) {
    if (cin % 8 || cout % 8 || !aligned16(x) || !aligned16(dy) || !tc_geometry_ok(h, w)) return PARAGAN_ERR_INVALID_ARG;
    const size_t out = (size_t)cout * ksz * ksz * cin;
    const size_t scratch_n = out * 64;
    float* scratch = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), scratch_n * sizeof(float), st) != cudaSuccess)
      return PARAGAN_ERR_CUDA;
    cudaError_t e = tc_conv_wgrad(x, dy, n, h, w, cin, cout, ksz, dw, 0, scratch, scratch_n, st, db);
    cudaFreeAsync(scratch, st);
    return cuda_status(e);
  }
  if (dt != PARAGAN_F32) return PARAGAN_ERR_INVALID_ARG;
  cudaError_t e;
  if (cout == 3 && ksz == 3 && cin % 4 == 0 && cin <= 128 && aligned16(x)) {
    const size_t scratch_n = (size_t)4 * 148 * 27 * cin;
    float* scratch = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), scratch_n * sizeof(float), st) != cudaSuccess)
      return PARAGAN_ERR_CUDA;
    e = thin_conv_wgrad(static_cast<const float*>(x), static_cast<const float*>(dy), n, h, w, cin, 3, dw, scratch,
                        scratch_n, st);
    cudaFreeAsync(scratch, st);
  } else {
    const size_t sn = (size_t)64 * cout * ksz * ksz * cin;
    float* scratch = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), sn * sizeof(float), st) != cudaSuccess)
      return PARAGAN_ERR_CUDA;
    e = simt_conv_wgrad<float, float>(static_cast<const float*>(x), static_cast<const float*>(dy), n, h, w, cin, cout,
                                      ksz, dw, 0, st, scratch, sn);
    cudaFreeAsync(scratch, st);
  }
  if (e == cudaSuccess && db) {
    double* part = nullptr;
    constexpr int kBlocks = 1024;
    if (cudaMallocAsync(reinterpret_cast<void**>(&part), (size_t)kBlocks * cout * sizeof(double), st) != cudaSuccess)
      return PARAGAN_ERR_CUDA;
    e = col_sum<float>(static_cast<const float*>(dy), (long long)n * h * w, cout, part, kBlocks, db, 0, st);
    cudaFreeAsync(part, st);
  }
  return cuda_status(e);
}

paragan_status paragan_op_conv_up2_fwd(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const float* wgt,
                                       const float* bias, int32_t cout, void* y, void* stream) {
  if (!x || !wgt || !y || n < 1 || h < 1 || w < 1 || cin % 8 || cout % 8 || cin < 8 || cout < 8 || !aligned16(x) ||
      !aligned16(y) || !tc_geometry_ok(h, w))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* buf = nullptr;
  const size_t wbytes = (size_t)16 * cout * cin * 2;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), wbytes + 256, st) != cudaSuccess) return PARAGAN_ERR_CUDA;
  float* one = reinterpret_cast<float*>(buf + wbytes);
  cudaError_t e = fill_const(one, 1, 1.0f, st);
  if (e == cudaSuccess) e = fold_up2_weights(wgt, one, cout, cin, reinterpret_cast<bf16*>(buf), st);
  TcEpilogue ep;
  ep.bias = bias;
  ep.out = y;
  if (e == cudaSuccess) e = tc_conv_fprop_up2(x, n, h, w, cin, buf, cout, ep, st);
  cudaFreeAsync(buf, st);
  return cuda_status(e);
}

paragan_status paragan_op_conv_up2_dgrad(const void* dy, int32_t n, int32_t h, int32_t w, int32_t cout,
                                         const float* wgt, int32_t cin, void* dx, void* stream) {
  if (!dy || !wgt || !dx || n < 1 || h < 1 || w < 1 || cin % 8 || cout % 8 || cin < 8 || cout < 8 || !aligned16(dy) ||
      !aligned16(dx) || !tc_geometry_ok(h, w))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* buf = nullptr;
  const size_t wbytes = (size_t)16 * cout * cin * 2;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), wbytes + 256, st) != cudaSuccess) return PARAGAN_ERR_CUDA;
  float* one = reinterpret_cast<float*>(buf + wbytes);
  cudaError_t e = fill_const(one, 1, 1.0f, st);
  if (e == cudaSuccess) e = fold_up2_weights(wgt, one, cout, cin, reinterpret_cast<bf16*>(buf), st, 1);
  TcEpilogue ep;
  ep.out = dx;
  if (e == cudaSuccess) e = tc_conv_dgrad_up2(dy, n, h, w, cout, buf, cin, ep, st);
  cudaFreeAsync(buf, st);
  return cuda_status(e);
}

paragan_status paragan_op_conv_up2_wgrad(const void* x, const void* dy, int32_t n, int32_t h, int32_t w, int32_t cin,
                                         int32_t cout, float* dw, float* db, void* stream) {
  if (!x || !dy || !dw || n < 1 || h < 1 || w < 1 || cin % 8 || cout % 8 || cin < 8 || cout < 8 || !aligned16(x) ||
      !aligned16(dy) || !tc_geometry_ok(h, w))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t scratch_n = (size_t)64 * (16 * (size_t)cout * cin + 4 * (size_t)cout);
  float* scratch = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), scratch_n * sizeof(float), st) != cudaSuccess)
    return PARAGAN_ERR_CUDA;
  cudaError_t e = tc_conv_wgrad_up2(x, dy, n, h, w, cin, cout, dw, scratch, scratch_n, st, db);
  cudaFreeAsync(scratch, st);
  return cuda_status(e);
}

paragan_status paragan_op_conv_dgrad(paragan_dtype dt, const void* dy, int32_t n, int32_t h, int32_t w, int32_t cout,
                                     const void* wgt, int32_t cin, int32_t ksz, void* dx, void* stream) {
  if (dt != PARAGAN_F32 || !dy || !wgt || !dx || n < 1 || h < 1 || w < 1 || cout != 3 || ksz != 3 || cin % 4 ||
      !aligned16(dx))
    return PARAGAN_ERR_INVALID_ARG;
  return cuda_status(thin_conv_dgrad(static_cast<const float*>(dy), n, h, w, cin, static_cast<const float*>(wgt), 3,
                                     static_cast<float*>(dx), static_cast<cudaStream_t>(stream)));
}

paragan_status paragan_op_attn_fwd(const void* qkv, const void* phi, const void* gp, int32_t n, int32_t hw,
                                   int32_t cq, int32_t c2, int32_t ct, void* o, float* o32, float* lse,
                                   void* stream) {
  if (!qkv || !phi || !gp || !o || !lse || n < 1 || hw % 4 || ct < 2 * cq + c2 || ct % 8 ||
      !tc_attn_ok(hw, hw / 4, cq, c2) || !aligned16(qkv) || !aligned16(phi) || !aligned16(gp) || !aligned16(o) ||
      (o32 && !aligned16(o32)))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* gT = nullptr;
  if (cudaMallocAsync(&gT, (size_t)n * (hw / 4) * c2 * 2 + 2 * (size_t)n * sizeof(float) + 256, st) != cudaSuccess)
    return PARAGAN_ERR_CUDA;
  float* phimax = reinterpret_cast<float*>(static_cast<char*>(gT) + (((size_t)n * (hw / 4) * c2 * 2 + 255) & ~size_t(255)));
  float* thetamax = phimax + n;
  const int flat_on = getenv("PARAGAN_ATTN_FLAT") ? atoi(getenv("PARAGAN_ATTN_FLAT")) : 1;   // per call (tests toggle it)
  TcAttnArgs a{};
  a.n = n;
  a.HW = hw;
  a.Q = hw / 4;
  a.Cq = cq;
  a.C2 = c2;
  a.Ct = ct;
  a.qkv = qkv;
  a.phi = phi;
  a.gp = gp;
  a.gT = gT;
  a.o = o;
  a.o32 = o32;
  a.lse = lse;
  a.phimax = phimax;
  a.thetamax = flat_on ? thetamax : nullptr;
  cudaError_t e = attn_transpose(gp, n, a.Q, c2, gT, st);
  if (e == cudaSuccess) e = attn_phimax(phi, n, a.Q, cq, phimax, st);
  if (e == cudaSuccess && flat_on) e = attn_thetamax(qkv, n, hw, cq, ct, thetamax, st);
  if (e == cudaSuccess) e = tc_attn_fwd(a, st);
  cudaFreeAsync(gT, st);
  return cuda_status(e);
}

paragan_status paragan_op_attn_bwd(const void* qkv, const void* phi, const void* gp, const void* dO,
                                   const float* o32, const float* lse, int32_t n, int32_t hw, int32_t cq,
                                   int32_t c2, int32_t ct, void* dqkv, float* dphi, float* dgp, void* stream) {
  if (!qkv || !phi || !gp || !dO || !o32 || !lse || !dqkv || !dphi || !dgp || n < 1 || hw % 4 ||
      ct < 2 * cq + c2 || ct % 8 || !tc_attn_ok(hw, hw / 4, cq, c2) || !aligned16(qkv) || !aligned16(phi) ||
      !aligned16(gp) || !aligned16(dO) || !aligned16(dqkv) || !aligned16(dphi) || !aligned16(dgp))
    return PARAGAN_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nkb = hw / 4 / 128;
  float *D = nullptr, *part = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&D), (size_t)n * hw * sizeof(float), st) != cudaSuccess)
    return PARAGAN_ERR_CUDA;
  if (cudaMallocAsync(reinterpret_cast<void**>(&part), (size_t)nkb * n * hw * cq * sizeof(float), st) !=
      cudaSuccess) {
    cudaFreeAsync(D, st);
    return PARAGAN_ERR_CUDA;
  }
  TcAttnArgs a{};
  a.n = n;
  a.HW = hw;
  a.Q = hw / 4;
  a.Cq = cq;
  a.C2 = c2;
  a.Ct = ct;
  a.qkv = qkv;
  a.phi = phi;
  a.gp = gp;
  a.lse = const_cast<float*>(lse);
  a.dO = dO;
  a.Dr = D;
  a.dgp = dgp;
  a.dphi = dphi;
  a.dth_part = part;
  cudaError_t e = attn_rowdot(dO, o32, (long long)n * hw, c2, D, st);
  if (e == cudaSuccess) e = tc_attn_bwd(a, st);
  if (e == cudaSuccess) e = attn_dtheta_reduce(part, nkb, (long long)n * hw, cq, dqkv, ct, st);
  cudaFreeAsync(part, st);
  cudaFreeAsync(D, st);
  return cuda_status(e);
}

}  // extern "C"
