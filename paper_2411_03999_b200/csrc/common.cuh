// Shared device/host helpers of libparagan (product path only; the oracle
// shares nothing with this file).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

namespace pg {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------
// error plumbing: every launcher returns cudaError_t; the engine records the
// first failure as a sticky error (include/paragan.h "Errors").
// ---------------------------------------------------------------------------
#define PG_CUDA(x)                                                            \
  do {                                                                        \
    cudaError_t e__ = (x);                                                    \
    if (e__ != cudaSuccess) return e__;                                       \
  } while (0)

#define PG_LAUNCH_CHECK() PG_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// element conversion (storage type T is float or bf16; math is fp32)
// ---------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

constexpr int kNumSMs = 148;  // B200

// SMs the persistent grids may occupy (kNumSMs, fewer while a gradient all-reduce overlaps compute, so the
// NCCL kernels find free SMs instead of waiting behind one-CTA-per-SM grids; engine.cu sets it)
extern int g_sm_cap;
inline int sm_cap() { return g_sm_cap; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is per device,
// so a process driving two GPUs sets it on each
template <auto K>
cudaError_t set_smem_once(int bytes) {
  static unsigned long long done = 0;   // bit per device; host-side, one host thread per context
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done |= bit;
  return e;
}

}  // namespace pg
