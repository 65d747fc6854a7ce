// Asymmetric optimisation policy kernels (see optim.h).  Rules follow the papers P:293 cites:
// AdaBelief (Zhuang et al. 2020, Alg. 2), RAdam (Liu et al. 2020, Alg. 2; rectified when rho_t > 5),
// LARS (You et al. 2017, per-tensor trust ratio of the inner step), Lookahead (Zhang et al. 2019,
// Alg. 1); R26-R30.  One thread per 4 consecutive elements of a chunk (16-byte accesses);
// one block per chunk, so every chunk-level sum has a fixed order.
#include <cuda_runtime.h>

#include "common.cuh"
#include "optim.h"

namespace pg {
namespace {

constexpr int kThreads = 256;

__device__ double block_sum_d(double v, double* sh) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < (int)(blockDim.x >> 5) ? sh[l] : 0.0;
    r = warp_sum_d(r);
  }
  __syncthreads();
  return r;   // valid in thread 0
}

// learning rate of update t (1-based): lr * warmup(t) * schedule(t)
__device__ float lr_at(const OptRule& r, double t) {
  double f = 1.0;
  if (r.warmup > 0) f *= fmin(1.0, t / r.warmup);
  if (r.total > 0) {
    if (r.schedule == 1) f *= 0.5 * (1.0 + cos(3.14159265358979323846 * fmin(t, (double)r.total) / r.total));
    else if (r.schedule == 2) f *= fmax(0.0, 1.0 - t / r.total);
  }
  return (float)(r.lr * f);
}

struct RuleScalars {
  float bc1, bc2, rect;   // 1 - b1^t, 1 - b2^t, RAdam rectification (0 = un-adapted step)
};

__device__ RuleScalars rule_scalars(const OptRule& r, double t) {
  RuleScalars s;
  s.bc1 = (float)(1.0 - pow((double)r.b1, t));
  s.bc2 = (float)(1.0 - pow((double)r.b2, t));
  s.rect = 0.0f;
  if (r.rule == 2) {
    const double b2 = r.b2, b2t = pow(b2, t);
    const double rinf = 2.0 / (1.0 - b2) - 1.0;
    const double rt = rinf - 2.0 * t * b2t / (1.0 - b2t);
    if (rt > 5.0) s.rect = (float)sqrt((rt - 4.0) * (rt - 2.0) * rinf / ((rinf - 4.0) * (rinf - 2.0) * rt));
  }
  return s;
}

// the rule's step direction u for one element (m, v updated in place)
__device__ __forceinline__ float direction(const OptRule& r, const RuleScalars& s, float g, float& m, float& v) {
  switch (r.rule) {
    case 3:   // SGD with heavy-ball momentum
      m = r.b1 * m + g;
      return m;
    case 1: {   // AdaBelief: s tracks (g - m_t)^2, eps inside and outside
      m = r.b1 * m + (1.0f - r.b1) * g;
      const float d = g - m;
      v = r.b2 * v + (1.0f - r.b2) * d * d + r.eps;
      return (m / s.bc1) / (sqrtf(v / s.bc2) + r.eps);
    }
    case 2: {   // RAdam
      m = r.b1 * m + (1.0f - r.b1) * g;
      v = r.b2 * v + (1.0f - r.b2) * g * g;
      const float mh = m / s.bc1;
      if (s.rect > 0.0f) return s.rect * mh * sqrtf(s.bc2) / (sqrtf(v) + r.eps);
      return mh;
    }
    default: {   // Adam
      m = r.b1 * m + (1.0f - r.b1) * g;
      v = r.b2 * v + (1.0f - r.b2) * g * g;
      return (m / s.bc1) / (sqrtf(v / s.bc2) + r.eps);
    }
  }
}

__global__ void k_opt_sumsq(const float* __restrict__ g, const OptChunk* __restrict__ chunks, float gscale,
                            double* __restrict__ part) {
  __shared__ double sh[32];
  const OptChunk c = chunks[blockIdx.x];
  double a = 0.0;
  for (int i = threadIdx.x; i < c.len; i += blockDim.x) {
    const double x = (double)(g[c.start + i] * gscale);
    a += x * x;
  }
  a = block_sum_d(a, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = a;
}

__global__ void k_opt_clip_finalize(const double* __restrict__ part, int n, float clip, float* scale, int* flag) {
  __shared__ double sh[32];
  double a = 0.0;
  // fixed order: each thread a strided slice in index order, then the block tree
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += part[i];
  a = block_sum_d(a, sh);
  if (threadIdx.x == 0) {
    if (!isfinite(a)) {
      atomicOr(flag, 1);
      *scale = 1.0f;
    } else {
      const double nrm = sqrt(a);
      *scale = nrm > clip ? (float)(clip / nrm) : 1.0f;
    }
  }
}

template <bool LARS>
__global__ void k_opt_update(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, float* __restrict__ u, const OptChunk* __restrict__ chunks,
                             OptRule r, const long long* __restrict__ t_dev, const float* __restrict__ clip_scale,
                             const int* __restrict__ flag, double* __restrict__ wpart, double* __restrict__ upart) {
  __shared__ double sh[32];
  if (*flag) return;
  const double t = (double)(*t_dev + 1);
  const RuleScalars s = rule_scalars(r, t);
  const float lr = lr_at(r, t);
  const float gs = r.gscale * (clip_scale ? *clip_scale : 1.0f);
  const OptChunk c = chunks[blockIdx.x];
  double aw = 0.0, au = 0.0;
  for (int i = threadIdx.x; i < c.len; i += blockDim.x) {
    const long long k = c.start + i;
    float mi = m[k], vi = v[k];
    const float d = direction(r, s, g[k] * gs, mi, vi);
    m[k] = mi;
    v[k] = vi;
    if (LARS) {
      const float wi = w[k];
      u[k] = d;
      aw += (double)wi * wi;
      au += (double)d * d;
    } else {
      w[k] -= lr * d;
    }
  }
  if (LARS) {
    aw = block_sum_d(aw, sh);
    au = block_sum_d(au, sh);
    if (threadIdx.x == 0) {
      wpart[blockIdx.x] = aw;
      upart[blockIdx.x] = au;
    }
  }
}

__global__ void k_opt_lars_apply(float* __restrict__ w, const float* __restrict__ u, const OptChunk* __restrict__ chunks,
                                 OptRule r, const long long* __restrict__ t_dev, const double* __restrict__ wpart,
                                 const double* __restrict__ upart, const int* __restrict__ flag) {
  __shared__ float lam;
  if (*flag) return;
  const OptChunk c = chunks[blockIdx.x];
  if (threadIdx.x == 0) {
    double aw = 0.0, au = 0.0;   // the tensor's chunks in order (identical in every block of the tensor)
    for (int j = 0; j < c.count; ++j) {
      aw += wpart[c.first + j];
      au += upart[c.first + j];
    }
    lam = (aw > 0.0 && au > 0.0) ? (float)(r.trust * sqrt(aw) / sqrt(au)) : 1.0f;
  }
  __syncthreads();
  const float lr = lr_at(r, (double)(*t_dev + 1)) * lam;
  for (int i = threadIdx.x; i < c.len; i += blockDim.x) w[c.start + i] -= lr * u[c.start + i];
}

__global__ void k_opt_lookahead(float* __restrict__ w, float* __restrict__ slow, long long n, int k, float alpha,
                                const long long* __restrict__ t_dev, const int* __restrict__ flag) {
  if (*flag || (*t_dev % k) != 0) return;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float s = slow[i] + alpha * (w[i] - slow[i]);
    slow[i] = s;
    w[i] = s;
  }
}

}  // namespace

cudaError_t opt_sumsq(const float* g, const OptChunk* chunks, int n_chunks, float gscale, double* part,
                      cudaStream_t st) {
  k_opt_sumsq<<<n_chunks, kThreads, 0, st>>>(g, chunks, gscale, part);
  return cudaGetLastError();
}
cudaError_t opt_clip_finalize(const double* part, int n_chunks, float clip, float* clip_scale, int* flag,
                              cudaStream_t st) {
  k_opt_clip_finalize<<<1, 1024, 0, st>>>(part, n_chunks, clip, clip_scale, flag);
  return cudaGetLastError();
}
cudaError_t opt_update(float* w, const float* g, float* m, float* v, float* u, const OptChunk* chunks, int n_chunks,
                       const OptRule& r, const long long* t_dev, const float* clip_scale, const int* flag,
                       double* wpart, double* upart, cudaStream_t st) {
  if (r.lars)
    k_opt_update<true><<<n_chunks, kThreads, 0, st>>>(w, g, m, v, u, chunks, r, t_dev, clip_scale, flag, wpart, upart);
  else
    k_opt_update<false><<<n_chunks, kThreads, 0, st>>>(w, g, m, v, u, chunks, r, t_dev, clip_scale, flag, wpart,
                                                        upart);
  return cudaGetLastError();
}
cudaError_t opt_lars_apply(float* w, const float* u, const OptChunk* chunks, int n_chunks, const OptRule& r,
                           const long long* t_dev, const double* wpart, const double* upart, const int* flag,
                           cudaStream_t st) {
  k_opt_lars_apply<<<n_chunks, kThreads, 0, st>>>(w, u, chunks, r, t_dev, wpart, upart, flag);
  return cudaGetLastError();
}
cudaError_t opt_lookahead(float* w, float* slow, long long n, int k, float alpha, const long long* t_dev,
                          const int* flag, cudaStream_t st) {
  long long b = (n + kThreads - 1) / kThreads;
  if (b > (long long)kNumSMs * 8) b = (long long)kNumSMs * 8;
  k_opt_lookahead<<<(int)b, kThreads, 0, st>>>(w, slow, n, k, alpha, t_dev, flag);
  return cudaGetLastError();
}

}  // namespace pg
