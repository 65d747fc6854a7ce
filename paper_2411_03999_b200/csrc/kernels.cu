// Memory-bound and SIMT kernels of libparagan (see kernels.h for contracts).
// Access pattern rules (B200): NHWC activations are read/written with one
// thread per 8-channel group of a pixel (16-byte vectors for bf16), grids are
// sized in multiples of the 148 SMs, reductions are warp-shuffle + shared
// memory with fp64 cross-block accumulation in a fixed order (deterministic).
#include <type_traits>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "../../include/paragan.h"
#include "tc_ptx.cuh"

namespace pg {

int g_sm_cap = kNumSMs;

namespace {

inline int grid_for(long long n, int threads, int max_waves = 8) {
  long long b = (n + threads - 1) / threads;
  long long cap = (long long)kNumSMs * max_waves;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

template <typename T> struct Vec8;
template <> struct Vec8<float> {
  __device__ static void load(const float* p, float (&v)[8]) {
    float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ static void store(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <> struct Vec8<bf16> {
  __device__ static void load(const bf16* p, float (&v)[8]) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  }
  __device__ static void store(bf16* p, const float (&v)[8]) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};

// ===================================================================== layout
template <typename TD>
__global__ void k_pack(const float* __restrict__ src, TD* __restrict__ dst, int n, int c, int h, int w, int cp) {
  const long long total = (long long)n * h * w * cp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % cp);
    long long p = i / cp;
    const int x = (int)(p % w);
    p /= w;
    const int y = (int)(p % h);
    const int b = (int)(p / h);
    float v = 0.0f;
    if (k < c) v = src[(((long long)b * c + k) * h + y) * w + x];
    dst[i] = from_f<TD>(v);
  }
}
template <typename TS>
__global__ void k_unpack(const TS* __restrict__ src, float* __restrict__ dst, int n, int c, int h, int w, int cp) {
  const long long total = (long long)n * c * h * w;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % w);
    long long p = i / w;
    const int y = (int)(p % h);
    p /= h;
    const int k = (int)(p % c);
    const int b = (int)(p / c);
    dst[i] = to_f<TS>(src[(((long long)b * h + y) * w + x) * cp + k]);
  }
}

// ===================================================================== small GEMM
// 64x64 tile, 256 threads, 4x4 per thread, K chunk 16
template <typename TI, typename TC>
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, const TI* __restrict__ A, long long sab,
                                              long long sam, long long sak, const TI* __restrict__ B, long long sbb,
                                              long long sbn, long long sbk, TC* __restrict__ C, long long scb,
                                              long long ldc, float beta, const float* __restrict__ bias) {
  __shared__ __align__(16) float As[16][68];
  __shared__ __align__(16) float Bs[16][68];
  const int b = blockIdx.z;
  A += b * sab;
  B += b * sbb;
  C += b * scb;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = tid; i < 1024; i += 256) {
      int mm, kk;
      if (sak == 1) { mm = i >> 4; kk = i & 15; } else { kk = i >> 6; mm = i & 63; }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? to_f<TI>(A[m * sam + k * sak]) : 0.0f;
      int nn, kb;
      if (sbk == 1) { nn = i >> 4; kb = i & 15; } else { kb = i >> 6; nn = i & 63; }
      const int n = n0 + nn, k2 = k0 + kb;
      Bs[kb][nn] = (n < N && k2 < K) ? to_f<TI>(B[n * sbn + k2 * sbk]) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (bias) v += bias[n];
      TC* cp = C + m * ldc + n;
      if (beta != 0.0f) v += beta * to_f<TC>(*cp);
      *cp = from_f<TC>(v);
    }
  }
}

// ===================================================================== grouped fp32 GEMM
// 64x64 tile, 256 threads (4x4 each), K chunks of 16 double-buffered through registers
__global__ void __launch_bounds__(256) k_gemm_grouped(const GemmProblem* __restrict__ probs, int nprob) {
  // rows padded to 68 floats: 16-byte aligned, so the inner loop reads each thread's 4 A and 4 B
  // values as one float4 each (2 shared loads per 16 FMAs instead of 8)
  __shared__ __align__(16) float As[2][16][68];
  __shared__ __align__(16) float Bs[2][16][68];
  const int bid = blockIdx.x;
  int pi = 0;
  while (pi + 1 < nprob && probs[pi + 1].tile0 <= bid) ++pi;
  const GemmProblem& P = probs[pi];
  const int tiles_n = (P.N + 63) / 64;
  const int lt = bid - P.tile0;
  const int m0 = (lt / tiles_n) * 64, n0 = (lt % tiles_n) * 64;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4] = {};
  // flatten (segment, k chunk) into one chunk sequence
  int nch = 0;
  for (int s = 0; s < P.nseg; ++s) nch += (P.seg[s].K + 15) / 16;
  float ra[4], rb[4];
  auto load = [&](int ch) {
    int s = 0, c = ch;
    while (c >= (P.seg[s].K + 15) / 16) { c -= (P.seg[s].K + 15) / 16; ++s; }
    const GemmSeg& G = P.seg[s];
    const int k0 = c * 16;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = tid + r * 256;
      int mm, kk;
      if (G.sak == 1) { mm = i >> 4; kk = i & 15; } else { kk = i >> 6; mm = i & 63; }
      const int m = m0 + mm, k = k0 + kk;
      ra[r] = (m < P.M && k < G.K) ? G.A[m * G.sam + k * G.sak] : 0.0f;
      int nn, kb;
      if (G.sbk == 1) { nn = i >> 4; kb = i & 15; } else { kb = i >> 6; nn = i & 63; }
      const int n = n0 + nn, k2 = k0 + kb;
      rb[r] = (n < P.N && k2 < G.K) ? G.B[n * G.sbn + k2 * G.sbk] : 0.0f;
    }
  };
  auto store = [&](int ch, int buf) {
    int s = 0, c = ch;
    while (c >= (P.seg[s].K + 15) / 16) { c -= (P.seg[s].K + 15) / 16; ++s; }
    const GemmSeg& G = P.seg[s];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = tid + r * 256;
      int mm, kk;
      if (G.sak == 1) { mm = i >> 4; kk = i & 15; } else { kk = i >> 6; mm = i & 63; }
      As[buf][kk][mm] = ra[r];
      int nn, kb;
      if (G.sbk == 1) { nn = i >> 4; kb = i & 15; } else { kb = i >> 6; nn = i & 63; }
      Bs[buf][kb][nn] = rb[r];
    }
  };
  if (nch > 0) {
    load(0);
    store(0, 0);
  }
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nch) load(ch + 1);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    if (ch + 1 < nch) store(ch + 1, buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= P.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= P.N) continue;
      float v = acc[i][j];
      if (P.bias) v += P.bias[n];
      float* cp = P.C + m * P.ldc + n;
      if (P.beta != 0.0f) v += P.beta * *cp;
      *cp = v;
    }
  }
}

// column sums of a short, wide matrix: one thread per column, fp64 over the rows
template <typename T>
__global__ void k_col_sum_tall(const T* __restrict__ x, long long M, int C, float* __restrict__ out, int accumulate) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (long long p = 0; p < M; ++p) s += (double)to_f<T>(x[p * C + c]);
  out[c] = accumulate ? out[c] + (float)s : (float)s;
}

// ===================================================================== gathers
__global__ void k_gather_rows(const float* __restrict__ table, const int32_t* __restrict__ idx, int n, int dim,
                              float* __restrict__ out, int ldo) {
  const long long total = (long long)n * dim;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / dim), j = (int)(i % dim);
    out[(long long)r * ldo + j] = table[(long long)idx[r] * dim + j];
  }
}
__global__ void k_copy_cols(const float* __restrict__ src, int lds, int n, int cols, float* __restrict__ dst,
                            int ldd) {
  const long long total = (long long)n * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), j = (int)(i % cols);
    dst[(long long)r * ldd + j] = src[(long long)r * lds + j];
  }
}
__global__ void k_scatter_add_rows(const float* __restrict__ src, int lds, const int32_t* __restrict__ idx, int n,
                                   int dim, float* __restrict__ dtable) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= dim) return;
  for (int i = 0; i < n; ++i) dtable[(long long)idx[i] * dim + j] += src[(long long)i * lds + j];
}
__global__ void k_scatter_add_rows_multi(const RowSrcs srcs, int lds, const int32_t* __restrict__ idx, int n, int dim,
                                         float* __restrict__ dtable) {
  const int r = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= dim) return;
  float acc = 0.0f;
  bool hit = false;
  for (int i = 0; i < n; ++i) {
    if (idx[i] != r) continue;
    hit = true;
    for (int s = 0; s < srcs.n; ++s) acc += srcs.p[s][(long long)i * lds + j];
  }
  if (hit) dtable[(long long)r * dim + j] += acc;
}
template <typename TD>
__global__ void k_convert(const float* __restrict__ s, TD* __restrict__ d, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = from_f<TD>(s[i]);
}
template <typename TS>
__global__ void k_to_f32(const TS* __restrict__ s, float* __restrict__ d, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = to_f<TS>(s[i]);
}

// ===================================================================== BN statistics
// block: 256 threads = R rows x G groups (8 channels each); each block covers a
// contiguous pixel range; per-thread fp32 partials, block combine in fp64.
template <typename T>
__global__ void __launch_bounds__(256) k_bn_stats(const T* __restrict__ x, long long M, int C,
                                                  double* __restrict__ partial, long long pix_per_blk) {
  extern __shared__ double sh[];  // [R][2C] doubles
  const int G = C >> 3;
  const int R = 256 / G;
  const int tid = threadIdx.x;
  const int g = tid % G, r = tid / G;
  const long long p0 = (long long)blockIdx.x * pix_per_blk;
  const long long p1 = min(M, p0 + pix_per_blk);
  float s[8] = {}, q[8] = {};
  if (r < R) {
    for (long long p = p0 + r; p < p1; p += R) {
      float v[8];
      Vec8<T>::load(x + p * C + g * 8, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[j] += v[j];
        q[j] = fmaf(v[j], v[j], q[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sh[r * 2 * C + g * 8 + j] = s[j];
      sh[r * 2 * C + C + g * 8 + j] = q[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < 2 * C; c += 256) {
    double a = 0.0;
    for (int rr = 0; rr < R; ++rr) a += sh[rr * 2 * C + c];
    partial[(long long)blockIdx.x * 2 * C + c] = a;
  }
}
__global__ void k_reduce_partials(const double* __restrict__ partial, int nblk, int width, double* __restrict__ out) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= width) return;
  double a = 0.0;
  for (int b = lane; b < nblk; b += 32) a += partial[(long long)b * width + c];
  a = warp_sum_d(a);
  if (lane == 0) out[c] = a;
}
__global__ void k_bn_finalize(const double* __restrict__ sums, int C, double count, float eps,
                              float* __restrict__ mean, float* __restrict__ rstd) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double mu = sums[c] / count;
  double var = sums[C + c] / count - mu * mu;
  if (var < 0) var = 0;
  mean[c] = (float)mu;
  rstd[c] = (float)(1.0 / sqrt(var + (double)eps));
}

// per (pixel, 8-channel group): gain/bias factors
struct BnAffine {
  const float* gain;   // [N][C] (conditional: factor 1 + gain)
  const float* bias;   // [N][C]
  const float* gamma;  // [C]    (plain BN)
  const float* beta;   // [C]
  // 8 consecutive channels c0..c0+7 (c0 % 8 == 0, 16-byte aligned rows)
  __device__ __forceinline__ void get8(int n, int c0, int C, float (&g)[8], float (&b)[8]) const {
    if (gain) {
      ld8(gain + (long long)n * C + c0, g);
      ld8(bias + (long long)n * C + c0, b);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] += 1.0f;
    } else {
      ld8(gamma + c0, g);
      ld8(beta + c0, b);
    }
  }
  // 8 floats; vector loads when 16-byte aligned (parameter slots inside the flat buffer may not be)
  __device__ __forceinline__ static void ld8(const float* p, float (&v)[8]) {
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(p + j);
    }
  }
};

template <typename TI, typename TO>
__global__ void k_bn_apply_relu(const TI* __restrict__ x, int N, int H, int W, int C, const float* __restrict__ mean,
                                const float* __restrict__ rstd, BnAffine af, TO* __restrict__ y, int up2) {
  // 32-bit index arithmetic (every tensor here has < 2^31 elements): 64-bit div/mod dominated the loop
  const unsigned G = C >> 3, HW = (unsigned)(H * W);
  const unsigned total = (unsigned)N * HW * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned g = i % G;
    const unsigned pp = i / G;
    const long long p = pp;
    const int n = (int)(pp / HW);
    float v[8], ga[8], be[8], mu[8], rs[8];
    Vec8<TI>::load(x + p * C + g * 8, v);
    af.get8(n, g * 8, C, ga, be);
    BnAffine::ld8(mean + g * 8, mu);
    BnAffine::ld8(rstd + g * 8, rs);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = (v[j] - mu[j]) * rs[j] * ga[j] + be[j];
      v[j] = t > 0.0f ? t : 0.0f;
    }
    if (!up2) {
      Vec8<TO>::store(y + p * C + g * 8, v);
    } else {
      const unsigned rem = pp - (unsigned)n * HW;
      const int h = (int)(rem / (unsigned)W), w = (int)(rem - (unsigned)h * W);
      const long long W2 = 2 * W;
      const long long base = ((long long)n * 2 * H + 2 * h) * W2 + 2 * w;
      Vec8<TO>::store(y + (base)*C + g * 8, v);
      Vec8<TO>::store(y + (base + 1) * C + g * 8, v);
      Vec8<TO>::store(y + (base + W2) * C + g * 8, v);
      Vec8<TO>::store(y + (base + W2 + 1) * C + g * 8, v);
    }
  }
}

// g0 (gradient w.r.t. the affine output z = x_hat*g + b, through relu) at pixel p
template <typename TG>
__device__ __forceinline__ void load_dy(const TG* dy, long long p, int n, int H, int W, int C, int g, int up2,
                                        float (&d)[8]) {
  if (!up2) {
    Vec8<TG>::load(dy + p * C + g * 8, d);
  } else {
    const unsigned rem = (unsigned)p - (unsigned)n * (unsigned)(H * W);
    const int h = (int)(rem / (unsigned)W), w = (int)(rem - (unsigned)h * W);
    const long long W2 = 2 * W;
    const long long base = ((long long)n * 2 * H + 2 * h) * W2 + 2 * w;
    float a[8], b[8], c[8], e[8];
    Vec8<TG>::load(dy + base * C + g * 8, a);
    Vec8<TG>::load(dy + (base + 1) * C + g * 8, b);
    Vec8<TG>::load(dy + (base + W2) * C + g * 8, c);
    Vec8<TG>::load(dy + (base + W2 + 1) * C + g * 8, e);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = (a[j] + b[j]) + (c[j] + e[j]);
  }
}

// grid: (chunks, N); each block sums over its chunk of sample n's pixels
template <typename TI, typename TG>
__global__ void __launch_bounds__(256) k_bn_bwd_reduce(const TI* __restrict__ x, const TG* __restrict__ dy, int N,
                                                       int H, int W, int C, const float* __restrict__ mean,
                                                       const float* __restrict__ rstd, BnAffine af, int up2,
                                                       float* __restrict__ partial, int chunks) {
  extern __shared__ float shf[];  // [R][2C]
  const int G = C >> 3;
  const int R = 256 / G;
  const int tid = threadIdx.x;
  const int g = tid % G, r = tid / G;
  const int n = blockIdx.y;
  const long long HW = (long long)H * W;
  const long long per = (HW + chunks - 1) / chunks;
  const long long q0 = blockIdx.x * per, q1 = min(HW, q0 + per);
  float sa[8] = {}, sb[8] = {};
  if (r < R) {
    float ga[8], be[8], mu[8], rs[8];
    af.get8(n, g * 8, C, ga, be);
    BnAffine::ld8(mean + g * 8, mu);
    BnAffine::ld8(rstd + g * 8, rs);
    for (long long q = q0 + r; q < q1; q += R) {
      const long long p = (long long)n * HW + q;
      float v[8], d[8];
      Vec8<TI>::load(x + p * C + g * 8, v);
      load_dy<TG>(dy, p, n, H, W, C, g, up2, d);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (v[j] - mu[j]) * rs[j];
        const float z = xh * ga[j] + be[j];
        const float g0 = z > 0.0f ? d[j] : 0.0f;
        sa[j] += g0;
        sb[j] = fmaf(g0, xh, sb[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      shf[r * 2 * C + g * 8 + j] = sa[j];
      shf[r * 2 * C + C + g * 8 + j] = sb[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < 2 * C; c += 256) {
    float a = 0.0f;
    for (int rr = 0; rr < R; ++rr) a += shf[rr * 2 * C + c];
    partial[((long long)n * chunks + blockIdx.x) * 2 * C + c] = a;
  }
}
// bulk-staged streaming (cp.async.bulk into a double-buffered smem ring) for the BN kernels below
constexpr int kBnChunkBytes = 16384;
__device__ __forceinline__ int bn_chunk_pix(int C, int esize) { return kBnChunkBytes / (C * esize); }

// bulk-staged version (no up2): this block's pixel range of image n streams through a double-
// buffered 2 x 16 KB ring (x and dy side by side), the per-thread sums are the register kernel's
template <typename TI, typename TG>
__global__ void __launch_bounds__(256) k_bn_bwd_reduce_bulk(const TI* __restrict__ x, const TG* __restrict__ dy,
                                                            int N, int H, int W, int C, int cpix,
                                                            const float* __restrict__ mean,
                                                            const float* __restrict__ rstd, BnAffine af,
                                                            float* __restrict__ partial, int chunks) {
  extern __shared__ float shf[];  // [R][2C]
  __shared__ __align__(128) uint8_t buf[2][kBnChunkBytes];
  __shared__ __align__(8) uint64_t full[2];
  const int G = C >> 3;
  const int R = 256 / G;
  const int tid = threadIdx.x;
  const int g = tid % G, r = tid / G;
  const int n = blockIdx.y;
  const long long HW = (long long)H * W;
  const long long per = (HW + chunks - 1) / chunks;
  const long long q0 = blockIdx.x * per, q1 = min(HW, q0 + per);
  const int nsub = q1 > q0 ? (int)((q1 - q0 + cpix - 1) / cpix) : 0;
  const uint32_t off_dy = (uint32_t)cpix * C * sizeof(TI);
  if (tid == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int sub, int b) {
    const long long p0 = (long long)n * HW + q0 + (long long)sub * cpix;
    const uint32_t np = (uint32_t)min((long long)cpix, q1 - q0 - (long long)sub * cpix);
    const uint32_t bx = np * C * sizeof(TI), bd = np * C * sizeof(TG);
    tc::mbar_expect_tx(&full[b], bx + bd);
    tc::bulk_load_1d(buf[b], x + p0 * C, bx, &full[b]);
    tc::bulk_load_1d(buf[b] + off_dy, dy + p0 * C, bd, &full[b]);
  };
  if (tid == 0) {
    if (nsub > 0) issue(0, 0);
    if (nsub > 1) issue(1, 1);
  }
  float sa[8] = {}, sb[8] = {};
  float ga[8], be[8], mu[8], rs[8];
  af.get8(n, g * 8, C, ga, be);
  BnAffine::ld8(mean + g * 8, mu);
  BnAffine::ld8(rstd + g * 8, rs);
  for (int sub = 0; sub < nsub; ++sub) {
    const int b = sub & 1;
    tc::mbar_wait(&full[b], (sub >> 1) & 1);
    const int np = (int)min((long long)cpix, q1 - q0 - (long long)sub * cpix);
    const TI* xs = reinterpret_cast<const TI*>(buf[b]);
    const TG* ds = reinterpret_cast<const TG*>(buf[b] + off_dy);
    if (r < R) {
      for (int q = r; q < np; q += R) {
        float v[8], d[8];
        Vec8<TI>::load(xs + q * C + g * 8, v);
        Vec8<TG>::load(ds + q * C + g * 8, d);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (v[j] - mu[j]) * rs[j];
          const float z = xh * ga[j] + be[j];
          const float g0 = z > 0.0f ? d[j] : 0.0f;
          sa[j] += g0;
          sb[j] = fmaf(g0, xh, sb[j]);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && sub + 2 < nsub) issue(sub + 2, b);
  }
  if (r < R) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      shf[r * 2 * C + g * 8 + j] = sa[j];
      shf[r * 2 * C + C + g * 8 + j] = sb[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < 2 * C; c += 256) {
    float a = 0.0f;
    for (int rr = 0; rr < R; ++rr) a += shf[rr * 2 * C + c];
    partial[((long long)n * chunks + blockIdx.x) * 2 * C + c] = a;
  }
}
__global__ void k_bn_bwd_fold(const float* __restrict__ partial, int N, int chunks, int C, float* __restrict__ AB) {
  const long long total = (long long)N * 2 * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i / (2 * C)), c = (int)(i % (2 * C));
    double a = 0.0;
    for (int k = 0; k < chunks; ++k) a += partial[((long long)n * chunks + k) * 2 * C + c];
    AB[i] = (float)a;
  }
}
// tot[c] = sum_n g(n, c) AB[n][c], tot[C + c] = sum_n g(n, c) AB[n][C + c]: block = 32 channels x 8
// sample groups (group j sums n = j, j + 8, .. in order), groups combined in order (deterministic)
__global__ void __launch_bounds__(256) k_bn_bwd_totals(const float* __restrict__ AB, int N, int C,
                                                       const float* __restrict__ gain, const float* __restrict__ gamma,
                                                       double* __restrict__ tot) {
  __shared__ double red[2][8][32];
  const int cx = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cx;
  double t0 = 0.0, t1 = 0.0;
  if (c < C) {
    const double g0 = gain ? 0.0 : (double)gamma[c];
    for (int n = j; n < N; n += 8) {
      const double g = gain ? 1.0 + (double)gain[(long long)n * C + c] : g0;
      t0 += g * AB[(long long)n * 2 * C + c];
      t1 += g * AB[(long long)n * 2 * C + C + c];
    }
  }
  red[0][j][cx] = t0;
  red[1][j][cx] = t1;
  __syncthreads();
  if (j == 0 && c < C) {
    double a0 = 0.0, a1 = 0.0;
    for (int k = 0; k < 8; ++k) {
      a0 += red[0][k][cx];
      a1 += red[1][k][cx];
    }
    tot[c] = a0;
    tot[C + c] = a1;
  }
}
template <typename TI, typename TG, typename TO>
__global__ void k_bn_bwd_apply(const TI* __restrict__ x, const TG* __restrict__ dy, int N, int H, int W, int C,
                               const float* __restrict__ mean, const float* __restrict__ rstd, BnAffine af, int up2,
                               const float* __restrict__ mgrad, const TO* __restrict__ add, TO* __restrict__ dx) {
  // mgrad[c] = mean over the global batch of g * g0, mgrad[C + c] = mean of g * g0 * x_hat
  const unsigned G = C >> 3, HW = (unsigned)(H * W);
  const unsigned total = (unsigned)N * HW * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned g = i % G;
    const long long p = i / G;
    const int n = (int)((unsigned)p / HW);
    float v[8], d[8], o[8], ga[8], be[8], mu[8], rs[8], mg[8], mgx[8];
    Vec8<TI>::load(x + p * C + g * 8, v);
    load_dy<TG>(dy, p, n, H, W, C, g, up2, d);
    af.get8(n, g * 8, C, ga, be);
    BnAffine::ld8(mean + g * 8, mu);
    BnAffine::ld8(rstd + g * 8, rs);
    BnAffine::ld8(mgrad + g * 8, mg);
    BnAffine::ld8(mgrad + C + g * 8, mgx);
    float ad[8];
    if (add) Vec8<TO>::load(add + p * C + g * 8, ad);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float xh = (v[j] - mu[j]) * rs[j];
      const float z = xh * ga[j] + be[j];
      const float g0 = z > 0.0f ? d[j] : 0.0f;
      o[j] = rs[j] * (ga[j] * g0 - mg[j] - xh * mgx[j]);
      if (add) o[j] += ad[j];
    }
    Vec8<TO>::store(dx + p * C + g * 8, o);
  }
}
__global__ void k_bn_bwd_means(const double* __restrict__ tot, int C, double count, float* __restrict__ mgrad) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= 2 * C) return;
  mgrad[c] = (float)(tot[c] / count);
}

// Channel-group-stationary variants (no upsample): thread (pixel lane, channel group g) keeps its 8 channels'
// statistics in registers and walks pixels, two per iteration; per-sample CBN gains are reloaded only
// when the image changes.  blockDim = G * P (G = C/8 groups, P pixel lanes).
template <typename TI, typename TO>
__global__ void __launch_bounds__(256) k_bn_apply_relu_cs(const TI* __restrict__ x, long long P_total, int HW, int C,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd, BnAffine af,
                                                          TO* __restrict__ y) {
  const int G = C >> 3;
  const int lanes = blockDim.x / G;
  const int g = threadIdx.x % G, lane = threadIdx.x / G;
  if (lane >= lanes) return;
  float mu[8], rs[8], ga[8], be[8];
  BnAffine::ld8(mean + g * 8, mu);
  BnAffine::ld8(rstd + g * 8, rs);
  int ncur = -1;
  if (!af.gain) af.get8(0, g * 8, C, ga, be);
  // each block owns a contiguous pixel range, so an image's CBN gains are reloaded ~once per block
  const long long chunk = (P_total + gridDim.x - 1) / gridDim.x;
  const long long p_end = min(P_total, (blockIdx.x + 1) * chunk);
  const long long step = lanes;
  for (long long p = blockIdx.x * chunk + lane; p < p_end; p += 2 * step) {
    const long long p2 = p + step;
    float v[8], v2[8];
    Vec8<TI>::load(x + p * C + g * 8, v);
    const bool has2 = p2 < p_end;
    if (has2) Vec8<TI>::load(x + p2 * C + g * 8, v2);
    if (af.gain) {
      const int n = (int)((unsigned)p / (unsigned)HW);   // pixel counts < 2^31
      if (n != ncur) {
        af.get8(n, g * 8, C, ga, be);
        ncur = n;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = (v[j] - mu[j]) * rs[j] * ga[j] + be[j];
      v[j] = t > 0.0f ? t : 0.0f;
    }
    Vec8<TO>::store(y + p * C + g * 8, v);
    if (has2) {
      if (af.gain) {
        const int n = (int)((unsigned)p2 / (unsigned)HW);
        if (n != ncur) {
          af.get8(n, g * 8, C, ga, be);
          ncur = n;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float t = (v2[j] - mu[j]) * rs[j] * ga[j] + be[j];
        v2[j] = t > 0.0f ? t : 0.0f;
      }
      Vec8<TO>::store(y + p2 * C + g * 8, v2);
    }
  }
}

template <typename TI, typename TG, typename TO>
__global__ void __launch_bounds__(256) k_bn_bwd_apply_cs(const TI* __restrict__ x, const TG* __restrict__ dy,
                                                         long long P_total, int HW, int C,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, BnAffine af,
                                                         const float* __restrict__ mgrad, const TO* __restrict__ add,
                                                         TO* __restrict__ dx) {
  const int G = C >> 3;
  const int lanes = blockDim.x / G;
  const int g = threadIdx.x % G, lane = threadIdx.x / G;
  if (lane >= lanes) return;
  float mu[8], rs[8], ga[8], be[8], mg[8], mgx[8];
  BnAffine::ld8(mean + g * 8, mu);
  BnAffine::ld8(rstd + g * 8, rs);
  BnAffine::ld8(mgrad + g * 8, mg);
  BnAffine::ld8(mgrad + C + g * 8, mgx);
  int ncur = -1;
  if (!af.gain) af.get8(0, g * 8, C, ga, be);
  const long long chunk = (P_total + gridDim.x - 1) / gridDim.x;
  const long long p_end = min(P_total, (blockIdx.x + 1) * chunk);
  for (long long p = blockIdx.x * chunk + lane; p < p_end; p += lanes) {
    float v[8], d[8], ad[8], o[8];
    Vec8<TI>::load(x + p * C + g * 8, v);
    Vec8<TG>::load(dy + p * C + g * 8, d);
    if (add) Vec8<TO>::load(add + p * C + g * 8, ad);
    if (af.gain) {
      const int n = (int)((unsigned)p / (unsigned)HW);   // pixel counts < 2^31
      if (n != ncur) {
        af.get8(n, g * 8, C, ga, be);
        ncur = n;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float xh = (v[j] - mu[j]) * rs[j];
      const float z = xh * ga[j] + be[j];
      const float g0 = z > 0.0f ? d[j] : 0.0f;
      o[j] = rs[j] * (ga[j] * g0 - mg[j] - xh * mgx[j]);
      if (add) o[j] += ad[j];
    }
    Vec8<TO>::store(dx + p * C + g * 8, o);
  }
}

// Bulk-staged variants (memory-level parallelism without registers): each block walks chunks
// of kBnChunkBytes of consecutive pixels; one thread issues cp.async.bulk copies of the chunk's
// input(s) into a double-buffered smem ring (mbarrier complete_tx), the threads compute from
// shared memory with their channel group's constants in registers and store with 16-byte
// stores.  (The register-staged kernels held 2 x 16 B per thread in flight at 68-90 registers,
// ~24 KB per SM: 4.1-4.5 TB/s.)

// TO = Bf16Split: the output is the two-term bf16 split of the fp32 result, y = [P][2C] with x1 = bf16(v) in
// channels [0, C) and x2 = bf16(v - x1) in [C, 2C) (the operand of G's tensor-core output layer, R36)
struct Bf16Split {};

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) k_bn_apply_relu_bulk(const TI* __restrict__ x, long long P_total, int HW, int C,
                                                            const float* __restrict__ mean,
                                                            const float* __restrict__ rstd, BnAffine af,
                                                            TO* __restrict__ y) {
  __shared__ __align__(128) uint8_t buf[2][kBnChunkBytes];
  __shared__ __align__(8) uint64_t full[2];
  const int G = C >> 3;
  const int lanes = blockDim.x / G;
  const int g = threadIdx.x % G, lane = threadIdx.x / G;
  // whole rounds of the block's pixel lanes per chunk
  const int cmax = bn_chunk_pix(C, (int)sizeof(TI));
  const int cpix = cmax >= lanes ? cmax / lanes * lanes : cmax;
  const long long nchunks = (P_total + cpix - 1) / cpix;
  if (threadIdx.x == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](long long t, int b) {
    const long long p0 = t * cpix;
    const int np = (int)min((long long)cpix, P_total - p0);
    const uint32_t bytes = (uint32_t)np * C * sizeof(TI);
    tc::mbar_expect_tx(&full[b], bytes);
    tc::bulk_load_1d(buf[b], x + p0 * C, bytes, &full[b]);
  };
  if (threadIdx.x == 0) {
    if (blockIdx.x < nchunks) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < nchunks) issue(blockIdx.x + gridDim.x, 1);
  }
  float mu[8], rs[8], ga[8], be[8];
  BnAffine::ld8(mean + g * 8, mu);
  BnAffine::ld8(rstd + g * 8, rs);
  int ncur = -1;
  if (!af.gain) af.get8(0, g * 8, C, ga, be);
  int it = 0;
  for (long long t = blockIdx.x; t < nchunks; t += gridDim.x, ++it) {
    const int b = it & 1;
    tc::mbar_wait(&full[b], (it >> 1) & 1);
    const long long p0 = t * cpix;
    const int np = (int)min((long long)cpix, P_total - p0);
    const TI* xs = reinterpret_cast<const TI*>(buf[b]);
    bool per_pixel = false;   // as in the backward apply: gains loaded once per chunk inside one image
    if (af.gain) {
      const int n0 = (int)((unsigned)p0 / (unsigned)HW), n1 = (int)((unsigned)(p0 + np - 1) / (unsigned)HW);
      if (n0 == n1) {
        if (n0 != ncur) {
          af.get8(n0, g * 8, C, ga, be);
          ncur = n0;
        }
      } else {
        per_pixel = true;
      }
    }
    if (lane < lanes) {
      for (int q = lane; q < np; q += lanes) {
        const long long p = p0 + q;
        float v[8];
        Vec8<TI>::load(xs + q * C + g * 8, v);
        if (per_pixel) {
          const int n = (int)((unsigned)p / (unsigned)HW);   // pixel counts < 2^31
          if (n != ncur) {
            af.get8(n, g * 8, C, ga, be);
            ncur = n;
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float tt = (v[j] - mu[j]) * rs[j] * ga[j] + be[j];
          v[j] = tt > 0.0f ? tt : 0.0f;
        }
        if constexpr (std::is_same<TO, Bf16Split>::value) {
          float lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) lo[j] = v[j] - __bfloat162float(__float2bfloat16_rn(v[j]));
          bf16* ys = reinterpret_cast<bf16*>(y) + p * 2 * C + g * 8;
          Vec8<bf16>::store(ys, v);
          Vec8<bf16>::store(ys + C, lo);
        } else {
          Vec8<TO>::store(y + p * C + g * 8, v);
        }
      }
    }
    __syncthreads();   // every thread is done with buf[b]
    if (threadIdx.x == 0 && t + 2LL * gridDim.x < nchunks) issue(t + 2LL * gridDim.x, b);
  }
}

// backward apply, bulk-staged: x, dy (and the optional residual gradient `add`) of a chunk of
// pixels land side by side in one 16 KB stage of the ring
template <typename TI, typename TG, typename TO>
__global__ void __launch_bounds__(256) k_bn_bwd_apply_bulk(const TI* __restrict__ x, const TG* __restrict__ dy,
                                                           long long P_total, int HW, int C, int cpix,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ rstd, BnAffine af,
                                                           const float* __restrict__ mgrad, const TO* __restrict__ add,
                                                           TO* __restrict__ dx) {
  __shared__ __align__(128) uint8_t buf[2][kBnChunkBytes];
  __shared__ __align__(8) uint64_t full[2];
  const int G = C >> 3;
  const int lanes = blockDim.x / G;
  const int g = threadIdx.x % G, lane = threadIdx.x / G;
  const long long nchunks = (P_total + cpix - 1) / cpix;
  const uint32_t off_dy = (uint32_t)cpix * C * sizeof(TI);
  const uint32_t off_add = off_dy + (uint32_t)cpix * C * sizeof(TG);
  if (threadIdx.x == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](long long t, int b) {
    const long long p0 = t * cpix;
    const uint32_t np = (uint32_t)min((long long)cpix, P_total - p0);
    const uint32_t bx = np * C * sizeof(TI), bd = np * C * sizeof(TG), ba = add ? np * C * sizeof(TO) : 0u;
    tc::mbar_expect_tx(&full[b], bx + bd + ba);
    tc::bulk_load_1d(buf[b], x + p0 * C, bx, &full[b]);
    tc::bulk_load_1d(buf[b] + off_dy, dy + p0 * C, bd, &full[b]);
    if (add) tc::bulk_load_1d(buf[b] + off_add, add + p0 * C, ba, &full[b]);
  };
  if (threadIdx.x == 0) {
    if (blockIdx.x < nchunks) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < nchunks) issue(blockIdx.x + gridDim.x, 1);
  }
  float mu[8], rs[8], ga[8], be[8], mg[8], mgx[8];
  BnAffine::ld8(mean + g * 8, mu);
  BnAffine::ld8(rstd + g * 8, rs);
  BnAffine::ld8(mgrad + g * 8, mg);
  BnAffine::ld8(mgrad + C + g * 8, mgx);
  int ncur = -1;
  if (!af.gain) af.get8(0, g * 8, C, ga, be);
  int it = 0;
  for (long long t = blockIdx.x; t < nchunks; t += gridDim.x, ++it) {
    const int b = it & 1;
    tc::mbar_wait(&full[b], (it >> 1) & 1);
    const long long p0 = t * cpix;
    const int np = (int)min((long long)cpix, P_total - p0);
    const TI* xs = reinterpret_cast<const TI*>(buf[b]);
    const TG* ds = reinterpret_cast<const TG*>(buf[b] + off_dy);
    const TO* as = reinterpret_cast<const TO*>(buf[b] + off_add);
    // conditional BN: the per-image gains change at most once inside a chunk; when the whole chunk lies in one
    // image they are loaded once here, outside the pixel loop (a per-pixel check kept a global load and its
    // latency inside the loop: 24% of the kernel's stall samples)
    bool per_pixel = false;
    if (af.gain) {
      const int n0 = (int)((unsigned)p0 / (unsigned)HW), n1 = (int)((unsigned)(p0 + np - 1) / (unsigned)HW);
      if (n0 == n1) {
        if (n0 != ncur) {
          af.get8(n0, g * 8, C, ga, be);
          ncur = n0;
        }
      } else {
        per_pixel = true;
      }
    }
    for (int q = lane; q < np; q += lanes) {
      const long long p = p0 + q;
      float v[8], d[8], ad[8], o[8];
      Vec8<TI>::load(xs + q * C + g * 8, v);
      Vec8<TG>::load(ds + q * C + g * 8, d);
      if (add) Vec8<TO>::load(as + q * C + g * 8, ad);
      if (per_pixel) {
        const int n = (int)((unsigned)p / (unsigned)HW);   // pixel counts < 2^31
        if (n != ncur) {
          af.get8(n, g * 8, C, ga, be);
          ncur = n;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (v[j] - mu[j]) * rs[j];
        const float z = xh * ga[j] + be[j];
        const float g0 = z > 0.0f ? d[j] : 0.0f;
        o[j] = rs[j] * (ga[j] * g0 - mg[j] - xh * mgx[j]);
        if (add) o[j] += ad[j];
      }
      Vec8<TO>::store(dx + p * C + g * 8, o);
    }
    __syncthreads();   // every thread is done with buf[b]
    if (threadIdx.x == 0 && t + 2LL * gridDim.x < nchunks) issue(t + 2LL * gridDim.x, b);
  }
}

// ===================================================================== elementwise
template <typename T>
__global__ void k_relu_copy(const T* __restrict__ x, T* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = to_f<T>(x[i]);
    y[i] = from_f<T>(v > 0.0f ? v : 0.0f);
  }
}
template <typename T>
__global__ void k_relu_bwd(const T* __restrict__ dy, const T* __restrict__ ref, const T* __restrict__ add,
                           T* __restrict__ dx, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v = to_f<T>(ref[i]) > 0.0f ? to_f<T>(dy[i]) : 0.0f;
    if (add) v += to_f<T>(add[i]);
    dx[i] = from_f<T>(v);
  }
}
// out pixel (n, ho, wo), channel c:  ((x00 + x01) + (x10 + x11)) * 0.25 (+ add)
template <typename T>
__global__ void k_avgpool2(const T* __restrict__ x, int N, int H, int W, int C, int ldx, const T* __restrict__ add,
                           T* __restrict__ y) {
  const int Ho = H >> 1, Wo = W >> 1;
  const long long total = (long long)N * Ho * Wo * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    long long p = i / C;
    const int wo = (int)(p % Wo);
    p /= Wo;
    const int ho = (int)(p % Ho);
    const int n = (int)(p / Ho);
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    const float s = (to_f<T>(x[b * ldx + c]) + to_f<T>(x[(b + 1) * ldx + c])) +
                    (to_f<T>(x[(b + W) * ldx + c]) + to_f<T>(x[(b + W + 1) * ldx + c]));
    float v = s * 0.25f;
    if (add) v += to_f<T>(add[i]);
    y[i] = from_f<T>(v);
  }
}
template <typename T>
__global__ void k_avgpool2_bwd(const T* __restrict__ dy, int N, int H, int W, int C, const T* __restrict__ add,
                               T* __restrict__ dx, int lddx) {
  const long long total = (long long)N * H * W * C;
  const int Ho = H >> 1, Wo = W >> 1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    long long p = i / C;
    const int w = (int)(p % W);
    p /= W;
    const int h = (int)(p % H);
    const int n = (int)(p / H);
    float v = 0.25f * to_f<T>(dy[(((long long)n * Ho + (h >> 1)) * Wo + (w >> 1)) * C + c]);
    const long long o = (((long long)n * H + h) * W + w);
    if (add) v += to_f<T>(add[o * C + c]);
    dx[o * lddx + c] = from_f<T>(v);
  }
}
template <typename T>
__global__ void k_up2_bwd(const T* __restrict__ dy, int N, int H, int W, int C, T* __restrict__ dx) {
  const long long total = (long long)N * H * W * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    long long p = i / C;
    const int w = (int)(p % W);
    p /= W;
    const int h = (int)(p % H);
    const int n = (int)(p / H);
    const long long W2 = 2 * W;
    const long long b = ((long long)n * 2 * H + 2 * h) * W2 + 2 * w;
    const float s = (to_f<T>(dy[b * C + c]) + to_f<T>(dy[(b + 1) * C + c])) +
                    (to_f<T>(dy[(b + W2) * C + c]) + to_f<T>(dy[(b + W2 + 1) * C + c]));
    dx[i] = from_f<T>(s);
  }
}
// column sums: scalar path (any C) and an 8-channel-vector path (C % 8 == 0, C/8 <= 256)
template <typename T>
__global__ void __launch_bounds__(256) k_col_sum(const T* __restrict__ x, long long M, int C,
                                                 double* __restrict__ partial, long long pix_per_blk) {
  extern __shared__ double sh[];  // [256]
  const long long p0 = (long long)blockIdx.x * pix_per_blk;
  const long long p1 = min(M, p0 + pix_per_blk);
  for (int c0 = 0; c0 < C; c0 += 32) {
    const int c = c0 + (threadIdx.x & 31);
    const int r = threadIdx.x >> 5;
    float s = 0.0f;
    if (c < C)
      for (long long p = p0 + r; p < p1; p += 8) s += to_f<T>(x[p * C + c]);
    sh[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < 32 && c < C) {
      double a = 0.0;
      for (int k = 0; k < 8; ++k) a += sh[k * 32 + threadIdx.x];
      partial[(long long)blockIdx.x * C + c] = a;
    }
    __syncthreads();
  }
}
// C <= 8: thread-private sums of all channels over a strided pixel range, block combine in fp64
template <typename T>
__global__ void __launch_bounds__(256) k_col_sum_small(const T* __restrict__ x, long long M, int C,
                                                       double* __restrict__ partial, long long pix_per_blk) {
  __shared__ double sh[8][33];
  const long long p0 = (long long)blockIdx.x * pix_per_blk;
  const long long p1 = min(M, p0 + pix_per_blk);
  float s[8] = {};
  for (long long p = p0 + threadIdx.x; p < p1; p += blockDim.x)
    for (int c = 0; c < C; ++c) s[c] += to_f<T>(x[p * C + c]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c = 0; c < C; ++c) {
    const double v = warp_sum_d((double)s[c]);
    if (lane == 0) sh[c][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < C) {
    double a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += sh[threadIdx.x][w];
    partial[(long long)blockIdx.x * C + threadIdx.x] = a;
  }
}
template <typename T>
__global__ void __launch_bounds__(256) k_col_sum_vec(const T* __restrict__ x, long long M, int C,
                                                     double* __restrict__ partial, long long pix_per_blk) {
  extern __shared__ float shs[];  // [R][C]
  const int G = C >> 3, R = 256 / G;
  const int g = threadIdx.x % G, r = threadIdx.x / G;
  const long long p0 = (long long)blockIdx.x * pix_per_blk;
  const long long p1 = min(M, p0 + pix_per_blk);
  float s[8] = {};
  if (r < R) {
    long long p = p0 + r;
    for (; p + 3 * R < p1; p += 4 * R) {   // four independent 16-byte loads in flight
      float v0[8], v1[8], v2[8], v3[8];
      Vec8<T>::load(x + p * C + g * 8, v0);
      Vec8<T>::load(x + (p + R) * C + g * 8, v1);
      Vec8<T>::load(x + (p + 2 * R) * C + g * 8, v2);
      Vec8<T>::load(x + (p + 3 * R) * C + g * 8, v3);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += (v0[j] + v1[j]) + (v2[j] + v3[j]);
    }
    for (; p < p1; p += R) {
      float v[8];
      Vec8<T>::load(x + p * C + g * 8, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += v[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) shs[r * C + g * 8 + j] = s[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += 256) {
    double a = 0.0;
    for (int rr = 0; rr < R; ++rr) a += shs[rr * C + c];
    partial[(long long)blockIdx.x * C + c] = a;
  }
}
__global__ void k_reduce_partials_f32(const double* __restrict__ partial, int nblk, int width, float* __restrict__ out,
                                      int accumulate) {
  // one warp per column: lane l sums blocks l, l+32, ... then a fixed shuffle tree (deterministic)
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= width) return;
  double a = 0.0;
  for (int b = lane; b < nblk; b += 32) a += partial[(long long)b * width + c];
  a = warp_sum_d(a);
  if (lane == 0) out[c] = (float)(accumulate ? (double)out[c] + a : a);
}

// ===================================================================== G output / tanh
template <typename T>
__global__ void k_tanh_to_image(const float* __restrict__ pre, float* __restrict__ img, T* __restrict__ dst,
                                long long M, int cp) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < M; p += (long long)gridDim.x * blockDim.x) {
    for (int k = 0; k < cp; ++k) {
      float v = 0.0f;
      if (k < 3) {
        v = tanhf(pre[p * 3 + k]);
        img[p * 3 + k] = v;
      }
      dst[p * cp + k] = from_f<T>(v);
    }
  }
}
template <typename T>
__global__ void k_tanh_bwd(const T* __restrict__ dimg, int cp, const float* __restrict__ img, float* __restrict__ dpre,
                           long long M) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < M * 3;
       i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / 3;
    const int k = (int)(i % 3);
    const float y = img[i];
    dpre[i] = to_f<T>(dimg[p * cp + k]) * (1.0f - y * y);
  }
}

// ===================================================================== SIMT conv
// y tile: TM pixels x TN output channels; K = taps x Cin in chunks of 8 channels
template <typename TI, typename TW, typename TO, int TM, int TN, int RM, int RN>
__global__ void __launch_bounds__(256) k_simt_conv(const TI* __restrict__ x, int N, int H, int W, int Cin,
                                                   const TW* __restrict__ w, int Cout, int ksz,
                                                   const float* __restrict__ bias, const float* __restrict__ alpha,
                                                   const TO* __restrict__ res, int res_mode, TO* __restrict__ y,
                                                   const TO* __restrict__ relu_ref) {
  constexpr int KC = 8;
  __shared__ float As[KC][TM + 1];
  __shared__ float Bs[KC][TN + 1];
  const long long M = (long long)N * H * W;
  const long long m0 = (long long)blockIdx.x * TM;
  const int n0 = blockIdx.y * TN;
  const int tid = threadIdx.x;
  constexpr int TX = TN / RN;   // threads along N
  const int tx = tid % TX, ty = tid / TX;
  const int taps = ksz * ksz, pad = ksz >> 1;
  // fp64 accumulation: this is the fp32 parity engine's conv (reference-grade; not the bf16 hot path)
  double acc[RM][RN] = {};
  for (int tap = 0; tap < taps; ++tap) {
    const int dy = tap / ksz - pad, dx = tap % ksz - pad;
    for (int c0 = 0; c0 < Cin; c0 += KC) {
      for (int i = tid; i < TM * KC; i += 256) {
        const int mm = i / KC, kk = i % KC;
        const long long m = m0 + mm;
        float v = 0.0f;
        const int c = c0 + kk;
        if (m < M && c < Cin) {
          const int n = (int)(m / ((long long)H * W));
          const int r = (int)(m - (long long)n * H * W);
          const int h = r / W + dy, ww = r % W + dx;
          if (h >= 0 && h < H && ww >= 0 && ww < W) v = to_f<TI>(x[(((long long)n * H + h) * W + ww) * Cin + c]);
        }
        As[kk][mm] = v;
      }
      for (int i = tid; i < TN * KC; i += 256) {
        const int nn = i / KC, kk = i % KC;
        const int o = n0 + nn, c = c0 + kk;
        Bs[kk][nn] = (o < Cout && c < Cin) ? to_f<TW>(w[((long long)o * taps + tap) * Cin + c]) : 0.0f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        float a[RM], b[RN];
#pragma unroll
        for (int i = 0; i < RM; ++i) a[i] = As[kk][ty * RM + i];
#pragma unroll
        for (int j = 0; j < RN; ++j) b[j] = Bs[kk][tx * RN + j];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = fma((double)a[i], (double)b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  const float al = alpha ? *alpha : 1.0f;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const long long m = m0 + ty * RM + i;
    if (m >= M) continue;
    long long rb = m * Cout;
    if (res && res_mode == 2) {
      const int n = (int)(m / ((long long)H * W));
      const int r = (int)(m - (long long)n * H * W);
      const int h = r / W, ww = r % W;
      rb = (((long long)n * (H >> 1) + (h >> 1)) * (W >> 1) + (ww >> 1)) * Cout;
    }
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int o = n0 + tx * RN + j;
      if (o >= Cout) continue;
      float v = (float)acc[i][j] * al;
      if (relu_ref && !(to_f<TO>(relu_ref[m * Cout + o]) > 0.0f)) v = 0.0f;
      if (bias) v += bias[o];
      if (res) v += to_f<TO>(res[rb + o]);
      y[m * Cout + o] = from_f<TO>(v);
    }
  }
}

// wgrad: block tile T_O x T_C over (o, c) for one tap; pixel range split over blockIdx.z;
// 256 threads = (T_O/RO) x (T_C/RC), each RO x RC outputs
template <typename TI, typename TG, int T_O, int T_C, int RO, int RC>
__global__ void __launch_bounds__(256) k_simt_wgrad(const TI* __restrict__ x, const TG* __restrict__ dy, int N, int H,
                                                    int W, int Cin, int Cout, int ksz, float* __restrict__ dw,
                                                    long long pix_per_split) {
  constexpr int KP = 16;
  constexpr int TXC = T_C / RC;   // threads along c
  __shared__ float As[KP][T_O + 1];
  __shared__ float Bs[KP][T_C + 1];
  const int taps = ksz * ksz, pad = ksz >> 1;
  const int cblocks = (Cin + T_C - 1) / T_C;
  const int tap = blockIdx.y / cblocks, cb = blockIdx.y % cblocks;
  const int o0 = blockIdx.x * T_O, c0 = cb * T_C;
  const int dyy = tap / ksz - pad, dxx = tap % ksz - pad;
  const long long M = (long long)N * H * W;
  const long long p0 = (long long)blockIdx.z * pix_per_split, p1 = min(M, p0 + pix_per_split);
  const int tid = threadIdx.x, tx = tid % TXC, ty = tid / TXC;
  double acc[RO][RC] = {};   // fp64: the fp32 parity engine's wgrad sums up to millions of pixels
  for (long long pb = p0; pb < p1; pb += KP) {
    for (int i = tid; i < KP * T_O; i += 256) {
      const int kk = i / T_O, oo = i % T_O;
      const long long p = pb + kk;
      const int o = o0 + oo;
      As[kk][oo] = (p < p1 && o < Cout) ? to_f<TG>(dy[p * Cout + o]) : 0.0f;
    }
    for (int i = tid; i < KP * T_C; i += 256) {
      const int kk = i / T_C, cc = i % T_C;
      const long long p = pb + kk;
      const int c = c0 + cc;
      float v = 0.0f;
      if (p < p1 && c < Cin) {
        const int n = (int)(p / ((long long)H * W));
        const int r = (int)(p - (long long)n * H * W);
        const int h = r / W + dyy, ww = r % W + dxx;
        if (h >= 0 && h < H && ww >= 0 && ww < W) v = to_f<TI>(x[(((long long)n * H + h) * W + ww) * Cin + c]);
      }
      Bs[kk][cc] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
      float a[RO], b[RC];
#pragma unroll
      for (int i = 0; i < RO; ++i) a[i] = As[kk][ty * RO + i];
#pragma unroll
      for (int j = 0; j < RC; ++j) b[j] = Bs[kk][tx * RC + j];
#pragma unroll
      for (int i = 0; i < RO; ++i)
#pragma unroll
        for (int j = 0; j < RC; ++j) acc[i][j] = fma((double)a[i], (double)b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RO; ++i) {
    const int o = o0 + ty * RO + i;
    if (o >= Cout) continue;
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      const int c = c0 + tx * RC + j;
      if (c >= Cin) continue;
      // one partial per pixel split, summed in split order afterwards (deterministic; no atomics)
      dw[(long long)blockIdx.z * Cout * taps * Cin + ((long long)o * taps + tap) * Cin + c] = (float)acc[i][j];
    }
  }
}
__global__ void k_simt_split_sum(const float* __restrict__ part, float* __restrict__ dst, long long n, int splits,
                                 int accumulate) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = accumulate ? dst[i] : 0.0;
    for (int k = 0; k < splits; ++k) a += part[(long long)k * n + i];
    dst[i] = (float)a;
  }
}

// ===================================================================== D head / hinge
template <typename T>
__global__ void k_d_head_fwd(const T* __restrict__ h, int HW, int C, const float* __restrict__ w_lin,
                             const float* __restrict__ b_lin, const float* __restrict__ embed,
                             const int32_t* __restrict__ y, float* __restrict__ feat, float* __restrict__ logits) {
  const int n = blockIdx.x;
  __shared__ double red[32];
  double part = 0.0;
  const float* e = embed + (long long)y[n] * C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.0f;
    for (int q = 0; q < HW; ++q) {
      const float v = to_f<T>(h[((long long)n * HW + q) * C + c]);
      s += v > 0.0f ? v : 0.0f;
    }
    feat[(long long)n * C + c] = s;
    part += (double)s * ((double)w_lin[c] + (double)e[c]);
  }
  part = warp_sum_d(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a += red[i];
    logits[n] = (float)(a + (double)b_lin[0]);
  }
}
__global__ void k_hinge(const float* __restrict__ logits, int B, int mode, float* __restrict__ dl,
                        float* __restrict__ out) {
  // single block
  __shared__ double s_loss, s_real, s_fake;
  __shared__ int s_bad;
  if (threadIdx.x == 0) { s_loss = 0; s_real = 0; s_fake = 0; s_bad = 0; }
  __syncthreads();
  const int total = mode == 0 ? 2 * B : B;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const float l = logits[i];
    if (!isfinite(l)) atomicOr(&s_bad, 1);
    double lo;
    float d;
    if (mode == 0) {
      if (i < B) {  // fake: relu(1 + l)
        lo = 1.0 + l > 0 ? 1.0 + l : 0.0;
        d = (1.0f + l > 0.0f) ? 1.0f / B : 0.0f;
        atomicAdd(&s_fake, (double)l);
      } else {      // real: relu(1 - l)
        lo = 1.0 - l > 0 ? 1.0 - l : 0.0;
        d = (1.0f - l > 0.0f) ? -1.0f / B : 0.0f;
        atomicAdd(&s_real, (double)l);
      }
    } else {
      lo = -(double)l;
      d = -1.0f / B;
      atomicAdd(&s_fake, (double)l);
    }
    dl[i] = d;
    atomicAdd(&s_loss, lo);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[0] = (float)(s_loss / B);
    out[1] = (float)(s_real / B);
    out[2] = (float)(s_fake / B);
    out[3] = s_bad ? 1.0f : 0.0f;
  }
}
template <typename T>
__global__ void k_d_head_bwd_dh(const T* __restrict__ h, int N, int HW, int C, const float* __restrict__ w_lin,
                                const float* __restrict__ embed, const int32_t* __restrict__ y,
                                const float* __restrict__ dl, T* __restrict__ dh) {
  const long long total = (long long)N * HW * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int n = (int)(i / ((long long)HW * C));
    const float df = dl[n] * (w_lin[c] + embed[(long long)y[n] * C + c]);
    dh[i] = from_f<T>(to_f<T>(h[i]) > 0.0f ? df : 0.0f);
  }
}
// dw_lin[c] = sum_n dl[n] feat[n][c];  dembed[y][c] += sum_{n : y[n] = y} dl[n] feat[n][c]  (each class's
// samples summed in n order by one thread: the samples are ranked by (class, n) in shared memory, the
// thread at the first rank of a class walks its run);  db_lin = sum_n dl[n].  Block = 32 channels.
constexpr int kHeadMaxN = 2048;
__global__ void __launch_bounds__(256) k_d_head_bwd_w(int N, int C, const float* __restrict__ feat,
                                                      const float* __restrict__ dl, const int32_t* __restrict__ y,
                                                      float* __restrict__ dw_lin, float* __restrict__ db_lin,
                                                      float* __restrict__ dembed) {
  __shared__ int ys[kHeadMaxN];
  __shared__ short perm[kHeadMaxN];
  __shared__ double red[8][32];
  for (int n = threadIdx.x; n < N; n += blockDim.x) ys[n] = y[n];
  __syncthreads();
  for (int n = threadIdx.x; n < N; n += blockDim.x) {   // stable rank by (class, n)
    const int yn = ys[n];
    int r = 0;
    for (int m = 0; m < N; ++m) {
      const int ym = ys[m];
      r += (ym < yn) || (ym == yn && m < n);
    }
    perm[r] = (short)n;
  }
  __syncthreads();
  const int cx = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cx;
  double a = 0.0;
  if (c < C) {
    for (int n = j; n < N; n += 8) a += (double)(dl[n] * feat[(long long)n * C + c]);
    for (int p = j; p < N; p += 8) {
      const int n0 = perm[p], k = ys[n0];
      if (p > 0 && ys[perm[p - 1]] == k) continue;   // not the first sample of its class
      float s = 0.0f;
      for (int q = p; q < N && ys[perm[q]] == k; ++q) {
        const int n = perm[q];
        s += dl[n] * feat[(long long)n * C + c];
      }
      dembed[(long long)k * C + c] += s;
    }
  }
  red[j][cx] = a;
  __syncthreads();
  if (j == 0 && c < C) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[k][cx];
    dw_lin[c] = (float)t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int n = 0; n < N; ++n) t += dl[n];
    db_lin[0] = (float)t;
  }
}

// ===================================================================== attention helpers
template <typename T>
__global__ void k_maxpool2_split(const T* __restrict__ x, int N, int H, int W, int ldx, int c_off, int C,
                                 T* __restrict__ pooled, T* __restrict__ pooledT) {
  const int Ho = H >> 1, Wo = W >> 1, Q = Ho * Wo;
  const long long total = (long long)N * Q * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const long long pq = i / C;
    const int q = (int)(pq % Q);
    const int n = (int)(pq / Q);
    const int ho = q / Wo, wo = q % Wo;
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    const float a0 = to_f<T>(x[b * ldx + c_off + c]), a1 = to_f<T>(x[(b + 1) * ldx + c_off + c]);
    const float a2 = to_f<T>(x[(b + W) * ldx + c_off + c]), a3 = to_f<T>(x[(b + W + 1) * ldx + c_off + c]);
    const float m = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
    pooled[i] = from_f<T>(m);
    if (pooledT) pooledT[((long long)n * C + c) * Q + q] = from_f<T>(m);
  }
}
template <typename T>
__global__ void k_maxpool2_split_bwd(const T* __restrict__ x, int N, int H, int W, int ldx, int c_off, int C,
                                     const float* __restrict__ dp, T* __restrict__ dx) {
  const int Ho = H >> 1, Wo = W >> 1, Q = Ho * Wo;
  const long long total = (long long)N * Q * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const long long pq = i / C;
    const int q = (int)(pq % Q);
    const int n = (int)(pq / Q);
    const int ho = q / Wo, wo = q % Wo;
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    const long long idx[4] = {b, b + 1, b + W, b + W + 1};
    // first maximum in row-major scan wins (R7)
    int arg = 0;
    float best = to_f<T>(x[idx[0] * ldx + c_off + c]);
    for (int k = 1; k < 4; ++k) {
      const float v = to_f<T>(x[idx[k] * ldx + c_off + c]);
      if (v > best) { best = v; arg = k; }
    }
    const float g = dp[i];
    for (int k = 0; k < 4; ++k) dx[idx[k] * ldx + c_off + c] = from_f<T>(k == arg ? g : 0.0f);
  }
}
// 8 channels per thread (C, ldx, c_off multiples of 8, 16-byte aligned): the same per-element
// arithmetic as k_maxpool2_split / k_maxpool2_split_bwd with 16-byte accesses and 32-bit indexing
template <typename T>
__global__ void k_maxpool2_split_v(const T* __restrict__ x, int N, int H, int W, int ldx, int c_off, int C,
                                   T* __restrict__ pooled) {
  const int Ho = H >> 1, Wo = W >> 1, Q = Ho * Wo, G = C >> 3;
  const unsigned total = (unsigned)N * Q * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = (int)(i % G);
    const unsigned pq = i / G;
    const int q = (int)(pq % Q), n = (int)(pq / Q);
    const int ho = q / Wo, wo = q - ho * Wo;
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    float a0[8], a1[8], a2[8], a3[8], m[8];
    Vec8<T>::load(x + b * ldx + c_off + 8 * g, a0);
    Vec8<T>::load(x + (b + 1) * ldx + c_off + 8 * g, a1);
    Vec8<T>::load(x + (b + W) * ldx + c_off + 8 * g, a2);
    Vec8<T>::load(x + (b + W + 1) * ldx + c_off + 8 * g, a3);
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = fmaxf(fmaxf(a0[k], a1[k]), fmaxf(a2[k], a3[k]));
    Vec8<T>::store(pooled + (long long)pq * C + 8 * g, m);
  }
}
template <typename T>
__global__ void k_maxpool2_split_bwd_v(const T* __restrict__ x, int N, int H, int W, int ldx, int c_off, int C,
                                       const float* __restrict__ dp, T* __restrict__ dx) {
  const int Ho = H >> 1, Wo = W >> 1, Q = Ho * Wo, G = C >> 3;
  const unsigned total = (unsigned)N * Q * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = (int)(i % G);
    const unsigned pq = i / G;
    const int q = (int)(pq % Q), n = (int)(pq / Q);
    const int ho = q / Wo, wo = q - ho * Wo;
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    const long long idx[4] = {b, b + 1, b + W, b + W + 1};
    float a[4][8], gv[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) Vec8<T>::load(x + idx[k] * ldx + c_off + 8 * g, a[k]);
    Vec8<float>::load(dp + (long long)pq * C + 8 * g, gv);
    int arg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {   // first maximum in row-major scan wins (R7)
      float best = a[0][e];
      arg[e] = 0;
#pragma unroll
      for (int k = 1; k < 4; ++k)
        if (a[k][e] > best) { best = a[k][e]; arg[e] = k; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = arg[e] == k ? gv[e] : 0.0f;
      Vec8<T>::store(dx + idx[k] * ldx + c_off + 8 * g, o);
    }
  }
}
// one warp per row
template <typename T>
__global__ void k_softmax_rows(const float* __restrict__ S, long long rows, int cols, T* __restrict__ P) {
  const long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* s = S + row * cols;
  float mx = -INFINITY;
  for (int j = lane; j < cols; j += 32) mx = fmaxf(mx, s[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.0f;
  for (int j = lane; j < cols; j += 32) sum += __expf(s[j] - mx);
  sum = warp_sum(sum);
  const float inv = 1.0f / sum;
  for (int j = lane; j < cols; j += 32) P[row * cols + j] = from_f<T>(__expf(s[j] - mx) * inv);
}
template <typename T>
__global__ void k_softmax_bwd_rows(const float* __restrict__ S, const float* __restrict__ dP, long long rows, int cols,
                                   T* __restrict__ dS) {
  const long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* s = S + row * cols;
  const float* d = dP + row * cols;
  float mx = -INFINITY;
  for (int j = lane; j < cols; j += 32) mx = fmaxf(mx, s[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.0f, dot = 0.0f;
  for (int j = lane; j < cols; j += 32) {
    const float e = __expf(s[j] - mx);
    sum += e;
    dot = fmaf(e, d[j], dot);
  }
  sum = warp_sum(sum);
  dot = warp_sum(dot);
  const float inv = 1.0f / sum;
  dot *= inv;
  for (int j = lane; j < cols; j += 32) {
    const float p = __expf(s[j] - mx) * inv;
    dS[row * cols + j] = from_f<T>(p * (d[j] - dot));
  }
}

// ===================================================================== SN
// pass 1a: part[rc][k] = sum_{r in chunk rc} W[r][k] u[r]   (block = 128 rows x sn_cols_per_block(K)
// columns of one job; with K % 4 == 0 each thread owns 4 consecutive columns: 16-byte row loads)
__global__ void __launch_bounds__(256) k_sn_wtu(const SnJob* __restrict__ jobs, const int* __restrict__ blk_job,
                                                const int* __restrict__ blk_k0, const int* __restrict__ blk_rc) {
  const SnJob j = jobs[blk_job[blockIdx.x]];
  const int rc = blk_rc[blockIdx.x];
  const int r0 = rc * 128, r1 = min(j.rows, r0 + 128);
  __shared__ float us[128];
  if (threadIdx.x < r1 - r0) us[threadIdx.x] = j.u[r0 + threadIdx.x];
  __syncthreads();
  if ((j.K & 3) == 0) {
    const int k = blk_k0[blockIdx.x] + 4 * threadIdx.x;
    if (k >= j.K) return;
    const float* w = j.w + (long long)r0 * j.K + k;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    int r = r0;
#pragma unroll 1
    for (; r + 4 <= r1; r += 4) {   // four rows in flight per thread
      const float4 w0 = __ldg(reinterpret_cast<const float4*>(w));
      const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + j.K));
      const float4 w2 = __ldg(reinterpret_cast<const float4*>(w + 2 * (long long)j.K));
      const float4 w3 = __ldg(reinterpret_cast<const float4*>(w + 3 * (long long)j.K));
      const float u0 = us[r - r0], u1 = us[r - r0 + 1], u2 = us[r - r0 + 2], u3 = us[r - r0 + 3];
      a.x = fmaf(w3.x, u3, fmaf(w2.x, u2, fmaf(w1.x, u1, fmaf(w0.x, u0, a.x))));
      a.y = fmaf(w3.y, u3, fmaf(w2.y, u2, fmaf(w1.y, u1, fmaf(w0.y, u0, a.y))));
      a.z = fmaf(w3.z, u3, fmaf(w2.z, u2, fmaf(w1.z, u1, fmaf(w0.z, u0, a.z))));
      a.w = fmaf(w3.w, u3, fmaf(w2.w, u2, fmaf(w1.w, u1, fmaf(w0.w, u0, a.w))));
      w += 4 * (long long)j.K;
    }
    for (; r < r1; ++r) {
      const float4 w0 = __ldg(reinterpret_cast<const float4*>(w));
      const float u0 = us[r - r0];
      a.x = fmaf(w0.x, u0, a.x);
      a.y = fmaf(w0.y, u0, a.y);
      a.z = fmaf(w0.z, u0, a.z);
      a.w = fmaf(w0.w, u0, a.w);
      w += j.K;
    }
    *reinterpret_cast<float4*>(j.part + (long long)rc * j.K + k) = a;
    return;
  }
  const int k = blk_k0[blockIdx.x] + threadIdx.x;
  if (k >= j.K) return;
  float a = 0.0f;
  for (int r = r0; r < r1; ++r) a = fmaf(j.w[(long long)r * j.K + k], us[r - r0], a);
  j.part[(long long)rc * j.K + k] = a;
}
// pass 1b: t[k] = sum_rc part[rc][k] (fixed order)
__global__ void __launch_bounds__(256) k_sn_wtu_reduce(const SnJob* __restrict__ jobs, const int* __restrict__ blk_job,
                                                       const int* __restrict__ blk_k0) {
  const SnJob j = jobs[blk_job[blockIdx.x]];
  if ((j.K & 3) == 0) {
    const int k = blk_k0[blockIdx.x] + 4 * threadIdx.x;
    if (k >= j.K) return;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8   // loads issued ahead, additions still in rc order
    for (int rc = 0; rc < j.nrc; ++rc) {
      const float4 p = __ldg(reinterpret_cast<const float4*>(j.part + (long long)rc * j.K + k));
      a.x += p.x;
      a.y += p.y;
      a.z += p.z;
      a.w += p.w;
    }
    *reinterpret_cast<float4*>(j.t + k) = a;
    return;
  }
  const int k = blk_k0[blockIdx.x] + threadIdx.x;
  if (k >= j.K) return;
  float a = 0.0f;
#pragma unroll 8
  for (int rc = 0; rc < j.nrc; ++rc) a += __ldg(j.part + (long long)rc * j.K + k);
  j.t[k] = a;
}
// pass 2: s[r] = sum_k W[r][k] t[k] / ||t||   (block = 8 rows, one warp per row, 16-byte loads)
__global__ void __launch_bounds__(256) k_sn_wv(const SnJob* __restrict__ jobs, const int* __restrict__ blk_job,
                                               const int* __restrict__ blk_r0) {
  const SnJob j = jobs[blk_job[blockIdx.x]];
  __shared__ float red[8];
  __shared__ float s_inv;
  const bool v4 = (j.K & 3) == 0;
  // ||t|| (every block recomputes it: K <= 14k floats from L2)
  float q = 0.0f;
  if (v4) {
    for (int k = threadIdx.x; k < (j.K >> 2); k += 256) {
      const float4 t = reinterpret_cast<const float4*>(j.t)[k];
      q = fmaf(t.x, t.x, fmaf(t.y, t.y, fmaf(t.z, t.z, fmaf(t.w, t.w, q))));
    }
  } else {
    for (int k = threadIdx.x; k < j.K; k += 256) q = fmaf(j.t[k], j.t[k], q);
  }
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.0f;
    for (int i = 0; i < 8; ++i) a += red[i];
    s_inv = 1.0f / fmaxf(sqrtf(a), j.eps);
  }
  __syncthreads();
  const float inv = s_inv;
  const int r = blk_r0[blockIdx.x] + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (blk_r0[blockIdx.x] == 0) {  // one block per job writes v
    for (int k = threadIdx.x; k < j.K; k += 256) j.v[k] = j.t[k] * inv;
  }
  if (r >= j.rows) return;
  float a = 0.0f;
  if (v4) {
    const float4* w = reinterpret_cast<const float4*>(j.w + (long long)r * j.K);
    const float4* t = reinterpret_cast<const float4*>(j.t);
    for (int k = lane; k < (j.K >> 2); k += 32) {
      const float4 x = __ldg(w + k), y = t[k];
      a = fmaf(x.x, y.x, fmaf(x.y, y.y, fmaf(x.z, y.z, fmaf(x.w, y.w, a))));
    }
  } else {
    for (int k = lane; k < j.K; k += 32) a = fmaf(j.w[(long long)r * j.K + k], j.t[k], a);
  }
  a = warp_sum(a);
  if (lane == 0) j.s[r] = a * inv;
}
// pass 3: sigma = ||s||, u = s / ||s||   (one block per job)
__global__ void k_sn_finish(const SnJob* __restrict__ jobs) {
  const SnJob j = jobs[blockIdx.x];
  __shared__ float red[8];
  __shared__ float s_n;
  float q = 0.0f;
  for (int r = threadIdx.x; r < j.rows; r += 256) q = fmaf(j.s[r], j.s[r], q);
  q = warp_sum(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.0f;
    for (int i = 0; i < 8; ++i) a += red[i];
    s_n = sqrtf(a);
    j.sigma[0] = s_n;   // sigma = u'^T W v = ||W v||
    j.sigma[1] = 1.0f / fmaxf(s_n, j.eps);
  }
  __syncthreads();
  const float inv = 1.0f / fmaxf(s_n, j.eps);
  for (int r = threadIdx.x; r < j.rows; r += 256) j.u[r] = j.s[r] * inv;
}
constexpr int kSnPackItems = 4;
__global__ void __launch_bounds__(256) k_sn_pack(const SnPack* __restrict__ jobs, const long long* __restrict__ blk_start,
                                                 int n_jobs) {
  // find job by binary search over block starts
  int lo = 0, hi = n_jobs - 1;
  const long long b = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (blk_start[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const SnPack J = jobs[lo];
  const int n = J.rows * J.taps * J.cin;   // < 2^31 for every weight of the model
  if (J.vec8) {   // 8 consecutive input channels per item: two float4 loads, one 16-byte bf16 store;
                  // kSnPackItems items per thread so the job search above is paid once per 8192 elements
    const float inv = J.sigma[1];
    const int base = (int)(b - blk_start[lo]) * (kSnPackItems * 256) + threadIdx.x;
    float4 a0[kSnPackItems], a1[kSnPackItems];
#pragma unroll
    for (int u = 0; u < kSnPackItems; ++u) {
      const int i = (base + u * 256) * 8;
      if (i < n) {
        a0[u] = *reinterpret_cast<const float4*>(J.w + i);
        a1[u] = *reinterpret_cast<const float4*>(J.w + i + 4);
      }
    }
#pragma unroll
    for (int u = 0; u < kSnPackItems; ++u) {
      const int i = (base + u * 256) * 8;
      if (i >= n) break;
      const int c = i % J.cin, rt = i / J.cin;
      const int t = rt % J.taps, o = rt / J.taps;
      const long long d = ((long long)(o + J.dst_row_offset) * J.taps + t) * J.dst_cin + c;
      uint4 q;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(a0[u].x * inv, a0[u].y * inv);
      __nv_bfloat162 h1 = __floats2bfloat162_rn(a0[u].z * inv, a0[u].w * inv);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(a1[u].x * inv, a1[u].y * inv);
      __nv_bfloat162 h3 = __floats2bfloat162_rn(a1[u].z * inv, a1[u].w * inv);
      q.x = *reinterpret_cast<uint32_t*>(&h0);
      q.y = *reinterpret_cast<uint32_t*>(&h1);
      q.z = *reinterpret_cast<uint32_t*>(&h2);
      q.w = *reinterpret_cast<uint32_t*>(&h3);
      *reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(J.dst) + d) = q;
    }
    return;
  }
  const int i = (int)(b - blk_start[lo]) * 256 + threadIdx.x;
  if (i >= n) return;
  const float v = J.w[i] * J.sigma[1];
  long long d;
  if (J.mode == 0 && J.dst_cin == J.cin) {   // same layout: a scaled, converted copy
    d = (long long)J.dst_row_offset * J.taps * J.cin + i;
  } else {
    const int c = i % J.cin;
    const int rt = i / J.cin;
    const int t = rt % J.taps;
    const int o = rt / J.taps;
    if (J.mode == 1) {  // dgrad layout [cin][taps-1-t][rows]
      d = ((long long)c * J.taps + (J.taps - 1 - t)) * J.dst_rows + (o + J.dst_row_offset);
    } else {
      d = ((long long)(o + J.dst_row_offset) * J.taps + t) * J.dst_cin + c;
    }
  }
  if (J.dst_bf16) reinterpret_cast<bf16*>(J.dst)[d] = __float2bfloat16_rn(v);
  else reinterpret_cast<float*>(J.dst)[d] = v;
}
// dgrad-layout pack: reads W[o][t][c] along c, writes Wt[c][T-1-t][o] along o (both coalesced).
// vec8 jobs (rows, dst_rows, row offset % 8 == 0, cin % 4 == 0, bf16): one block = (job, t, 64-o tile,
// 64-c tile) staged through shared memory, 16-byte float4 loads and 16-byte (8 x bf16) stores; other
// jobs: 32x32 tiles, scalar.
__global__ void __launch_bounds__(256) k_sn_pack_t(const SnPack* __restrict__ jobs, const long long* __restrict__ blk_start,
                                                   int n_jobs) {
  __shared__ float tile[64][65];
  int lo = 0, hi = n_jobs - 1;
  const long long b = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (blk_start[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const SnPack J = jobs[lo];
  const float inv = J.sigma[1];
  long long r = b - blk_start[lo];
  if (J.vec8) {
    const int ot = (J.rows + 63) / 64, ct = (J.cin + 63) / 64;
    const int cti = (int)(r % ct);
    r /= ct;
    const int oti = (int)(r % ot);
    const int t = (int)(r / ot);
    const int o0 = oti * 64, c0 = cti * 64;
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int ol = i >> 4, c4 = (i & 15) * 4;
      const int o = o0 + ol, c = c0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (o < J.rows && c < J.cin) v = __ldg(reinterpret_cast<const float4*>(J.w + ((long long)o * J.taps + t) * J.cin + c));
      tile[ol][c4] = v.x * inv;
      tile[ol][c4 + 1] = v.y * inv;
      tile[ol][c4 + 2] = v.z * inv;
      tile[ol][c4 + 3] = v.w * inv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * 8; i += 256) {
      const int cl = i >> 3, og = (i & 7) * 8;
      const int c = c0 + cl, o = o0 + og;
      if (c < J.cin && o < J.rows) {
        uint4 q;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(tile[og][cl], tile[og + 1][cl]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(tile[og + 2][cl], tile[og + 3][cl]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(tile[og + 4][cl], tile[og + 5][cl]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(tile[og + 6][cl], tile[og + 7][cl]);
        q.x = *reinterpret_cast<uint32_t*>(&h0);
        q.y = *reinterpret_cast<uint32_t*>(&h1);
        q.z = *reinterpret_cast<uint32_t*>(&h2);
        q.w = *reinterpret_cast<uint32_t*>(&h3);
        const long long d = ((long long)c * J.taps + (J.taps - 1 - t)) * J.dst_rows + (o + J.dst_row_offset);
        *reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(J.dst) + d) = q;
      }
    }
    return;
  }
  const int ot = (J.rows + 31) / 32, ct = (J.cin + 31) / 32;
  const int cti = (int)(r % ct);
  r /= ct;
  const int oti = (int)(r % ot);
  const int t = (int)(r / ot);
  const int o0 = oti * 32, c0 = cti * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int o = o0 + k, c = c0 + tx;
    tile[k][tx] = (o < J.rows && c < J.cin) ? J.w[((long long)o * J.taps + t) * J.cin + c] * inv : 0.0f;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int c = c0 + k, o = o0 + tx;
    if (c < J.cin && o < J.rows) {
      const long long d = ((long long)c * J.taps + (J.taps - 1 - t)) * J.dst_rows + (o + J.dst_row_offset);
      const float v = tile[tx][k];
      if (J.dst_bf16) reinterpret_cast<bf16*>(J.dst)[d] = __float2bfloat16_rn(v);
      else reinterpret_cast<float*>(J.dst)[d] = v;
    }
  }
}
// SN backward, pass a: per-block fp64 partial of <g, W> over 4096 elements of one job
__device__ __forceinline__ int find_job(const long long* __restrict__ start, int n, long long b) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}
__global__ void __launch_bounds__(256) k_snb_dot(const SnJob* __restrict__ jobs, const long long* __restrict__ start,
                                                 int n_jobs, double* __restrict__ dotp) {
  __shared__ double red[8];
  const int ji = find_job(start, n_jobs, blockIdx.x);
  const SnJob j = jobs[ji];
  const long long n = (long long)j.rows * j.K;
  const long long e0 = (blockIdx.x - start[ji]) * 4096;
  double a = 0.0;
  for (long long i = e0 + threadIdx.x; i < min(n, e0 + 4096); i += 256) a += (double)j.grad[i] * (double)j.w[i];
  a = warp_sum_d(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    dotp[blockIdx.x] = t;
  }
}
// pass b: coef = <g, W> / sigma^2; one warp per job: lane l sums partials l, l + 32, ... in order,
// then a fixed shuffle tree (deterministic)
__global__ void k_snb_coef(const SnJob* __restrict__ jobs, int n_jobs, const double* __restrict__ dotp) {
  const int ji = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (ji >= n_jobs) return;
  const SnJob j = jobs[ji];
  double t = 0.0;
  for (long long b = lane; b < j.bwd_nblk; b += 32) t += dotp[j.bwd_blk0 + b];
  t = warp_sum_d(t);
  if (lane == 0) {
    const double is = (double)j.sigma[1];
    j.coef[0] = t * is * is;
  }
}
// pass c: g = g / sigma - coef * u[r] * v[k]   (float4 when K % 4 == 0: the 4 elements share a row)
__global__ void __launch_bounds__(256) k_snb_apply(const SnJob* __restrict__ jobs, const long long* __restrict__ start,
                                                   int n_jobs) {
  const int ji = find_job(start, n_jobs, blockIdx.x);
  const SnJob j = jobs[ji];
  const int n = j.rows * j.K;   // < 2^31 for every weight of the model
  const int e0 = (int)(blockIdx.x - start[ji]) * 4096;
  const int e1 = min(n, e0 + 4096);
  const float c = (float)j.coef[0], inv = j.sigma[1];
  if ((j.K & 3) == 0 && ((reinterpret_cast<uintptr_t>(j.grad) | reinterpret_cast<uintptr_t>(j.v)) & 15) == 0) {
    for (int i = e0 + 4 * threadIdx.x; i < e1; i += 1024) {
      const int r = i / j.K, k = i - r * j.K;
      float4 g = *reinterpret_cast<float4*>(j.grad + i);
      const float4 vv = *reinterpret_cast<const float4*>(j.v + k);
      const float cu = c * j.u[r];
      g.x = g.x * inv - cu * vv.x;
      g.y = g.y * inv - cu * vv.y;
      g.z = g.z * inv - cu * vv.z;
      g.w = g.w * inv - cu * vv.w;
      *reinterpret_cast<float4*>(j.grad + i) = g;
    }
    return;
  }
  for (int i = e0 + threadIdx.x; i < e1; i += 256) {
    const int r = i / j.K, k = i - r * j.K;
    j.grad[i] = j.grad[i] * inv - c * j.u[r] * j.v[k];
  }
}

// ===================================================================== Adam / finite / init
__global__ void k_check_finite(const float* __restrict__ g, long long n, int* flag) {
  int bad = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}
__global__ void k_check_finite_scalar(const float* loss, int* flag) {
  if (!isfinite(loss[0]) || loss[3] != 0.0f) atomicOr(flag, 1);
}
__device__ __forceinline__ float adam_one(float& w, float g, float& m, float& v, float lr, float b1, float b2,
                                          float eps, float gscale, float bc1, float bc2) {
  const float gi = g * gscale;
  const float mi = b1 * m + (1.0f - b1) * gi;
  const float vi = b2 * v + (1.0f - b2) * gi * gi;
  m = mi;
  v = vi;
  w -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  return w;
}
__global__ void k_adam(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                       long long n, float lr, float b1, float b2, float eps, const long long* __restrict__ t_dev,
                       float gscale, const int* __restrict__ flag) {
  if (*flag) return;
  const double t = (double)(*t_dev + 1);
  const float bc1 = (float)(1.0 - pow((double)b1, t)), bc2 = (float)(1.0 - pow((double)b2, t));
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(m) |
                     reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  long long done = 0;
  if (vec) {   // float4 body, scalar tail (same arithmetic per element)
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nth) {
      float4 W = reinterpret_cast<float4*>(w)[i], M = reinterpret_cast<float4*>(m)[i], V = reinterpret_cast<float4*>(v)[i];
      const float4 Gv = reinterpret_cast<const float4*>(g)[i];
      adam_one(W.x, Gv.x, M.x, V.x, lr, b1, b2, eps, gscale, bc1, bc2);
      adam_one(W.y, Gv.y, M.y, V.y, lr, b1, b2, eps, gscale, bc1, bc2);
      adam_one(W.z, Gv.z, M.z, V.z, lr, b1, b2, eps, gscale, bc1, bc2);
      adam_one(W.w, Gv.w, M.w, V.w, lr, b1, b2, eps, gscale, bc1, bc2);
      reinterpret_cast<float4*>(w)[i] = W;
      reinterpret_cast<float4*>(m)[i] = M;
      reinterpret_cast<float4*>(v)[i] = V;
    }
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nth) adam_one(w[i], g[i], m[i], v[i], lr, b1, b2, eps, gscale, bc1, bc2);
}
__global__ void k_adam_bookkeep(long long* t_dev, const int* flag, int* sticky) {
  if (*flag) *sticky = 1;
  else *t_dev += 1;
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_fill_normal(float* p, long long n, float std, uint64_t seed, uint64_t off) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed ^ mix64(off + (uint64_t)i));
    const double u1 = ((h >> 11) + 1.0) * (1.0 / 9007199254740993.0);
    const double u2 = (mix64(h) >> 11) * (1.0 / 9007199254740992.0);
    p[i] = (float)(std * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
  }
}
__global__ void k_fill_const(float* p, long long n, float v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_normalize(float* p, int n) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += (double)p[i] * p[i];
  a = warp_sum_d(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    red[0] = t;
  }
  __syncthreads();
  const float inv = (float)(1.0 / sqrt(red[0]));
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] *= inv;
}
__global__ void k_oihw_ohwi(const float* __restrict__ s, float* __restrict__ d, int O, int I, int taps, int to_ohwi) {
  const long long n = (long long)O * I * taps;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // i indexes OIHW: o, c, t
    const int t = (int)(i % taps);
    const long long oc = i / taps;
    const int c = (int)(oc % I);
    const int o = (int)(oc / I);
    const long long j = ((long long)o * taps + t) * I + c;   // OHWI
    if (to_ohwi) d[j] = s[i];
    else d[i] = s[j];
  }
}
__global__ void k_scale_dev(float* p, long long n, const float* s) {
  const float f = *s;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] *= f;
}
template <typename TA>
__global__ void k_dot(const TA* __restrict__ a, const float* __restrict__ b, long long n, float* out, int acc) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += (double)to_f<TA>(a[i]) * (double)b[i];
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    out[0] = (float)(acc ? (double)out[0] + t : t);
  }
}
__global__ void k_copy_rows_cols(const float* __restrict__ src, long long lds, long long rows, int cols,
                                 float* __restrict__ dst, long long ldd, int acc) {
  const long long total = rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols;
    const int j = (int)(i % cols);
    const float v = src[r * lds + j];
    dst[r * ldd + j] = acc ? dst[r * ldd + j] + v : v;
  }
}
__global__ void k_scale(float* p, long long n, float s) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] *= s;
}

// ---- 8-channel vector variants of the resampling kernels (C % 8 == 0, 16-byte rows)
template <typename T>
__global__ void k_relu_copy_v(const T* __restrict__ x, T* __restrict__ y, long long n8) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    float v[8];
    Vec8<T>::load(x + i * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
    Vec8<T>::store(y + i * 8, v);
  }
}
template <typename T>
__global__ void k_avgpool2_v(const T* __restrict__ x, int N, int H, int W, int C, int ldx, const T* __restrict__ add,
                             T* __restrict__ y, T* __restrict__ y_relu, T* __restrict__ x_relu) {
  const unsigned Ho = H >> 1, Wo = W >> 1, G = C >> 3;
  const unsigned total = (unsigned)N * Ho * Wo * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned g = i % G;
    unsigned p = i / G;
    const unsigned wo = p % Wo;
    p /= Wo;
    const unsigned ho = p % Ho;
    const unsigned n = p / Ho;
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    float a0[8], a1[8], a2[8], a3[8], o[8];
    Vec8<T>::load(x + b * ldx + g * 8, a0);
    Vec8<T>::load(x + (b + 1) * ldx + g * 8, a1);
    Vec8<T>::load(x + (b + W) * ldx + g * 8, a2);
    Vec8<T>::load(x + (b + W + 1) * ldx + g * 8, a3);
    if (x_relu) {   // relu(x) at full resolution from the same loads (the block's conv1 input)
      float r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = a0[j] > 0.0f ? a0[j] : 0.0f;
      Vec8<T>::store(x_relu + b * ldx + g * 8, r);
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = a1[j] > 0.0f ? a1[j] : 0.0f;
      Vec8<T>::store(x_relu + (b + 1) * ldx + g * 8, r);
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = a2[j] > 0.0f ? a2[j] : 0.0f;
      Vec8<T>::store(x_relu + (b + W) * ldx + g * 8, r);
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = a3[j] > 0.0f ? a3[j] : 0.0f;
      Vec8<T>::store(x_relu + (b + W + 1) * ldx + g * 8, r);
    }
    float ad[8];
    if (add) Vec8<T>::load(add + (long long)i * 8, ad);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      o[j] = ((a0[j] + a1[j]) + (a2[j] + a3[j])) * 0.25f;
      if (add) o[j] += ad[j];
    }
    Vec8<T>::store(y + (long long)i * 8, o);
    if (y_relu) {
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = o[j] > 0.0f ? o[j] : 0.0f;   // relu commutes with the rounding
      Vec8<T>::store(y_relu + (long long)i * 8, o);
    }
  }
}
template <typename T>
__global__ void k_avgpool2_bwd_v(const T* __restrict__ dy, int N, int H, int W, int C, const T* __restrict__ add,
                                 T* __restrict__ dx, int lddx) {
  // one thread per (output-grad pixel of the pooled map, 8 channels): writes its 2x2 block
  const unsigned Ho = H >> 1, Wo = W >> 1, G = C >> 3;
  const unsigned total = (unsigned)N * Ho * Wo * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned g = i % G;
    unsigned p = i / G;
    const unsigned wo = p % Wo;
    p /= Wo;
    const unsigned ho = p % Ho;
    const unsigned n = p / Ho;
    float v[8];
    Vec8<T>::load(dy + (long long)i * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] *= 0.25f;
    const long long b = ((long long)n * H + 2 * ho) * W + 2 * wo;
    const long long q[4] = {b, b + 1, b + W, b + W + 1};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float o[8];
      if (add) {
        Vec8<T>::load(add + q[k] * C + g * 8, o);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += v[j];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = v[j];
      }
      Vec8<T>::store(dx + q[k] * lddx + g * 8, o);
    }
  }
}
template <typename T>
__global__ void k_up2_bwd_v(const T* __restrict__ dy, int N, int H, int W, int C, T* __restrict__ dx) {
  const unsigned G = C >> 3;
  const unsigned total = (unsigned)N * H * W * G;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned g = i % G;
    unsigned p = i / G;
    const unsigned w = p % (unsigned)W;
    p /= (unsigned)W;
    const unsigned h = p % (unsigned)H;
    const unsigned n = p / (unsigned)H;
    const long long W2 = 2 * W;
    const long long b = ((long long)n * 2 * H + 2 * h) * W2 + 2 * w;
    float a0[8], a1[8], a2[8], a3[8], o[8];
    Vec8<T>::load(dy + b * C + g * 8, a0);
    Vec8<T>::load(dy + (b + 1) * C + g * 8, a1);
    Vec8<T>::load(dy + (b + W2) * C + g * 8, a2);
    Vec8<T>::load(dy + (b + W2 + 1) * C + g * 8, a3);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (a0[j] + a1[j]) + (a2[j] + a3[j]);
    Vec8<T>::store(dx + (long long)i * 8, o);
  }
}

}  // namespace

// ============================================================================ launchers
template <typename TD>
cudaError_t layout_pack(const float* src, TD* dst, int n, int c, int h, int w, int c_pad, long long off,
                        cudaStream_t st) {
  const long long total = (long long)n * h * w * c_pad;
  k_pack<TD><<<grid_for(total, 256), 256, 0, st>>>(src, dst + off, n, c, h, w, c_pad);
  return cudaGetLastError();
}
template <typename TS>
cudaError_t layout_unpack(const TS* src, float* dst, int n, int c, int h, int w, int c_pad, cudaStream_t st) {
  const long long total = (long long)n * h * w * c;
  k_unpack<TS><<<grid_for(total, 256), 256, 0, st>>>(src, dst, n, c, h, w, c_pad);
  return cudaGetLastError();
}
template cudaError_t layout_pack<float>(const float*, float*, int, int, int, int, int, long long, cudaStream_t);
template cudaError_t layout_pack<bf16>(const float*, bf16*, int, int, int, int, int, long long, cudaStream_t);
template cudaError_t layout_unpack<float>(const float*, float*, int, int, int, int, int, cudaStream_t);
template cudaError_t layout_unpack<bf16>(const bf16*, float*, int, int, int, int, int, cudaStream_t);

cudaError_t gemm_f32(int M, int N, int K, const float* A, long long sam, long long sak, const float* B, long long sbn,
                     long long sbk, float* C, long long ldc, float beta, const float* bias, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 g(ceil_div(N, 64), ceil_div(M, 64), 1);
  k_gemm<float, float><<<g, 256, 0, st>>>(M, N, K, A, 0, sam, sak, B, 0, sbn, sbk, C, 0, ldc, beta, bias);
  return cudaGetLastError();
}
int gemm_grouped_plan(GemmProblem* probs, int nprob) {
  int t = 0;
  for (int i = 0; i < nprob; ++i) {
    probs[i].tile0 = t;
    t += ceil_div(probs[i].M, 64) * ceil_div(probs[i].N, 64);
  }
  return t;
}
cudaError_t gemm_f32_grouped(const GemmProblem* probs_dev, int nprob, int total_tiles, cudaStream_t st) {
  if (total_tiles <= 0) return cudaSuccess;
  k_gemm_grouped<<<total_tiles, 256, 0, st>>>(probs_dev, nprob);
  return cudaGetLastError();
}
cudaError_t gemm_f32_batched(int batch, int M, int N, int K, const float* A, long long sab, long long sam,
                             long long sak, const float* B, long long sbb, long long sbn, long long sbk, float* C,
                             long long scb, long long ldc, float beta, cudaStream_t st) {
  dim3 g(ceil_div(N, 64), ceil_div(M, 64), batch);
  k_gemm<float, float><<<g, 256, 0, st>>>(M, N, K, A, sab, sam, sak, B, sbb, sbn, sbk, C, scb, ldc, beta, nullptr);
  return cudaGetLastError();
}
cudaError_t gemm_bf16_batched(int batch, int M, int N, int K, const bf16* A, long long sab, long long sam,
                              long long sak, const bf16* B, long long sbb, long long sbn, long long sbk, void* C,
                              bool c_f32, long long scb, long long ldc, cudaStream_t st) {
  dim3 g(ceil_div(N, 64), ceil_div(M, 64), batch);
  if (c_f32)
    k_gemm<bf16, float><<<g, 256, 0, st>>>(M, N, K, A, sab, sam, sak, B, sbb, sbn, sbk, static_cast<float*>(C), scb,
                                           ldc, 0.0f, nullptr);
  else
    k_gemm<bf16, bf16><<<g, 256, 0, st>>>(M, N, K, A, sab, sam, sak, B, sbb, sbn, sbk, static_cast<bf16*>(C), scb,
                                          ldc, 0.0f, nullptr);
  return cudaGetLastError();
}

template <typename TD>
cudaError_t convert_f32(const float* s, TD* d, long long n, cudaStream_t st) {
  k_convert<TD><<<grid_for(n, 256), 256, 0, st>>>(s, d, n);
  return cudaGetLastError();
}
template cudaError_t convert_f32<float>(const float*, float*, long long, cudaStream_t);
template cudaError_t convert_f32<bf16>(const float*, bf16*, long long, cudaStream_t);
template <typename TS>
cudaError_t to_f32(const TS* s, float* d, long long n, cudaStream_t st) {
  k_to_f32<TS><<<grid_for(n, 256), 256, 0, st>>>(s, d, n);
  return cudaGetLastError();
}
template cudaError_t to_f32<float>(const float*, float*, long long, cudaStream_t);
template cudaError_t to_f32<bf16>(const bf16*, float*, long long, cudaStream_t);

cudaError_t gather_rows(const float* table, const int32_t* idx, int n, int dim, float* out, int ldo, cudaStream_t st) {
  k_gather_rows<<<grid_for((long long)n * dim, 256), 256, 0, st>>>(table, idx, n, dim, out, ldo);
  return cudaGetLastError();
}
cudaError_t copy_cols(const float* src, int lds, int n, int cols, float* dst, int ldd, cudaStream_t st) {
  k_copy_cols<<<grid_for((long long)n * cols, 256), 256, 0, st>>>(src, lds, n, cols, dst, ldd);
  return cudaGetLastError();
}
cudaError_t scatter_add_rows_multi(const RowSrcs& srcs, int lds, const int32_t* idx, int n, int dim, int table_rows,
                                   float* dtable, cudaStream_t st) {
  if (srcs.n < 1 || srcs.n > 8) return cudaErrorInvalidValue;
  dim3 g(ceil_div(dim, 128), table_rows);
  k_scatter_add_rows_multi<<<g, 128, 0, st>>>(srcs, lds, idx, n, dim, dtable);
  return cudaGetLastError();
}
cudaError_t scatter_add_rows(const float* src, int lds, const int32_t* idx, int n, int dim, float* dtable,
                             cudaStream_t st) {
  k_scatter_add_rows<<<ceil_div(dim, 128), 128, 0, st>>>(src, lds, idx, n, dim, dtable);
  return cudaGetLastError();
}

template <typename T>
cudaError_t bn_stats(const T* x, long long M, int C, double* partial, int max_blocks, double* sums, cudaStream_t st) {
  if (C % 8 || C / 8 > 256) return cudaErrorInvalidValue;
  const int R = 256 / (C / 8);
  // ~8 pixels per thread row: wide layers at low resolution (C = 1536, R = 1) get enough blocks
  long long nb = M / (8LL * R);
  if (nb < 1) nb = 1;
  if (nb > max_blocks) nb = max_blocks;
  const int nblk = (int)nb;
  const long long per = (M + nblk - 1) / nblk;
  const size_t sm = (size_t)R * 2 * C * sizeof(double);
  if (sm > 48 * 1024) PG_CUDA(cudaFuncSetAttribute(k_bn_stats<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_bn_stats<T><<<nblk, 256, sm, st>>>(x, M, C, partial, per);
  PG_LAUNCH_CHECK();
  k_reduce_partials<<<ceil_div(2 * C, 8), 256, 0, st>>>(partial, nblk, 2 * C, sums);
  return cudaGetLastError();
}
template cudaError_t bn_stats<float>(const float*, long long, int, double*, int, double*, cudaStream_t);
template cudaError_t bn_stats<bf16>(const bf16*, long long, int, double*, int, double*, cudaStream_t);

cudaError_t bn_finalize(const double* sums, int C, double count, float eps, float* mean, float* rstd, cudaStream_t st) {
  k_bn_finalize<<<ceil_div(C, 256), 256, 0, st>>>(sums, C, count, eps, mean, rstd);
  return cudaGetLastError();
}

template <typename TI, typename TO>
cudaError_t bn_apply_relu(const TI* x, int N, int H, int W, int C, const float* mean, const float* rstd,
                          const float* gain, const float* bias, const float* gamma, const float* beta, TO* y, bool up2,
                          cudaStream_t st) {
  const long long total = (long long)N * H * W * (C / 8);
  const int G = C / 8;
  static const int bulk_on = getenv("PARAGAN_BN_BULK") ? atoi(getenv("PARAGAN_BN_BULK")) : 1;
  if (bulk_on && !up2 && C % 8 == 0 && G <= 256 && (long long)C * sizeof(TI) <= kBnChunkBytes &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
    const int lanes = 256 / G;
    const long long P = (long long)N * H * W;
    const long long cmax = kBnChunkBytes / ((long long)C * sizeof(TI));
    const long long cpix = cmax >= lanes ? cmax / lanes * lanes : cmax;
    long long blocks = (P + cpix - 1) / cpix;
    if (blocks > 4LL * sm_cap()) blocks = 4LL * sm_cap();
    k_bn_apply_relu_bulk<TI, TO><<<(unsigned)blocks, lanes * G, 0, st>>>(x, P, H * W, C, mean, rstd,
                                                                         BnAffine{gain, bias, gamma, beta}, y);
    return cudaGetLastError();
  }
  if (!up2 && C % 8 == 0 && G <= 256) {
    const int lanes = 256 / G;
    const long long P = (long long)N * H * W;
    long long blocks = (P + 2LL * lanes - 1) / (2LL * lanes);
    if (blocks > 8LL * sm_cap()) blocks = 8LL * sm_cap();
    k_bn_apply_relu_cs<TI, TO><<<(unsigned)blocks, lanes * G, 0, st>>>(x, P, H * W, C, mean, rstd,
                                                                       BnAffine{gain, bias, gamma, beta}, y);
    return cudaGetLastError();
  }
  k_bn_apply_relu<TI, TO><<<grid_for(total, 256), 256, 0, st>>>(x, N, H, W, C, mean, rstd,
                                                                BnAffine{gain, bias, gamma, beta}, y, up2 ? 1 : 0);
  return cudaGetLastError();
}
template cudaError_t bn_apply_relu<float, float>(const float*, int, int, int, int, const float*, const float*,
                                                 const float*, const float*, const float*, const float*, float*, bool,
                                                 cudaStream_t);
template cudaError_t bn_apply_relu<bf16, bf16>(const bf16*, int, int, int, int, const float*, const float*,
                                               const float*, const float*, const float*, const float*, bf16*, bool,
                                               cudaStream_t);
template cudaError_t bn_apply_relu<bf16, float>(const bf16*, int, int, int, int, const float*, const float*,
                                                const float*, const float*, const float*, const float*, float*, bool,
                                                cudaStream_t);

cudaError_t bn_apply_relu_split(const bf16* x, int N, int H, int W, int C, const float* mean, const float* rstd,
                                const float* gamma, const float* beta, bf16* y2, cudaStream_t st) {
  const int G = C / 8;
  if (C % 8 || G > 256 || (long long)C * 2 > kBnChunkBytes ||
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y2)) & 15))
    return cudaErrorInvalidValue;
  const int lanes = 256 / G;
  const long long P = (long long)N * H * W;
  const long long cmax = kBnChunkBytes / ((long long)C * 2);
  const long long cpix = cmax >= lanes ? cmax / lanes * lanes : cmax;
  long long blocks = (P + cpix - 1) / cpix;
  if (blocks > 4LL * sm_cap()) blocks = 4LL * sm_cap();
  k_bn_apply_relu_bulk<bf16, Bf16Split><<<(unsigned)blocks, lanes * G, 0, st>>>(
      x, P, H * W, C, mean, rstd, BnAffine{nullptr, nullptr, gamma, beta}, reinterpret_cast<Bf16Split*>(y2));
  return cudaGetLastError();
}

template <typename TI, typename TG>
cudaError_t bn_bwd_reduce(const TI* x, const TG* dy, int N, int H, int W, int C, const float* mean, const float* rstd,
                          const float* gain, const float* bias, const float* gamma, const float* beta, bool up2,
                          float* partial, int chunks, float* AB, cudaStream_t st) {
  if (C % 8 || C / 8 > 256) return cudaErrorInvalidValue;
  const int R = 256 / (C / 8);
  const size_t sm = (size_t)R * 2 * C * sizeof(float);
  if (sm > 48 * 1024)
    PG_CUDA(cudaFuncSetAttribute(k_bn_bwd_reduce<TI, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  dim3 g(chunks, N);
  static const int bulk_on = getenv("PARAGAN_BN_BULK") ? atoi(getenv("PARAGAN_BN_BULK")) : 1;
  const long long per_pix = (long long)C * (sizeof(TI) + sizeof(TG));
  if (bulk_on && !up2 && per_pix <= kBnChunkBytes && sm <= 32 * 1024 &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) & 15) == 0) {
    // (each thread's pixel order restarts per 16 KB sub-chunk: a different, still fixed, summation order)
    PG_CUDA(cudaFuncSetAttribute(k_bn_bwd_reduce_bulk<TI, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int cmax = (int)(kBnChunkBytes / per_pix);
    const int cpix = cmax >= R ? cmax / R * R : cmax;   // whole rounds of the R pixel lanes
    k_bn_bwd_reduce_bulk<TI, TG><<<g, 256, sm, st>>>(x, dy, N, H, W, C, cpix, mean, rstd,
                                                     BnAffine{gain, bias, gamma, beta}, partial, chunks);
  } else {
    k_bn_bwd_reduce<TI, TG><<<g, 256, sm, st>>>(x, dy, N, H, W, C, mean, rstd, BnAffine{gain, bias, gamma, beta},
                                                up2 ? 1 : 0, partial, chunks);
  }
  PG_LAUNCH_CHECK();
  k_bn_bwd_fold<<<grid_for((long long)N * 2 * C, 256), 256, 0, st>>>(partial, N, chunks, C, AB);
  return cudaGetLastError();
}
template cudaError_t bn_bwd_reduce<float, float>(const float*, const float*, int, int, int, int, const float*,
                                                 const float*, const float*, const float*, const float*, const float*,
                                                 bool, float*, int, float*, cudaStream_t);
template cudaError_t bn_bwd_reduce<bf16, bf16>(const bf16*, const bf16*, int, int, int, int, const float*, const float*,
                                               const float*, const float*, const float*, const float*, bool, float*, int,
                                               float*, cudaStream_t);
template cudaError_t bn_bwd_reduce<bf16, float>(const bf16*, const float*, int, int, int, int, const float*,
                                                const float*, const float*, const float*, const float*, const float*,
                                                bool, float*, int, float*, cudaStream_t);

cudaError_t bn_bwd_totals(const float* AB, int N, int C, const float* gain, const float* gamma, double* tot,
                          cudaStream_t st) {
  k_bn_bwd_totals<<<ceil_div(C, 32), 256, 0, st>>>(AB, N, C, gain, gamma, tot);
  return cudaGetLastError();
}

template <typename TI, typename TG, typename TO>
cudaError_t bn_bwd_apply(const TI* x, const TG* dy, int N, int H, int W, int C, const float* mean, const float* rstd,
                         const float* gain, const float* bias, const float* gamma, const float* beta, bool up2,
                         const double* tot, double count, const TO* add, TO* dx, cudaStream_t st) {
  // tot (all-reduced channel sums, fp64) -> per-channel means in fp32, kept in the tail of tot's buffer
  float* mgrad = reinterpret_cast<float*>(const_cast<double*>(tot) + 2 * C);
  k_bn_bwd_means<<<ceil_div(2 * C, 256), 256, 0, st>>>(tot, C, count, mgrad);
  PG_LAUNCH_CHECK();
  const long long total = (long long)N * H * W * (C / 8);
  const int G = C / 8;
  static const int bulk_on = getenv("PARAGAN_BN_BULK") ? atoi(getenv("PARAGAN_BN_BULK")) : 1;
  const long long per_pix = (long long)C * (sizeof(TI) + sizeof(TG) + (add ? sizeof(TO) : 0));
  if (bulk_on && !up2 && C % 8 == 0 && G <= 256 && per_pix <= kBnChunkBytes &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(add) |
        reinterpret_cast<uintptr_t>(dx)) & 15) == 0) {
    const int lanes = 256 / G;
    const long long P = (long long)N * H * W;
    const int cmax = (int)(kBnChunkBytes / per_pix);
    const int cpix = cmax >= lanes ? cmax / lanes * lanes : cmax;   // whole rounds of the pixel lanes
    long long blocks = (P + cpix - 1) / cpix;
    if (blocks > 4LL * sm_cap()) blocks = 4LL * sm_cap();
    k_bn_bwd_apply_bulk<TI, TG, TO><<<(unsigned)blocks, lanes * G, 0, st>>>(
        x, dy, P, H * W, C, cpix, mean, rstd, BnAffine{gain, bias, gamma, beta}, mgrad, add, dx);
    return cudaGetLastError();
  }
  if (!up2 && C % 8 == 0 && G <= 256) {
    const int lanes = 256 / G;
    const long long P = (long long)N * H * W;
    long long blocks = (P + lanes - 1) / lanes;
    if (blocks > 8LL * sm_cap()) blocks = 8LL * sm_cap();
    k_bn_bwd_apply_cs<TI, TG, TO><<<(unsigned)blocks, lanes * G, 0, st>>>(
        x, dy, P, H * W, C, mean, rstd, BnAffine{gain, bias, gamma, beta}, mgrad, add, dx);
    return cudaGetLastError();
  }
  k_bn_bwd_apply<TI, TG, TO><<<grid_for(total, 256), 256, 0, st>>>(
      x, dy, N, H, W, C, mean, rstd, BnAffine{gain, bias, gamma, beta}, up2 ? 1 : 0, mgrad, add, dx);
  return cudaGetLastError();
}
template cudaError_t bn_bwd_apply<float, float, float>(const float*, const float*, int, int, int, int, const float*,
                                                       const float*, const float*, const float*, const float*,
                                                       const float*, bool, const double*, double, const float*, float*,
                                                       cudaStream_t);
template cudaError_t bn_bwd_apply<bf16, bf16, bf16>(const bf16*, const bf16*, int, int, int, int, const float*,
                                                    const float*, const float*, const float*, const float*,
                                                    const float*, bool, const double*, double, const bf16*, bf16*,
                                                    cudaStream_t);
template cudaError_t bn_bwd_apply<bf16, float, bf16>(const bf16*, const float*, int, int, int, int, const float*,
                                                     const float*, const float*, const float*, const float*,
                                                     const float*, bool, const double*, double, const bf16*, bf16*,
                                                     cudaStream_t);

#define PG_INST_T(T)                                                                                               \
  template cudaError_t relu_copy<T>(const T*, T*, long long, cudaStream_t);                                        \
  template cudaError_t relu_bwd<T>(const T*, const T*, const T*, T*, long long, cudaStream_t);                     \
  template cudaError_t avgpool2<T>(const T*, int, int, int, int, int, const T*, T*, cudaStream_t, T*, T*);                 \
  template cudaError_t avgpool2_bwd<T>(const T*, int, int, int, int, const T*, T*, int, cudaStream_t);             \
  template cudaError_t up2_bwd<T>(const T*, int, int, int, int, T*, cudaStream_t);                                 \
  template cudaError_t col_sum<T>(const T*, long long, int, double*, int, float*, int, cudaStream_t);              \
  template cudaError_t tanh_to_image<T>(const float*, float*, T*, long long, int, cudaStream_t);                   \
  template cudaError_t tanh_bwd<T>(const T*, int, const float*, float*, long long, cudaStream_t);                  \
  template cudaError_t d_head_fwd<T>(const T*, int, int, int, const float*, const float*, const float*,            \
                                     const int32_t*, float*, float*, cudaStream_t);                                \
  template cudaError_t d_head_bwd<T>(const T*, int, int, int, const float*, const float*, const int32_t*,          \
                                     const float*, const float*, T*, float*, float*, float*, int, bool,            \
                                     cudaStream_t);                                                                \
  template cudaError_t maxpool2_split<T>(const T*, int, int, int, int, int, int, T*, T*, cudaStream_t);            \
  template cudaError_t maxpool2_split_bwd<T>(const T*, int, int, int, int, int, int, const float*, T*,             \
                                             cudaStream_t);                                                        \
  template cudaError_t softmax_rows<T>(const float*, long long, int, T*, cudaStream_t);                            \
  template cudaError_t softmax_bwd_rows<T>(const float*, const float*, long long, int, T*, cudaStream_t);

template <typename T>
cudaError_t relu_copy(const T* x, T* y, long long n, cudaStream_t st) {
  if (n % 8 == 0 && !((uintptr_t)x & 15) && !((uintptr_t)y & 15)) {
    k_relu_copy_v<T><<<grid_for(n / 8, 256), 256, 0, st>>>(x, y, n / 8);
    return cudaGetLastError();
  }
  k_relu_copy<T><<<grid_for(n, 256), 256, 0, st>>>(x, y, n);
  return cudaGetLastError();
}
template <typename T>
cudaError_t relu_bwd(const T* dy, const T* ref, const T* add, T* dx, long long n, cudaStream_t st) {
  k_relu_bwd<T><<<grid_for(n, 256), 256, 0, st>>>(dy, ref, add, dx, n);
  return cudaGetLastError();
}
template <typename T>
cudaError_t avgpool2(const T* x, int N, int H, int W, int C, int ldx, const T* add, T* y, cudaStream_t st,
                     T* y_relu, T* x_relu) {
  const long long total = (long long)N * (H / 2) * (W / 2) * C;
  if (C % 8 == 0 && ldx % 8 == 0) {
    k_avgpool2_v<T><<<grid_for(total / 8, 256), 256, 0, st>>>(x, N, H, W, C, ldx, add, y, y_relu, x_relu);
    return cudaGetLastError();
  }
  k_avgpool2<T><<<grid_for(total, 256), 256, 0, st>>>(x, N, H, W, C, ldx, add, y);
  PG_LAUNCH_CHECK();
  if (y_relu) {
    const cudaError_t e = relu_copy<T>(y, y_relu, total, st);
    if (e != cudaSuccess) return e;
  }
  if (x_relu) return relu_copy<T>(x, x_relu, (long long)N * H * W * C, st);   // (scalar path: ldx == C only)
  return cudaGetLastError();
}
template <typename T>
cudaError_t avgpool2_bwd(const T* dy, int N, int H, int W, int C, const T* add, T* dx, int lddx, cudaStream_t st) {
  const long long total = (long long)N * H * W * C;
  if (C % 8 == 0 && lddx % 8 == 0 && H % 2 == 0 && W % 2 == 0) {
    k_avgpool2_bwd_v<T><<<grid_for(total / 32, 256), 256, 0, st>>>(dy, N, H, W, C, add, dx, lddx);
    return cudaGetLastError();
  }
  k_avgpool2_bwd<T><<<grid_for(total, 256), 256, 0, st>>>(dy, N, H, W, C, add, dx, lddx);
  return cudaGetLastError();
}
template <typename T>
cudaError_t up2_bwd(const T* dy, int N, int H, int W, int C, T* dx, cudaStream_t st) {
  const long long total = (long long)N * H * W * C;
  if (C % 8 == 0) {
    k_up2_bwd_v<T><<<grid_for(total / 8, 256), 256, 0, st>>>(dy, N, H, W, C, dx);
    return cudaGetLastError();
  }
  k_up2_bwd<T><<<grid_for(total, 256), 256, 0, st>>>(dy, N, H, W, C, dx);
  return cudaGetLastError();
}
template <typename T>
cudaError_t col_sum(const T* dy, long long M, int C, double* partial, int max_blocks, float* db, int accumulate,
                    cudaStream_t st) {
  if (M <= 1024 && C >= 1024) {   // short and wide (e.g. the G linear's bias): a thread per column
    k_col_sum_tall<T><<<ceil_div(C, 256), 256, 0, st>>>(dy, M, C, db, accumulate);
    return cudaGetLastError();
  }
  int nblk = (int)((M + 1023) / 1024);
  if (nblk > max_blocks) nblk = max_blocks;
  const long long per = (M + nblk - 1) / nblk;
  if (C <= 8) {
    k_col_sum_small<T><<<nblk, 256, 0, st>>>(dy, M, C, partial, per);
  } else if (C % 8 == 0 && C / 8 <= 256) {
    const int R = 256 / (C / 8);
    const size_t sm = (size_t)R * C * sizeof(float);
    if (sm > 48 * 1024)
      PG_CUDA(cudaFuncSetAttribute(k_col_sum_vec<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_col_sum_vec<T><<<nblk, 256, sm, st>>>(dy, M, C, partial, per);
  } else {
    k_col_sum<T><<<nblk, 256, 256 * sizeof(double), st>>>(dy, M, C, partial, per);
  }
  PG_LAUNCH_CHECK();
  k_reduce_partials_f32<<<ceil_div(C, 8), 256, 0, st>>>(partial, nblk, C, db, accumulate);
  return cudaGetLastError();
}
template <typename T>
cudaError_t tanh_to_image(const float* pre, float* img, T* dst, long long M, int c_pad, cudaStream_t st) {
  k_tanh_to_image<T><<<grid_for(M, 256), 256, 0, st>>>(pre, img, dst, M, c_pad);
  return cudaGetLastError();
}
template <typename T>
cudaError_t tanh_bwd(const T* dimg, int c_pad, const float* img, float* dpre, long long M, cudaStream_t st) {
  k_tanh_bwd<T><<<grid_for(M * 3, 256), 256, 0, st>>>(dimg, c_pad, img, dpre, M);
  return cudaGetLastError();
}
template <typename T>
cudaError_t d_head_fwd(const T* h, int N, int HW, int C, const float* w_lin, const float* b_lin, const float* embed,
                       const int32_t* y, float* feat, float* logits, cudaStream_t st) {
  k_d_head_fwd<T><<<N, 256, 0, st>>>(h, HW, C, w_lin, b_lin, embed, y, feat, logits);
  return cudaGetLastError();
}
cudaError_t hinge_loss(const float* logits, int B, int mode, float* dlogits, float* loss_out, cudaStream_t st) {
  k_hinge<<<1, 256, 0, st>>>(logits, B, mode, dlogits, loss_out);
  return cudaGetLastError();
}
template <typename T>
cudaError_t d_head_bwd(const T* h, int N, int HW, int C, const float* w_lin, const float* embed, const int32_t* y,
                       const float* feat, const float* dlogits, T* dh, float* dw_lin, float* db_lin, float* dembed,
                       int n_classes, bool want_wgrad, cudaStream_t st) {
  (void)n_classes;
  const long long total = (long long)N * HW * C;
  k_d_head_bwd_dh<T><<<grid_for(total, 256), 256, 0, st>>>(h, N, HW, C, w_lin, embed, y, dlogits, dh);
  PG_LAUNCH_CHECK();
  if (want_wgrad) {
    if (N > kHeadMaxN) return cudaErrorInvalidValue;
    k_d_head_bwd_w<<<ceil_div(C, 32), 256, 0, st>>>(N, C, feat, dlogits, y, dw_lin, db_lin, dembed);
    PG_LAUNCH_CHECK();
  }
  return cudaSuccess;
}
template <typename T>
cudaError_t maxpool2_split(const T* x, int N, int H, int W, int ldx, int c_off, int C, T* pooled, T* pooledT,
                           cudaStream_t st) {
  const long long total = (long long)N * (H / 2) * (W / 2) * C;
  const bool vec = !pooledT && C % 8 == 0 && ldx % 8 == 0 && c_off % 8 == 0 &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(pooled)) & 15) == 0 && total < (1LL << 32);
  if (vec) {
    k_maxpool2_split_v<T><<<grid_for(total / 8, 256), 256, 0, st>>>(x, N, H, W, ldx, c_off, C, pooled);
    return cudaGetLastError();
  }
  k_maxpool2_split<T><<<grid_for(total, 256), 256, 0, st>>>(x, N, H, W, ldx, c_off, C, pooled, pooledT);
  return cudaGetLastError();
}
template <typename T>
cudaError_t maxpool2_split_bwd(const T* x, int N, int H, int W, int ldx, int c_off, int C, const float* dpooled, T* dx,
                               cudaStream_t st) {
  const long long total = (long long)N * (H / 2) * (W / 2) * C;
  const bool vec = C % 8 == 0 && ldx % 8 == 0 && c_off % 8 == 0 &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dx) |
                     reinterpret_cast<uintptr_t>(dpooled)) & 15) == 0 && total < (1LL << 32);
  if (vec) {
    k_maxpool2_split_bwd_v<T><<<grid_for(total / 8, 256), 256, 0, st>>>(x, N, H, W, ldx, c_off, C, dpooled, dx);
    return cudaGetLastError();
  }
  k_maxpool2_split_bwd<T><<<grid_for(total, 256), 256, 0, st>>>(x, N, H, W, ldx, c_off, C, dpooled, dx);
  return cudaGetLastError();
}
template <typename T>
cudaError_t softmax_rows(const float* S, long long rows, int cols, T* P, cudaStream_t st) {
  k_softmax_rows<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(S, rows, cols, P);
  return cudaGetLastError();
}
template <typename T>
cudaError_t softmax_bwd_rows(const float* S, const float* dP, long long rows, int cols, T* dS, cudaStream_t st) {
  k_softmax_bwd_rows<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(S, dP, rows, cols, dS);
  return cudaGetLastError();
}
PG_INST_T(float)
PG_INST_T(bf16)

template <typename TI, typename TW, typename TO>
cudaError_t simt_conv_fwd(const TI* x, int N, int H, int W, int Cin, const TW* w, int Cout, int ksz, const float* bias,
                          const float* alpha, const TO* residual, int res_mode, TO* y, cudaStream_t st,
                          const TO* relu_ref) {
  const long long M = (long long)N * H * W;
  if (Cout <= 8) {
    dim3 g(ceil_div(M, 256), ceil_div(Cout, 4));
    k_simt_conv<TI, TW, TO, 256, 4, 1, 4><<<g, 256, 0, st>>>(x, N, H, W, Cin, w, Cout, ksz, bias, alpha, residual,
                                                             res_mode, y, relu_ref);
  } else {
    dim3 g(ceil_div(M, 64), ceil_div(Cout, 64));
    k_simt_conv<TI, TW, TO, 64, 64, 4, 4><<<g, 256, 0, st>>>(x, N, H, W, Cin, w, Cout, ksz, bias, alpha, residual,
                                                             res_mode, y, relu_ref);
  }
  return cudaGetLastError();
}
template cudaError_t simt_conv_fwd<float, float, float>(const float*, int, int, int, int, const float*, int, int,
                                                        const float*, const float*, const float*, int, float*,
                                                        cudaStream_t, const float*);

template <typename TI, typename TG>
cudaError_t simt_conv_wgrad(const TI* x, const TG* dy, int N, int H, int W, int Cin, int Cout, int ksz, float* dw,
                            int accumulate, cudaStream_t st, float* scratch, size_t scratch_floats) {
  const long long M = (long long)N * H * W;
  const int taps = ksz * ksz;
  const long long n_out = (long long)Cout * taps * Cin;
  const bool small = Cout <= 4;
  const int TO = small ? 4 : 64, TC = small ? 256 : 64;
  const int cblocks = ceil_div(Cin, TC);
  const int tiles = ceil_div(Cout, TO) * taps * cblocks;
  int splits = ceil_div(4 * kNumSMs, tiles);
  const long long max_splits = (M + 255) / 256;
  if (splits > max_splits) splits = (int)max_splits;
  if (splits < 1) splits = 1;
  if (!scratch) splits = 1;
  while (splits > 1 && (size_t)splits * n_out > scratch_floats) --splits;
  const long long per = ((M + splits - 1) / splits + 15) / 16 * 16;
  splits = (int)((M + per - 1) / per);
  // partials [splits][n_out] in scratch (or dw directly when one split and no accumulation)
  const bool direct = splits == 1 && !accumulate;
  float* out = direct ? dw : scratch;
  if (!direct && (size_t)splits * n_out > scratch_floats) return cudaErrorInvalidValue;
  dim3 g(ceil_div(Cout, TO), taps * cblocks, splits);
  if (small)
    k_simt_wgrad<TI, TG, 4, 256, 1, 4><<<g, 256, 0, st>>>(x, dy, N, H, W, Cin, Cout, ksz, out, per);
  else
    k_simt_wgrad<TI, TG, 64, 64, 4, 4><<<g, 256, 0, st>>>(x, dy, N, H, W, Cin, Cout, ksz, out, per);
  PG_LAUNCH_CHECK();
  if (!direct) {
    k_simt_split_sum<<<grid_for(n_out, 256), 256, 0, st>>>(scratch, dw, n_out, splits, accumulate);
    PG_LAUNCH_CHECK();
  }
  return cudaSuccess;
}
template cudaError_t simt_conv_wgrad<float, float>(const float*, const float*, int, int, int, int, int, int, float*,
                                                   int, cudaStream_t, float*, size_t);

cudaError_t sn_power(const SnJob* jobs, int n_jobs, const int* b1_job, const int* b1_k0, const int* b1_rc, int n_b1,
                     const int* b1b_job, const int* b1b_k0, int n_b1b, const int* b2_job, const int* b2_r0, int n_b2,
                     cudaStream_t st) {
  k_sn_wtu<<<n_b1, 256, 0, st>>>(jobs, b1_job, b1_k0, b1_rc);
  PG_LAUNCH_CHECK();
  k_sn_wtu_reduce<<<n_b1b, 256, 0, st>>>(jobs, b1b_job, b1b_k0);
  PG_LAUNCH_CHECK();
  k_sn_wv<<<n_b2, 256, 0, st>>>(jobs, b2_job, b2_r0);
  PG_LAUNCH_CHECK();
  k_sn_finish<<<n_jobs, 256, 0, st>>>(jobs);
  return cudaGetLastError();
}
long long sn_pack_prepare(SnPack& j) {
  const long long n = (long long)j.rows * j.taps * j.cin;
  j.vec8 = j.mode == 0 && j.dst_bf16 && j.cin % 8 == 0 && j.dst_cin % 8 == 0 &&
           ((reinterpret_cast<uintptr_t>(j.w) | reinterpret_cast<uintptr_t>(j.dst)) & 15) == 0;
  return ceil_div(n, j.vec8 ? 2048 * kSnPackItems : 256);
}
long long sn_pack_t_prepare(SnPack& j) {
  j.vec8 = j.mode == 1 && j.dst_bf16 && j.rows % 8 == 0 && j.dst_rows % 8 == 0 && j.dst_row_offset % 8 == 0 &&
           j.cin % 4 == 0 && ((reinterpret_cast<uintptr_t>(j.w) | reinterpret_cast<uintptr_t>(j.dst)) & 15) == 0;
  if (j.vec8) return (long long)j.taps * ceil_div(j.rows, 64) * ceil_div(j.cin, 64);
  return (long long)j.taps * ceil_div(j.rows, 32) * ceil_div(j.cin, 32);
}
cudaError_t sn_pack(const SnPack* jobs, const long long* blk_start, int n_jobs, long long total_blocks,
                    cudaStream_t st) {
  k_sn_pack<<<(unsigned)total_blocks, 256, 0, st>>>(jobs, blk_start, n_jobs);
  return cudaGetLastError();
}
cudaError_t sn_pack_t(const SnPack* jobs, const long long* blk_start, int n_jobs, long long total_blocks,
                      cudaStream_t st) {
  k_sn_pack_t<<<(unsigned)total_blocks, 256, 0, st>>>(jobs, blk_start, n_jobs);
  return cudaGetLastError();
}
cudaError_t sn_backward(const SnJob* jobs, int n_jobs, const long long* blk_start, long long total_blocks,
                        double* dotp, cudaStream_t st) {
  k_snb_dot<<<(unsigned)total_blocks, 256, 0, st>>>(jobs, blk_start, n_jobs, dotp);
  PG_LAUNCH_CHECK();
  k_snb_coef<<<ceil_div(n_jobs, 4), 128, 0, st>>>(jobs, n_jobs, dotp);
  PG_LAUNCH_CHECK();
  k_snb_apply<<<(unsigned)total_blocks, 256, 0, st>>>(jobs, blk_start, n_jobs);
  return cudaGetLastError();
}
cudaError_t check_finite(const float* g, long long n, int* flag, cudaStream_t st) {
  k_check_finite<<<grid_for(n, 256, 4), 256, 0, st>>>(g, n, flag);
  return cudaGetLastError();
}
cudaError_t check_finite_scalar(const float* loss, int* flag, cudaStream_t st) {
  k_check_finite_scalar<<<1, 1, 0, st>>>(loss, flag);
  return cudaGetLastError();
}
cudaError_t adam_flat(float* w, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
                      float eps, const long long* t_dev, float gscale, const int* flag, cudaStream_t st) {
  k_adam<<<grid_for(n, 256, 4), 256, 0, st>>>(w, g, m, v, n, lr, b1, b2, eps, t_dev, gscale, flag);
  return cudaGetLastError();
}
cudaError_t adam_bookkeep(long long* t_dev, const int* flag, int* sticky, cudaStream_t st) {
  k_adam_bookkeep<<<1, 1, 0, st>>>(t_dev, flag, sticky);
  return cudaGetLastError();
}
cudaError_t fill_normal(float* p, long long n, float std, uint64_t seed, uint64_t off, cudaStream_t st) {
  k_fill_normal<<<grid_for(n, 256), 256, 0, st>>>(p, n, std, seed, off);
  return cudaGetLastError();
}
cudaError_t fill_const(float* p, long long n, float v, cudaStream_t st) {
  k_fill_const<<<grid_for(n, 256), 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}
cudaError_t normalize_vec(float* p, int n, cudaStream_t st) {
  k_normalize<<<1, 1024, 0, st>>>(p, n);
  return cudaGetLastError();
}
cudaError_t oihw_to_ohwi(const float* s, float* d, int O, int I, int taps, cudaStream_t st) {
  k_oihw_ohwi<<<grid_for((long long)O * I * taps, 256), 256, 0, st>>>(s, d, O, I, taps, 1);
  return cudaGetLastError();
}
cudaError_t ohwi_to_oihw(const float* s, float* d, int O, int I, int taps, cudaStream_t st) {
  k_oihw_ohwi<<<grid_for((long long)O * I * taps, 256), 256, 0, st>>>(s, d, O, I, taps, 0);
  return cudaGetLastError();
}
cudaError_t scale_dev(float* p, long long n, const float* s, cudaStream_t st) {
  k_scale_dev<<<grid_for(n, 256), 256, 0, st>>>(p, n, s);
  return cudaGetLastError();
}
cudaError_t dot_f32(const float* a, const float* b, long long n, float* out, int accumulate, cudaStream_t st) {
  k_dot<float><<<1, 1024, 0, st>>>(a, b, n, out, accumulate);
  return cudaGetLastError();
}
cudaError_t dot_bf16_f32(const bf16* a, const float* b, long long n, float* out, int accumulate, cudaStream_t st) {
  k_dot<bf16><<<1, 1024, 0, st>>>(a, b, n, out, accumulate);
  return cudaGetLastError();
}
cudaError_t copy_rows_cols(const float* src, long long lds, long long rows, int cols, float* dst, long long ldd,
                           int accumulate, cudaStream_t st) {
  k_copy_rows_cols<<<grid_for(rows * cols, 256), 256, 0, st>>>(src, lds, rows, cols, dst, ldd, accumulate);
  return cudaGetLastError();
}
cudaError_t scale_f32(float* p, long long n, float s, cudaStream_t st) {
  k_scale<<<grid_for(n, 256), 256, 0, st>>>(p, n, s);
  return cudaGetLastError();
}

}  // namespace pg

// ============================================================================
// Thin fp32 convolution (C_out <= 4): G's output layer 96 -> 3 (P:202 keeps it
// fp32).  A 3x3 halo tile of the input is staged once per channel chunk in
// shared memory (channel-major planes, padded to a bank-conflict-free stride),
// so each input element is read from HBM once per tile instead of once per tap.
// ============================================================================
namespace pg {
namespace {
// ---------------------------------------------------------------------------
// fprop: y[m][o] = bias[o] + sum_{tap,c} x[m+tap][c] w[o][tap][c]
// tile 32 rows x 64 cols, thread = 8 consecutive pixels of one row (acc[8][CO] in registers);
// 4-channel halo chunks staged in smem ([c][row][68] planes), software-pipelined: the global loads of
// chunk c+1 (9 x 16 bytes per thread, held in registers) are in flight while chunk c is computed, so
// the DRAM latency hides behind the FMA loop; weights as [c][28] so each channel's 27 taps x outputs
// come in 7 broadcast float4 loads; rows slide through 3 float4s.
constexpr int kFTH = 32, kFTW = 64, kFCC = 4, kFRS = 68;
constexpr int kFPlane = (kFTH + 2) * kFRS;
constexpr int kFItems = (kFTH + 2) * (kFTW + 2);          // 16-byte items per chunk (one per halo pixel)
constexpr int kFPre = (kFItems + 255) / 256;              // per thread
template <int CO>
__global__ void __launch_bounds__(256, 2) k_thin_fwd(const float* __restrict__ x, int N, int H, int W, int C,
                                                  const float* __restrict__ w, const float* __restrict__ bias,
                                                  float* __restrict__ y) {
  extern __shared__ float4 sm4[];
  float* ws = reinterpret_cast<float*>(sm4);   // [C][28]
  float* xs = ws + C * 28;                      // [kFCC][kFPlane]
  const int tiles_w = (W + kFTW - 1) / kFTW, tiles_h = (H + kFTH - 1) / kFTH;
  int t = blockIdx.x;
  const int tw = t % tiles_w;
  t /= tiles_w;
  const int th = t % tiles_h;
  const int n = t / tiles_h;
  const int h0 = th * kFTH, w0 = tw * kFTW;
  for (int i = threadIdx.x; i < C * 28; i += blockDim.x) {
    const int c = i / 28, k = i - c * 28;
    ws[i] = k < CO * 9 ? w[(long long)k * C + c] : 0.0f;
  }
  const int py = threadIdx.x >> 3, px0 = (threadIdx.x & 7) * 8;
  float acc[8][CO];
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int o = 0; o < CO; ++o) acc[p][o] = 0.0f;
  float4 pre[kFPre];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int u = 0; u < kFPre; ++u) {
      const int i = threadIdx.x + u * 256;
      pre[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < kFItems) {
        const int sx = i % (kFTW + 2), r = i / (kFTW + 2);
        const int h = h0 - 1 + r, ww = w0 - 1 + sx;
        if (h >= 0 && h < H && ww >= 0 && ww < W && c0 < C)
          pre[u] = __ldg(reinterpret_cast<const float4*>(x + (((long long)n * H + h) * W + ww) * C + c0));
      }
    }
  };
  fetch(0);
  for (int c0 = 0; c0 < C; c0 += kFCC) {
    __syncthreads();   // the previous chunk's planes are no longer read
#pragma unroll
    for (int u = 0; u < kFPre; ++u) {
      const int i = threadIdx.x + u * 256;
      if (i < kFItems) {
        const int sx = i % (kFTW + 2), r = i / (kFTW + 2);
        float* d = xs + r * kFRS + sx;
        d[0] = pre[u].x;
        d[kFPlane] = pre[u].y;
        d[2 * kFPlane] = pre[u].z;
        d[3 * kFPlane] = pre[u].w;
      }
    }
    __syncthreads();
    if (c0 + kFCC < C) fetch(c0 + kFCC);   // in flight during the FMA loop below
    const int cc = min(kFCC, C - c0);
    for (int c = 0; c < cc; ++c) {
      const float* plane = xs + c * kFPlane;
      float wv[28];
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const float4 q = *reinterpret_cast<const float4*>(ws + (c0 + c) * 28 + 4 * k);
        wv[4 * k] = q.x;
        wv[4 * k + 1] = q.y;
        wv[4 * k + 2] = q.z;
        wv[4 * k + 3] = q.w;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        float xr[12];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float4 q = *reinterpret_cast<const float4*>(plane + (py + r) * kFRS + px0 + 4 * k);
          xr[4 * k] = q.x;
          xr[4 * k + 1] = q.y;
          xr[4 * k + 2] = q.z;
          xr[4 * k + 3] = q.w;
        }
#pragma unroll
        for (int sx = 0; sx < 3; ++sx)
#pragma unroll
          for (int p = 0; p < 8; ++p)
#pragma unroll
            for (int o = 0; o < CO; ++o) acc[p][o] = fmaf(xr[p + sx], wv[o * 9 + r * 3 + sx], acc[p][o]);
      }
    }
  }
  const int h = h0 + py;
  if (h >= H) return;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int ww = w0 + px0 + p;
    if (ww >= W) break;
    const long long m = ((long long)n * H + h) * W + ww;
#pragma unroll
    for (int o = 0; o < CO; ++o) y[m * CO + o] = acc[p][o] + (bias ? bias[o] : 0.0f);
  }
}

// ---------------------------------------------------------------------------
// dgrad: dx[m][c] = sum_{o,r,s} dy[h+1-r][w+1-s][o] w[o][r][s][c]  (transposed 3x3, pad 1)
// Thread = (input channel c, pixel group): its 27 weights w[.][.][.][c] live in registers and it
// walks 4-pixel row chunks of the tile; the dy halo ([10][34] pixels x 4, the 3 channels padded) is
// staged per tile with cp.async (double-buffered) and read as broadcast float4s (18 per chunk for
// 108 FMAs).  A warp's stores cover 32 consecutive channels of one pixel: fully coalesced.
constexpr int kDTH = 8, kDTW = 32;
__device__ __forceinline__ void cp_async4_zfill(float* dst, const float* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
// CPT channels per thread (c and c + C/CPT): each broadcast dy load then feeds CPT x 27 FMAs
template <int CO, int CPT>
__global__ void __launch_bounds__(CPT == 1 ? 384 : 192, CPT == 1 ? 2 : 3) k_thin_dgrad(const float* __restrict__ dy, int N, int H, int W, int C,
                                                       const float* __restrict__ w, float* __restrict__ dx) {
  constexpr int HR = kDTH + 2, HC = kDTW + 2, kHalo = HR * HC;
  __shared__ float4 ds[2][kHalo];
  const int tiles_w = (W + kDTW - 1) / kDTW, tiles_h = (H + kDTH - 1) / kDTH;
  const int tiles = N * tiles_h * tiles_w;
  const int Ct = C / CPT;   // threads per pixel group
  const int c = threadIdx.x % Ct, pg = threadIdx.x / Ct, npg = blockDim.x / Ct;
  float wv[CPT][CO * 9];   // wv[j][o*9 + r*3 + s] = w[o][r][s][c + j*Ct]
#pragma unroll
  for (int j = 0; j < CPT; ++j)
#pragma unroll
    for (int k = 0; k < CO * 9; ++k) wv[j][k] = w[(long long)k * C + c + j * Ct];
  auto stage = [&](int t, int buf) {
    int u = t;
    const int tw = u % tiles_w;
    u /= tiles_w;
    const int th = u % tiles_h;
    const int n = u / tiles_h;
    const int h0 = th * kDTH, w0 = tw * kDTW;
    float* d = reinterpret_cast<float*>(ds[buf]);
    for (int i = threadIdx.x; i < kHalo * CO; i += blockDim.x) {
      const int o = i % CO, rs = i / CO;
      const int sx = rs % HC, r = rs / HC;
      const int h = h0 - 1 + r, ww = w0 - 1 + sx;
      const bool ok = h >= 0 && h < H && ww >= 0 && ww < W;
      cp_async4_zfill(d + rs * 4 + o, ok ? dy + (((long long)n * H + h) * W + ww) * CO + o : dy, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  if (blockIdx.x < tiles) stage(blockIdx.x, 0);
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, buf ^= 1) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();   // tile t landed for every thread; the other buffer's readers are done
    if (t + (int)gridDim.x < tiles) stage(t + gridDim.x, buf ^ 1);
    int u = t;
    const int tw = u % tiles_w;
    u /= tiles_w;
    const int th = u % tiles_h;
    const int n = u / tiles_h;
    const int h0 = th * kDTH, w0 = tw * kDTW;
    const float4* hal = ds[buf];
    for (int q = pg; q < kDTH * (kDTW / 4); q += npg) {
      const int row = q / (kDTW / 4), x0 = (q % (kDTW / 4)) * 4;
      float acc[CPT][4];
#pragma unroll
      for (int j = 0; j < CPT; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0.0f;
      // output (row, x0 + i) reads halo (row + 2 - r, x0 + i + 2 - s)
#pragma unroll
      for (int hr = 0; hr < 3; ++hr) {        // halo row row + hr  <->  r = 2 - hr
        const int r = 2 - hr;
#pragma unroll
        for (int cc = 0; cc < 6; ++cc) {      // halo column x0 + cc  <->  s = i + 2 - cc
          const float4 g = hal[(row + hr) * HC + x0 + cc];
          const float gv[3] = {g.x, g.y, g.z};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int sx = i + 2 - cc;
            if (sx >= 0 && sx <= 2) {
#pragma unroll
              for (int j = 0; j < CPT; ++j)
#pragma unroll
                for (int o = 0; o < CO; ++o) acc[j][i] = fmaf(gv[o], wv[j][o * 9 + r * 3 + sx], acc[j][i]);
            }
          }
        }
      }
      const int h = h0 + row;
      if (h < H) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ww = w0 + x0 + i;
          if (ww < W) {
#pragma unroll
            for (int j = 0; j < CPT; ++j) dx[(((long long)n * H + h) * W + ww) * C + c + j * Ct] = acc[j][i];
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// wgrad partials: dW[o][tap][c] over one block's pixel tiles.  Persistent blocks walk 4 x 16
// pixel tiles; thread = (channel c, tile row) keeps all 27 (o, tap) sums in registers; x is staged
// channel-innermost ([6][18][C], the global NHWC order, so 16-byte cp.async copies with zero fill
// for the padding), dy as [64][4] (one broadcast float4 per pixel), double-buffered so the next
// tile's copies fly during this tile's FMAs; the 3x3 neighbourhood slides along the row.
constexpr int kWTH = 4, kWTW = 16;
__device__ __forceinline__ void cp_async_zfill(void* dst, const void* src, int bytes_valid, int size) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (size == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes_valid) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(bytes_valid) : "memory");
}
// SPLIT: x is the two-term bf16 split [P][2C] of the fp32 activation (R36) — the same 4C bytes per pixel as
// fp32, so the staging is unchanged and each read sums the pair, x = x1 + x2, in fp32
template <int CO, bool SPLIT>
__global__ void __launch_bounds__(512) k_thin_wgrad(const float* __restrict__ x, const float* __restrict__ dy, int N,
                                                    int H, int W, int C, float* __restrict__ partial) {
  extern __shared__ float4 sm4[];
  constexpr int HC = kWTW + 2;
  const int xs_floats = (kWTH + 2) * HC * C;
  float* xs0 = reinterpret_cast<float*>(sm4);                 // 2 x [kWTH+2][kWTW+2][C]
  float* dys0 = xs0 + 2 * xs_floats;                          // 2 x [kWTH*kWTW][4]
  float* red = xs0;                                           // [kWTH-1][C][CO*9] after the loop
  const int tiles_w = (W + kWTW - 1) / kWTW, tiles_h = (H + kWTH - 1) / kWTH;
  const int tiles = N * tiles_h * tiles_w;
  const int c = threadIdx.x % C, py = threadIdx.x / C;        // blockDim = kWTH * C
  auto stage = [&](int t, int buf) {
    int u = t;
    const int tw = u % tiles_w;
    u /= tiles_w;
    const int th = u % tiles_h;
    const int n = u / tiles_h;
    const int h0 = th * kWTH, w0 = tw * kWTW;
    float* xs = xs0 + buf * xs_floats;
    // blockDim = kWTH * C = 16 * (C / 4): the vector index cv is fixed per thread, rs advances by 16
    const int cv = threadIdx.x % (C / 4);
    for (int rs = threadIdx.x / (C / 4); rs < (kWTH + 2) * HC; rs += 4 * kWTH) {
      const int sx = rs % HC, r = rs / HC;
      const int h = h0 - 1 + r, ww = w0 - 1 + sx;
      const bool ok = h >= 0 && h < H && ww >= 0 && ww < W;
      const float* src = ok ? x + (((long long)n * H + h) * W + ww) * C + cv * 4 : x;
      cp_async_zfill(xs + rs * C + cv * 4, src, ok ? 16 : 0, 16);
    }
    float* dys = dys0 + buf * kWTH * kWTW * 4;
    for (int i = threadIdx.x; i < kWTH * kWTW * CO; i += blockDim.x) {
      const int o = i % CO, p = i / CO;
      const int h = h0 + p / kWTW, ww = w0 + p % kWTW;
      const bool ok = h < H && ww < W;
      cp_async_zfill(dys + p * 4 + o, ok ? dy + (((long long)n * H + h) * W + ww) * CO + o : dy, ok ? 4 : 0, 4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float acc[CO * 9];
#pragma unroll
  for (int k = 0; k < CO * 9; ++k) acc[k] = 0.0f;
  // x at staged pixel slot q (row-major over the [kWTH+2][kWTW+2] halo), channel c
  auto xat = [&](const float* xs, int q) -> float {
    if constexpr (SPLIT) {
      const bf16* xb = reinterpret_cast<const bf16*>(xs) + (size_t)q * 2 * C + c;
      return __bfloat162float(xb[0]) + __bfloat162float(xb[C]);
    } else {
      return xs[q * C + c];
    }
  };
  int buf = 0;
  if (blockIdx.x < tiles) stage(blockIdx.x, 0);
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, buf ^= 1) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();   // this tile landed for every thread; the other buffer's readers are done
    if (t + (int)gridDim.x < tiles) stage(t + gridDim.x, buf ^ 1);
    const float* xs = xs0 + buf * xs_floats;
    const float* dys = dys0 + buf * kWTH * kWTW * 4;
    // window xw[r][s] = x[py + r][px + s][c] for the current px
    float xw[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      xw[r][0] = xat(xs, (py + r) * HC + 0);
      xw[r][1] = xat(xs, (py + r) * HC + 1);
    }
#pragma unroll
    for (int px = 0; px < kWTW; ++px) {   // fully unrolled: the window slide is register renaming, not moves
#pragma unroll
      for (int r = 0; r < 3; ++r) xw[r][2] = xat(xs, (py + r) * HC + px + 2);
      const float4 g = *reinterpret_cast<const float4*>(dys + (py * kWTW + px) * 4);
      const float gv[3] = {g.x, g.y, g.z};
#pragma unroll
      for (int o = 0; o < CO; ++o)
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int sx = 0; sx < 3; ++sx) acc[o * 9 + r * 3 + sx] = fmaf(gv[o], xw[r][sx], acc[o * 9 + r * 3 + sx]);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        xw[r][0] = xw[r][1];
        xw[r][1] = xw[r][2];
      }
    }
  }
  // combine the row groups in order 0, 1, .., kWTH-1; write this block's partial [CO*9][C]
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (py > 0)
#pragma unroll
    for (int k = 0; k < CO * 9; ++k) red[((py - 1) * C + c) * CO * 9 + k] = acc[k];
  __syncthreads();
  if (py == 0) {
    float* pb = partial + (long long)blockIdx.x * CO * 9 * C;
#pragma unroll
    for (int k = 0; k < CO * 9; ++k) {
      float s = acc[k];
      for (int g = 1; g < kWTH; ++g) s += red[((g - 1) * C + c) * CO * 9 + k];
      pb[k * C + c] = s;
    }
  }
}
__global__ void k_reduce_rows_f32(const float* __restrict__ partial, int rows, int n, float* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int r = 0; r < rows; ++r) a += partial[(long long)r * n + i];
    out[i] = (float)a;
  }
}
}  // namespace

cudaError_t sum_slices(const float* part, int nslices, int n, float* dst, cudaStream_t st) {
  k_reduce_rows_f32<<<ceil_div(n, 256), 256, 0, st>>>(part, nslices, n, dst);
  return cudaGetLastError();
}

// one thread per (o, c): the nine 3x3 taps read once, the sixteen folded (phase, tap) weights written.
// layout 0: c fastest across threads (coalesced reads and writes); layout 1: o fastest (coalesced writes)
__global__ void k_fold_up2(const float* __restrict__ w, const float* __restrict__ inv_sigma, int Cout, int Cin,
                           bf16* __restrict__ dst, int layout) {
  const long long n = (long long)Cout * Cin;
  const float is = inv_sigma[0];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int o, c;
    if (layout == 0) {
      o = (int)(i / Cin);
      c = (int)(i - (long long)o * Cin);
    } else {
      c = (int)(i / Cout);
      o = (int)(i - (long long)c * Cout);
    }
    float t9[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) t9[k] = w[((long long)o * 9 + k) * Cin + c];
#pragma unroll
    for (int ph = 0; ph < 4; ++ph) {
      const int a = ph >> 1, b = ph & 1;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int p = t >> 1, q = t & 1;
        // rows of the 3x3 kernel landing on input row offset p for phase a (same for columns)
        const int r0 = (a == 0) ? (p == 0 ? 0 : 1) : (p == 0 ? 0 : 2);
        const int r1 = (a == 0) ? (p == 0 ? 0 : 2) : (p == 0 ? 1 : 2);
        const int s0 = (b == 0) ? (q == 0 ? 0 : 1) : (q == 0 ? 0 : 2);
        const int s1 = (b == 0) ? (q == 0 ? 0 : 2) : (q == 0 ? 1 : 2);
        float acc = 0.0f;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
          for (int ss = 0; ss < 3; ++ss)
            if (rr >= r0 && rr <= r1 && ss >= s0 && ss <= s1) acc += t9[rr * 3 + ss];
        const bf16 v = __float2bfloat16_rn(acc * is);
        if (layout == 0) dst[(((long long)ph * Cout + o) * 4 + t) * Cin + c] = v;
        else dst[((long long)c * 16 + ph * 4 + t) * Cout + o] = v;
      }
    }
  }
}

// All of G's conv1 folds of one forward in one launch: 32 (o) x 32 (c) tiles; each thread reads its 9 taps
// coalesced over c, writes the fprop layout coalesced over c and stages the 16 folded values so that the
// dgrad layout ([Cin][16][Cout]) is written coalesced over o (the per-block kernel read it with a 9*Cin stride).
// Same arithmetic and summation order as k_fold_up2 (bit-identical).
__global__ void __launch_bounds__(256) k_fold_up2_grouped(const FoldJob* __restrict__ jobs, int njobs, int dgrad) {
  __shared__ bf16 st[16][32][34];
  int j = 0;
  while (j + 1 < njobs && (int)blockIdx.x >= jobs[j + 1].tile0) ++j;
  const FoldJob jb = jobs[j];
  const int t = blockIdx.x - jb.tile0;
  const int tc = (jb.Cin + 31) / 32;
  const int o0 = (t / tc) * 32, c0 = (t % tc) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const float is = jb.inv_sigma[0];
  const int c = c0 + tx;
  for (int oo = ty; oo < 32; oo += 8) {
    const int o = o0 + oo;
    if (o >= jb.Cout || c >= jb.Cin) continue;
    float t9[9];
#pragma unroll
    for (int k = 0; k < 9; ++k)
      t9[k] = jb.tf ? jb.w[((long long)c * 9 + (8 - k)) * jb.Cout + o] : jb.w[((long long)o * 9 + k) * jb.Cin + c];
#pragma unroll
    for (int ph = 0; ph < 4; ++ph) {
      const int a = ph >> 1, b = ph & 1;
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) {
        const int p = tp >> 1, q = tp & 1;
        const int r0 = (a == 0) ? (p == 0 ? 0 : 1) : (p == 0 ? 0 : 2);
        const int r1 = (a == 0) ? (p == 0 ? 0 : 2) : (p == 0 ? 1 : 2);
        const int s0 = (b == 0) ? (q == 0 ? 0 : 1) : (q == 0 ? 0 : 2);
        const int s1 = (b == 0) ? (q == 0 ? 0 : 2) : (q == 0 ? 1 : 2);
        float acc = 0.0f;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
          for (int ss = 0; ss < 3; ++ss)
            if (rr >= r0 && rr <= r1 && ss >= s0 && ss <= s1) acc += t9[rr * 3 + ss];
        const bf16 v = __float2bfloat16_rn(acc * is);
        jb.dst0[(((long long)ph * jb.Cout + o) * 4 + tp) * jb.Cin + c] = v;
        st[ph * 4 + tp][oo][tx] = v;
      }
    }
  }
  if (!dgrad) return;
  __syncthreads();
  const int o = o0 + tx;
  if (o >= jb.Cout) return;
  for (int cc = ty; cc < 32; cc += 8) {
    if (c0 + cc >= jb.Cin) break;
#pragma unroll
    for (int pt = 0; pt < 16; ++pt) jb.dst1[((long long)(c0 + cc) * 16 + pt) * jb.Cout + o] = st[pt][tx][cc];
  }
}

cudaError_t fold_up2_grouped(const FoldJob* jobs_d, int njobs, int tiles, bool dgrad, cudaStream_t st) {
  k_fold_up2_grouped<<<tiles, 256, 0, st>>>(jobs_d, njobs, dgrad ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t fold_up2_weights(const float* w, const float* inv_sigma, int Cout, int Cin, bf16* dst, cudaStream_t st,
                             int layout) {
  k_fold_up2<<<grid_for((long long)Cout * Cin, 256), 256, 0, st>>>(w, inv_sigma, Cout, Cin, dst, layout);
  return cudaGetLastError();
}

// ===================================================================== SN-DCGAN generic fp32 kernels
namespace {
__global__ void k_gconv_fwd(const float* __restrict__ x, int N, int H, int W, int Cin, const float* __restrict__ w,
                            int ldw, int Cout, int k, int s, int p, int Ho, int Wo, const float* __restrict__ bias,
                            float* __restrict__ y) {
  const long long total = (long long)N * Ho * Wo * Cout;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int co = (int)(i % Cout);
    long long r = i / Cout;
    const int ox = (int)(r % Wo);
    r /= Wo;
    const int oy = (int)(r % Ho);
    const int n = (int)(r / Ho);
    // fp64 accumulation: this config-1 path is the exact reference-grade SIMT path (R25)
    double acc = bias ? bias[co] : 0.0;
    for (int ky = 0; ky < k; ++ky) {
      const int iy = oy * s - p + ky;
      if (iy < 0 || iy >= H) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int ix = ox * s - p + kx;
        if (ix < 0 || ix >= W) continue;
        const float* xp = x + (((long long)n * H + iy) * W + ix) * Cin;
        const float* wp = w + ((long long)(co * k + ky) * k + kx) * ldw;
        for (int ci = 0; ci < Cin; ++ci) acc += (double)xp[ci] * wp[ci];
      }
    }
    y[i] = (float)acc;
  }
}
__global__ void k_gconv_dgrad(const float* __restrict__ dy, int N, int Ho, int Wo, int Cout,
                              const float* __restrict__ w, int ldw, int Cin, int k, int s, int p, int H, int W,
                              const float* __restrict__ bias, float* __restrict__ dx) {
  const long long total = (long long)N * H * W * Cin;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(i % Cin);
    long long r = i / Cin;
    const int ix = (int)(r % W);
    r /= W;
    const int iy = (int)(r % H);
    const int n = (int)(r / H);
    double acc = bias ? bias[ci] : 0.0;
    for (int ky = 0; ky < k; ++ky) {
      const int ty = iy + p - ky;
      if (ty < 0 || ty % s) continue;
      const int oy = ty / s;
      if (oy >= Ho) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int tx = ix + p - kx;
        if (tx < 0 || tx % s) continue;
        const int ox = tx / s;
        if (ox >= Wo) continue;
        const float* dp = dy + (((long long)n * Ho + oy) * Wo + ox) * Cout;
        for (int co = 0; co < Cout; ++co) acc += (double)dp[co] * w[((long long)(co * k + ky) * k + kx) * ldw + ci];
      }
    }
    dx[i] = (float)acc;
  }
}
// one block per weight element group: thread-strided sum over pixels in fp64, block reduce
__global__ void k_gconv_wgrad(const float* __restrict__ x, int N, int H, int W, int Cin, const float* __restrict__ dy,
                              int Ho, int Wo, int Cout, int k, int s, int p, float* __restrict__ dw) {
  __shared__ double red[256];
  const long long widx = blockIdx.x;   // (co, ky, kx, ci)
  const int ci = (int)(widx % Cin);
  long long r = widx / Cin;
  const int kx = (int)(r % k);
  r /= k;
  const int ky = (int)(r % k);
  const int co = (int)(r / k);
  const long long P = (long long)N * Ho * Wo;
  double acc = 0.0;
  for (long long q = threadIdx.x; q < P; q += blockDim.x) {
    const int ox = (int)(q % Wo);
    const long long t = q / Wo;
    const int oy = (int)(t % Ho);
    const int n = (int)(t / Ho);
    const int iy = oy * s - p + ky, ix = ox * s - p + kx;
    if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
    acc += (double)dy[q * Cout + co] * (double)x[(((long long)n * H + iy) * W + ix) * Cin + ci];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) dw[widx] = (float)red[0];
}
__global__ void k_lrelu_fwd(const float* __restrict__ x, float* __restrict__ y, long long n, float slope) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = x[i];
    y[i] = v > 0.0f ? v : slope * v;
  }
}
__global__ void k_lrelu_bwd(const float* __restrict__ dy, const float* __restrict__ pre, float* __restrict__ dx,
                            long long n, float slope) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dx[i] = pre[i] > 0.0f ? dy[i] : slope * dy[i];
}
// one block per channel, fp64 block reduction over the rows
__global__ void k_bn_sums_generic(const float* __restrict__ x, long long M, int C, double* __restrict__ sums) {
  __shared__ double r1[256], r2[256];
  const int c = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (long long m = threadIdx.x; m < M; m += blockDim.x) {
    const double v = x[m * C + c];
    a += v;
    b += v * v;
  }
  r1[threadIdx.x] = a;
  r2[threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      r1[threadIdx.x] += r1[threadIdx.x + o];
      r2[threadIdx.x] += r2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sums[c] = r1[0];
    sums[C + c] = r2[0];
  }
}
__global__ void k_bn_apply_generic(const float* __restrict__ x, long long M, int C, const float* __restrict__ mean,
                                   const float* __restrict__ rstd, const float* __restrict__ gamma,
                                   const float* __restrict__ beta, int relu, float* __restrict__ y) {
  const long long n = M * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    float v = (x[i] - mean[c]) * rstd[c] * gamma[c] + beta[c];
    y[i] = relu ? fmaxf(v, 0.0f) : v;
  }
}
__global__ void k_bn_bwd_sums_generic(const float* __restrict__ x, const float* __restrict__ dy, long long M, int C,
                                      const float* __restrict__ mean, const float* __restrict__ rstd,
                                      const float* __restrict__ gamma, const float* __restrict__ beta, int relu,
                                      double* __restrict__ tot, float* __restrict__ dgamma,
                                      float* __restrict__ dbeta) {
  __shared__ double r1[256], r2[256];
  const int c = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (long long m = threadIdx.x; m < M; m += blockDim.x) {
    const float xh = (x[m * C + c] - mean[c]) * rstd[c];
    float g = dy[m * C + c];
    if (relu && xh * gamma[c] + beta[c] <= 0.0f) g = 0.0f;
    a += g;
    b += (double)g * xh;
  }
  r1[threadIdx.x] = a;
  r2[threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      r1[threadIdx.x] += r1[threadIdx.x + o];
      r2[threadIdx.x] += r2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tot[c] = r1[0];
    tot[C + c] = r2[0];
    if (dbeta) dbeta[c] = (float)r1[0];
    if (dgamma) dgamma[c] = (float)r2[0];
  }
}
__global__ void k_bn_bwd_apply_generic(const float* __restrict__ x, const float* __restrict__ dy, long long M, int C,
                                       const float* __restrict__ mean, const float* __restrict__ rstd,
                                       const float* __restrict__ gamma, const float* __restrict__ beta, int relu,
                                       const double* __restrict__ tot, double count, float* __restrict__ dx) {
  const long long n = M * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const float xh = (x[i] - mean[c]) * rstd[c];
    float g = dy[i];
    if (relu && xh * gamma[c] + beta[c] <= 0.0f) g = 0.0f;
    const float mg = (float)(tot[c] / count), mgx = (float)(tot[C + c] / count);
    dx[i] = gamma[c] * rstd[c] * (g - mg - xh * mgx);
  }
}
}  // namespace

cudaError_t gconv_fwd(const float* x, int N, int H, int W, int Cin, const float* w, int ldw, int Cout, int k, int s,
                      int p, int Ho, int Wo, const float* bias, float* y, cudaStream_t st) {
  k_gconv_fwd<<<grid_for((long long)N * Ho * Wo * Cout, 256), 256, 0, st>>>(x, N, H, W, Cin, w, ldw, Cout, k, s, p, Ho,
                                                                           Wo, bias, y);
  return cudaGetLastError();
}
cudaError_t gconv_dgrad(const float* dy, int N, int Ho, int Wo, int Cout, const float* w, int ldw, int Cin, int k,
                        int s, int p, int H, int W, const float* bias, float* dx, cudaStream_t st) {
  k_gconv_dgrad<<<grid_for((long long)N * H * W * Cin, 256), 256, 0, st>>>(dy, N, Ho, Wo, Cout, w, ldw, Cin, k, s, p,
                                                                           H, W, bias, dx);
  return cudaGetLastError();
}
cudaError_t gconv_wgrad(const float* x, int N, int H, int W, int Cin, const float* dy, int Ho, int Wo, int Cout,
                        int k, int s, int p, float* dw, cudaStream_t st) {
  const long long nw = (long long)Cout * k * k * Cin;
  k_gconv_wgrad<<<(unsigned)nw, 256, 0, st>>>(x, N, H, W, Cin, dy, Ho, Wo, Cout, k, s, p, dw);
  return cudaGetLastError();
}
cudaError_t lrelu_fwd(const float* x, float* y, long long n, float slope, cudaStream_t st) {
  k_lrelu_fwd<<<grid_for(n, 256), 256, 0, st>>>(x, y, n, slope);
  return cudaGetLastError();
}
cudaError_t lrelu_bwd(const float* dy, const float* pre, float* dx, long long n, float slope, cudaStream_t st) {
  k_lrelu_bwd<<<grid_for(n, 256), 256, 0, st>>>(dy, pre, dx, n, slope);
  return cudaGetLastError();
}
cudaError_t bn_sums_generic(const float* x, long long M, int C, double* sums, cudaStream_t st) {
  k_bn_sums_generic<<<C, 256, 0, st>>>(x, M, C, sums);
  return cudaGetLastError();
}
cudaError_t bn_apply_generic(const float* x, long long M, int C, const float* mean, const float* rstd,
                             const float* gamma, const float* beta, int relu, float* y, cudaStream_t st) {
  k_bn_apply_generic<<<grid_for(M * C, 256), 256, 0, st>>>(x, M, C, mean, rstd, gamma, beta, relu, y);
  return cudaGetLastError();
}
cudaError_t bn_bwd_sums_generic(const float* x, const float* dy, long long M, int C, const float* mean,
                                const float* rstd, const float* gamma, const float* beta, int relu, double* tot,
                                float* dgamma, float* dbeta, cudaStream_t st) {
  k_bn_bwd_sums_generic<<<C, 256, 0, st>>>(x, dy, M, C, mean, rstd, gamma, beta, relu, tot, dgamma, dbeta);
  return cudaGetLastError();
}
cudaError_t bn_bwd_apply_generic(const float* x, const float* dy, long long M, int C, const float* mean,
                                 const float* rstd, const float* gamma, const float* beta, int relu, const double* tot,
                                 double count, float* dx, cudaStream_t st) {
  k_bn_bwd_apply_generic<<<grid_for(M * C, 256), 256, 0, st>>>(x, dy, M, C, mean, rstd, gamma, beta, relu, tot,
                                                               count, dx);
  return cudaGetLastError();
}

cudaError_t thin_conv_fwd(const float* x, int N, int H, int W, int C, const float* w, int CO, const float* bias,
                          float* y, cudaStream_t st) {
  if (CO != 3 || C % 4 || ((uintptr_t)x & 15)) return cudaErrorInvalidValue;
  const int tiles = N * ((H + kFTH - 1) / kFTH) * ((W + kFTW - 1) / kFTW);
  const size_t sm = (size_t)(C * 28 + kFCC * kFPlane) * sizeof(float);
  PG_CUDA(cudaFuncSetAttribute(k_thin_fwd<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_thin_fwd<3><<<tiles, 256, sm, st>>>(x, N, H, W, C, w, bias, y);
  return cudaGetLastError();
}
cudaError_t thin_conv_dgrad(const float* dy, int N, int H, int W, int C, const float* w, int CO, float* dx,
                            cudaStream_t st) {
  if (CO != 3 || C > 384) return cudaErrorInvalidValue;
  const int tiles = N * ((H + kDTH - 1) / kDTH) * ((W + kDTW - 1) / kDTW);
  static const int cpt_env = getenv("PARAGAN_THIN_DG_CPT") ? atoi(getenv("PARAGAN_THIN_DG_CPT")) : 2;
  const int cpt = (cpt_env == 2 && C % 2 == 0 && 192 % (C / 2) == 0) ? 2 : 1;
  const int Ct = C / cpt, npg = (cpt == 2 ? 192 : 384) / Ct;
  int per_sm = 1;
  if (cpt == 2) PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_thin_dgrad<3, 2>, npg * Ct, 0));
  else PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_thin_dgrad<3, 1>, npg * Ct, 0));
  if (per_sm < 1) per_sm = 1;
  const int grid = tiles < per_sm * sm_cap() ? tiles : per_sm * sm_cap();
  if (cpt == 2) k_thin_dgrad<3, 2><<<grid, npg * Ct, 0, st>>>(dy, N, H, W, C, w, dx);
  else k_thin_dgrad<3, 1><<<grid, npg * Ct, 0, st>>>(dy, N, H, W, C, w, dx);
  return cudaGetLastError();
}
cudaError_t thin_conv_wgrad(const void* x, const float* dy, int N, int H, int W, int C, int CO, float* dw,
                            float* scratch, size_t scratch_floats, cudaStream_t st, bool split) {
  if (CO != 3 || C % 4 || C > 128 || ((uintptr_t)x & 15)) return cudaErrorInvalidValue;
  const int tiles = N * ((H + kWTH - 1) / kWTH) * ((W + kWTW - 1) / kWTW);
  const size_t sm = (size_t)(2 * (kWTH + 2) * (kWTW + 2) * C + 2 * kWTH * kWTW * 4) * sizeof(float);
  int per_sm = (int)(200 * 1024 / sm);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  int grid = per_sm * kNumSMs;
  if (grid > tiles) grid = tiles;
  const int n = CO * 9 * C;
  while ((size_t)grid * n > scratch_floats && grid > 1) grid /= 2;
  const float* xf = static_cast<const float*>(x);
  if (split) {   // (the smem size depends on C: set on every call)
    PG_CUDA(cudaFuncSetAttribute(k_thin_wgrad<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_thin_wgrad<3, true><<<grid, kWTH * C, sm, st>>>(xf, dy, N, H, W, C, scratch);
  } else {
    PG_CUDA(cudaFuncSetAttribute(k_thin_wgrad<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_thin_wgrad<3, false><<<grid, kWTH * C, sm, st>>>(xf, dy, N, H, W, C, scratch);
  }
  PG_LAUNCH_CHECK();
  k_reduce_rows_f32<<<ceil_div(n, 256), 256, 0, st>>>(scratch, grid, n, dw);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Operands of G's output layer on the tensor cores (R36; tc_outconv.cu).  x (fp32) -> [x1 | x2],
// x1 = bf16(x), x2 = bf16(x - x1); w (fp32 [CO = 3][9][C]) -> w1 + w2 + w3 (w1 = bf16(w), w2 = bf16(w - w1),
// w3 = bf16(w - w1 - w2)) laid out as the B operand [96][2C] over the split A = [x1 | x2]: row
// t * 9 + term * 3 + o holds, for tap t and output o,
//   term 0: [w1 | w1]  -> x1 w1 + x2 w1
//   term 1: [w2 | w2]  -> x1 w2 + x2 w2
//   term 2: [w3 | 0 ]  -> x1 w3
// (rows 81..95 zero), so the three terms' sum drops only x2 w3 (< 2^-25 |x w|) and the split residual of x
// (|x - x1 - x2| <= 2^-18 |x|).
__global__ void k_split_planes(const float* __restrict__ x, long long P, int C, bf16* __restrict__ y) {
  const long long n = P * (C / 4);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / (C / 4);
    const int c = (int)(i - p * (C / 4)) * 4;
    const float4 v = *reinterpret_cast<const float4*>(x + p * C + c);
    const float f[4] = {v.x, v.y, v.z, v.w};
    __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      hi[j] = __float2bfloat16_rn(f[j]);
      lo[j] = __float2bfloat16_rn(f[j] - __bfloat162float(hi[j]));
    }
    *reinterpret_cast<uint2*>(y + p * 2 * C + c) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(y + p * 2 * C + C + c) = *reinterpret_cast<const uint2*>(lo);
  }
}
__global__ void k_split_out_weights(const float* __restrict__ w, int C, bf16* __restrict__ ws) {
  const int n = 96 * 2 * C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = i % (2 * C), row = i / (2 * C);
    const int t = row / 9, term = (row % 9) / 3, o = row % 3, c = k < C ? k : k - C;
    float out = 0.0f;
    if (row < 81 && !(term == 2 && k >= C)) {
      const float v = w[((size_t)o * 9 + t) * C + c];
      const float w1 = __bfloat162float(__float2bfloat16_rn(v));
      const float w2 = __bfloat162float(__float2bfloat16_rn(v - w1));
      out = term == 0 ? w1 : term == 1 ? w2 : v - w1 - w2;
    }
    ws[i] = __float2bfloat16_rn(out);
  }
}

// dgrad operand of the same layer (tc_outconv.cu): wd[c][j], j = blk * 27 + t * 3 + o over the A~ columns
// [dy1 | dy2 | dy1 | dy1], holds [w1 | w1 | w2 | w3][o][t][c]; j >= 108 and rows c >= C are zero
__global__ void k_split_out_weights_dgrad(const float* __restrict__ w, int C, int C16, bf16* __restrict__ wd) {
  const int n = C16 * 128;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = i % 128, c = i / 128;
    float out = 0.0f;
    if (j < 108 && c < C) {
      const int blk = j / 27, m = j % 27, t = m / 3, o = m % 3;
      const float v = w[((size_t)o * 9 + t) * C + c];
      const float w1 = __bfloat162float(__float2bfloat16_rn(v));
      const float w2 = __bfloat162float(__float2bfloat16_rn(v - w1));
      out = blk <= 1 ? w1 : blk == 2 ? w2 : v - w1 - w2;
    }
    wd[i] = __float2bfloat16_rn(out);
  }
}

cudaError_t split_out_weights_dgrad(const float* w, int C, int C16, bf16* wd, cudaStream_t st) {
  k_split_out_weights_dgrad<<<ceil_div(C16 * 128, 256), 256, 0, st>>>(w, C, C16, wd);
  return cudaGetLastError();
}

__global__ void k_pack_stats(const float* __restrict__ ld, const float* __restrict__ lg,
                             const long long* __restrict__ td, const long long* __restrict__ tg,
                             const int* __restrict__ nf, float inv, paragan_stats* __restrict__ out) {
  if (threadIdx.x != 0) return;
  out->d_loss = ld[0] * inv;
  out->d_real_mean = ld[1] * inv;
  out->d_fake_mean = ld[2] * inv;
  out->g_loss = lg[0] * inv;
  out->nonfinite = *nf;
  out->t_d = *td;
  out->t_g = *tg;
}
cudaError_t pack_stats(const float* ld, const float* lg, const long long* td, const long long* tg, const int* nf,
                       float inv, paragan_stats* out, cudaStream_t st) {
  k_pack_stats<<<1, 32, 0, st>>>(ld, lg, td, tg, nf, inv, out);
  return cudaGetLastError();
}

cudaError_t split_planes(const float* x, long long P, int C, bf16* y, cudaStream_t st) {
  if (C % 4 || ((uintptr_t)x & 15) || ((uintptr_t)y & 7)) return cudaErrorInvalidValue;
  k_split_planes<<<grid_for(P * (C / 4), 256), 256, 0, st>>>(x, P, C, y);
  return cudaGetLastError();
}
cudaError_t split_out_weights(const float* w, int C, bf16* ws, cudaStream_t st) {
  k_split_out_weights<<<ceil_div(96 * 2 * C, 256), 256, 0, st>>>(w, C, ws);
  return cudaGetLastError();
}

}  // namespace pg

// ============================================================================
// First D layer as a K = 27 (padded to 32) GEMM: im2col of the 3-channel image
// and its adjoint.  out[p][tap*3 + c] = x[p + delta_tap][c] (zero padding), 0 for k >= 27.
// ============================================================================
namespace pg {
namespace {
template <typename T>
__global__ void k_im2col3(const T* __restrict__ x, int N, int H, int W, int cx, T* __restrict__ out) {
  const long long total = (long long)N * H * W;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(p % W);
    const long long q = p / W;
    const int h = (int)(q % H);
    const int n = (int)(q / H);
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = 0.0f;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int hh = h + t / 3 - 1, ww = w + t % 3 - 1;
      if (hh >= 0 && hh < H && ww >= 0 && ww < W) {
        const T* src = x + (((long long)n * H + hh) * W + ww) * cx;
        if (cx == 8) {   // the padded image: one 16-byte load per neighbour (8 bf16 channels, 3 used)
          float e[8];
          Vec8<T>::load(src, e);
#pragma unroll
          for (int c = 0; c < 3; ++c) v[t * 3 + c] = e[c];
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) v[t * 3 + c] = to_f<T>(src[c]);
        }
      }
    }
    T* dst = out + p * 32;
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
      float u[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = v[k + j];
      Vec8<T>::store(dst + k, u);
    }
  }
}
// dx[p][c] = sum_tap dxi[p - delta_tap][tap*3 + c] (+ add[p][c]); channels 3..cx-1 = add or 0
template <typename T>
__global__ void k_col2im3(const T* __restrict__ dxi, int N, int H, int W, int cx, const T* __restrict__ add,
                          T* __restrict__ dx) {
  const long long total = (long long)N * H * W;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(p % W);
    const long long q = p / W;
    const int h = (int)(q % H);
    const int n = (int)(q / H);
    float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      // x[p] feeds output pixel p - delta_tap through slot tap
      const int hh = h - (t / 3 - 1), ww = w - (t % 3 - 1);
      if (hh >= 0 && hh < H && ww >= 0 && ww < W) {
        const T* src = dxi + (((long long)n * H + hh) * W + ww) * 32 + t * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += to_f<T>(src[c]);
      }
    }
    for (int c = 0; c < cx; ++c) {
      float v = c < 3 ? acc[c] : 0.0f;
      if (add) v += to_f<T>(add[p * cx + c]);
      dx[p * cx + c] = from_f<T>(v);
    }
  }
}
}  // namespace

template <typename T>
cudaError_t im2col3(const T* x, int N, int H, int W, int cx, T* out, cudaStream_t st) {
  const long long total = (long long)N * H * W;
  k_im2col3<T><<<(unsigned)std::min<long long>((total + 255) / 256, 8LL * kNumSMs), 256, 0, st>>>(x, N, H, W, cx, out);
  return cudaGetLastError();
}
template <typename T>
cudaError_t col2im3(const T* dxi, int N, int H, int W, int cx, const T* add, T* dx, cudaStream_t st) {
  const long long total = (long long)N * H * W;
  k_col2im3<T><<<(unsigned)std::min<long long>((total + 255) / 256, 8LL * kNumSMs), 256, 0, st>>>(dxi, N, H, W, cx, add,
                                                                                                  dx);
  return cudaGetLastError();
}
template cudaError_t im2col3<bf16>(const bf16*, int, int, int, int, bf16*, cudaStream_t);
template cudaError_t col2im3<bf16>(const bf16*, int, int, int, int, const bf16*, bf16*, cudaStream_t);
template cudaError_t im2col3<float>(const float*, int, int, int, int, float*, cudaStream_t);
template cudaError_t col2im3<float>(const float*, int, int, int, int, const float*, float*, cudaStream_t);

}  // namespace pg
