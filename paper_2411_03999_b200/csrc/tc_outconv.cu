// G's fp32 output layer (3x3 conv, C_out = 3) on the tcgen05 tensor cores through bf16 splits
// (reading R36 in DESIGN.md).
//
// A 3x3 conv with three outputs is a poor implicit GEMM: with N = 3 (x3 split terms) every MMA re-reads a
// 128-pixel A tile per filter tap, so the layer would be bound by the tensor core's shared-memory reads
// (9 taps x K / 16 MMAs of 4 KB each per tile).  Here the taps go into N instead:
//
//   Z[p][t][j] = sum_c xs[p][c] * ws[t*9 + j][c]          (one GEMM per 128-pixel image row, N = 81 -> 96)
//
// with xs = [x1 | x2] the two-term bf16 split of the fp32 activation (K = 2C) and ws the three-term split
// of the weight (j = term * 3 + o; term 0: [w1 | w1], 1: [w2 | w2], 2: [w3 | 0]).  A is read once per pixel
// row and per 16-wide K step.  The epilogue then does the convolution's spatial sum ("col2im"):
//
//   v[p][t][o] = Z[p][t][o] + Z[p][t][3 + o] + Z[p][t][6 + o]
//   y[h][w][o] = bias[o] + sum_{r,s} v[(h + r - 1, w + s - 1)][r*3 + s][o]
//
// Horizontal neighbours are neighbouring TMEM lanes (warp shuffles, a shared-memory hand-off between the
// four lane quadrants).  Vertical neighbours are consecutive tiles: each CTA walks a strip of kStrip output
// rows of one image top to bottom (x rows h0-1 .. h1), keeping the two open output rows' partial sums in
// registers, so every output is complete when written and nothing is re-read.  Fixed summation order
// (deterministic).  Requires W = 128 (one image row = one M tile).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_outconv.h"
#include "tc_ptx.cuh"

namespace pg {
namespace {

constexpr int kW = 128;                   // image width = M tile
constexpr int kStrip = 32;                // output rows per work unit
constexpr int kNCols = 96;                // 9 taps x 9 (term, output) columns = 81, padded to a multiple of 16
constexpr int kStages = 8;                // A ring
constexpr uint32_t kABytes = 128 * 128;   // [128 px][64 ch] bf16, SW128 K-major
constexpr uint32_t kBChunk = kNCols * 128;  // [96 rows][64 ch] bf16, SW128 K-major
constexpr int kMaxChunks = 4;             // C2 <= 256
constexpr int kThreads = 192;             // w0 TMA, w1 MMA, w2-5 epilogue (one per TMEM lane quadrant)
constexpr size_t kSmem = 1024 + kMaxChunks * kBChunk + kStages * kABytes + 2 * 4 * 2 * 9 * sizeof(float) + 256;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  return reinterpret_cast<uint8_t*>((a + 1023) & ~uintptr_t(1023));
}

struct OcArgs {
  int N, H, c_chunks, last_ksteps, strips;
  const float* bias;
  float* y;   // [N][H][128][3]
};

// unit u = (image n, strip s): x rows [max(h0 - 1, 0), min(h1, H - 1)] for output rows [h0, h1)
__device__ __forceinline__ void unit_rows(const OcArgs& a, int u, int& n, int& h0, int& h1, int& hs, int& he) {
  n = u / a.strips;
  h0 = (u - n * a.strips) * kStrip;
  h1 = min(h0 + kStrip, a.H);
  hs = max(h0 - 1, 0);
  he = min(h1, a.H - 1);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_out_conv_fwd(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const OcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sB = smem;
  uint8_t* sA = sB + kMaxChunks * kBChunk;
  float* sedge = reinterpret_cast<float*>(sA + kStages * kABytes);   // [2 bufs][4 quadrants][2 sides][9]
  uint64_t* full = reinterpret_cast<uint64_t*>(sedge + 2 * 4 * 2 * 9);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 4);
    }
    tc::mbar_init(bfull, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int units = a.N * a.strips;

  if (warp == 0) {
    if (lane == 0) {
      // the whole split weight stays resident
      tc::mbar_expect_tx(bfull, a.c_chunks * kBChunk);
      for (int cc = 0; cc < a.c_chunks; ++cc) tc::tma_load_3d(sB + cc * kBChunk, &tmB, bfull, cc * 64, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int n, h0, h1, hs, he;
        unit_rows(a, u, n, h0, h1, hs, he);
        for (int hq = hs; hq <= he; ++hq) {
          for (int cc = 0; cc < a.c_chunks; ++cc) {
            tc::mbar_wait(&empty[stage], phase ^ 1);
            tc::mbar_expect_tx(&full[stage], kABytes);
            tc::tma_load_3d(sA + stage * kABytes, &tmA, &full[stage], cc * 64, 0, n * a.H + hq);
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, kNCols, false, false);
    const bool issuer = tc::elect_one();
    tc::mbar_wait(bfull, 0);
    tc::tc_fence_after();
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int n, h0, h1, hs, he;
      unit_rows(a, u, n, h0, h1, hs, he);
      for (int hq = hs; hq <= he; ++hq, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + buf * kNCols;
        for (int cc = 0; cc < a.c_chunks; ++cc) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const int ksteps = cc == a.c_chunks - 1 ? a.last_ksteps : 4;
          if (issuer) {
            const uint64_t ad = tc::sdesc_sw128(sA0 + stage * kABytes, 16, 1024);
            const uint64_t bd = tc::sdesc_sw128(sB0 + cc * kBChunk, 16, 1024);
            for (int k = 0; k < ksteps; ++k)   // +32 bytes per K = 16 step (= 2 in the >>4 address field)
              tc::mma_bf16(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (cc | k) != 0 ? 1u : 0u);
            tc::mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (issuer) tc::mma_commit(&tfull[buf]);
        __syncwarp();
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) ..; thread = pixel column px of the current x row
    const int q = warp & 3;
    const int px = q * 32 + lane;
    float bias[3];
#pragma unroll
    for (int o = 0; o < 3; ++o) bias[o] = a.bias ? a.bias[o] : 0.0f;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int n, h0, h1, hs, he;
      unit_rows(a, u, n, h0, h1, hs, he);
      float R0[3] = {0.f, 0.f, 0.f}, R1[3] = {0.f, 0.f, 0.f};   // open output rows hq and hq + 1
      for (int hq = hs; hq <= he; ++hq, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&tfull[buf], (it >> 1) & 1);
        tc::tc_fence_after();
        float v[9][3];
        {
          float z[32];
#pragma unroll
          for (int g = 0; g < 3; ++g) {
            tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * kNCols + g * 32, z);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = g * 32 + j;
              if (col < 81) {
                const int t = col / 9, r = col % 9;
                if (r < 3) v[t][r] = z[j];
                else v[t][r % 3] += z[j];
              }
            }
          }
        }
        // the accumulator is in registers: hand the TMEM buffer back to the MMA warp
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[buf]);
        // horizontal neighbours: output px takes tap s = 0 from px - 1, s = 2 from px + 1
        float* ed = sedge + (it & 1) * (4 * 2 * 9);
        if (lane == 31) {
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int o = 0; o < 3; ++o) ed[(q * 2 + 0) * 9 + r * 3 + o] = v[r * 3 + 0][o];   // to quadrant q+1's lane 0
        }
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int o = 0; o < 3; ++o) ed[(q * 2 + 1) * 9 + r * 3 + o] = v[r * 3 + 2][o];   // to quadrant q-1's lane 31
        }
        tc::named_bar(1, 128);
        float acc[3][3];   // [r][o]: this x row's contribution to output row hq - r + 1
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int o = 0; o < 3; ++o) {
            float left = __shfl_up_sync(0xffffffffu, v[r * 3 + 0][o], 1);
            float right = __shfl_down_sync(0xffffffffu, v[r * 3 + 2][o], 1);
            if (lane == 0) left = q > 0 ? ed[((q - 1) * 2 + 0) * 9 + r * 3 + o] : 0.0f;
            if (lane == 31) right = q < 3 ? ed[((q + 1) * 2 + 1) * 9 + r * 3 + o] : 0.0f;
            acc[r][o] = (v[r * 3 + 1][o] + left) + right;
          }
        // output row hq - 1 is complete (x rows hq - 2, hq - 1, hq)
        const int ho = hq - 1;
        if (ho >= h0 && ho < h1) {
          float* yp = a.y + (((long long)n * a.H + ho) * kW + px) * 3;
#pragma unroll
          for (int o = 0; o < 3; ++o) yp[o] = (R0[o] + acc[2][o]) + bias[o];
        }
#pragma unroll
        for (int o = 0; o < 3; ++o) {
          R0[o] = R1[o] + acc[1][o];
          R1[o] = acc[0][o];
        }
      }
      if (h1 == a.H) {   // the last row has no x row below it (zero padding)
        float* yp = a.y + (((long long)n * a.H + (a.H - 1)) * kW + px) * 3;
#pragma unroll
        for (int o = 0; o < 3; ++o) yp[o] = R0[o] + bias[o];
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 256);
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;

cudaError_t encoder() {
  if (g_enc) return cudaSuccess;
  cudaDriverEntryPointQueryResult qr;
  PG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_enc), cudaEnableDefault,
                                  &qr));
  if (qr != cudaDriverEntryPointSuccess || !g_enc) return cudaErrorNotSupported;
  return cudaSuccess;
}

// 3-D bf16 map over [d2][d1][d0] (d0 contiguous), box {64, b1, 1}, 128-byte swizzle
cudaError_t map3(CUtensorMap* m, const void* base, long long d0, long long d1, long long d2, int b1) {
  PG_CUDA(encoder());
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)d0 * 2, (cuuint64_t)(d0 * d1 * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

bool out_conv_tc_ok(int H, int W, int C) { return W == kW && H >= 1 && C % 8 == 0 && 2 * C <= 64 * kMaxChunks; }

cudaError_t out_conv_fwd_tc(const void* xs, int N, int H, int W, int C, const void* ws, const float* bias, float* y,
                            cudaStream_t st) {
  if (!out_conv_tc_ok(H, W, C) || ((uintptr_t)xs & 15) || ((uintptr_t)ws & 15)) return cudaErrorInvalidValue;
  const int C2 = 2 * C;
  OcArgs a{};
  a.N = N;
  a.H = H;
  a.c_chunks = ceil_div(C2, 64);
  a.last_ksteps = ceil_div(C2 - (a.c_chunks - 1) * 64, 16);
  a.strips = ceil_div(H, kStrip);
  a.bias = bias;
  a.y = y;
  CUtensorMap ma, mb;
  PG_CUDA(map3(&ma, xs, C2, kW, (long long)N * H, kW));
  PG_CUDA(map3(&mb, ws, C2, kNCols, 1, kNCols));
  PG_CUDA((set_smem_once<k_out_conv_fwd>((int)kSmem)));
  const int units = N * a.strips;
  const int grid = units < sm_cap() ? units : sm_cap();
  k_out_conv_fwd<<<grid, kThreads, kSmem, st>>>(ma, mb, a);
  return cudaGetLastError();
}

}  // namespace pg
