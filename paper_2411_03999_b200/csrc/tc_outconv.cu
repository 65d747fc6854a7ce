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
//
// The backward shares one operand: the "im2col" of the (tiny, 3-channel) output gradient,
//   A~[q][j] = dy_b[q - d_t][o],  j = blk * 27 + t * 3 + o,  blk 0..3 = dy1, dy2, dy1, dy1   (108 -> 128)
// (dy1 = bf16(dy), dy2 = bf16(dy - dy1); d_t the tap offset; zero outside the image), built per 128-pixel
// row tile by four warps straight into shared memory, where the tensor core reads it both ways:
//   wgrad  D_w[j][n] += sum_q A~[q][j] xs[q][n]   (A MN-major over the tile's pixels, M = 128, N = 2C;
//                                                 rows j < 54 are used: dy1 and dy2 against x1 and x2)
//   dgrad  dx[q][c]   = sum_j A~[q][j] wd[c][j]   (A K-major, K = 112, N = C; wd = [w1 | w1 | w2 | w3])
// so one pass over the activation serves both gradients: x is read once, dx written once, dy read from L2.
// D_w stays in TMEM over all of a CTA's tiles; the per-CTA partials are summed (and the four split
// products folded) in a fixed order by k_out_wgrad_reduce.  (D_w is flushed into the CTA's partial every 16
// tiles: the tensor core's fp32 accumulation over a CTA's ~28k pixels otherwise drifts to ~3e-5.)
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

// the dynamic shared-memory base rounded up to 1024 bytes by pointer arithmetic on the shared array itself, so
// the compiler keeps the shared address space (LDS/STS, not generic LD/ST) for every access derived from it
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (tc::smem_u32(p) & 1023u)) & 1023u);
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

// ---------------------------------------------------------------------------------------------- backward
constexpr int kBwdThreads = 320;          // w0 TMA, w1 MMA, w2-5 build A~, w6-9 dx epilogue / dW readout
constexpr uint32_t kAtBytes = 2 * 16384;  // A~ stage: two [128 px][64] SW128 atoms (j 0..63, 64..127)
constexpr int kBlk = 4, kJ = 27 * kBlk;   // 108 real A~ columns
constexpr int kDgK = 112;                 // dgrad K (7 steps of 16; columns 108..111 are zero)
constexpr int kWRows = 54;                // D_w rows used: dy1 (27) and dy2 (27)

struct OcBwdArgs {
  int N, H, C, C16, c_chunks, tiles, tma_store;   // tma_store: dx leaves through SW128 staging + TMA stores
  // D_w flush: every `flush` tiles the accumulator (one of dw_bufs TMEM buffers) is added into the CTA's
  // partial in global memory (L2-resident), bounding the fp32 accumulation chain in TMEM; D_x has dx_bufs
  // buffers
  int flush, dw_bufs, dx_bufs;
  const float* dy;     // [N][H][128][3] fp32
  float* dx;           // [N][H][128][C] fp32
  float* partial;      // [gridDim.x][54][2C]
};

constexpr uint32_t kDxStage = 128 * 128;   // [128 px][32 fp32] SW128 dx staging tile
__host__ __device__ constexpr size_t bwd_smem(int C16, int c_chunks, int tma_store) {
  return 1024 + (size_t)2 * C16 * 128 + (size_t)2 * c_chunks * 16384 + 2 * kAtBytes + (tma_store ? 2 * kDxStage : 0) +
         256;
}

// the 27 output-gradient values A~ needs at pixel (h, px): dy at (h - rr + 1, px - ss + 1), zero outside
__device__ __forceinline__ void load_dy_window(const float* __restrict__ dy, int n, int h, int H, int px, float (&v)[27]) {
#pragma unroll
  for (int rr = 0; rr < 3; ++rr)
#pragma unroll
    for (int ss = 0; ss < 3; ++ss) {
      const int hh = h - rr + 1, ww = px - ss + 1;
      const bool ok = hh >= 0 && hh < H && ww >= 0 && ww < kW;
      const float* src = dy + (((long long)n * H + (ok ? hh : 0)) * kW + (ok ? ww : 0)) * 3;
#pragma unroll
      for (int o = 0; o < 3; ++o) v[(rr * 3 + ss) * 3 + o] = ok ? __ldg(src + o) : 0.0f;
    }
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    k_out_conv_bwd(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                   const __grid_constant__ CUtensorMap tmDX, const OcBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sW = smem;                                       // [2 atoms][C16 rows][128 B]
  uint8_t* sX = sW + 2 * a.C16 * 128;                       // 2 stages x c_chunks x [128 px][64 ch]
  const uint32_t x_stage = (uint32_t)a.c_chunks * 16384;
  uint8_t* sAt = sX + 2 * x_stage;                          // 2 stages x A~
  uint8_t* sDx = sAt + 2 * kAtBytes;                        // 2 dx staging tiles (tma_store)
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sDx + (a.tma_store ? 2 * kDxStage : 0));
  uint64_t* xempty = xfull + 2;
  uint64_t* afull = xempty + 2;
  uint64_t* aempty = afull + 2;
  uint64_t* dfull = aempty + 2;
  uint64_t* dempty = dfull + 2;
  uint64_t* wfull = dempty + 2;
  uint64_t* wempty = wfull + 2;
  uint64_t* bfull = wempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = a.C, C2 = 2 * a.C;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmW);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 1);
      tc::mbar_init(&afull[s], 4);
      tc::mbar_init(&aempty[s], 1);
      tc::mbar_init(&dfull[s], 1);
      tc::mbar_init(&dempty[s], 4);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&wfull[s], 1);
      tc::mbar_init(&wempty[s], 4);
    }
    tc::mbar_init(bfull, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // D_w buffers at b * 2C, D_x after them (dw_bufs = 2, one D_x buffer), or D_w at 0 and two D_x at 256
  const uint32_t tm_dw = tmem, tm_dx = tmem + (a.dw_bufs == 2 ? 2 * C2 : 256);
  auto ntiles = [&]() { return blockIdx.x < a.tiles ? (a.tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0; };

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_expect_tx(bfull, 2 * a.C16 * 128);
      tc::tma_load_3d(sW, &tmW, bfull, 0, 0, 0);
      tc::tma_load_3d(sW + a.C16 * 128, &tmW, bfull, 64, 0, 0);
      int it = 0;
      for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        tc::mbar_wait(&xempty[s], ((it >> 1) & 1) ^ 1);
        tc::mbar_expect_tx(&xfull[s], x_stage);
        for (int cc = 0; cc < a.c_chunks; ++cc)
          tc::tma_load_3d(sX + s * x_stage + cc * 16384, &tmX, &xfull[s], cc * 64, 0, t);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idw = tc::idesc_bf16(128, 0, true, true);   // N patched below
    const uint32_t id_w = idw | ((uint32_t)(C2 >> 3) << 17);
    const uint32_t id_x = tc::idesc_bf16(128, 0, false, false) | ((uint32_t)(a.C16 >> 3) << 17);
    const bool issuer = tc::elect_one();
    tc::mbar_wait(bfull, 0);
    tc::tc_fence_after();
    const uint32_t sX0 = tc::smem_u32(sX), sA0 = tc::smem_u32(sAt), sW0 = tc::smem_u32(sW);
    const int nt = ntiles();
    int it = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++it) {
      const int s = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const int g = it / a.flush, gi = it - g * a.flush;
      const int wb = g % a.dw_bufs, db = it % a.dx_bufs;
      tc::mbar_wait(&xfull[s], ph);
      tc::mbar_wait(&afull[s], ph);
      tc::mbar_wait(&dempty[db], ((it / a.dx_bufs) & 1) ^ 1);
      if (gi == 0) tc::mbar_wait(&wempty[wb], ((g / a.dw_bufs) & 1) ^ 1);
      tc::tc_fence_after();
      if (issuer) {
        const uint32_t ab = sA0 + s * kAtBytes, xb = sX0 + s * x_stage;
        // wgrad: K = the tile's 128 pixels, 8 steps of 16 pixel rows (2048 B)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc::mma_bf16(tm_dw + wb * C2, tc::sdesc_sw128(ab + k * 2048, 16384, 1024),
                       tc::sdesc_sw128(xb + k * 2048, 16384, 1024), id_w, (gi > 0 || k > 0) ? 1u : 0u);
        // dgrad: K = 112 A~ columns, 16 per step (32 B within a 128-B row; atom 1 from step 4)
#pragma unroll
        for (int k = 0; k < kDgK / 16; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          tc::mma_bf16(tm_dx + db * a.C16, tc::sdesc_sw128(ab + off, 16, 1024),
                       tc::sdesc_sw128(sW0 + (k >> 2) * a.C16 * 128 + (k & 3) * 32, 16, 1024), id_x,
                       k > 0 ? 1u : 0u);
        }
        tc::mma_commit(&xempty[s]);
        tc::mma_commit(&aempty[s]);
        tc::mma_commit(&dfull[db]);
        if (gi == a.flush - 1 || it == nt - 1) tc::mma_commit(&wfull[wb]);
      }
      __syncwarp();
    }
  } else if (warp < 6) {
    // build A~ for pixel (h, px) of each tile: thread = pixel; the next tile's dy window is loaded
    // before this tile's stage is written, so its L2 latency overlaps the wait and the stores
    const int px = (warp - 2) * 32 + lane;
    float raw[27], nxt[27];
    if (blockIdx.x < a.tiles) load_dy_window(a.dy, blockIdx.x / a.H, blockIdx.x % a.H, a.H, px, raw);
    int it = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++it) {
      const int s = it & 1;
      const int tn = t + gridDim.x;
      if (tn < a.tiles) load_dy_window(a.dy, tn / a.H, tn % a.H, a.H, px, nxt);
      float d1[27], d2[27];
#pragma unroll
      for (int m = 0; m < 27; ++m) {
        d1[m] = __bfloat162float(__float2bfloat16_rn(raw[m]));
        d2[m] = raw[m] - d1[m];
      }
      tc::mbar_wait(&aempty[s], ((it >> 1) & 1) ^ 1);
      uint8_t* at = sAt + s * kAtBytes;
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) {   // 16 chunks of 8 columns j
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = ch * 8 + e;
          const int blk = j / 27, m = j - blk * 27;
          f[e] = j >= kJ ? 0.0f : (blk == 1 ? d2[m < 27 ? m : 0] : d1[m < 27 ? m : 0]);
        }
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) hp[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
        const int atom = ch >> 3, c = ch & 7;
        *reinterpret_cast<uint4*>(at + atom * 16384 + px * 128 + ((c ^ (px & 7)) << 4)) = u;
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&afull[s]);
      if (tn < a.tiles) {
#pragma unroll
        for (int m = 0; m < 27; ++m) raw[m] = nxt[m];
      }
    }
  } else {
    // dx epilogue: warp w reads TMEM lanes 32 (w % 4) ..; thread = pixel
    const int q = warp & 3;
    const int px = q * 32 + lane;
    const int nt = ntiles();
    const int j = q * 32 + lane;   // D_w row of this thread (rows < 54 are used; quadrants 0 and 1)
    // D_w buffer of group g -> the CTA's partial: stored (g = 0) or added in fp32 (each thread owns its row,
    // so the read-modify-write is race-free and its order fixed)
    auto flush_dw = [&](int g) {
      const int wb = g % a.dw_bufs;
      tc::mbar_wait(&wfull[wb], (g / a.dw_bufs) & 1);
      tc::tc_fence_after();
      if (q < 2) {
        float* pp = a.partial + ((long long)blockIdx.x * kWRows + (j < kWRows ? j : 0)) * C2;
#pragma unroll 1
        for (int cb = 0; cb < C2; cb += 16) {
          float v[16];
          tc::tmem_ld16(tm_dw + wb * C2 + ((uint32_t)(q * 32) << 16) + cb, v);
          if (j < kWRows) {
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
              float4 r = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
              if (g > 0) {
                const float4 o = *reinterpret_cast<const float4*>(pp + cb + e);
                r = make_float4(o.x + r.x, o.y + r.y, o.z + r.z, o.w + r.w);
              }
              *reinterpret_cast<float4*>(pp + cb + e) = r;
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&wempty[wb]);
    };
    int it = 0, sb = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++it) {
      const int s = it % a.dx_bufs;
      tc::mbar_wait(&dfull[s], (it / a.dx_bufs) & 1);
      tc::tc_fence_after();
      if (a.tma_store) {
        // 32-column chunks through two SW128 staging tiles (row r's 16-byte chunk c at c ^ (r & 7)) and TMA
        // bulk stores (columns >= C clipped by the tensor map)
        const bool leader = (threadIdx.x & 127) == 0;
#pragma unroll 1
        for (int cb = 0; cb < a.C16; cb += 32) {
          float v[32];
          if (cb + 32 <= a.C16) {
            tc::tmem_ld32(tm_dx + ((uint32_t)(q * 32) << 16) + s * a.C16 + cb, v);
          } else {
            float h16[16];
            tc::tmem_ld16(tm_dx + ((uint32_t)(q * 32) << 16) + s * a.C16 + cb, h16);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              v[j] = h16[j];
              v[16 + j] = 0.0f;
            }
          }
          if (leader) tc::bulk_wait_read<1>();   // the store that last used this staging tile has read it
          tc::named_bar(1, 128);
          uint8_t* stg = sDx + (sb & 1) * kDxStage;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(stg + px * 128 + ((c ^ (px & 7)) << 4)) =
                make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          tc::fence_async_smem();
          tc::named_bar(1, 128);
          if (leader) {
            tc::tma_store_2d(&tmDX, stg, cb, t * kW);
            tc::bulk_commit();
          }
          ++sb;
        }
      } else {
        float* op = a.dx + ((long long)t * kW + px) * C;
#pragma unroll 1
        for (int cb = 0; cb < a.C16; cb += 16) {
          float v[16];
          tc::tmem_ld16(tm_dx + ((uint32_t)(q * 32) << 16) + s * a.C16 + cb, v);
          if (cb + 16 <= C) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(op + cb + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (cb + j < C) op[cb + j] = v[j];
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dempty[s]);
      if ((it + 1) % a.flush == 0 || it == nt - 1) flush_dw(it / a.flush);
    }
    if (a.tma_store && (threadIdx.x & 127) == 0) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// dW[o][t][c] = sum_b (P[b][t*3+o][c] + P[b][t*3+o][C+c]) + (P[b][27+t*3+o][c] + P[b][27+t*3+o][C+c]), b in order
// (one warp per output: lane l sums blocks l, l + 32, ... in order, then a fixed shuffle tree)
__global__ void k_out_wgrad_reduce(const float* __restrict__ part, int blocks, int C, float* __restrict__ dw) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= 27 * C) return;
  const int c = i % C, ot = i / C, o = ot / 9, t = ot - o * 9;
  const int m = t * 3 + o;
  float s = 0.0f;
  for (int b = lane; b < blocks; b += 32) {
    const float* p = part + (size_t)b * kWRows * 2 * C;
    s += (p[m * 2 * C + c] + p[m * 2 * C + C + c]) + (p[(27 + m) * 2 * C + c] + p[(27 + m) * 2 * C + C + c]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) dw[i] = s;
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

// 2-D fp32 map over [rows][cols], box {32, 128}, 128-byte swizzle (the dx stores)
cudaError_t map2_f32(CUtensorMap* m, void* base, long long cols, long long rows) {
  PG_CUDA(encoder());
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

constexpr int kFlush = 16;   // tiles per D_w accumulation chain (8 MMAs each) when two D_w buffers fit in TMEM

size_t out_conv_bwd_scratch_floats(int C) { return (size_t)kNumSMs * kWRows * 2 * C; }

cudaError_t out_conv_bwd_tc(const void* xs, const float* dy, int N, int H, int W, int C, const void* wd, float* dx,
                            float* dw, float* scratch, size_t scratch_floats, cudaStream_t st) {
  if (!out_conv_tc_ok(H, W, C) || ((uintptr_t)xs & 15) || ((uintptr_t)wd & 15) || ((uintptr_t)dx & 15) ||
      ((uintptr_t)scratch & 15))
    return cudaErrorInvalidValue;
  OcBwdArgs a{};
  a.N = N;
  a.H = H;
  a.C = C;
  a.C16 = (C + 15) / 16 * 16;
  a.c_chunks = ceil_div(2 * C, 64);
  a.tiles = N * H;
  a.dy = dy;
  a.dx = dx;
  int grid = a.tiles < sm_cap() ? a.tiles : sm_cap();
  a.dw_bufs = 2 * (2 * C) + a.C16 <= 512 ? 2 : 1;
  a.dx_bufs = a.dw_bufs == 2 ? 1 : 2;
  a.flush = a.dw_bufs == 2 ? kFlush : a.tiles;
  if ((size_t)grid * kWRows * 2 * C > scratch_floats) return cudaErrorInvalidValue;
  a.partial = scratch;
  CUtensorMap mx, mw, mdx;
  PG_CUDA(map3(&mx, xs, 2 * C, kW, (long long)N * H, kW));
  PG_CUDA(map3(&mw, wd, 128, a.C16, 1, a.C16));
  a.tma_store = (C % 4 == 0 && bwd_smem(a.C16, a.c_chunks, 1) <= 232448) ? 1 : 0;
  if (a.tma_store) PG_CUDA(map2_f32(&mdx, dx, C, (long long)N * H * W));
  else mdx = mx;   // unused
  const size_t smem = bwd_smem(a.C16, a.c_chunks, a.tma_store);
  PG_CUDA(cudaFuncSetAttribute(k_out_conv_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_out_conv_bwd<<<grid, kBwdThreads, smem, st>>>(mx, mw, mdx, a);
  PG_CUDA(cudaGetLastError());
  k_out_wgrad_reduce<<<ceil_div(27 * C * 32, 256), 256, 0, st>>>(scratch, grid, C, dw);
  return cudaGetLastError();
}

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
