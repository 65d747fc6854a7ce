// tcgen05 implicit-GEMM convolution for sm_100a.
//
// Activations are NHWC bf16 ("hardware-aware layout").  A
// 3x3 / 1x1 stride-1 'same' convolution is a GEMM over M = N*H*W output
// pixels, N = C_out, K = taps * C_in.  No im2col is materialised: the A tile
// of one K-block (one filter tap x 64 input channels) is a single 4-D TMA box
// {64 ch, bw, bh, bn} of the input at coordinates shifted by the tap offset;
// TMA's out-of-bounds zero fill *is* the zero padding, per image and per edge.
//
//   fprop : A = X (K-major), B = W^  [C_out][taps][C_in]          -> Y
//   dgrad : A = dY (K-major), B = W^T [C_in][taps'][C_out] (flip) -> dX
//   wgrad : A = dY (MN-major, M = C_out), B = X shifted (MN-major,
//           N = C_in of one tap), K = pixels, split-K with fp32 partials
//
// Warp roles (192 threads, 1 CTA/SM, persistent over tiles):
//   warp 0 lane 0 : TMA producer over a STAGES-deep smem ring (mbarriers)
//   warp 1        : TMEM allocation; lane 0 issues tcgen05.mma and commits
//   warps 2..5    : epilogue, TMEM -> registers -> global (bias / residual /
//                   scale fused), double-buffered accumulators in TMEM so the
//                   epilogue of tile i overlaps the main loop of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_conv.h"
#include "tc_ptx.cuh"

#include <cstdlib>

namespace pg {

namespace {

constexpr int kTileM = 128;
constexpr uint32_t kAtomBytes = 128 * 128;   // 128 rows x 128 B (64 bf16)
// 227 KB per CTA minus alignment slack, barriers and the 2 x 16 KB epilogue staging tiles
constexpr uint32_t kStageBytes = 128 * 128;   // one [128 rows][64 bf16] SW128 output tile
constexpr int kStageBufs = 4;                 // two per epilogue half: a store drains one while the other fills
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;   // producer warp, MMA warp, 8 epilogue warps
constexpr int kMaxBiasSmem = 2048;              // floats of bias staged in shared memory
constexpr int kSmemBudget = 232448 - 1024 - kStageBufs * (int)kStageBytes - 1024 - 4 * kMaxBiasSmem;

template <int BN>
struct FpropCfg {
  static constexpr uint32_t A_BYTES = kAtomBytes;
  static constexpr uint32_t B_BYTES = BN * 128;
  static constexpr int STAGES_RAW = kSmemBudget / (A_BYTES + B_BYTES);
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + kStageBufs * kStageBytes + 512 + 4 * kMaxBiasSmem;
};

template <int BN>
struct WgradCfg {
  static constexpr int NB = (BN + 63) / 64;           // 64-wide MN atoms of B
  static constexpr uint32_t A_BYTES = 2 * kAtomBytes;  // M = 128 output channels
  static constexpr uint32_t B_BYTES = NB * kAtomBytes;
  static constexpr uint32_t ONES_BYTES = kAtomBytes;    // constant bf16 1.0 tile: bias-gradient B operand
  static constexpr int STAGES_RAW = (232448 - 2048 - (int)ONES_BYTES) / (A_BYTES + B_BYTES);
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  // dW accumulator in columns [0, BN), bias sums in [BN, BN + 16) (read as one 32-column load)
  static constexpr uint32_t TMEM_COLS = (BN + 32 <= 64) ? 64 : (BN + 32 <= 128) ? 128 : (BN + 32 <= 256) ? 256 : 512;
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + ONES_BYTES + 256;
};

template <int BN>
struct WgradCg2Cfg {   // per CTA: 128 dY channels x 128 pixels (A), BN / 2 input channels (B half)
  static constexpr int NB = BN / 128;                  // 64-wide MN atoms of this CTA's B half
  static constexpr uint32_t A_BYTES = 2 * kAtomBytes;
  static constexpr uint32_t B_BYTES = NB * kAtomBytes;
  static constexpr uint32_t ONES_BYTES = kAtomBytes;
  static constexpr int STAGES_RAW = (232448 - 2048 - (int)ONES_BYTES) / (A_BYTES + B_BYTES);
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = (BN + 32 <= 128) ? 128 : (BN + 32 <= 256) ? 256 : 512;
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + ONES_BYTES + 256;
  static_assert(BN % 128 == 0, "each CTA's B half must be whole 64-channel atoms");
};

template <int BN>
struct Wgrad3Cfg {
  static constexpr int NB = (BN + 63) / 64;            // 64-channel chunks of the X halo
  static constexpr uint32_t XCH = 18432;               // one chunk: up to 144 halo pixel rows x 128 B
  static constexpr uint32_t A_BYTES = 2 * kAtomBytes;
  static constexpr uint32_t B_BYTES = NB * XCH;
  static constexpr uint32_t ONES_BYTES = kAtomBytes;
  static constexpr int STAGES_RAW = (232448 - 2048 - (int)ONES_BYTES) / (A_BYTES + B_BYTES);
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  // three taps' accumulators in [0, 3 BN), bias sums at 3 BN
  static constexpr uint32_t TMEM_COLS = (3 * BN + 32 <= 256) ? 256 : 512;
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + ONES_BYTES + 256;
  static_assert(3 * BN + 32 <= 512, "three taps must fit TMEM");
  static_assert(STAGES >= 2, "pipeline needs two stages");
};

// the dynamic shared-memory base rounded up to 1024 bytes by pointer arithmetic on the shared array itself, so
// the compiler keeps the shared address space (LDS/STS, not generic LD/ST) for every access derived from it
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (tc::smem_u32(p) & 1023u)) & 1023u);
}

// pixel index -> (n, h, w) origin of a 128-pixel tile
__device__ __forceinline__ void pix_origin(int p0, int H, int W, int& n0, int& h0, int& w0) {
  int hw = H * W;
  n0 = p0 / hw;
  int r = p0 - n0 * hw;
  h0 = r / W;
  w0 = r - h0 * W;
}

// the first N (multiple of 8) of v as bf16, 16-byte stores
template <int N>
__device__ __forceinline__ void store_row32_bf16_n(bf16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < N / 8; ++q) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 t = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&t);
    }
    d[q] = u;
  }
}

__device__ __forceinline__ void store_row32_bf16(bf16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 t = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&t);
    }
    d[q] = u;
  }
}

// Epilogue: 8 warps (2..9), two per TMEM lane quadrant (warp w may only read lanes
// 32*(w%4)..+31); half h = (w-2)/4 takes the 64-column groups g with g % 2 == h.  Thread =
// output row.  bias / gamma scale / ReLU-backward mask / residual (same or half resolution)
// are fused before a single rounding; the bias vector is staged in shared memory once.
// bf16 outputs go through one 16 KB SW128 staging tile per half (row r's 16-byte chunk j at
// j ^ (r & 7): conflict-free) and leave as 64-column TMA bulk stores (rows >= M and columns
// >= C_out clipped by the tensor map).

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* r) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 f = __bfloat1622float2(h[j]);
    r[2 * j] = f.x;
    r[2 * j + 1] = f.y;
  }
}

// CG = 2: tiles are CTA-pair tiles (M = 256); this CTA owns M rows [rank * 128, rank * 128 + 128)
// and releases the accumulator on the leader CTA's barrier.
template <int BN, int CG = 1>
__device__ __forceinline__ void epilogue_loop(const TcFpropArgs& a, const CUtensorMap* tmO, uint8_t* stage,
                                              float* sbias, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                              int num_tiles, int tile0 = -1, int tile_step = 0, int rank = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;
  const int half = (warp - 2) >> 2;
  const int row = q * 32 + lane;
  const int etid = threadIdx.x - 64;                    // 0..255
  const bool leader = (etid & 127) == 0;                // one store-issuing thread per half
  const float alpha = a.alpha ? *a.alpha : 1.0f;
  const bool scale = a.alpha != nullptr;
  // bias -> shared memory (all epilogue threads; named barrier over the 256 of them)
  const int cpad = a.n_tiles * BN;   // the tiles' columns; those >= C_out get a zero bias
  const bool bias_smem = a.bias && cpad <= kMaxBiasSmem;
  if (bias_smem) {
    for (int c = etid; c < cpad; c += 32 * kEpiWarps) sbias[c] = c < a.Cout ? a.bias[c] : 0.0f;
  }
  // a ragged chunk (C_out not a multiple of 32) takes the vectorised path too when nothing per element needs
  // masking: its extra columns are zero accumulators (B rows >= C_out are TMA zero fill) plus a zero bias, and
  // the TMA store clips them (the masked path below made C_out = 48 layers 2.6x slower than C_out = 64)
  const bool ragged_fast = a.tma_store && !a.relu_ref && !a.residual && (!a.bias || bias_smem);
  tc::named_bar(3, 32 * kEpiWarps);
  if (tile0 < 0) {
    tile0 = blockIdx.x;
    tile_step = gridDim.x;
  }
  int sb = 0;   // which of this half's two staging tiles the next 64-column group fills
  int it = 0;
  bool pending = false;
  // BN <= 192: the two halves take alternate TILES (whole accumulators: half h always reads buffer h) rather than
  // alternate 64-column groups of each tile, so no half idles when a tile has one or one-and-a-half groups
  constexpr bool kSplitTiles = BN <= 192;
  constexpr int kG0Step = kSplitTiles ? 64 : 128;
  const int g0 = kSplitTiles ? 0 : half * 64;
  for (int tile = tile0; tile < num_tiles; tile += tile_step, ++it) {
    if (kSplitTiles && (it & 1) != half) continue;
    const int buf = it & 1;
    const int nt = tile % a.n_tiles;
    int mt = CG == 2 ? (tile / a.n_tiles) * 2 + rank : tile / a.n_tiles;
    int phase = 0;
    if (CG == 2 && a.phases > 1) {   // tile = (phase * mpairs + pair) * n_tiles + nt
      const int mpairs = (a.m_tiles + 1) / 2;
      phase = (tile / a.n_tiles) / mpairs;
      mt = ((tile / a.n_tiles) - phase * mpairs) * 2 + rank;
    }
    const long long m = (long long)mt * kTileM + row;
    const bool valid = m < a.M;
    // the ReLU-mask reference row: the output pixel itself, or in sub-pixel mode the full-resolution pixel
    // (2i + a, 2j + b) that low-resolution pixel m writes in output phase (a, b)
    long long rrow = m;
    if (CG == 2 && a.phases > 1 && a.relu_ref && valid) {
      const int hw = a.H * a.W;
      const int n = (int)(m / hw);
      const int r = (int)(m - (long long)n * hw);
      const int i = r / a.W, jj = r - i * a.W;
      rrow = ((long long)(n * 2 * a.H + 2 * i + (phase >> 1)) * (2 * a.W)) + 2 * jj + (phase & 1);
    }
    long long rbase = 0;
    if (valid && a.residual) {
      if (a.res_mode == 2) {   // residual stored at half resolution (nearest x2 upsample)
        const int hw = a.H * a.W;
        const int n = (int)(m / hw);
        const int r = (int)(m - (long long)n * hw);
        const int h = r / a.W, w = r - h * a.W;
        rbase = ((long long)(n * (a.H >> 1) + (h >> 1)) * (a.W >> 1) + (w >> 1)) * a.ldr;
      } else {
        rbase = m * a.ldr;
      }
    }
    // one bf16 side input per chunk (the ReLU mask reference, else the residual) is loaded one chunk
    // ahead — the first before the accumulator wait — so its global latency overlaps the pipeline
    const bf16* side = nullptr;
    long long sbase = 0;
    if (valid) {
      if (a.relu_ref) {
        side = reinterpret_cast<const bf16*>(a.relu_ref);
        sbase = rrow * a.ldo;
      } else if (a.residual) {
        side = reinterpret_cast<const bf16*>(a.residual);
        sbase = rbase;
      }
    }
    auto load_side = [&](int cb, uint4 (&dst)[4]) {
      const int col0 = nt * BN + cb;
      if (side && cb >= 0 && col0 + 32 <= a.Cout) {
        const uint4* p = reinterpret_cast<const uint4*>(side + sbase + col0);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) dst[qq] = p[qq];
      }
    };
    auto next_cb = [&](int cb) {   // this thread's chunk after cb: within the 64-wide group, else the next group
      const int g = cb & ~63;
      if (cb + 32 < g + 64 && cb + 32 < BN) return cb + 32;
      return g + kG0Step < BN ? g + kG0Step : -1;
    };
    uint4 scur[4] = {};
    load_side(g0 < BN ? g0 : -1, scur);
    tc::mbar_wait(&tfull[buf], (it >> 1) & 1);
    tc::tc_fence_after();
#pragma unroll 1
    for (int g = g0; g < BN; g += kG0Step) {
      uint8_t* st = stage + (half * 2 + sb) * kStageBytes;
      if (a.tma_store) {
        // the store that last used this staging tile (two groups ago) has read it; the previous
        // group's store may still be draining the other tile
        if (leader && pending) tc::bulk_wait_read<1>();
        tc::named_bar(1 + half, 128);
      }
#pragma unroll 1
      for (int cb = g; cb < g + 64 && cb < BN; cb += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + cb, v);
        uint4 snext[4] = {};
        load_side(next_cb(cb), snext);
        const int col0 = nt * BN + cb;
        if (valid && (col0 + 32 <= a.Cout || (ragged_fast && col0 < a.Cout))) {
          // ---- full 32-column chunk: straight-line, vectorised
          if (scale) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= alpha;
          }
          if (a.relu_ref) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              float r[8];
              bf16x8_to_f32(scur[qq], r);
#pragma unroll
              for (int j = 0; j < 8; ++j) v[qq * 8 + j] = r[j] > 0.0f ? v[qq * 8 + j] : 0.0f;
            }
          }
          if (a.bias) {
            if (bias_smem) {
              const float4* b4 = reinterpret_cast<const float4*>(sbias + col0);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 b = b4[j];
                v[4 * j] += b.x;
                v[4 * j + 1] += b.y;
                v[4 * j + 2] += b.z;
                v[4 * j + 3] += b.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += __ldg(a.bias + col0 + j);
            }
          }
          if (a.residual) {
            const uint4* rp = reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(a.residual) + rbase + col0);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              float r[8];
              bf16x8_to_f32(a.relu_ref ? rp[qq] : scur[qq], r);
#pragma unroll
              for (int j = 0; j < 8; ++j) v[qq * 8 + j] += r[j];
            }
          }
          if (a.relu_out) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
          }
          if (!a.tma_store) {
            if (a.out_f32) {
              float* op = reinterpret_cast<float*>(a.out) + m * a.ldo + col0;
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(op + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
              store_row32_bf16(reinterpret_cast<bf16*>(a.out) + m * a.ldo + col0, v);
            }
          }
        } else if (valid && col0 < a.Cout) {
          // ---- ragged tail (C_out not a multiple of 32): masked, compile-time indices only; the bias from
          // shared memory (a per-element global load here made C_out = 48 layers 2.6x slower than 64)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int c = col0 + j;
            const bool ok = c < a.Cout;
            float t = v[j] * alpha;
            if (a.relu_ref && ok)
              t = __bfloat162float(reinterpret_cast<const bf16*>(a.relu_ref)[rrow * a.ldo + c]) > 0.0f ? t : 0.0f;
            if (a.bias && ok) t += bias_smem ? sbias[c] : __ldg(a.bias + c);
            if (a.residual && ok) t += __bfloat162float(reinterpret_cast<const bf16*>(a.residual)[rbase + c]);
            if (a.relu_out) t = fmaxf(t, 0.0f);
            v[j] = t;
            if (!a.tma_store && ok) {
              if (a.out_f32) reinterpret_cast<float*>(a.out)[m * a.ldo + c] = t;
              else reinterpret_cast<bf16*>(a.out)[m * a.ldo + c] = __float2bfloat16_rn(t);
            }
          }
        }
        if (a.tma_store) {
          // 4 x 16-byte chunks of this row into the swizzled staging tile
          const int c0 = (cb - g) >> 3;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint4 u;
            uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __nv_bfloat162 t2 = __floats2bfloat162_rn(v[qq * 8 + 2 * j], v[qq * 8 + 2 * j + 1]);
              w[j] = *reinterpret_cast<uint32_t*>(&t2);
            }
            const int chunk = (c0 + qq) ^ (row & 7);
            *reinterpret_cast<uint4*>(st + row * 128 + chunk * 16) = u;
          }
        }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) scur[qq] = snext[qq];
      }
      if (a.tma_store && a.pool_out) {
        // fused 2x2 average pooling (D blocks with a downsample): the tile holds whole row pairs, its 32 pooled
        // pixels are contiguous in the pooled map (base m0 / 4); thread t of the half -> pooled pixel t / 4,
        // 16 columns; same arithmetic as k_avgpool2_v on the bf16 values (bit-identical)
        tc::named_bar(1 + half, 128);
        const int tt = etid & 127;
        const int pp = tt >> 2, c16 = (tt & 3) * 16;
        const int hw2 = a.W >> 1;
        const int r0 = (pp / hw2) * 2 * a.W + (pp % hw2) * 2;
        const long long pm = (long long)mt * (kTileM / 4) + pp;
        const int col = nt * BN + g + c16;
        if ((long long)mt * kTileM + r0 + a.W + 1 < a.M + 0 && g + c16 < BN && col < a.Cout) {
          float o[16];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {   // two 16-byte chunks of 8 columns
            const int ch = (c16 >> 3) + hh;
            float q[4][8];
            const int rr[4] = {r0, r0 + 1, r0 + a.W, r0 + a.W + 1};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint4 u = *reinterpret_cast<const uint4*>(st + rr[k] * 128 + ((ch ^ (rr[k] & 7)) << 4));
              bf16x8_to_f32(u, q[k]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) o[hh * 8 + j] = ((q[0][j] + q[1][j]) + (q[2][j] + q[3][j])) * 0.25f;
          }
          float t16[32];
#pragma unroll
          for (int j = 0; j < 16; ++j) t16[j] = o[j];
          bf16* dst = reinterpret_cast<bf16*>(a.pool_out) + pm * a.ldo + col;
          store_row32_bf16_n<16>(dst, t16);
          if (a.pool_relu) {
#pragma unroll
            for (int j = 0; j < 16; ++j) t16[j] = o[j] > 0.0f ? o[j] : 0.0f;
            store_row32_bf16_n<16>(reinterpret_cast<bf16*>(a.pool_relu) + pm * a.ldo + col, t16);
          }
        }
      } else if (a.tma_store) {
        tc::fence_async_smem();
        tc::named_bar(1 + half, 128);
        if (leader) {
          if (CG == 2 && a.phases > 1) {
            int n0, h0, w0;
            pix_origin(mt * kTileM, a.H, a.W, n0, h0, w0);
            tc::tma_store_5d(tmO, st, nt * BN + g, phase & 1, w0, phase >> 1, n0 * a.H + h0);
          } else {
            tc::tma_store_2d(tmO, st, nt * BN + g, mt * kTileM);
          }
          tc::bulk_commit();
          pending = true;
        }
      }
      sb ^= 1;
    }
    // one arrival per warp (the barrier counts warps): every lane's tcgen05.ld has completed
    // (wait::ld) and is ordered before lane 0's arrive by the fence + warp sync
    tc::tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (CG == 2 && rank != 0) tc::mbar_arrive_cluster(tc::map_to_rank(&tempty[buf], 0));
      else tc::mbar_arrive(&tempty[buf]);
    }
  }
  if (a.tma_store && leader) tc::bulk_wait_all();
}

// ===========================================================================
// fprop / dgrad kernel
// ===========================================================================
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_fprop(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmO, const TcFpropArgs a) {
  using C = FpropCfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sO = sB + STAGES * C::B_BYTES;            // 2 epilogue staging tiles
  uint64_t* full = reinterpret_cast<uint64_t*>(sO + kStageBufs * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], BN <= 192 ? kEpiWarps / 2 : kEpiWarps);   // one half per tile when BN <= 192
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int num_tiles = a.m_tiles * a.n_tiles;
  const int num_kb = a.taps * a.c_chunks;
  const int pad = a.ksz >> 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile / a.n_tiles, nt = tile - mt * a.n_tiles;
        int n0, h0, w0;
        pix_origin(mt * kTileM, a.H, a.W, n0, h0, w0);
        for (int kb = 0; kb < num_kb; ++kb) {
          const int tap = kb / a.c_chunks, cc = kb - tap * a.c_chunks;
          const int dy = tap / a.ksz - pad, dx = tap % a.ksz - pad;
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
          tc::tma_load_4d(sA + stage * C::A_BYTES, &tmA, &full[stage], cc * 64, w0 + dx, h0 + dy, n0);
          tc::tma_load_3d(sB + stage * C::B_BYTES, &tmB, &full[stage], cc * 64, tap, nt * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(kTileM, BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + buf * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a_base = tc::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_base = tc::smem_u32(sB + stage * C::B_BYTES);
          // the last channel chunk may hold fewer than 64 real channels (e.g. 96 = 64 + 32, or the
          // 8-channel RGB image): issue only the K=16 steps that cover them
          const int cc = kb % a.c_chunks;
          const int ksteps = (cc == a.c_chunks - 1) ? a.last_ksteps : 4;
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t ad = tc::sdesc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bd = tc::sdesc_sw128(b_base + k * 32, 16, 1024);
            tc::mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull[buf]);
      }
    }
  } else {
    epilogue_loop<BN>(a, &tmO, sO, sbias, tmem, tfull, tempty, num_tiles);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ===========================================================================
// wgrad kernel: dW[o][tap][c] = sum_p dY[p][o] * X[p + delta_tap][c]
// ===========================================================================
template <int BN>
__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmX,
                 const TcWgradArgs a, const __grid_constant__ TmaQuad tq) {
  using C = WgradCfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sOnes = sB + STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the CTAs of tap 0 / channel block 0 also sum dY over their pixels: db[o] = sum_p dY[p][o]
  // (an extra N = 16 MMA per K step against a constant all-ones B tile)
  const int nt_ = (int)(blockIdx.x % (a.m_tiles * a.n_tiles)) % a.n_tiles;
  const bool do_bias = a.bias_out != nullptr &&
                       (a.phases > 1 ? (nt_ % a.c_blocks == 0 && (nt_ / a.c_blocks) % 4 == 0) : nt_ == 0);
  if (do_bias) {
    uint4* o4 = reinterpret_cast<uint4*>(sOnes);
    for (int i = threadIdx.x; i < (int)(C::ONES_BYTES / 16); i += blockDim.x)
      o4[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    tc::fence_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmDY);
    tc::tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&tfull[0], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // work unit -> (split, m tile over C_out, n tile over (tap, C_in block)); the split (pixel
  // range) is the slowest index so that the CTAs resident together read the same dY / X
  // pixels for all taps and channel blocks (L2 reuse instead of one DRAM pass per tap)
  const int tiles = a.m_tiles * a.n_tiles;
  const int split = blockIdx.x / tiles;
  const int u = blockIdx.x - split * tiles;
  const int nt = u % a.n_tiles;
  const int mt = u / a.n_tiles;
  const int tap = nt / a.c_blocks, cb = nt - tap * a.c_blocks;
  const int pad = a.ksz >> 1;
  int dy = tap / a.ksz - pad, dx = tap % a.ksz - pad;
  const int ph = a.phases > 1 ? tap >> 2 : 0;   // phase wgrad: tap = phase * 4 + p * 2 + q
  if (a.phases > 1) {
    dy = ((tap >> 1) & 1) - 1 + (ph >> 1);
    dx = (tap & 1) - 1 + (ph & 1);
  }
  const CUtensorMap* mdy = a.phases > 1 ? &tq.m[ph] : &tmDY;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.total_kb, kb0 + a.kb_per_split);
  const int o0 = mt * 128, c0 = cb * BN;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        int n0, h0, w0;
        pix_origin(kb * kTileM, a.H, a.W, n0, h0, w0);
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
        uint8_t* da = sA + stage * C::A_BYTES;
        tc::tma_load_4d(da, mdy, &full[stage], o0, w0, h0, n0);
        tc::tma_load_4d(da + kAtomBytes, mdy, &full[stage], o0 + 64, w0, h0, n0);
        uint8_t* db = sB + stage * C::B_BYTES;
#pragma unroll
        for (int j = 0; j < C::NB; ++j)
          tc::tma_load_4d(db + j * kAtomBytes, &tmX, &full[stage], c0 + 64 * j, w0 + dx, h0 + dy, n0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    {   // the whole (converged) warp runs the loop; one elected lane issues (uniform descriptors)
      constexpr uint32_t idesc = tc::idesc_bf16(128, BN, true, true);
      const bool issuer = tc::elect_one();
      const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB), o_base = tc::smem_u32(sOnes);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t a_base = sA0 + stage * C::A_BYTES;
        const uint32_t b_base = sB0 + stage * C::B_BYTES;
        if (issuer) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {   // 8 x K=16 pixels; each K=16 step = two 8-row groups = 2048 B
            const uint64_t ad = tc::sdesc_sw128(a_base + k * 2048, kAtomBytes, 1024);
            const uint64_t bd = tc::sdesc_sw128(b_base + k * 2048, kAtomBytes, 1024);
            tc::mma_bf16(tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
          }
          if (do_bias) {
            constexpr uint32_t idb = tc::idesc_bf16(128, 16, true, true);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              tc::mma_bf16(tmem + BN, tc::sdesc_sw128(a_base + k * 2048, kAtomBytes, 1024),
                           tc::sdesc_sw128(o_base + k * 2048, kAtomBytes, 1024), idb, (kb != kb0) || (k != 0));
          }
          tc::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (issuer) tc::mma_commit(&tfull[0]);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    tc::mbar_wait(&tfull[0], 0);
    tc::tc_fence_after();
    const int o = o0 + row;
    if (do_bias) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + BN, v);
      if (o < a.Cout) a.bias_out[((long long)split * (a.phases > 1 ? 4 : 1) + ph) * a.Cout + o] = v[0];
    }
#pragma unroll 1
    for (int cbk = 0; cbk < BN; cbk += 32) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + cbk, v);
      const int col0 = c0 + cbk;
      if (o >= a.Cout || col0 >= a.Cin) continue;
      float* op = a.out + (((long long)split * a.Cout + o) * a.taps + tap) * a.Cin + col0;
      if (col0 + 32 <= a.Cin && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(op + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < a.Cin) op[j] = v[j];
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ===========================================================================
// wgrad, CTA pair (cta_group::2): M = 256 output channels per pair tile — each CTA stages its own
// 128 dY channels (A) and HALF of the B tile (BN / 2 input channels of X), the leader issues
// tcgen05.mma.cta_group::2 over both CTAs' shared memory and each CTA's TMEM holds its 128 rows.
// Per SM this halves the B traffic (TMA writes and tensor-core reads), the shared-memory
// bandwidth the one-CTA kernel saturates at C_in, C_out >= 256.  Same work units / split-K
// partials / phase (sub-pixel) taps as k_conv_wgrad, with unit = (split, pair tile, n tile).
// ===========================================================================
template <int BN>
__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad_cg2(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmX,
                     const TcWgradArgs a, const __grid_constant__ TmaQuad tq) {
  using C = WgradCg2Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sOnes = sB + STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool is_leader = rank == 0;
  const int unit = (int)tc::cluster_id_x();
  const int mpairs = (a.m_tiles + 1) / 2;
  const int tiles = mpairs * a.n_tiles;
  const int split = unit / tiles;
  const int uu = unit - split * tiles;
  const int nt = uu % a.n_tiles;
  const int mp = uu / a.n_tiles;
  const bool do_bias = a.bias_out != nullptr &&
                       (a.phases > 1 ? (nt % a.c_blocks == 0 && (nt / a.c_blocks) % 4 == 0) : nt == 0);
  if (do_bias) {
    uint4* o4 = reinterpret_cast<uint4*>(sOnes);
    for (int i = threadIdx.x; i < (int)(C::ONES_BYTES / 16); i += blockDim.x)
      o4[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    tc::fence_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmDY);
    tc::tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&tfull[0], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int tap = nt / a.c_blocks, cb = nt - tap * a.c_blocks;
  const int pad = a.ksz >> 1;
  int dy = tap / a.ksz - pad, dx = tap % a.ksz - pad;
  const int ph = a.phases > 1 ? tap >> 2 : 0;
  if (a.phases > 1) {
    dy = ((tap >> 1) & 1) - 1 + (ph >> 1);
    dx = (tap & 1) - 1 + (ph & 1);
  }
  const CUtensorMap* mdy = a.phases > 1 ? &tq.m[ph] : &tmDY;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.total_kb, kb0 + a.kb_per_split);
  const int o0 = mp * 256 + (int)rank * 128;          // this CTA's 128 output channels
  const int c0 = cb * BN + (int)rank * (BN / 2);      // this CTA's half of the input channels

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        int n0, h0, w0;
        pix_origin(kb * kTileM, a.H, a.W, n0, h0, w0);
        tc::mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t fbar = tc::map_to_rank(&full[stage], 0);
        if (is_leader) tc::mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
        uint8_t* da = sA + stage * C::A_BYTES;
        tc::tma_load_4d_cg2(da, mdy, fbar, o0, w0, h0, n0);
        tc::tma_load_4d_cg2(da + kAtomBytes, mdy, fbar, o0 + 64, w0, h0, n0);
        uint8_t* db = sB + stage * C::B_BYTES;
#pragma unroll
        for (int j = 0; j < C::NB; ++j)
          tc::tma_load_4d_cg2(db + j * kAtomBytes, &tmX, fbar, c0 + 64 * j, w0 + dx, h0 + dy, n0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (is_leader) {   // whole (converged) warp runs the loop; one elected lane issues
      constexpr uint32_t idesc = tc::idesc_bf16(256, BN, true, true);
      constexpr uint32_t idb = tc::idesc_bf16(256, 16, true, true);
      const bool issuer = tc::elect_one();
      const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB), o_base = tc::smem_u32(sOnes);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t a_base = sA0 + stage * C::A_BYTES;
        const uint32_t b_base = sB0 + stage * C::B_BYTES;
        if (issuer) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {   // 8 x K=16 pixels
            const uint64_t ad = tc::sdesc_sw128(a_base + k * 2048, kAtomBytes, 1024);
            const uint64_t bd = tc::sdesc_sw128(b_base + k * 2048, kAtomBytes, 1024);
            tc::mma_bf16_cg2(tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
          }
          if (do_bias) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              tc::mma_bf16_cg2(tmem + BN, tc::sdesc_sw128(a_base + k * 2048, kAtomBytes, 1024),
                               tc::sdesc_sw128(o_base + k * 2048, kAtomBytes, 1024), idb, (kb != kb0) || (k != 0));
          }
          tc::mma_commit_cg2(&empty[stage], 3);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (issuer) tc::mma_commit_cg2(&tfull[0], 3);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    tc::mbar_wait(&tfull[0], 0);
    tc::tc_fence_after();
    const int o = o0 + row;
    if (do_bias) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + BN, v);
      if (o < a.Cout) a.bias_out[((long long)split * (a.phases > 1 ? 4 : 1) + ph) * a.Cout + o] = v[0];
    }
    const int cbase = cb * BN;
#pragma unroll 1
    for (int cbk = 0; cbk < BN; cbk += 32) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + cbk, v);
      const int col0 = cbase + cbk;
      if (o >= a.Cout || col0 >= a.Cin) continue;
      float* op = a.out + (((long long)split * a.Cout + o) * a.taps + tap) * a.Cin + col0;
      if (col0 + 32 <= a.Cin && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(op + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < a.Cin) op[j] = v[j];
      }
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 1) tc::tmem_dealloc_cg2(tmem, C::TMEM_COLS);
}

// ===========================================================================
// wgrad, 3x3, one filter row per CTA: the three taps (r, 0..2) of a row share the dY tile (A,
// loaded once instead of three times) and one X halo box {64 ch, Wt + 2, 128 / Wt rows, 1}
// (Wt = min(W, 128)) per 64-channel chunk, which each tap reads through a descriptor shifted by
// s pixel rows (the SW128 swizzle is a function of the absolute address; the MN-major K=16
// step of 16 pixels stays inside one image row because W >= 16).  L2 -> SM traffic per K-block
// drops from 3 x (dY + X) to dY + X(1 + 2 / Wt), which is what bounded the 96/192-channel layers.
// ===========================================================================
template <int BN>
__global__ void __launch_bounds__(192, 1)
    k_conv_wgrad3(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmXh,
                  const TcWgradArgs a) {
  using C = Wgrad3Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sOnes = sB + STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOnes + C::ONES_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = a.m_tiles * a.n_tiles;   // n_tiles = 3 rows x c_blocks
  const int split = blockIdx.x / tiles;
  const int u = blockIdx.x - split * tiles;
  const int nt = u % a.n_tiles;
  const int mt = u / a.n_tiles;
  const int r = nt / a.c_blocks, cb = nt - r * a.c_blocks;
  const bool do_bias = a.bias_out != nullptr && nt == 0;
  if (do_bias) {
    uint4* o4 = reinterpret_cast<uint4*>(sOnes);
    for (int i = threadIdx.x; i < (int)(C::ONES_BYTES / 16); i += blockDim.x)
      o4[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    tc::fence_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmDY);
    tc::tma_prefetch(&tmXh);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&tfull[0], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int Wt = a.W < 128 ? a.W : 128;          // pixels of one tile row
  const int rowsT = 128 / Wt;                    // image rows per tile
  const uint32_t x_tx = (uint32_t)(C::NB * (Wt + 2) * rowsT * 128);
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(a.total_kb, kb0 + a.kb_per_split);
  const int o0 = mt * 128, c0 = cb * BN;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        int n0, h0, w0;
        pix_origin(kb * kTileM, a.H, a.W, n0, h0, w0);
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_expect_tx(&full[stage], C::A_BYTES + x_tx);
        uint8_t* da = sA + stage * C::A_BYTES;
        tc::tma_load_4d(da, &tmDY, &full[stage], o0, w0, h0, n0);
        tc::tma_load_4d(da + kAtomBytes, &tmDY, &full[stage], o0 + 64, w0, h0, n0);
        uint8_t* db = sB + stage * C::B_BYTES;
#pragma unroll
        for (int j = 0; j < C::NB; ++j)
          tc::tma_load_4d(db + j * C::XCH, &tmXh, &full[stage], c0 + 64 * j, w0 - 1, h0 + r - 1, n0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    {   // the whole (converged) warp runs the loop; one elected lane issues (uniform descriptors)
      constexpr uint32_t idesc = tc::idesc_bf16(128, BN, true, true);
      const bool issuer = tc::elect_one();
      const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB), o_base = tc::smem_u32(sOnes);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t a_base = sA0 + stage * C::A_BYTES;
        const uint32_t b_base = sB0 + stage * C::B_BYTES;
        if (issuer) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {   // 8 x K=16 pixels
            const uint64_t ad = tc::sdesc_sw128(a_base + k * 2048, kAtomBytes, 1024);
            const int p0 = 16 * k, ir = p0 / Wt, jc = p0 - ir * Wt;
            const uint32_t hrow = (uint32_t)(ir * (Wt + 2) + jc);   // halo row of tap s = 0
#pragma unroll
            for (int sx = 0; sx < 3; ++sx) {
              const uint64_t bd = tc::sdesc_sw128(b_base + (hrow + sx) * 128, C::XCH, 1024);
              tc::mma_bf16(tmem + sx * BN, ad, bd, idesc, (kb != kb0) || (k != 0));
            }
          }
          if (do_bias) {
            constexpr uint32_t idb = tc::idesc_bf16(128, 16, true, true);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              tc::mma_bf16(tmem + 3 * BN, tc::sdesc_sw128(a_base + k * 2048, kAtomBytes, 1024),
                           tc::sdesc_sw128(o_base + k * 2048, kAtomBytes, 1024), idb, (kb != kb0) || (k != 0));
          }
          tc::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (issuer) tc::mma_commit(&tfull[0]);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    tc::mbar_wait(&tfull[0], 0);
    tc::tc_fence_after();
    const int o = o0 + row;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    if (do_bias) {
      float v[32];
      tc::tmem_ld32(lane_base + 3 * BN, v);
      if (o < a.Cout) a.bias_out[(long long)split * a.Cout + o] = v[0];
    }
#pragma unroll 1
    for (int sx = 0; sx < 3; ++sx) {
      const int tap = r * 3 + sx;
#pragma unroll 1
      for (int cbk = 0; cbk < BN; cbk += 32) {
        float v[32];
        tc::tmem_ld32(lane_base + sx * BN + cbk, v);
        const int col0 = c0 + cbk;
        if (o >= a.Cout || col0 >= a.Cin) continue;
        float* op = a.out + (((long long)split * a.Cout + o) * a.taps + tap) * a.Cin + col0;
        if (col0 + 32 <= a.Cin && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(op + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < a.Cin) op[j] = v[j];
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ===========================================================================
// fprop / dgrad, 3x3: halo variants.  The A operand of the 9 taps is staged in
// "units" that several taps share, each tap reading its unit through a descriptor
// whose start address is shifted by whole 128-byte pixel rows (the SW128 swizzle is
// a function of the absolute smem address, so any row offset is valid — verified
// bit-exact, base-offset field 0):
//   MODE 0 (W % 128 == 0, tile = 128 pixels of one row): one unit per 64-channel
//          chunk = box {64, 130, 3, 1}; tap (r, s) starts at row r*130 + s
//          (2.95x less A traffic than one box per tap);
//   MODE 1 (16 <= W <= 64, tile = 128/W whole rows): three units per chunk, one per
//          filter column s = box {64, W, 128/W + 2, 1} shifted by s - 1; tap (r, s)
//          starts at row r*W of unit s (1.5x / 2x / 2.4x less A traffic at W = 64/32/16).
// ===========================================================================
template <int BN, int MODE>
struct HaloCfg {
  static constexpr uint32_t UNIT_BYTES = MODE == 0 ? 50176 : 32768;   // 390 rows / (128/W + 2) * W rows
  static constexpr int NA = MODE == 0 ? 2 : 3;
  static constexpr uint32_t B_BYTES = BN * 128;
  static constexpr int STAGES_RAW = (kSmemBudget - NA * (int)UNIT_BYTES) / (int)B_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = FpropCfg<BN>::TMEM_COLS;
  static constexpr size_t SMEM = 1024 + NA * UNIT_BYTES + STAGES * B_BYTES + kStageBufs * kStageBytes + 512 + 4 * kMaxBiasSmem;
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_fprop_halo(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, const TcFpropArgs a, const uint32_t unit_tx) {
  using C = HaloCfg<BN, MODE>;
  constexpr int STAGES = C::STAGES, NA = C::NA;
  constexpr int UNITS = MODE == 0 ? 1 : 3, TAPS_PER_UNIT = MODE == 0 ? 9 : 3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sH = smem;
  uint8_t* sB = smem + NA * C::UNIT_BYTES;
  uint8_t* sO = sB + STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sO + kStageBufs * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* hfull = empty + STAGES;
  uint64_t* hempty = hfull + NA;
  uint64_t* tfull = hempty + NA;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NA; ++b) {
      tc::mbar_init(&hfull[b], 1);
      tc::mbar_init(&hempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], BN <= 192 ? kEpiWarps / 2 : kEpiWarps);   // one half per tile when BN <= 192
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int num_tiles = a.m_tiles * a.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0, hs = 0;
      uint32_t phase = 0, hphase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile / a.n_tiles, nt = tile - mt * a.n_tiles;
        int n0, h0, w0;
        pix_origin(mt * kTileM, a.H, a.W, n0, h0, w0);
        for (int cc = 0; cc < a.c_chunks; ++cc) {
          for (int u = 0; u < UNITS; ++u) {
            tc::mbar_wait(&hempty[hs], hphase ^ 1);
            tc::mbar_expect_tx(&hfull[hs], unit_tx);
            tc::tma_load_4d(sH + hs * C::UNIT_BYTES, &tmA, &hfull[hs], cc * 64, w0 - 1 + (MODE == 0 ? 0 : u), h0 - 1,
                            n0);
            for (int j = 0; j < TAPS_PER_UNIT; ++j) {
              const int tap = MODE == 0 ? j : j * 3 + u;
              tc::mbar_wait(&empty[stage], phase ^ 1);
              tc::mbar_expect_tx(&full[stage], C::B_BYTES);
              tc::tma_load_3d(sB + stage * C::B_BYTES, &tmB, &full[stage], cc * 64, tap, nt * BN);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            if (++hs == NA) { hs = 0; hphase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(kTileM, BN, false, false);
      int stage = 0, hs = 0;
      uint32_t phase = 0, hphase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + buf * BN;
        bool first = true;
        for (int cc = 0; cc < a.c_chunks; ++cc) {
          const int ksteps = (cc == a.c_chunks - 1) ? a.last_ksteps : 4;
          for (int u = 0; u < UNITS; ++u) {
            tc::mbar_wait(&hfull[hs], hphase);
            tc::tc_fence_after();
            const uint32_t h_base = tc::smem_u32(sH + hs * C::UNIT_BYTES);
            for (int j = 0; j < TAPS_PER_UNIT; ++j) {
              tc::mbar_wait(&full[stage], phase);
              tc::tc_fence_after();
              const uint32_t row = MODE == 0 ? (uint32_t)((j / 3) * 130 + (j % 3)) : (uint32_t)(j * a.W);
              const uint32_t a_base = h_base + row * 128;
              const uint32_t b_base = tc::smem_u32(sB + stage * C::B_BYTES);
              for (int k = 0; k < ksteps; ++k) {
                const uint64_t ad = tc::sdesc_sw128(a_base + k * 32, 16, 1024);
                const uint64_t bd = tc::sdesc_sw128(b_base + k * 32, 16, 1024);
                tc::mma_bf16(d_tmem, ad, bd, idesc, first ? 0u : 1u);
                first = false;
              }
              tc::mma_commit(&empty[stage]);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            tc::mma_commit(&hempty[hs]);
            if (++hs == NA) { hs = 0; hphase ^= 1; }
          }
        }
        tc::mma_commit(&tfull[buf]);
      }
    }
  } else {
    epilogue_loop<BN>(a, &tmO, sO, sbias, tmem, tfull, tempty, num_tiles);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ===========================================================================
// CTA-pair (cta_group::2) fprop / dgrad.  Two CTAs of a cluster share one M = 256 x BN
// tile: each stages its own 128 pixel rows of A and HALF of the B tile (BN/2 weight rows),
// the leader issues tcgen05.mma.cta_group::2 over both CTAs' shared memory, and each
// CTA's TMEM holds its 128 accumulator rows.  Per SM this halves the B traffic at the
// same MMA rate.  A is staged in "units" as in the halo kernels; MODE 2 is the plain
// one-box-per-tap layout (any geometry).
// ===========================================================================
template <int BN, int MODE>
struct Cg2Cfg {
  // MODE 3: MODE 0's halo units with the whole weight resident in shared memory (this CTA's BN/2 rows of all
  // 9 taps x 2 channel chunks, loaded once per CTA) and direct stores from the epilogue (no staging tiles):
  // the C_in = C_out = 96 layers, where re-streaming the weights per tile was half of the per-tile TMA bytes
  static constexpr bool RESB = MODE == 3;
  static constexpr uint32_t UNIT_BYTES = (MODE == 0 || RESB) ? 50176 : (MODE == 1 ? 32768 : kAtomBytes);
  static constexpr int NA = (MODE == 0 || RESB) ? 2 : (MODE == 1 ? 3 : 4);
  static constexpr uint32_t B_BYTES = (BN / 2) * 128;
  static constexpr int SBUFS = RESB ? 0 : kStageBufs;
  static constexpr int STAGES_RAW = RESB ? 18 : (kSmemBudget - NA * (int)UNIT_BYTES) / (int)B_BYTES;
  static constexpr int STAGES = RESB ? 18 : (STAGES_RAW > 12 ? 12 : STAGES_RAW);   // RESB: 9 taps x 2 chunks
  static_assert(STAGES >= 2, "CTA-pair conv needs a >= 2 stage B ring");
  static constexpr uint32_t TMEM_COLS = FpropCfg<BN>::TMEM_COLS;
  static constexpr size_t SMEM = 1024 + NA * UNIT_BYTES + STAGES * B_BYTES + SBUFS * kStageBytes + 512 + 4 * kMaxBiasSmem;
  static_assert(SMEM <= 232448, "CTA-pair conv: shared memory");
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_fprop_cg2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmO, const TcFpropArgs a, const uint32_t unit_tx,
                     const __grid_constant__ TmaQuad tq) {
  using C = Cg2Cfg<BN, MODE>;
  constexpr int STAGES = C::STAGES, NA = C::NA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sH = smem;
  uint8_t* sB = smem + NA * C::UNIT_BYTES;
  uint8_t* sO = sB + STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sO + C::SBUFS * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* hfull = empty + STAGES;
  uint64_t* hempty = hfull + NA;
  uint64_t* tfull = hempty + NA;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool is_leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NA; ++b) {
      tc::mbar_init(&hfull[b], 1);
      tc::mbar_init(&hempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], (BN <= 192 ? 1 : 2) * kEpiWarps);   // both CTAs' epilogue warps (leader's copy)
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int mpairs = (a.m_tiles + 1) / 2;
  const int num_tiles = mpairs * a.n_tiles * (a.phases > 1 ? a.phases : 1);
  const int cid = (int)tc::cluster_id_x(), ncl = (int)tc::num_clusters_x();
  constexpr int M0 = C::RESB ? 0 : MODE;   // the halo geometry of MODE 3 is MODE 0's
  constexpr int UNITS_PER_CHUNK_FIXED = M0 == 0 ? 1 : (M0 == 1 ? 3 : 0);
  const int units_per_chunk = M0 == 2 ? a.taps : UNITS_PER_CHUNK_FIXED;
  const int taps_per_unit = M0 == 0 ? 9 : (M0 == 1 ? 3 : 1);
  const int pad = a.ksz >> 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0, hs = 0;
      uint32_t phase = 0, hphase = 0;
      if constexpr (C::RESB) {   // the whole weight (this CTA's half of the rows), once: stage = cc * 9 + tap
        const uint32_t fbar = tc::map_to_rank(&full[0], 0);
        if (is_leader) tc::mbar_expect_tx(&full[0], 2 * C::STAGES * C::B_BYTES);
        for (int cc = 0; cc < a.c_chunks; ++cc)
          for (int tap = 0; tap < 9; ++tap)
            tc::tma_load_3d_cg2(sB + (cc * 9 + tap) * C::B_BYTES, &tmB, fbar, cc * 64, tap, (int)rank * (BN / 2));
      }
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        const int nt = tile % a.n_tiles;
        const int mp = tile / a.n_tiles;
        const int oph = a.phases > 1 ? mp / mpairs : 0;   // output phase (sub-pixel mode)
        const int mt = (mp - oph * mpairs) * 2 + (int)rank;
        const int pa = oph >> 1, pb = oph & 1;         // its row / column parity
        const int wrow = oph * a.Cout;                 // its weight rows
        int n0, h0, w0;
        pix_origin(mt * kTileM, a.H, a.W, n0, h0, w0);
        for (int cc = 0; cc < a.c_chunks; ++cc) {
          for (int u = 0; u < units_per_chunk; ++u) {
            tc::mbar_wait(&hempty[hs], hphase ^ 1);
            const uint32_t hbar = tc::map_to_rank(&hfull[hs], 0);
            if (is_leader) tc::mbar_expect_tx(&hfull[hs], 2 * unit_tx);
            if (M0 == 0) {
              tc::tma_load_4d_cg2(sH + hs * C::UNIT_BYTES, &tmA, hbar, cc * 64, w0 - 1, h0 - 1, n0);
            } else if (M0 == 1) {
              tc::tma_load_4d_cg2(sH + hs * C::UNIT_BYTES, &tmA, hbar, cc * 64, w0 - 1 + u, h0 - 1, n0);
            } else if (a.phase_dgrad) {   // tap u = phase * 4 + p * 2 + q: dY of phase (a, b) at (i+1-a-p, j+1-b-q)
              const int ph = u >> 2, ta = ph >> 1, tb = ph & 1, p = (u >> 1) & 1, q = u & 1;
              tc::tma_load_4d_cg2(sH + hs * C::UNIT_BYTES, &tq.m[ph], hbar, cc * 64, w0 + 1 - tb - q, h0 + 1 - ta - p,
                                  n0);
            } else if (a.phases > 1) {   // 2x2 taps (p, q) of phase (pa, pb): offsets p - 1 + pa, q - 1 + pb
              const int dy = (u >> 1) - 1 + pa, dx = (u & 1) - 1 + pb;
              tc::tma_load_4d_cg2(sH + hs * C::UNIT_BYTES, &tmA, hbar, cc * 64, w0 + dx, h0 + dy, n0);
            } else {
              const int dy = u / a.ksz - pad, dx = u % a.ksz - pad;
              tc::tma_load_4d_cg2(sH + hs * C::UNIT_BYTES, &tmA, hbar, cc * 64, w0 + dx, h0 + dy, n0);
            }
            for (int j = 0; j < taps_per_unit && !C::RESB; ++j) {
              const int tap = MODE == 0 ? j : (MODE == 1 ? j * 3 + u : u);
              tc::mbar_wait(&empty[stage], phase ^ 1);
              const uint32_t fbar = tc::map_to_rank(&full[stage], 0);
              if (is_leader) tc::mbar_expect_tx(&full[stage], 2 * C::B_BYTES);
              tc::tma_load_3d_cg2(sB + stage * C::B_BYTES, &tmB, fbar, cc * 64, tap,
                                  wrow + nt * BN + (int)rank * (BN / 2));
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            if (++hs == NA) { hs = 0; hphase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (is_leader) {   // the whole (converged) warp runs the loop; one elected lane issues
      constexpr uint32_t idesc = tc::idesc_bf16(256, BN, false, false);
      const bool issuer = tc::elect_one();
      const uint32_t sH0 = tc::smem_u32(sH), sB0 = tc::smem_u32(sB);
      int stage = 0, hs = 0;
      uint32_t phase = 0, hphase = 0;
      int it = 0;
      if constexpr (C::RESB) {
        tc::mbar_wait(&full[0], 0);   // the resident weight has landed in both CTAs
        tc::tc_fence_after();
      }
      for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem + buf * BN;
        uint32_t acc = 0u;
        for (int cc = 0; cc < a.c_chunks; ++cc) {
          const int ksteps = (cc == a.c_chunks - 1) ? a.last_ksteps : 4;
          for (int u = 0; u < units_per_chunk; ++u) {
            tc::mbar_wait(&hfull[hs], hphase);
            tc::tc_fence_after();
            const uint32_t h_base = sH0 + hs * C::UNIT_BYTES;
            for (int j = 0; j < taps_per_unit; ++j) {
              if constexpr (!C::RESB) {
                tc::mbar_wait(&full[stage], phase);
                tc::tc_fence_after();
              }
              const uint32_t row =
                  M0 == 0 ? (uint32_t)((j / 3) * 130 + (j % 3)) : (M0 == 1 ? (uint32_t)(j * a.W) : 0u);
              // descriptors advance by 32 bytes (= 2 in the >>4 address field) per K=16 step
              const uint64_t ad0 = tc::sdesc_sw128(h_base + row * 128, 16, 1024);
              const uint32_t bstage = C::RESB ? (uint32_t)(cc * 9 + j) : (uint32_t)stage;
              const uint64_t bd0 = tc::sdesc_sw128(sB0 + bstage * C::B_BYTES, 16, 1024);
              if (issuer) {
                tc::mma_bf16_cg2(d_tmem, ad0, bd0, idesc, acc);
                if (ksteps > 1) tc::mma_bf16_cg2(d_tmem, ad0 + 2, bd0 + 2, idesc, 1u);
                if (ksteps > 2) tc::mma_bf16_cg2(d_tmem, ad0 + 4, bd0 + 4, idesc, 1u);
                if (ksteps > 3) tc::mma_bf16_cg2(d_tmem, ad0 + 6, bd0 + 6, idesc, 1u);
                if constexpr (!C::RESB) tc::mma_commit_cg2(&empty[stage], 3);
              }
              __syncwarp();
              acc = 1u;
              if constexpr (!C::RESB) {
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
              }
            }
            if (issuer) tc::mma_commit_cg2(&hempty[hs], 3);
            __syncwarp();
            if (++hs == NA) { hs = 0; hphase ^= 1; }
          }
        }
        if (issuer) tc::mma_commit_cg2(&tfull[buf], 3);
        __syncwarp();
      }
    }
  } else {
    epilogue_loop<BN, 2>(a, &tmO, sO, sbias, tmem, tfull, tempty, num_tiles, cid, ncl, (int)rank);
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 1) tc::tmem_dealloc_cg2(tmem, C::TMEM_COLS);
}

// deterministic split-K reduction: dst[i] (+)= sum_s part[s][i] in split order
__global__ void k_split_reduce(const float* __restrict__ part, float* __restrict__ dst, long long n, int splits,
                               int accumulate) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    float s = accumulate ? dst[i] : 0.0f;
    for (int k = 0; k < splits; ++k) s += part[(long long)k * n + i];
    dst[i] = s;
  }
}

// bias-gradient reduction: dst[c] (+)= sum_k part[k][c] for the few output channels of a wgrad launch with
// many splits — one warp per channel, lane l sums splits l, l + 32, ... in order, then a fixed shuffle tree
// (deterministic; replaces a serial per-thread loop that was latency-bound)
__global__ void k_bias_reduce(const float* __restrict__ part, float* __restrict__ dst, int n, int splits,
                              int accumulate) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= n) return;
  float s = 0.0f;
  for (int k = lane; k < splits; k += 32) s += __ldg(part + (long long)k * n + c);
  s = warp_sum(s);
  if (lane == 0) dst[c] = accumulate ? dst[c] + s : s;
}

// the same sum, four consecutive outputs per thread (16-byte loads); per element the order is unchanged
// (dst or 0, then split 0, 1, ...), so the result is bit-identical to k_split_reduce
__global__ void k_split_reduce4(const float4* __restrict__ part, float4* __restrict__ dst, long long n4, int splits,
                                int accumulate) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n4; i += stride) {
    float4 s = accumulate ? dst[i] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int k = 0; k < splits; ++k) {
      const float4 q = __ldg(part + (long long)k * n4 + i);
      s.x += q.x;
      s.y += q.y;
      s.z += q.z;
      s.w += q.w;
    }
    dst[i] = s;
  }
}

// phase wgrad reduction: dW[o][r*3+s][c] = sum_splits sum over the four (phase, tap) pairs whose folded
// 2x2 tap covers (r, s) of part[split][o][phase*4 + p*2 + q][c]  (the adjoint of fold_up2_weights)
__global__ void k_split_reduce_unfold(const float* __restrict__ part, float* __restrict__ dw, int Cout, int Cin,
                                      int splits) {
  const long long n = 9LL * Cout * Cin;
  const long long pstride = 16LL * Cout * Cin;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cin);
    const long long r9 = i / Cin;
    const int rs = (int)(r9 % 9);
    const int o = (int)(r9 / 9);
    const int r = rs / 3, sc = rs % 3;
    // (a, p) pairs whose row set R(a, p) contains r (R(0,0)={0}, R(0,1)={1,2}, R(1,0)={0,1}, R(1,1)={2})
    const int ra[2] = {r == 0 ? 0 : 0, r == 0 ? 1 : 1};
    const int rp[2] = {r == 0 ? 0 : 1, r == 2 ? 1 : 0};
    const int sa[2] = {0, 1};
    const int sp[2] = {sc == 0 ? 0 : 1, sc == 2 ? 1 : 0};
    float acc = 0.0f;
    for (int k = 0; k < splits; ++k) {
      const float* pk = part + k * pstride + (long long)o * 16 * Cin + c;
#pragma unroll
      for (int i1 = 0; i1 < 2; ++i1)
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          const int ph = ra[i1] * 2 + sa[i2], t = rp[i1] * 2 + sp[i2];
          acc += pk[(long long)(ph * 4 + t) * Cin];
        }
    }
    dw[i] = acc;
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

cudaError_t get_encoder() {
  if (g_encode) return cudaSuccess;
  cudaDriverEntryPointQueryResult qr;
  PG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_encode), cudaEnableDefault,
                                  &qr));
  if (qr != cudaDriverEntryPointSuccess || !g_encode) return cudaErrorNotSupported;
  return cudaSuccess;
}

void tile_box(int N, int H, int W, int& bw, int& bh, int& bn) {
  bw = W < 128 ? W : 128;
  bh = H < 128 / bw ? H : 128 / bw;
  bn = 128 / (bw * bh);
  (void)N;
}

cudaError_t act_map(CUtensorMap* m, const void* base, int N, int H, int W, int C) {
  PG_CUDA(get_encoder());
  int bw, bh, bn;
  tile_box(N, H, W, bw, bh, bn);
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bn};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t weight_map(CUtensorMap* m, const void* base, int rows, int taps, int C, int box_rows) {
  PG_CUDA(get_encoder());
  cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)taps, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)C * 2, (cuuint64_t)taps * C * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t out_map(CUtensorMap* m, const void* base, long long M, int C, int ld) {
  PG_CUDA(get_encoder());
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BN>
cudaError_t launch_fprop_bn(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const TcFpropArgs& a,
                            int num_sms, cudaStream_t st) {
  using C = FpropCfg<BN>;
  PG_CUDA((set_smem_once<k_conv_fprop<BN>>((int)C::SMEM)));
  const int tiles = a.m_tiles * a.n_tiles;
  const int grid = tiles < num_sms ? tiles : num_sms;
  k_conv_fprop<BN><<<grid, kThreads, C::SMEM, st>>>(ma, mb, mo, a);
  return cudaGetLastError();
}

cudaError_t halo_map(CUtensorMap* m, const void* base, int N, int H, int W, int C, int bw, int bh) {
  PG_CUDA(get_encoder());
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BN, int MODE>
cudaError_t launch_halo_bn(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const TcFpropArgs& a,
                           uint32_t unit_tx, cudaStream_t st) {
  using C = HaloCfg<BN, MODE>;
  PG_CUDA((set_smem_once<k_conv_fprop_halo<BN, MODE>>((int)C::SMEM)));
  const int tiles = a.m_tiles * a.n_tiles;
  const int grid = tiles < sm_cap() ? tiles : sm_cap();
  k_conv_fprop_halo<BN, MODE><<<grid, kThreads, C::SMEM, st>>>(ma, mb, mo, a, unit_tx);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_halo(int bn, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                        const TcFpropArgs& a, uint32_t unit_tx, cudaStream_t st) {
  switch (bn) {
    case 32: return launch_halo_bn<32, MODE>(ma, mb, mo, a, unit_tx, st);
    case 64: return launch_halo_bn<64, MODE>(ma, mb, mo, a, unit_tx, st);
    case 96: return launch_halo_bn<96, MODE>(ma, mb, mo, a, unit_tx, st);
    case 128: return launch_halo_bn<128, MODE>(ma, mb, mo, a, unit_tx, st);
    case 192: return launch_halo_bn<192, MODE>(ma, mb, mo, a, unit_tx, st);
    default: return launch_halo_bn<256, MODE>(ma, mb, mo, a, unit_tx, st);
  }
}

template <int BN, int MODE>
cudaError_t launch_cg2_bn(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const TcFpropArgs& a,
                          uint32_t unit_tx, cudaStream_t st, const TmaQuad* quad) {
  using C = Cg2Cfg<BN, MODE>;
  PG_CUDA((set_smem_once<k_conv_fprop_cg2<BN, MODE>>((int)C::SMEM)));
  const int tiles = ((a.m_tiles + 1) / 2) * a.n_tiles * (a.phases > 1 ? a.phases : 1);
  int clusters = tiles < sm_cap() / 2 ? tiles : sm_cap() / 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  TmaQuad tq;
  for (int i = 0; i < 4; ++i) tq.m[i] = quad ? quad->m[i] : ma;
  return cudaLaunchKernelEx(&cfg, k_conv_fprop_cg2<BN, MODE>, ma, mb, mo, a, unit_tx, tq);
}

template <int MODE>
cudaError_t launch_cg2(int bn, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                       const TcFpropArgs& a, uint32_t unit_tx, cudaStream_t st, const TmaQuad* quad = nullptr) {
  switch (bn) {
    case 32: return launch_cg2_bn<32, MODE>(ma, mb, mo, a, unit_tx, st, quad);
    case 64: return launch_cg2_bn<64, MODE>(ma, mb, mo, a, unit_tx, st, quad);
    case 96: return launch_cg2_bn<96, MODE>(ma, mb, mo, a, unit_tx, st, quad);
    case 128: return launch_cg2_bn<128, MODE>(ma, mb, mo, a, unit_tx, st, quad);
    case 192: return launch_cg2_bn<192, MODE>(ma, mb, mo, a, unit_tx, st, quad);
    default: return launch_cg2_bn<256, MODE>(ma, mb, mo, a, unit_tx, st, quad);
  }
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <int BN>
cudaError_t launch_wgrad_bn(const CUtensorMap& ma, const CUtensorMap& mb, const TcWgradArgs& a, cudaStream_t st,
                            const TmaQuad* quad = nullptr) {
  using C = WgradCfg<BN>;
  PG_CUDA((set_smem_once<k_conv_wgrad<BN>>((int)C::SMEM)));
  const int units = a.m_tiles * a.n_tiles * a.splits;
  TmaQuad tq;
  for (int i = 0; i < 4; ++i) tq.m[i] = quad ? quad->m[i] : ma;
  k_conv_wgrad<BN><<<units, 192, C::SMEM, st>>>(ma, mb, a, tq);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_wgrad_cg2_bn(const CUtensorMap& ma, const CUtensorMap& mb, const TcWgradArgs& a, cudaStream_t st,
                                const TmaQuad* quad = nullptr) {
  using C = WgradCg2Cfg<BN>;
  PG_CUDA((set_smem_once<k_conv_wgrad_cg2<BN>>((int)C::SMEM)));
  const int units = ((a.m_tiles + 1) / 2) * a.n_tiles * a.splits;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * units, 1, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  TmaQuad tq;
  for (int i = 0; i < 4; ++i) tq.m[i] = quad ? quad->m[i] : ma;
  return cudaLaunchKernelEx(&cfg, k_conv_wgrad_cg2<BN>, ma, mb, a, tq);
}

template <int BN>
cudaError_t launch_wgrad3_bn(const CUtensorMap& ma, const CUtensorMap& mb, const TcWgradArgs& a, cudaStream_t st) {
  using C = Wgrad3Cfg<BN>;
  PG_CUDA((set_smem_once<k_conv_wgrad3<BN>>((int)C::SMEM)));
  k_conv_wgrad3<BN><<<a.m_tiles * a.n_tiles * a.splits, 192, C::SMEM, st>>>(ma, mb, a);
  return cudaGetLastError();
}

int pick_bn(int cout) {
  if (cout % 256 == 0) return 256;
  if (cout % 192 == 0) return 192;
  if (cout % 128 == 0) return 128;
  if (cout == 96) return 96;
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 96) return 96;
  return 128;
}

// The 128-pixel M tile must be one TMA box {bw, bh, bn} in pixel order:
// W a power of two, and either W >= 128 (row segments) or whole rows that tile H
// (or whole images when H*W < 128).
bool tileable(int H, int W) {
  auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  if (!pow2(W) || H < 1) return false;
  if (W >= 128) return true;
  const int rows = 128 / W;
  if (H >= rows) return H % rows == 0;
  return pow2(H);
}

}  // namespace

int tc_fprop_bn(int cout) { return pick_bn(cout); }
bool tc_geometry_ok(int H, int W) { return tileable(H, W); }

cudaError_t tc_conv_fprop(const void* x, int N, int H, int W, int Cin, const void* wpack, int Cout, int ksz,
                          const TcEpilogue& epi, cudaStream_t st) {
  if (Cin % 8 || ((uintptr_t)x & 15) || ((uintptr_t)wpack & 15) || !tileable(H, W)) return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  const int bn = pick_bn(Cout);
  PG_CUDA(act_map(&ma, x, N, H, W, Cin));
  PG_CUDA(weight_map(&mb, wpack, Cout, ksz * ksz, Cin, bn));
  TcFpropArgs a{};
  a.M = (long long)N * H * W;
  a.H = H;
  a.W = W;
  a.ksz = ksz;
  a.taps = ksz * ksz;
  a.c_chunks = ceil_div(Cin, 64);
  a.last_ksteps = ceil_div(Cin - (a.c_chunks - 1) * 64, 16);
  a.Cout = Cout;
  a.m_tiles = ceil_div(a.M, kTileM);
  a.n_tiles = ceil_div(Cout, bn);
  a.bias = epi.bias;
  a.alpha = epi.alpha;
  a.residual = epi.residual;
  a.res_mode = epi.res_mode;
  a.ldr = epi.ldr ? epi.ldr : Cout;
  a.relu_ref = epi.relu_ref;
  a.out = epi.out;
  a.out_f32 = epi.out_f32;
  a.ldo = epi.ldo ? epi.ldo : Cout;
  a.relu_out = epi.relu_out;
  a.pool_out = epi.pool_out;
  a.pool_relu = epi.pool_relu;
  const int sms = sm_cap();
  static const int halo_on = env_int("PARAGAN_HALO", 1), tma_st = env_int("PARAGAN_TMA_STORE", 1),
                   cg2_on = env_int("PARAGAN_CG2", 1);
  CUtensorMap mo;
  a.tma_store = tma_st && !a.out_f32 && (bn % 64 == 0 || a.n_tiles == 1) && a.ldo % 8 == 0 &&
                !((uintptr_t)epi.out & 15);
  if (a.pool_out) {   // the pooled epilogue reads the staging tiles: whole row pairs per 128-pixel tile
    if (!a.tma_store || a.out_f32 || W > 64 || (W & 1) || (H & 1) || !tileable(H, W) || Cout % 16 ||
        ((uintptr_t)epi.pool_out & 15) || ((uintptr_t)epi.pool_relu & 15))
      return cudaErrorInvalidValue;
  }
  if (a.tma_store && !a.pool_out) PG_CUDA(out_map(&mo, epi.out, a.M, Cout, a.ldo));
  else mo = mb;   // unused
  if (cg2_on && a.tma_store && a.m_tiles >= 2) {
    CUtensorMap mb2;
    PG_CUDA(weight_map(&mb2, wpack, Cout, ksz * ksz, Cin, bn / 2));
    if (halo_on && ksz == 3 && W % 128 == 0) {
      CUtensorMap mh;
      PG_CUDA(halo_map(&mh, x, N, H, W, Cin, 130, 3));
      static const int resb_on = env_int("PARAGAN_RESB", 1);
      if (resb_on && bn == 96 && Cout == 96 && a.n_tiles == 1 && a.c_chunks == 2) {
        TcFpropArgs a3 = a;   // resident weight, direct-store epilogue
        a3.tma_store = 0;
        return launch_cg2_bn<96, 3>(mh, mb2, mo, a3, 390u * 128u, st, nullptr);
      }
      return launch_cg2<0>(bn, mh, mb2, mo, a, 390u * 128u, st);
    }
    if (halo_on && ksz == 3 && W >= 16 && W <= 64 && H % (128 / W) == 0) {
      const int rows = 128 / W + 2;
      CUtensorMap mh;
      PG_CUDA(halo_map(&mh, x, N, H, W, Cin, W, rows));
      return launch_cg2<1>(bn, mh, mb2, mo, a, (uint32_t)(rows * W * 128), st);
    }
    return launch_cg2<2>(bn, ma, mb2, mo, a, kAtomBytes, st);
  }
  if (halo_on && ksz == 3 && W % 128 == 0) {
    CUtensorMap mh;
    PG_CUDA(halo_map(&mh, x, N, H, W, Cin, 130, 3));
    return launch_halo<0>(bn, mh, mb, mo, a, 390u * 128u, st);
  }
  if (halo_on && ksz == 3 && W >= 16 && W <= 64 && H % (128 / W) == 0) {
    const int rows = 128 / W + 2;
    CUtensorMap mh;
    PG_CUDA(halo_map(&mh, x, N, H, W, Cin, W, rows));
    return launch_halo<1>(bn, mh, mb, mo, a, (uint32_t)(rows * W * 128), st);
  }
  switch (bn) {
    case 32: return launch_fprop_bn<32>(ma, mb, mo, a, sms, st);
    case 64: return launch_fprop_bn<64>(ma, mb, mo, a, sms, st);
    case 96: return launch_fprop_bn<96>(ma, mb, mo, a, sms, st);
    case 128: return launch_fprop_bn<128>(ma, mb, mo, a, sms, st);
    case 192: return launch_fprop_bn<192>(ma, mb, mo, a, sms, st);
    default: return launch_fprop_bn<256>(ma, mb, mo, a, sms, st);
  }
}

cudaError_t tc_conv_fprop_up2(const void* x, int N, int H, int W, int Cin, const void* wpack4, int Cout,
                              const TcEpilogue& epi, cudaStream_t st) {
  if (Cin % 8 || Cout % 8 || ((uintptr_t)x & 15) || ((uintptr_t)wpack4 & 15) || ((uintptr_t)epi.out & 15) ||
      !tileable(H, W) || epi.residual || epi.out_f32 || (epi.ldo && epi.ldo != Cout) ||
      ((uintptr_t)epi.relu_ref & 15))
    return cudaErrorInvalidValue;
  const int bn = pick_bn(Cout);
  TcFpropArgs a{};
  a.M = (long long)N * H * W;
  a.H = H;
  a.W = W;
  a.ksz = 2;
  a.taps = 4;
  a.c_chunks = ceil_div(Cin, 64);
  a.last_ksteps = ceil_div(Cin - (a.c_chunks - 1) * 64, 16);
  a.Cout = Cout;
  a.m_tiles = ceil_div(a.M, kTileM);
  a.n_tiles = ceil_div(Cout, bn);
  a.bias = epi.bias;
  a.alpha = epi.alpha;
  a.relu_ref = epi.relu_ref;   // full-resolution [N][2H][2W][Cout] (the epilogue maps each phase's pixel)
  a.out = epi.out;
  a.ldo = Cout;
  a.ldr = Cout;
  a.tma_store = 1;
  a.phases = 4;
  if (!(bn % 64 == 0 || a.n_tiles == 1)) return cudaErrorInvalidValue;
  CUtensorMap ma, mb2, mo;
  PG_CUDA(act_map(&ma, x, N, H, W, Cin));
  PG_CUDA(weight_map(&mb2, wpack4, 4 * Cout, 4, Cin, bn / 2));
  {
    // output [N][2H][2W][C] viewed as {C, 2 (column phase), W, 2 (row phase), N*H}
    PG_CUDA(get_encoder());
    int bw, bh, bnn;
    tile_box(N, H, W, bw, bh, bnn);
    cuuint64_t dims[5] = {(cuuint64_t)Cout, 2, (cuuint64_t)W, 2, (cuuint64_t)N * H};
    cuuint64_t strides[4] = {(cuuint64_t)Cout * 2, (cuuint64_t)Cout * 4, (cuuint64_t)W * Cout * 4,
                             (cuuint64_t)W * Cout * 8};
    cuuint32_t box[5] = {64, 1, (cuuint32_t)bw, 1, (cuuint32_t)(bh * bnn)};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = g_encode(&mo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, epi.out, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return launch_cg2<2>(bn, ma, mb2, mo, a, kAtomBytes, st);
}

cudaError_t tc_conv_dgrad_up2(const void* dy, int N, int H, int W, int Cout, const void* wt4, int Cin,
                              const TcEpilogue& epi, cudaStream_t st) {
  if (Cin % 8 || Cout % 8 || ((uintptr_t)dy & 15) || ((uintptr_t)wt4 & 15) || ((uintptr_t)epi.out & 15) ||
      !tileable(H, W) || epi.out_f32)
    return cudaErrorInvalidValue;
  const int bn = pick_bn(Cin);
  TcFpropArgs a{};
  a.M = (long long)N * H * W;
  a.H = H;
  a.W = W;
  a.ksz = 2;
  a.taps = 16;
  a.c_chunks = ceil_div(Cout, 64);
  a.last_ksteps = ceil_div(Cout - (a.c_chunks - 1) * 64, 16);
  a.Cout = Cin;
  a.m_tiles = ceil_div(a.M, kTileM);
  a.n_tiles = ceil_div(Cin, bn);
  a.bias = epi.bias;
  a.alpha = epi.alpha;
  a.residual = epi.residual;
  a.res_mode = epi.res_mode;
  a.ldr = epi.ldr ? epi.ldr : Cin;
  a.relu_ref = epi.relu_ref;
  a.out = epi.out;
  a.ldo = epi.ldo ? epi.ldo : Cin;
  a.tma_store = (bn % 64 == 0 || a.n_tiles == 1) && a.ldo % 8 == 0;
  a.phases = 1;
  a.phase_dgrad = 1;
  if (!a.tma_store) return cudaErrorInvalidValue;
  CUtensorMap mb2, mo;
  PG_CUDA(weight_map(&mb2, wt4, Cin, 16, Cout, bn / 2));
  PG_CUDA(out_map(&mo, epi.out, a.M, Cin, a.ldo));
  TmaQuad tq;
  {
    PG_CUDA(get_encoder());
    int bw, bh, bnn;
    tile_box(N, H, W, bw, bh, bnn);
    for (int ph = 0; ph < 4; ++ph) {
      // dY of output phase (a, b) as a low-resolution [N][H][W][Cout] tensor
      const int pa = ph >> 1, pb = ph & 1;
      const char* base = static_cast<const char*>(dy) + ((size_t)pa * 2 * W + pb) * Cout * 2;
      cuuint64_t dims[4] = {(cuuint64_t)Cout, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t strides[3] = {(cuuint64_t)Cout * 4, (cuuint64_t)W * Cout * 8, (cuuint64_t)H * W * Cout * 8};
      cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bnn};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = g_encode(&tq.m[ph], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<char*>(base), dims, strides,
                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
  }
  return launch_cg2<2>(bn, tq.m[0], mb2, mo, a, kAtomBytes, st, &tq);
}

// Split-K factor for the wgrad grid (one CTA per SM, one work unit per CTA): minimise
//   waves(s) * (K-blocks per split + prologue/epilogue) * t_kb + the split reduction's traffic,
// waves(s) = ceil(tiles * s / #SMs).  (Taking the smallest s that fills the SMs twice can leave a
// third wave with a handful of CTAs — e.g. 9 taps x 33 splits = 297 CTAs on 148 SMs.)
int choose_wgrad_splits(int tiles, long long total_kb, int bn, size_t part_floats, size_t scratch_floats,
                        bool reduce_always) {
  const double t_kb = 2.0 * 128 * bn * 128 / 7.0e6;   // us per K-block per SM (~7 TFLOP/s per SM)
  long long smax = total_kb / 4;
  if (smax < 1) smax = 1;
  if (smax > 4096) smax = 4096;
  int best = 1;
  double best_cost = 1e300;
  for (long long s = 1; s <= smax; ++s) {
    if (s > 1 && (size_t)s * part_floats > scratch_floats) break;
    const long long units = (long long)tiles * s;
    const long long waves = (units + kNumSMs - 1) / kNumSMs;
    const long long kb = (total_kb + s - 1) / s;
    double cost = (double)waves * (double)(kb + 3) * t_kb;
    if (s > 1 || reduce_always) cost += (double)s * part_floats * 8.0 / 6.0e6;   // write + read partials
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = (int)s;
    }
  }
  return best;
}

cudaError_t tc_conv_wgrad_up2(const void* x, const void* dy, int N, int H, int W, int Cin, int Cout, float* dw,
                              float* scratch, size_t scratch_floats, cudaStream_t st, float* dbias) {
  if (Cin % 8 || Cout % 8 || ((uintptr_t)x & 15) || ((uintptr_t)dy & 15) || !tileable(H, W))
    return cudaErrorInvalidValue;
  int bn;
  if (Cin % 256 == 0) bn = 256;
  else if (Cin % 192 == 0) bn = 192;
  else if (Cin % 128 == 0) bn = 128;
  else if (Cin <= 32) bn = 32;
  else if (Cin <= 64) bn = 64;
  else if (Cin <= 96) bn = 96;
  else bn = 128;
  CUtensorMap mx;
  PG_CUDA(act_map(&mx, x, N, H, W, Cin));
  TmaQuad tq;
  {
    PG_CUDA(get_encoder());
    int bw, bh, bnn;
    tile_box(N, H, W, bw, bh, bnn);
    for (int ph = 0; ph < 4; ++ph) {   // dY of output phase (a, b) as a low-resolution tensor
      const char* base = static_cast<const char*>(dy) + ((size_t)(ph >> 1) * 2 * W + (ph & 1)) * Cout * 2;
      cuuint64_t dims[4] = {(cuuint64_t)Cout, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t strides[3] = {(cuuint64_t)Cout * 4, (cuuint64_t)W * Cout * 8, (cuuint64_t)H * W * Cout * 8};
      cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bnn};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = g_encode(&tq.m[ph], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<char*>(base), dims, strides,
                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
  }
  TcWgradArgs a{};
  a.H = H;
  a.W = W;
  a.ksz = 2;
  a.taps = 16;
  a.Cin = Cin;
  a.Cout = Cout;
  a.c_blocks = ceil_div(Cin, bn);
  a.m_tiles = ceil_div(Cout, 128);
  a.n_tiles = a.taps * a.c_blocks;
  a.total_kb = ceil_div((long long)N * H * W, kTileM);
  a.phases = 4;
  const int tiles = a.m_tiles * a.n_tiles;
  const size_t out_floats = (size_t)Cout * a.taps * Cin;
  const size_t bias_floats = dbias ? (size_t)4 * Cout : 0;
  const int splits = choose_wgrad_splits(tiles, a.total_kb, bn, out_floats + bias_floats, scratch_floats, true);
  if ((size_t)splits * (out_floats + bias_floats) > scratch_floats) return cudaErrorMemoryAllocation;
  a.kb_per_split = ceil_div(a.total_kb, splits);
  a.splits = ceil_div(a.total_kb, a.kb_per_split);
  a.out = scratch;
  a.bias_out = dbias ? scratch + (size_t)a.splits * out_floats : nullptr;
  static const int wg_cg2 = env_int("PARAGAN_WGRAD_CG2", 2);
  cudaError_t e;
  if (wg_cg2 && bn == 256 && Cout % 256 == 0) e = launch_wgrad_cg2_bn<256>(tq.m[0], mx, a, st, &tq);
  else switch (bn) {
    case 32: e = launch_wgrad_bn<32>(tq.m[0], mx, a, st, &tq); break;
    case 64: e = launch_wgrad_bn<64>(tq.m[0], mx, a, st, &tq); break;
    case 96: e = launch_wgrad_bn<96>(tq.m[0], mx, a, st, &tq); break;
    case 128: e = launch_wgrad_bn<128>(tq.m[0], mx, a, st, &tq); break;
    case 192: e = launch_wgrad_bn<192>(tq.m[0], mx, a, st, &tq); break;
    default: e = launch_wgrad_bn<256>(tq.m[0], mx, a, st, &tq); break;
  }
  PG_CUDA(e);
  {
    const long long n = 9LL * Cout * Cin;
    int blocks = ceil_div(n, 256);
    if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
    k_split_reduce_unfold<<<blocks, 256, 0, st>>>(scratch, dw, Cout, Cin, a.splits);
    PG_LAUNCH_CHECK();
  }
  if (dbias) {
    k_bias_reduce<<<ceil_div(Cout, 8), 256, 0, st>>>(a.bias_out, dbias, Cout, a.splits * 4, 0);
    PG_LAUNCH_CHECK();
  }
  return cudaSuccess;
}

size_t tc_wgrad_workspace_floats(int N, int H, int W, int Cin, int Cout, int ksz) {
  // upper bound used by the engine to size its split-K scratch
  (void)N; (void)H; (void)W;
  return (size_t)32 * Cout * ksz * ksz * Cin;
}

cudaError_t tc_conv_wgrad(const void* x, const void* dy, int N, int H, int W, int Cin, int Cout, int ksz,
                          float* dw, int accumulate, float* scratch, size_t scratch_floats, cudaStream_t st,
                          float* dbias) {
  if (Cin % 8 || Cout % 8 || ((uintptr_t)x & 15) || ((uintptr_t)dy & 15) || !tileable(H, W))
    return cudaErrorInvalidValue;
  int bn;
  if (Cin % 256 == 0) bn = 256;
  else if (Cin % 192 == 0) bn = 192;
  else if (Cin % 128 == 0) bn = 128;
  else if (Cin <= 32) bn = 32;
  else if (Cin <= 64) bn = 64;
  else if (Cin <= 96) bn = 96;
  else bn = 128;
  // one filter row per CTA (k_conv_wgrad3) for 3x3 convs whose tile rows are >= 16 pixels
  static const int row3_on = env_int("PARAGAN_WGRAD3", 1), wg_cg2 = env_int("PARAGAN_WGRAD_CG2", 2);
  // CTA-pair kernel for C_in, C_out multiples of 256 (measured in the bench step: 1536 -> 1536 at 8x8
  // 1093 -> 1394 TFLOP/s, 768 -> 768 at 16x16 1421 (one-row kernel) -> 1520); PARAGAN_WGRAD_CG2=1 keeps
  // the one-row kernel for 3x3 layers with W >= 16, 0 disables the pair kernel
  const bool pair = wg_cg2 && Cin % 256 == 0 && Cout % 256 == 0 && (wg_cg2 == 2 || ksz != 3 || W < 16);
  int bn3 = 0;
  // (measured in the bench step, B200: 96 -> 96 at 128x128 665 -> 816 TFLOP/s, 192 -> 192 at 64x64 828 -> 872
  // as two 96-channel blocks, 384 -> 384 at 32x32 1185 -> 1342)
  if (row3_on && ksz == 3 && W >= 16 && !pair) {
    if (Cin <= 64) bn3 = 64;
    else if (Cin <= 96) bn3 = 96;
    else if (Cin % 128 == 0) bn3 = 128;
    else if (Cin % 96 == 0) bn3 = 96;
  }
  CUtensorMap mdy, mx;
  PG_CUDA(act_map(&mdy, dy, N, H, W, Cout));
  if (bn3) {
    const int Wt = W < 128 ? W : 128;
    PG_CUDA(halo_map(&mx, x, N, H, W, Cin, Wt + 2, 128 / Wt));
    bn = bn3;
  } else {
    PG_CUDA(act_map(&mx, x, N, H, W, Cin));
  }
  TcWgradArgs a{};
  a.H = H;
  a.W = W;
  a.ksz = ksz;
  a.taps = ksz * ksz;
  a.Cin = Cin;
  a.Cout = Cout;
  a.c_blocks = ceil_div(Cin, bn);
  a.m_tiles = ceil_div(Cout, 128);
  a.n_tiles = (bn3 ? 3 : a.taps) * a.c_blocks;
  a.total_kb = ceil_div((long long)N * H * W, kTileM);
  const int tiles = a.m_tiles * a.n_tiles;
  const size_t out_floats = (size_t)Cout * a.taps * Cin;
  const size_t bias_floats = dbias ? (size_t)Cout : 0;
  const int splits = choose_wgrad_splits(tiles, a.total_kb, bn3 ? 3 * bn3 : bn, out_floats + bias_floats,
                                         scratch_floats, accumulate != 0);
  const bool direct = (splits == 1 && !accumulate);
  if (!direct && (size_t)splits * (out_floats + bias_floats) > scratch_floats) return cudaErrorMemoryAllocation;
  a.kb_per_split = ceil_div(a.total_kb, splits);
  a.splits = ceil_div(a.total_kb, a.kb_per_split);
  a.out = direct ? dw : scratch;
  a.bias_out = dbias ? (direct ? dbias : scratch + (size_t)a.splits * out_floats) : nullptr;
  cudaError_t e;
  if (pair) {
    e = launch_wgrad_cg2_bn<256>(mdy, mx, a, st);
  } else if (bn3) {
    // the cost model's per-K-block time covers the three taps
    switch (bn3) {
      case 64: e = launch_wgrad3_bn<64>(mdy, mx, a, st); break;
      case 96: e = launch_wgrad3_bn<96>(mdy, mx, a, st); break;
      default: e = launch_wgrad3_bn<128>(mdy, mx, a, st); break;
    }
  } else switch (bn) {
    case 32: e = launch_wgrad_bn<32>(mdy, mx, a, st); break;
    case 64: e = launch_wgrad_bn<64>(mdy, mx, a, st); break;
    case 96: e = launch_wgrad_bn<96>(mdy, mx, a, st); break;
    case 128: e = launch_wgrad_bn<128>(mdy, mx, a, st); break;
    case 192: e = launch_wgrad_bn<192>(mdy, mx, a, st); break;
    default: e = launch_wgrad_bn<256>(mdy, mx, a, st); break;
  }
  PG_CUDA(e);
  if (!direct) {
    const long long n = (long long)out_floats;
    if (n % 4 == 0 && (((uintptr_t)scratch | (uintptr_t)dw) & 15) == 0) {
      int blocks = ceil_div(n / 4, 256);
      if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
      k_split_reduce4<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(scratch), reinterpret_cast<float4*>(dw),
                                              n / 4, a.splits, accumulate);
    } else {
      int blocks = ceil_div(n, 256);
      if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
      k_split_reduce<<<blocks, 256, 0, st>>>(scratch, dw, n, a.splits, accumulate);
    }
    PG_LAUNCH_CHECK();
    if (dbias) {
      k_bias_reduce<<<ceil_div(Cout, 8), 256, 0, st>>>(a.bias_out, dbias, Cout, a.splits, accumulate);
      PG_LAUNCH_CHECK();
    }
  }
  return cudaSuccess;
}

}  // namespace pg
