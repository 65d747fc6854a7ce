// Fused tcgen05 attention for the BigGAN non-local block (reading
// R8: beta = softmax_rows(theta^T phi) with no 1/sqrt(d) scale, o = beta g).
//
// The [HW x Q] score matrix of an image (4096 x 1024 at 64x64) never reaches HBM:
//
//   forward  — persistent CTAs walk the (image, 128-query tile) list.  Pass 1 streams
//              128-key chunks of phi, S = theta phi^T lands in TMEM and the softmax
//              warps take the row max m (no exponentials).  Pass 2 recomputes each S
//              chunk, writes P~ = exp(S - m) <= 1 as bf16 into a SW128 smem tile and sums
//              l = sum P~ in fp32, while the MMA warp accumulates O += P~ g in TMEM; the
//              epilogue scales by 1/l (reading R21: the bf16 storage point of beta is taken
//              before the normalisation).  Outputs: o (bf16), o32 (fp32, optional) and
//              lse = m + log l per row.
//   backward — one CTA per (image, 128-key block), looping over the query tiles:
//              S^T and dP^T = g dO^T in TMEM, P = exp(S - lse) recomputed in fp32,
//              dS = P (dP - D) with D = rowsum(dO * o32) (= rowsum(dP * P)), then
//                dg   += P^T dO      (TMEM accumulator, per key)
//                dphi += dS^T theta  (TMEM accumulator, per key)
//                dtheta_part = dS phi (per query tile; one fp32 partial per key block,
//                                      summed in a fixed order by the caller)
//              so every reduction is deterministic.
//
// Operands are staged by TMA with 128-byte swizzle; the MMA reads the P / dS tiles
// both K-major (P^T dO, dS^T theta) and MN-major (dS phi).
#include "tc_attn.h"

#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace pg {
namespace {

constexpr int kT = 128;                 // query rows per tile = keys per chunk
constexpr uint32_t kAtom = 16384;       // 128 rows x 128 B, one SW128 operand atom
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSpan = 16.0f;          // single-pass forward when every row's score bound is within e^16 of chunk 0's max
constexpr float kFlat = 40.0f;          // "flat" tiles: every score of the image lies in [-U, U] with U <= 40, so the
                                        // constant offset U (exp(S - U) in [e^-80, 1], normal in fp32 / bf16) needs
                                        // no per-tile max and no decision round-trip
constexpr int kFwdKStages = 3, kFwdVMax = 4;   // V ring: as many stages (2..4) as fit
constexpr int kFwdThreads = 320;        // w0 TMA, w1 MMA, w2-9 softmax / epilogue
constexpr int kSoftThreads = 256;
constexpr int kBwdThreads = 320;        // w0 TMA, w1 MMA, w2-9 softmax / epilogue

// the dynamic shared-memory base rounded up to 1024 bytes by pointer arithmetic on the shared array itself, so
// the compiler keeps the shared address space (LDS/STS, not generic LD/ST) for every access derived from it
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (tc::smem_u32(p) & 1023u)) & 1023u);
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 16-byte chunk c (0..7) of row r of a K-major SW128 atom
__device__ __forceinline__ void st_sw128(uint8_t* atom, int r, int c, uint4 v) {
  *reinterpret_cast<uint4*>(atom + r * 128 + ((c ^ (r & 7)) << 4)) = v;
}

__device__ __forceinline__ uint64_t kdesc(const void* p) {   // K-major operand
  return tc::sdesc_sw128(tc::smem_u32(p), 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc(const void* p) {  // MN-major operand, 64-wide atoms kAtom apart
  return tc::sdesc_sw128(tc::smem_u32(p), kAtom, 1024);
}

// ===========================================================================
// forward (persistent: one CTA per SM walks the (image, query tile) list)
// ===========================================================================
__global__ void __launch_bounds__(kFwdThreads, 1)
    k_attn_fwd(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const TcAttnArgs a, const int nvs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int C2 = a.C2;
  const uint32_t v_bytes = 2u * C2 * 128;       // two boxes [C2][64 keys]
  uint8_t* sQ = smem;                           // 2 buffers: the next tile's theta loads during this tile
  uint8_t* sK = sQ + 2 * kAtom;
  uint8_t* sP = sK + kFwdKStages * kAtom;       // 2 buffers x 2 atoms
  uint8_t* sV = sP + 4 * kAtom;
  float* red = reinterpret_cast<float*>(sV + nvs * v_bytes);   // [2 tiles][2 halves][128] row max
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * 2 * kT);
  uint64_t* qfull = bars;        // [2]
  uint64_t* qempty = bars + 2;   // [2]
  uint64_t* kfull = bars + 4;
  uint64_t* kempty = kfull + kFwdKStages;
  uint64_t* vfull = kempty + kFwdKStages;
  uint64_t* vempty = vfull + kFwdVMax;
  uint64_t* sfull = vempty + kFwdVMax;
  uint64_t* sempty = sfull + 2;
  uint64_t* pfull = sempty + 2;
  uint64_t* pempty = pfull + 2;
  uint64_t* ofull = pempty + 2;   // [2] O double-buffered in TMEM: a tile's epilogue runs during the next tile
  uint64_t* oempty = ofull + 2;   // [2]
  uint64_t* decbar = oempty + 2;                                    // per tile: single- or two-pass decided
  uint32_t* dec = reinterpret_cast<uint32_t*>(decbar + 1);
  uint32_t* tmem_slot = dec + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmQ);
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmV);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&qfull[s], 1);
      tc::mbar_init(&qempty[s], 1);
    }
    for (int s = 0; s < kFwdKStages; ++s) {
      tc::mbar_init(&kfull[s], 1);
      tc::mbar_init(&kempty[s], 1);
    }
    for (int s = 0; s < nvs; ++s) {
      tc::mbar_init(&vfull[s], 1);
      tc::mbar_init(&vempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&sfull[s], 1);
      tc::mbar_init(&sempty[s], kSoftThreads);
      tc::mbar_init(&pfull[s], kSoftThreads);
      tc::mbar_init(&pempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&ofull[s], 1);
      tc::mbar_init(&oempty[s], kSoftThreads);
    }
    tc::mbar_init(decbar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;   // S buffers at columns 0 / 128, O buffers at 256 / 256 + C2

  const int tiles_per_img = a.HW / kT;
  const int num_tiles = a.n * tiles_per_img;
  const int NC = a.Q / kT;
  // the image-wide Cauchy-Schwarz bound U = max_i |theta_i| max_j |phi_j| (every role evaluates the same
  // expression on the same global values, so they agree without communicating)
  auto flat_bound = [&](int b) -> float {
    if (!a.thetamax || !a.phimax || NC < 2) return -1.0f;
    const float U = a.thetamax[b] * a.phimax[b] * 1.001f + 1e-3f;
    return U <= kFlat ? U : -1.0f;   // false for NaN / inf
  };

  if (warp == 0) {
    if (lane == 0) {
      int ks = 0, vs = 0, it = 0, dit = 0;
      uint32_t kph = 0, vph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int b = tile / tiles_per_img;
        const int q0 = (tile - b * tiles_per_img) * kT;
        const int qb = it & 1;
        tc::mbar_wait(&qempty[qb], ((it >> 1) & 1) ^ 1);
        tc::mbar_expect_tx(&qfull[qb], kAtom);
        tc::tma_load_3d(sQ + qb * kAtom, &tmQ, &qfull[qb], 0, q0, b);
        auto load_k = [&](int c) {
          tc::mbar_wait(&kempty[ks], kph ^ 1);
          tc::mbar_expect_tx(&kfull[ks], kAtom);
          tc::tma_load_3d(sK + ks * kAtom, &tmK, &kfull[ks], 0, c * kT, b);
          if (++ks == kFwdKStages) { ks = 0; kph ^= 1; }
        };
        auto load_v = [&](int c) {
          tc::mbar_wait(&vempty[vs], vph ^ 1);
          tc::mbar_expect_tx(&vfull[vs], v_bytes);
          uint8_t* dv = sV + vs * v_bytes;
          tc::tma_load_3d(dv, &tmV, &vfull[vs], c * kT, 0, b);
          tc::tma_load_3d(dv + C2 * 128, &tmV, &vfull[vs], c * kT + 64, 0, b);
          if (++vs == nvs) { vs = 0; vph ^= 1; }
        };
        // K(0), K(1) and V(0), V(1) come first in both schedules (the V ring is consumed in chunk order by
        // either); the rest depends on the tile's decision
        load_k(0);
        if (NC > 1) load_k(1);
        const int vpre = NC < 2 ? NC : 2;
        for (int c = 0; c < vpre; ++c) load_v(c);
        bool single = true;
        if (flat_bound(b) < 0.0f) {
          tc::mbar_wait(decbar, dit & 1);
          single = *reinterpret_cast<volatile uint32_t*>(dec) != 0;
          ++dit;
        }
        if (single) {   // single pass: V(c), then K(c + 2)
          for (int c = 0; c < NC; ++c) {
            if (c >= vpre) load_v(c);
            if (c + 2 < NC) load_k(c + 2);
          }
        } else {                                            // two passes: the rest of pass 1, then pass 2
          for (int c = 2; c < NC; ++c) load_k(c);
          for (int c = 0; c < NC; ++c) {
            load_k(c);
            if (c >= vpre) load_v(c);
          }
        }
      }
    }
  } else if (warp == 1) {
    {   // whole (converged) warp runs the loop, one elected lane issues: uniform descriptors
      const bool issuer = tc::elect_one();
      const uint32_t idS = tc::idesc_bf16(kT, kT, false, false);
      const uint32_t idO = tc::idesc_bf16(kT, C2, false, false);
      const int ksteps = a.Cq / 16;
      int ks = 0, vs = 0, it = 0, dit = 0;
      uint32_t kph = 0, vph = 0;
      uint32_t su = 0, pc = 0;   // running S-buffer use / P-buffer use counters
      int qb = 0;                // theta buffer of the current tile
      auto issue_s = [&](bool last) {
        const int sb = su & 1;
        tc::mbar_wait(&sempty[sb], ((su >> 1) & 1) ^ 1);
        tc::mbar_wait(&kfull[ks], kph);
        tc::tc_fence_after();
        if (issuer) {
          for (int k = 0; k < ksteps; ++k)
            tc::mma_bf16(tmem + sb * kT, kdesc(sQ + qb * kAtom + k * 32), kdesc(sK + ks * kAtom + k * 32), idS, k > 0);
          tc::mma_commit(&kempty[ks]);
          tc::mma_commit(&sfull[sb]);
          if (last) tc::mma_commit(&qempty[qb]);
        }
        __syncwarp();
        if (++ks == kFwdKStages) { ks = 0; kph ^= 1; }
        ++su;
      };
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        qb = it & 1;
        tc::mbar_wait(&qfull[qb], (it >> 1) & 1);
        tc::tc_fence_after();
        issue_s(false);                                     // chunk 0 (its max decides the schedule)
        bool single = true;
        if (flat_bound(tile / tiles_per_img) < 0.0f) {
          tc::mbar_wait(decbar, dit & 1);
          single = *reinterpret_cast<volatile uint32_t*>(dec) != 0;
          ++dit;
        }
        if (!single) {
          for (int u = 1; u < NC; ++u) issue_s(false);      // rest of pass 1
          issue_s(NC == 1);                                 // pass 2 starts again at chunk 0
        }
        const int ob = it & 1;
        tc::mbar_wait(&oempty[ob], ((it >> 1) & 1) ^ 1);   // the O buffer of two tiles ago has been read out
        for (int c = 0; c < NC; ++c) {
          if (c + 1 < NC) issue_s(c + 2 == NC);
          const int pb = pc & 1;
          tc::mbar_wait(&pfull[pb], (pc >> 1) & 1);
          tc::mbar_wait(&vfull[vs], vph);
          tc::tc_fence_after();
          const uint8_t* p = sP + pb * 2 * kAtom;
          const uint8_t* v = sV + vs * v_bytes;
          if (issuer) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              tc::mma_bf16(tmem + 256 + ob * C2, kdesc(p + (k >> 2) * kAtom + (k & 3) * 32),
                           kdesc(v + (k >> 2) * C2 * 128 + (k & 3) * 32), idO, (c | k) != 0);
            tc::mma_commit(&pempty[pb]);
            tc::mma_commit(&vempty[vs]);
          }
          __syncwarp();
          if (++vs == nvs) { vs = 0; vph ^= 1; }
          ++pc;
        }
        if (issuer) tc::mma_commit(&ofull[ob]);
        __syncwarp();
      }
    }
  } else {
    // 8 softmax warps: TMEM lane quadrant qd = warp % 4, half h = 64 of the 128 columns of a chunk
    const int qd = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = qd * 32 + lane;
    const uint32_t lrow = tmem + ((uint32_t)(qd * 32) << 16);
    uint32_t su = 0, pc = 0;
    // epilogue of a finished tile, deferred into the next tile (after its chunk 0's P~ is handed to the MMA
    // warp), so the wait for the tile's last P~ g MMA and the O stores overlap the next tile's MMAs
    struct Pending {
      int valid, ob, ob2ph;
      long long grow;
      float m, l;
    } pend{0, 0, 0, 0, 0.0f, 0.0f};
    auto epilogue = [&]() {
      if (!pend.valid) return;
      pend.valid = 0;
      const int ob = pend.ob;
      const float inv_l = 1.0f / pend.l;
      tc::mbar_wait(&ofull[ob], pend.ob2ph);
      tc::tc_fence_after();
      bf16* op = static_cast<bf16*>(a.o) + pend.grow * C2;
      float* op32 = a.o32 ? a.o32 + pend.grow * C2 : nullptr;
#pragma unroll 1
      for (int cb = h * 32; cb < C2; cb += 64) {
        float v[32];
        tc::tmem_ld32(lrow + 256 + ob * C2 + cb, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= inv_l;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (cb + j * 8 < C2) {
            *reinterpret_cast<uint4*>(op + cb + j * 8) =
                make_uint4(pack2(v[j * 8], v[j * 8 + 1]), pack2(v[j * 8 + 2], v[j * 8 + 3]),
                           pack2(v[j * 8 + 4], v[j * 8 + 5]), pack2(v[j * 8 + 6], v[j * 8 + 7]));
            if (op32) {
              *reinterpret_cast<float4*>(op32 + cb + j * 8) =
                  make_float4(v[j * 8], v[j * 8 + 1], v[j * 8 + 2], v[j * 8 + 3]);
              *reinterpret_cast<float4*>(op32 + cb + j * 8 + 4) =
                  make_float4(v[j * 8 + 4], v[j * 8 + 5], v[j * 8 + 6], v[j * 8 + 7]);
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&oempty[ob]);
      if (h == 0) a.lse[pend.grow] = pend.m + logf(pend.l);
    };
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int b = tile / tiles_per_img;
      const int q0 = (tile - b * tiles_per_img) * kT;
      // chunk 0: its row max m0 and the Cauchy-Schwarz bound U = |theta_i| max_j |phi_j| >= every score of
      // the row.  When U - m0 <= kSpan for every row of the tile, m0 serves as the softmax offset for all
      // chunks (P~ = exp(S - m0) <= e^kSpan: no overflow, and bf16 / fp32 keep their relative precision at
      // any magnitude), so the scores are computed and exponentiated once (single pass); otherwise pass 1
      // finds the exact row max first (two passes).  Either way O = (P~ g) / l and lse = m + log l exactly.
      // Flat images (flat_bound): the offset is the image-wide bound U itself, every chunk is loaded in the loop
      // below and there is neither a chunk-0 max nor a decision.
      float v[32], w[32];
      float* rb = red + (it & 1) * 2 * kT;
      const float uflat = flat_bound(b);
      float m = uflat;
      uint32_t single = 1;
      bool have0 = false;   // chunk 0's scores already in v / w
      if (uflat < 0.0f) {
      {
        const int sb = su & 1;
        tc::mbar_wait(&sfull[sb], (su >> 1) & 1);
        tc::tc_fence_after();
        tc::tmem_ld32(lrow + sb * kT + h * 64, v);
        tc::tmem_ld32(lrow + sb * kT + h * 64 + 32, w);
        tc::tc_fence_before();
        tc::mbar_arrive(&sempty[sb]);
        ++su;
      }
      m = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) m = fmaxf(m, fmaxf(v[j], w[j]));
      rb[h * kT + row] = m;
      tc::named_bar(1, kSoftThreads);
      m = fmaxf(rb[row], rb[kT + row]);
      uint32_t ok = 0;
      if (a.phimax && NC > 1) {
        tc::mbar_wait(&qfull[it & 1], (it >> 1) & 1);   // theta's tile (already landed: the chunk-0 MMA read it)
        const uint8_t* qrow = sQ + (it & 1) * kAtom + row * 128;
        float t2 = 0.0f;
        for (int c = 0; c < a.Cq / 8; ++c) {
          const uint4 u4 = *reinterpret_cast<const uint4*>(qrow + ((c ^ (row & 7)) << 4));
          const __nv_bfloat162* hp = reinterpret_cast<const __nv_bfloat162*>(&u4);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(hp[k]);
            t2 = fmaf(f.x, f.x, fmaf(f.y, f.y, t2));
          }
        }
        const float U = sqrtf(t2) * a.phimax[b] * 1.001f + 1e-3f;
        ok = (U - m <= kSpan) ? 1u : 0u;   // false for NaN / inf
      }
      asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.and.pred q, 2, %2, p;\n\t"
                   "selp.u32 %0, 1, 0, q;\n\t}"
                   : "=r"(single) : "r"(ok), "r"(kSoftThreads) : "memory");
      have0 = single != 0;
      if (threadIdx.x == 64) {   // warp 2 lane 0 publishes the decision to the TMA and MMA warps
        *dec = single;
        tc::mbar_arrive(decbar);
      }
      if (!single) {
        // pass 1 (rest): exact row max (no exponentials)
        for (int u = 1; u < NC; ++u, ++su) {
          const int sb = su & 1;
          tc::mbar_wait(&sfull[sb], (su >> 1) & 1);
          tc::tc_fence_after();
          float x[32], y[32];
          tc::tmem_ld32(lrow + sb * kT + h * 64, x);
          tc::tmem_ld32(lrow + sb * kT + h * 64 + 32, y);
          tc::tc_fence_before();
          tc::mbar_arrive(&sempty[sb]);
#pragma unroll
          for (int j = 0; j < 32; ++j) m = fmaxf(m, fmaxf(x[j], y[j]));
        }
        tc::named_bar(1, kSoftThreads);   // every thread has read m0 from rb
        rb[h * kT + row] = m;
        tc::named_bar(1, kSoftThreads);
        m = fmaxf(rb[row], rb[kT + row]);
      }
      }   // (not flat)
      // P~ = exp(S - m) -> bf16 smem tile for the P~ g MMA; l = sum of P~ in fp32
      const float ml = m * kLog2e;
      float l = 0.0f;
      for (int c = 0; c < NC; ++c, ++pc) {
        const int pb = pc & 1;
        if (c > 0 || !have0) {   // single pass after a decision: chunk 0's scores are still in registers
          const int sb = su & 1;
          tc::mbar_wait(&sfull[sb], (su >> 1) & 1);
          tc::tc_fence_after();
          tc::tmem_ld32(lrow + sb * kT + h * 64, v);
          tc::tmem_ld32(lrow + sb * kT + h * 64 + 32, w);
          tc::tc_fence_before();
          tc::mbar_arrive(&sempty[sb]);
          ++su;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] = tc::ex2(fmaf(v[j], kLog2e, -ml));
          w[j] = tc::ex2(fmaf(w[j], kLog2e, -ml));
          l += v[j] + w[j];
        }
        tc::mbar_wait(&pempty[pb], ((pc >> 1) & 1) ^ 1);
        uint8_t* atom = sP + pb * 2 * kAtom + h * kAtom;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_sw128(atom, row, j, make_uint4(pack2(v[j * 8], v[j * 8 + 1]), pack2(v[j * 8 + 2], v[j * 8 + 3]),
                                            pack2(v[j * 8 + 4], v[j * 8 + 5]), pack2(v[j * 8 + 6], v[j * 8 + 7])));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_sw128(atom, row, 4 + j, make_uint4(pack2(w[j * 8], w[j * 8 + 1]), pack2(w[j * 8 + 2], w[j * 8 + 3]),
                                                pack2(w[j * 8 + 4], w[j * 8 + 5]), pack2(w[j * 8 + 6], w[j * 8 + 7])));
        tc::fence_async_smem();
        tc::mbar_arrive(&pfull[pb]);
        if (c == 0) epilogue();   // the previous tile's
      }
      // combine the two halves' sums
      float* lb = rb + 0;   // reuse: max already consumed by both halves after this barrier
      tc::named_bar(1, kSoftThreads);
      lb[h * kT + row] = l;
      tc::named_bar(1, kSoftThreads);
      l = lb[row] + lb[kT + row];
      // epilogue (O = (P~ g) / l -> bf16 (+ fp32); lse = m + log l) deferred into the next tile
      pend.valid = 1;
      pend.ob = it & 1;
      pend.ob2ph = (it >> 1) & 1;
      pend.grow = (long long)b * a.HW + q0 + row;
      pend.m = m;
      pend.l = l;
    }
    epilogue();   // the last tile's
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ===========================================================================
// backward (key-block outer loop)
// ===========================================================================
// 10 warps: the fullest SM sub-partition holds 3, so <= 168 registers per thread
__global__ void __launch_bounds__(kBwdThreads, 1)
    k_attn_bwd(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmO,
               const TcAttnArgs a, const int NS, const int NP) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;   // the layout needs 1024-byte alignment (checked on the host, see bwd_stages)
  if (threadIdx.x == 0 && (tc::smem_u32(smem) & 1023u)) __trap();
  const int C2 = a.C2, Cq = a.Cq;
  const int g_atoms = C2 > 64 ? 2 : 1;
  // one stage = {theta atom, dO g_atoms atoms, lse[128], D[128]}; NS stages (2..4, host-chosen)
  const uint32_t stage_bytes = (1 + g_atoms) * kAtom + 1024;
  const uint32_t ld_off = (1 + g_atoms) * kAtom;   // lse / D inside a stage
  uint8_t* sPhi = smem;                       // [128 keys][64]        1 atom
  uint8_t* sG = sPhi + kAtom;                 // [128 keys][64 x g]    g_atoms atoms
  // NP buffers of {P^T [128 keys][128 q] 2 atoms, dS^T 2 atoms}: with two, the softmax warps fill tile t+1
  // while the MMAs of tile t still read theirs
  uint8_t* sPD = sG + g_atoms * kAtom;
  uint8_t* sStage = sPD + NP * 4 * kAtom;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + NS * stage_bytes);
  uint64_t* kvfull = bars;
  uint64_t* qfull = bars + 1;      // [4]
  uint64_t* qempty = bars + 5;     // [4]
  uint64_t* sfull = bars + 9;
  uint64_t* sempty = bars + 10;
  uint64_t* pfull = bars + 11;     // [2]
  uint64_t* pempty = bars + 13;    // [2]
  uint64_t* dtfull = bars + 15;    // [2]
  uint64_t* dtempty = bars + 17;   // [2]
  uint64_t* accfull = bars + 19;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmQ);
    tc::tma_prefetch(&tmK);
    tc::tma_prefetch(&tmG);
    tc::tma_prefetch(&tmO);
    tc::mbar_init(kvfull, 1);
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(&qfull[s], 1);
      tc::mbar_init(&qempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&dtfull[s], 1);
      tc::mbar_init(&dtempty[s], 256);
    }
    tc::mbar_init(sfull, 1);
    tc::mbar_init(sempty, 256);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&pfull[s], 256);
      tc::mbar_init(&pempty[s], 1);
    }
    tc::mbar_init(accfull, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // TMEM columns: S^T 0..127, dP^T 128..255, dg 256.., dphi 384.., dtheta partial 448 / 480
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t cS = 0, cDP = 128, cDG = 256, cDPH = 384, cDT = 448;

  const int NC = a.Q / kT;
  const int b = blockIdx.x / NC;
  const int kb = blockIdx.x - b * NC;
  const int T = a.HW / kT;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_expect_tx(kvfull, (1 + g_atoms) * kAtom);
      tc::tma_load_3d(sPhi, &tmK, kvfull, 0, kb * kT, b);
      tc::tma_load_3d(sG, &tmG, kvfull, 0, kb * kT, b);
      if (g_atoms == 2) tc::tma_load_3d(sG + kAtom, &tmG, kvfull, 64, kb * kT, b);
      int st = 0;
      uint32_t ph = 0;
      for (int t = 0; t < T; ++t) {
        // warm L2 with the tile NS ahead (the stage ring hides L2, not DRAM, latency)
        if (t + NS < T) {
          tc::tma_prefetch_l2_3d(&tmQ, 0, (t + NS) * kT, b);
          tc::tma_prefetch_l2_3d(&tmO, 0, (t + NS) * kT, b);
          if (g_atoms == 2) tc::tma_prefetch_l2_3d(&tmO, 64, (t + NS) * kT, b);
        }
        tc::mbar_wait(&qempty[st], ph ^ 1);
        uint8_t* sb = sStage + st * stage_bytes;
        tc::mbar_expect_tx(&qfull[st], (1 + g_atoms) * kAtom + 1024);
        tc::tma_load_3d(sb, &tmQ, &qfull[st], 0, t * kT, b);
        tc::tma_load_3d(sb + kAtom, &tmO, &qfull[st], 0, t * kT, b);
        if (g_atoms == 2) tc::tma_load_3d(sb + 2 * kAtom, &tmO, &qfull[st], 64, t * kT, b);
        const long long r0 = (long long)b * a.HW + t * kT;
        tc::bulk_load_1d(sb + ld_off, a.lse + r0, 512, &qfull[st]);
        tc::bulk_load_1d(sb + ld_off + 512, a.Dr + r0, 512, &qfull[st]);
        if (++st == NS) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    {   // whole (converged) warp runs the loop, one elected lane issues: uniform descriptors
      const bool issuer = tc::elect_one();
      const uint32_t idS = tc::idesc_bf16(kT, kT, false, false);
      const uint32_t idDG = tc::idesc_bf16(kT, C2, false, true);
      const uint32_t idDPH = tc::idesc_bf16(kT, Cq, false, true);
      const uint32_t idDT = tc::idesc_bf16(kT, Cq, true, true);
      const int qsteps = Cq / 16, gsteps = C2 / 16;
      tc::mbar_wait(kvfull, 0);
      auto issue_s = [&](int t) {
        const int st = t % NS;
        tc::mbar_wait(&qfull[st], (t / NS) & 1);
        tc::mbar_wait(sempty, (t & 1) ^ 1);
        tc::tc_fence_after();
        const uint8_t* sb = sStage + st * stage_bytes;
        if (issuer) {
          for (int k = 0; k < qsteps; ++k)
            tc::mma_bf16(tmem + cS, kdesc(sPhi + k * 32), kdesc(sb + k * 32), idS, k > 0);
          for (int k = 0; k < gsteps; ++k) {
            const uint32_t off = (k >> 2) * kAtom + (k & 3) * 32;
            tc::mma_bf16(tmem + cDP, kdesc(sG + off), kdesc(sb + kAtom + off), idS, k > 0);
          }
          tc::mma_commit(sfull);
        }
        __syncwarp();
      };
      issue_s(0);
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) issue_s(t + 1);
        const int st = t % NS, db = t & 1, pb = t % NP;
        const uint8_t* sb = sStage + st * stage_bytes;
        const uint8_t* sPT = sPD + pb * 4 * kAtom;
        const uint8_t* sDS = sPT + 2 * kAtom;
        tc::mbar_wait(&pfull[pb], (t / NP) & 1);
        tc::mbar_wait(&dtempty[db], ((t >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        if (issuer) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {   // K = 128 queries in steps of 16
            const uint32_t koff = (k >> 2) * kAtom + (k & 3) * 32;
            tc::mma_bf16(tmem + cDG, kdesc(sPT + koff), mndesc(sb + kAtom + k * 2048), idDG, (t | k) != 0);
            tc::mma_bf16(tmem + cDPH, kdesc(sDS + koff), mndesc(sb + k * 2048), idDPH, (t | k) != 0);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)     // K = 128 keys in steps of 16
            tc::mma_bf16(tmem + cDT + db * 32, mndesc(sDS + k * 2048), mndesc(sPhi + k * 2048), idDT, k > 0);
          tc::mma_commit(&pempty[pb]);
          tc::mma_commit(&qempty[st]);
          tc::mma_commit(&dtfull[db]);
        }
        __syncwarp();
      }
      if (issuer) tc::mma_commit(accfull);
      __syncwarp();
    }
  } else {
    const int qd = warp & 3;
    const int h = (warp - 2) >> 2;           // which 64 of the 128 columns
    const int row = qd * 32 + lane;          // key row (S^T, dP^T, dg, dphi) / query row (dtheta)
    const uint32_t lrow = tmem + ((uint32_t)(qd * 32) << 16);
    float* part_base = a.dth_part + ((long long)kb * a.n + b) * a.HW * Cq;
    auto drain_dt = [&](int t) {   // dtheta partial of tile t -> global
      const int st = t & 1;
      tc::mbar_wait(&dtfull[st], (t >> 1) & 1);
      tc::tc_fence_after();
      if (h * 16 < Cq) {
        float v[16];
        tc::tmem_ld16(lrow + cDT + st * 32 + h * 16, v);
        float* dst = part_base + ((long long)t * kT + row) * Cq + h * 16;
#pragma unroll
        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&dtempty[st]);
    };
    for (int t = 0; t < T; ++t) {
      const int st = t % NS;
      const uint8_t* sb = sStage + st * stage_bytes;
      const float* sl = reinterpret_cast<const float*>(sb + ld_off) + h * 64;
      const float* sd = reinterpret_cast<const float*>(sb + ld_off + 512) + h * 64;
      tc::mbar_wait(sfull, t & 1);
      tc::mbar_wait(&qfull[st], (t / NS) & 1);   // lse / D of this tile are in smem
      tc::tc_fence_after();
      // P recomputed in fp32 from the scores; dS = P (dP - D); both packed to bf16 pairs at once.
      // Two 32-column halves keep the register footprint under the 168-register cap.
      uint32_t pk[32], dk[32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float s[32], dp[32];
        tc::tmem_ld32(lrow + cS + h * 64 + half * 32, s);
        tc::tmem_ld32(lrow + cDP + h * 64 + half * 32, dp);
        if (half == 1) {
          tc::tc_fence_before();
          tc::mbar_arrive(sempty);
        }
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int jj = half * 32 + j;
          const float p0 = tc::ex2(fmaf(s[j], kLog2e, -sl[jj] * kLog2e));
          const float p1 = tc::ex2(fmaf(s[j + 1], kLog2e, -sl[jj + 1] * kLog2e));
          pk[jj >> 1] = pack2(p0, p1);
          dk[jj >> 1] = pack2(p0 * (dp[j] - sd[jj]), p1 * (dp[j + 1] - sd[jj + 1]));
        }
      }
      const int pb = t % NP;
      tc::mbar_wait(&pempty[pb], ((t / NP) & 1) ^ 1);
      uint8_t* pa = sPD + pb * 4 * kAtom + h * kAtom;
      uint8_t* da = pa + 2 * kAtom;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        st_sw128(pa, row, c, make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]));
        st_sw128(da, row, c, make_uint4(dk[c * 4], dk[c * 4 + 1], dk[c * 4 + 2], dk[c * 4 + 3]));
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&pfull[pb]);
      if (t > 0) drain_dt(t - 1);
    }
    drain_dt(T - 1);
    // per-key accumulators -> global fp32
    tc::mbar_wait(accfull, 0);
    tc::tc_fence_after();
    const long long krow = (long long)b * a.Q + kb * kT + row;
    float* dg = a.dgp + krow * C2;
#pragma unroll 1
    for (int cb = h * 64; cb < C2 && cb < h * 64 + 64; cb += 32) {
      float v[32];
      tc::tmem_ld32(lrow + cDG + cb, v);
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        if (cb + j < C2) *reinterpret_cast<float4*>(dg + cb + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
    if (h * 16 < Cq) {
      float v[16];
      tc::tmem_ld16(lrow + cDPH + h * 16, v);
      float* dph = a.dphi + krow * Cq + h * 16;
#pragma unroll
      for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dph + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;

cudaError_t encoder() {
  if (g_enc) return cudaSuccess;
  cudaDriverEntryPointQueryResult qr;
  PG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_enc), cudaEnableDefault,
                                  &qr));
  if (qr != cudaDriverEntryPointSuccess || !g_enc) return cudaErrorNotSupported;
  return cudaSuccess;
}

// 3-D bf16 map over [d2][d1][d0] (d0 contiguous), box {b0, b1, 1}, 128-byte swizzle
cudaError_t map3(CUtensorMap* m, const void* base, long long d0, long long d1, long long d2, int b0, int b1) {
  PG_CUDA(encoder());
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)d0 * 2, (cuuint64_t)(d0 * d1 * 2)};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

constexpr size_t kSmemMax = 232448;   // 227 KB opt-in per CTA
size_t fwd_smem(int C2, int nvs) {
  return 1024 + (2 + kFwdKStages + 4) * kAtom + nvs * 2u * C2 * 128 + 4 * kT * sizeof(float) + 256;
}
int fwd_vstages(int C2) {
  static const int cap = getenv("PARAGAN_ATTN_VSTAGES") ? atoi(getenv("PARAGAN_ATTN_VSTAGES")) : kFwdVMax;
  int n = cap < 2 ? 2 : (cap > kFwdVMax ? kFwdVMax : cap);
  while (n > 2 && fwd_smem(C2, n) > kSmemMax) --n;
  return n;
}
// fixed part (phi, g, P^T, dS^T) + NS stages; the largest NS <= 4 that fits
// NP (P/dS buffers) = 2 only when a 3-stage theta/dO ring still fits (measured: NP 2 with a 2-stage ring is
// slower than NP 1 with 3 stages for D's block, 2.4 vs 2.2 ms), else 1; then the largest NS <= 4
int bwd_stages(int C2, size_t* smem, int* np) {
  const size_t g = C2 > 64 ? 2 : 1;
  const size_t stage = (1 + g) * kAtom + 1024;
  for (int p = 2; p >= 1; --p) {
    const size_t fixed = (1 + g + 4 * (size_t)p) * kAtom + 256;
    int ns = (int)((kSmemMax - fixed) / stage);
    if (ns > 4) ns = 4;
    if (ns >= 3 || p == 1) {
      *np = p;
      *smem = fixed + ns * stage;
      return ns;
    }
  }
  return 0;
}

}  // namespace

bool tc_attn_ok(int HW, int Q, int Cq, int C2) {
  return HW % kT == 0 && Q % kT == 0 && (Cq == 16 || Cq == 32) && C2 % 16 == 0 && C2 >= 16 && C2 <= 128;
}

cudaError_t tc_attn_fwd(const TcAttnArgs& a, cudaStream_t st) {
  if (!tc_attn_ok(a.HW, a.Q, a.Cq, a.C2) || a.Ct % 8) return cudaErrorInvalidValue;
  CUtensorMap mq, mk, mv;
  PG_CUDA(map3(&mq, a.qkv, a.Ct, a.HW, a.n, 64, kT));
  PG_CUDA(map3(&mk, a.phi, a.Cq, a.Q, a.n, 64, kT));
  PG_CUDA(map3(&mv, a.gT, a.Q, a.C2, a.n, 64, a.C2));
  const int nvs = fwd_vstages(a.C2);
  const size_t smem = fwd_smem(a.C2, nvs);
  const int sms = sm_cap();
  const int tiles = a.n * (a.HW / kT);
  PG_CUDA(cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_attn_fwd<<<tiles < sms ? tiles : sms, kFwdThreads, smem, st>>>(mq, mk, mv, a, nvs);
  return cudaGetLastError();
}

cudaError_t tc_attn_bwd(const TcAttnArgs& a, cudaStream_t st) {
  if (!tc_attn_ok(a.HW, a.Q, a.Cq, a.C2) || a.Ct % 8) return cudaErrorInvalidValue;
  CUtensorMap mq, mk, mg, mo;
  PG_CUDA(map3(&mq, a.qkv, a.Ct, a.HW, a.n, 64, kT));
  PG_CUDA(map3(&mk, a.phi, a.Cq, a.Q, a.n, 64, kT));
  PG_CUDA(map3(&mg, a.gp, a.C2, a.Q, a.n, 64, kT));
  PG_CUDA(map3(&mo, a.dO, a.C2, a.HW, a.n, 64, kT));
  size_t smem = 0;
  int np = 1;
  const int ns = bwd_stages(a.C2, &smem, &np);
  if (ns < 2) return cudaErrorInvalidValue;
  PG_CUDA(cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_attn_bwd<<<a.n * (a.Q / kT), kBwdThreads, smem, st>>>(mq, mk, mg, mo, a, ns, np);
  return cudaGetLastError();
}

namespace {
__global__ void k_attn_transpose(const bf16* __restrict__ in, int Q, int C, bf16* __restrict__ out) {
  __shared__ bf16 tile[32][33];
  const int b = blockIdx.z;
  const int q0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const bf16* src = in + (long long)b * Q * C;
  bf16* dst = out + (long long)b * Q * C;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int q = q0 + i, c = c0 + threadIdx.x;
    if (q < Q && c < C) tile[i][threadIdx.x] = src[(long long)q * C + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, q = q0 + threadIdx.x;
    if (q < Q && c < C) dst[(long long)c * Q + q] = tile[threadIdx.x][i];
  }
}

// four lanes per row, 8 channels (one 16-byte bf16 load, two float4 loads) per lane per step
__global__ void k_attn_rowdot(const bf16* __restrict__ dO, const float* __restrict__ o32, long long rows, int C,
                              float* __restrict__ D) {
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 2;
  const int l = threadIdx.x & 3;
  float s = 0.0f;
  if (r < rows) {
    for (int c = 8 * l; c < C; c += 32) {
      const uint4 u = *reinterpret_cast<const uint4*>(dO + r * C + c);
      const float4 a = *reinterpret_cast<const float4*>(o32 + r * C + c);
      const float4 b = *reinterpret_cast<const float4*>(o32 + r * C + c + 4);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
      const float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
      const float2 f2 = __bfloat1622float2(h[2]), f3 = __bfloat1622float2(h[3]);
      s += f0.x * a.x + f0.y * a.y + f1.x * a.z + f1.y * a.w + f2.x * b.x + f2.y * b.y + f3.x * b.z + f3.y * b.w;
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (r < rows && l == 0) D[r] = s;
}

__global__ void k_attn_dtheta_reduce(const float* __restrict__ part, int nkb, long long rows, int Cq,
                                     bf16* __restrict__ dqkv, int ld) {
  const long long n4 = rows * (Cq / 4);
  const long long stride = rows * Cq;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / (Cq / 4);
    const int c = (int)(i - r * (Cq / 4)) * 4;
    float4 acc = *reinterpret_cast<const float4*>(part + r * Cq + c);
    for (int k = 1; k < nkb; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(part + k * stride + r * Cq + c);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dqkv + r * ld + c) = pk;
  }
}
}  // namespace

// out[b] = max over the `rows` rows of image b of the L2 norm of the row's first `cols` entries (row stride ld):
// grid (images, row slices), 16-byte loads; the slices combine through an integer atomicMax on the (non-negative)
// squared norm's bits, which is order-independent; `out` is zeroed first, the square root taken by k_sqrt_inplace
__global__ void k_attn_rowmaxnorm(const bf16* __restrict__ x, int rows, int cols, int ld, float* __restrict__ out) {
  __shared__ float red[8];
  const bf16* p = x + (long long)blockIdx.x * rows * ld;
  const int per = (rows + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float mx = 0.0f;
  for (int j = r0 + threadIdx.x; j < r1; j += blockDim.x) {
    float t = 0.0f;
    const uint4* rp = reinterpret_cast<const uint4*>(p + (long long)j * ld);
    for (int c = 0; c < cols / 8; ++c) {
      const uint4 u = __ldg(rp + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        t = fmaf(f.x, f.x, fmaf(f.y, f.y, t));
      }
    }
    mx = fmaxf(mx, t);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, red[i]);
    atomicMax(reinterpret_cast<int*>(out) + blockIdx.x, __float_as_int(m));
  }
}
__global__ void k_sqrt_inplace(float* __restrict__ v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = sqrtf(v[i]);
}
cudaError_t rowmaxnorm(const void* x, int n, int rows, int cols, int ld, float* out, cudaStream_t st) {
  if (cols % 8 || ld % 8 || (reinterpret_cast<uintptr_t>(x) & 15)) return cudaErrorInvalidValue;
  PG_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * n, st));
  const int slices = rows >= 2048 ? 8 : 1;
  k_attn_rowmaxnorm<<<dim3(n, slices), 256, 0, st>>>(static_cast<const bf16*>(x), rows, cols, ld, out);
  PG_CUDA(cudaGetLastError());
  k_sqrt_inplace<<<ceil_div(n, 256), 256, 0, st>>>(out, n);
  return cudaGetLastError();
}

cudaError_t attn_phimax(const void* phi, int n, int Q, int Cq, float* phimax, cudaStream_t st) {
  return rowmaxnorm(phi, n, Q, Cq, Cq, phimax, st);
}
cudaError_t attn_thetamax(const void* qkv, int n, int HW, int Cq, int Ct, float* thetamax, cudaStream_t st) {
  return rowmaxnorm(qkv, n, HW, Cq, Ct, thetamax, st);
}

cudaError_t attn_transpose(const void* gp, int n, int Q, int C, void* gT, cudaStream_t st) {
  dim3 grid((Q + 31) / 32, (C + 31) / 32, n);
  k_attn_transpose<<<grid, dim3(32, 8), 0, st>>>(static_cast<const bf16*>(gp), Q, C, static_cast<bf16*>(gT));
  return cudaGetLastError();
}

cudaError_t attn_rowdot(const void* dO, const float* o32, long long rows, int C, float* D, cudaStream_t st) {
  if (C % 8 || ((uintptr_t)dO & 15) || ((uintptr_t)o32 & 15)) return cudaErrorInvalidValue;
  const long long blocks = (rows + 63) / 64;
  k_attn_rowdot<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const bf16*>(dO), o32, rows, C, D);
  return cudaGetLastError();
}

cudaError_t attn_dtheta_reduce(const float* part, int nkb, long long rows, int Cq, void* dqkv, int ld,
                               cudaStream_t st) {
  if (Cq % 4 || ld % 4 || ((uintptr_t)dqkv & 7)) return cudaErrorInvalidValue;
  const long long n4 = rows * (Cq / 4);
  long long blocks = (n4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_attn_dtheta_reduce<<<(unsigned)blocks, 256, 0, st>>>(part, nkb, rows, Cq, static_cast<bf16*>(dqkv), ld);
  return cudaGetLastError();
}

}  // namespace pg
