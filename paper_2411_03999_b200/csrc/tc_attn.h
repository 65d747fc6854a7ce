// Internal interface of the fused tcgen05 attention kernels (tc_attn.cu): the
// non-local block of BigGAN (reading R8) for one image at a time,
// scores beta = softmax_rows(theta^T phi) never leaving the SM.
#pragma once
#include <cuda_runtime.h>

namespace pg {

struct TcAttnArgs {
  int n, HW, Q, Cq, C2, Ct;
  const void* qkv;     // bf16 [n][HW][Ct]; theta = channels [0, Cq) (zero beyond C/8)
  const void* phi;     // bf16 [n][Q][Cq]  max-pooled phi, zero-padded channels
  const void* gp;      // bf16 [n][Q][C2]  max-pooled g
  const void* gT;      // bf16 [n][C2][Q]  max-pooled g, transposed (forward B operand)
  void* o;             // bf16 [n][HW][C2] forward output  o = beta g
  float* o32;          // fp32 [n][HW][C2] the same before rounding (optional; for the backward's D)
  float* lse;          // fp32 [n][HW]     row log-sum-exp of the scores (forward out, backward in)
  const float* phimax; // fp32 [n]         max_j |phi_j| per image (forward; enables the single-pass
                       //                  schedule, see k_attn_fwd), or null = always two passes
  const float* thetamax; // fp32 [n]       max_i |theta_i| per image (forward; with phimax enables the flat
                         //                schedule for images whose score bound is <= 40), or null
  // backward
  const void* dO;      // bf16 [n][HW][C2]
  const float* Dr;     // fp32 [n][HW]     rowsum(dO * o) = rowsum(dP * beta)
  float* dgp;          // fp32 [n][Q][C2]  d(pooled g)
  float* dphi;         // fp32 [n][Q][Cq]  d(pooled phi)
  float* dth_part;     // fp32 [Q/128][n][HW][Cq] per-key-block partials of d theta
};

// true when the shapes fit the kernels (HW, Q multiples of 128, Cq in {16, 32, 48, 64},
// C2 a multiple of 16 and <= 128)
bool tc_attn_ok(int HW, int Q, int Cq, int C2);
// o, lse from qkv, phi, gT
cudaError_t tc_attn_fwd(const TcAttnArgs& a, cudaStream_t st);
// dgp, dphi, dth_part from qkv, phi, gp, dO, lse, Dr
cudaError_t tc_attn_bwd(const TcAttnArgs& a, cudaStream_t st);

}  // namespace pg

namespace pg {
// small helpers of the fused path (tc_attn.cu)
// gT[b][c][q] = gp[b][q][c]   (bf16, [n][Q][C] -> [n][C][Q])
cudaError_t attn_transpose(const void* gp, int n, int Q, int C, void* gT, cudaStream_t st);
// phimax[b] = max_j ||phi[b][j][0:Cq]||_2 (fp32; one block per image)
cudaError_t attn_phimax(const void* phi, int n, int Q, int Cq, float* phimax, cudaStream_t st);
// thetamax[b] = max_i |theta_i| over image b (theta = channels [0, Cq) of qkv [n][HW][Ct])
cudaError_t attn_thetamax(const void* qkv, int n, int HW, int Cq, int Ct, float* thetamax, cudaStream_t st);
// D[r] = sum_c dO[r][c] * o32[r][c]   (one warp per row)
cudaError_t attn_rowdot(const void* dO, const float* o32, long long rows, int C, float* D, cudaStream_t st);
// dqkv[r][0:Cq] = bf16( sum_{kb < nkb} part[kb][r][0:Cq] ), summed in kb order (deterministic)
cudaError_t attn_dtheta_reduce(const float* part, int nkb, long long rows, int Cq, void* dqkv, int ld,
                               cudaStream_t st);
}  // namespace pg
