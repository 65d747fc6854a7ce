// Launchers of the memory-bound and SIMT kernels of libparagan.  Storage
// type T is float (F32 mode) or bf16 (BF16 mode); arithmetic is fp32, global
// reductions are accumulated in fp64.  Activations are NHWC, [M = N*H*W][C].
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace pg {

// ---------------- layout (A1)
template <typename TD>
cudaError_t layout_pack(const float* src, TD* dst, int n, int c, int h, int w, int c_pad, long long dst_batch_offset,
                        cudaStream_t st);
template <typename TS>
cudaError_t layout_unpack(const TS* src, float* dst, int n, int c, int h, int w, int c_pad, cudaStream_t st);

// ---------------- small fp32 GEMM: C[m][n] = beta*C + sum_k A(m,k) B(n,k) (+ bias[n])
// A(m,k) = A[m*sam + k*sak]; B(n,k) = B[n*sbn + k*sbk]; C[m*ldc + n]
// Grouped fp32 GEMM: every problem p computes
//   C_p[M][N] = beta * C_p + bias_p[n] + sum_{s < nseg} A_s[M][K_s] B_s[N][K_s]^T
// (general strides), all problems in one launch; the table lives in device memory and
// tile0 is the prefix sum of the problems' 64x64 tile counts (see gemm_grouped_plan).
struct GemmSeg {
  const float* A;
  long long sam, sak;
  const float* B;
  long long sbn, sbk;
  int K;
};
struct GemmProblem {
  int M, N, nseg, tile0;
  GemmSeg seg[4];
  float* C;
  long long ldc;
  float beta;
  const float* bias;
};
// dst[i] = sum_{j < nslices} part[j * n + i]   (fp64 sum in slice order: deterministic)
cudaError_t sum_slices(const float* part, int nslices, int n, float* dst, cudaStream_t st);
// fills tile0 and returns the total tile count
int gemm_grouped_plan(GemmProblem* probs, int nprob);
cudaError_t gemm_f32_grouped(const GemmProblem* probs_dev, int nprob, int total_tiles, cudaStream_t st);
cudaError_t gemm_f32(int M, int N, int K, const float* A, long long sam, long long sak, const float* B,
                     long long sbn, long long sbk, float* C, long long ldc, float beta, const float* bias,
                     cudaStream_t st);

// ---------------- conversion / gathers
template <typename TD>
cudaError_t convert_f32(const float* src, TD* dst, long long n, cudaStream_t st);
template <typename TS>
cudaError_t to_f32(const TS* src, float* dst, long long n, cudaStream_t st);
cudaError_t gather_rows(const float* table, const int32_t* idx, int n, int dim, float* out, int ldo, cudaStream_t st);
cudaError_t copy_cols(const float* src, int lds, int n, int cols, float* dst, int ldd, cudaStream_t st);
// dtable[idx[i]][j] += src[i*lds + j]; deterministic (sequential over i per column)
// dtable[r][j] += sum_{i: idx[i] == r} sum_s srcs.p[s][i][j]  for up to 8 sources; one thread per
// (table row, j), rows i visited in order (deterministic, no atomics)
struct RowSrcs {
  const float* p[8];
  int n;
};
cudaError_t scatter_add_rows_multi(const RowSrcs& srcs, int lds, const int32_t* idx, int n, int dim, int table_rows,
                                   float* dtable, cudaStream_t st);
cudaError_t scatter_add_rows(const float* src, int lds, const int32_t* idx, int n, int dim, float* dtable,
                             cudaStream_t st);

// ---------------- batch norm (A4, A11)
// partial sums over pixel blocks -> sums[2C] (fp64: sum x, sum x^2)
template <typename T>
cudaError_t bn_stats(const T* x, long long M, int C, double* partial, int max_blocks, double* sums, cudaStream_t st);
// sums (all-reduced) -> mean, rstd (fp32)
cudaError_t bn_finalize(const double* sums, int C, double count, float eps, float* mean, float* rstd,
                        cudaStream_t st);
// y = relu(x_hat * g + b), g = 1 + gain[n][c] (conditional) or gamma[c]; b = bias[n][c] or beta[c];
// up2: write each output pixel to its 2x2 block of a [N,2H,2W,C] tensor
template <typename TI, typename TO>
cudaError_t bn_apply_relu(const TI* x, int N, int H, int W, int C, const float* mean, const float* rstd,
                          const float* gain, const float* bias, const float* gamma, const float* beta, TO* y, bool up2,
                          cudaStream_t st);
// backward, pass 1: per sample sums A[n][c] = sum g0, Bv[n][c] = sum g0*x_hat (g0 = dy * relu')
// dy is [N,2H,2W,C] when up2 (summed over each 2x2 block)
template <typename TI, typename TG>
cudaError_t bn_bwd_reduce(const TI* x, const TG* dy, int N, int H, int W, int C, const float* mean, const float* rstd,
                          const float* gain, const float* bias, const float* gamma, const float* beta, bool up2,
                          float* partial, int chunks, float* AB, cudaStream_t st);
// channel totals tot[2C] = sum_n g[n][c]*A[n][c], sum_n g[n][c]*Bv[n][c]  (fp64)
cudaError_t bn_bwd_totals(const float* AB, int N, int C, const float* gain, const float* gamma, double* tot,
                          cudaStream_t st);
// pass 2: dx = rstd*(g*g0 - tot0/cnt - x_hat*tot1/cnt) (+ add)
template <typename TI, typename TG, typename TO>
cudaError_t bn_bwd_apply(const TI* x, const TG* dy, int N, int H, int W, int C, const float* mean, const float* rstd,
                         const float* gain, const float* bias, const float* gamma, const float* beta, bool up2,
                         const double* tot, double count, const TO* add, TO* dx, cudaStream_t st);

// ---------------- elementwise / resampling (A7, A11)
template <typename T>
cudaError_t relu_copy(const T* x, T* y, long long n, cudaStream_t st);
// dx = dy * [ref > 0] (+ add)
template <typename T>
cudaError_t relu_bwd(const T* dy, const T* ref, const T* add, T* dx, long long n, cudaStream_t st);
// y[N,H/2,W/2,C] = avgpool2(x) (+ add[N,H/2,W/2,C])
template <typename T>
cudaError_t avgpool2(const T* x, int N, int H, int W, int C, int ldx, const T* add, T* y, cudaStream_t st,
                     T* y_relu = nullptr,    // y_relu (optional): relu(y) as well (the next D block's conv1 input)
                     T* x_relu = nullptr);   // x_relu (optional): relu(x) [N,H,W,ldx] from the same loads
// dx[N,H,W,C] = 0.25 * dy[n,h/2,w/2,c]   (avgpool adjoint); optional add (same shape as dx)
template <typename T>
cudaError_t avgpool2_bwd(const T* dy, int N, int H, int W, int C, const T* add, T* dx, int lddx, cudaStream_t st);
// dx[N,H,W,C] = sum of the 2x2 block of dy[N,2H,2W,C]   (nearest-upsample adjoint)
template <typename T>
cudaError_t up2_bwd(const T* dy, int N, int H, int W, int C, T* dx, cudaStream_t st);
// column sums: db[c] (+)= sum_m dy[m][c]   (bias gradients; fp64 partials, fixed order;
// 16-byte vectors over 8-channel groups when C % 8 == 0)
template <typename T>
cudaError_t col_sum(const T* dy, long long M, int C, double* partial, int max_blocks, float* db, int accumulate,
                    cudaStream_t st);

// ---------------- G output layer (fp32) and image buffer
// img = tanh(pre[M][3]); writes fp32 img and T copy into dst[M][c_pad] (pad channels zero)
template <typename T>
cudaError_t tanh_to_image(const float* pre, float* img, T* dst, long long M, int c_pad, cudaStream_t st);
// dpre[m][k] = dimg[m][k] * (1 - img^2), k < 3
template <typename T>
cudaError_t tanh_bwd(const T* dimg, int c_pad, const float* img, float* dpre, long long M, cudaStream_t st);

// ---------------- SIMT convolution (F32 path; G output conv in both modes)
// y[m][o] = alpha*sum + bias[o] + residual; w[Cout][k*k][Cin]
template <typename TI, typename TW, typename TO>
cudaError_t simt_conv_fwd(const TI* x, int N, int H, int W, int Cin, const TW* w, int Cout, int ksz,
                          const float* bias, const float* alpha, const TO* residual, int res_mode, TO* y,
                          cudaStream_t st, const TO* relu_ref = nullptr);
// dw[o][tap][c] (+)= sum_m dy[m][o] * x[m+tap][c]   (fp32 per pixel split; the split partials, kept in
// scratch, are summed in split order in fp64 — deterministic.  scratch == nullptr: a single split)
template <typename TI, typename TG>
cudaError_t simt_conv_wgrad(const TI* x, const TG* dy, int N, int H, int W, int Cin, int Cout, int ksz, float* dw,
                            int accumulate, cudaStream_t st, float* scratch = nullptr, size_t scratch_floats = 0);

// ---------------- first D layer as a K=27 GEMM: xi[p][tap*3+c] (K padded to 32) and its adjoint
template <typename T>
cudaError_t im2col3(const T* x, int N, int H, int W, int cx, T* out, cudaStream_t st);
template <typename T>
cudaError_t col2im3(const T* dxi, int N, int H, int W, int cx, const T* add, T* dx, cudaStream_t st);

// Sub-pixel weight fold for a 3x3 conv applied to a x2-nearest-upsampled input:
// dst[a*2+b][o][p*2+q][c] = bf16( inv_sigma[0] * sum_{r in R(a,p), s in R(b,q)} w[o][r*3+s][c] ),
// R(0,0) = {0}, R(0,1) = {1,2}, R(1,0) = {0,1}, R(1,1) = {2}  (output phase a reads input row i-1+a+p)
// layout 0: fprop operand [phase][Cout][tap][Cin]; layout 1: dgrad operand [Cin][phase * 4 + tap][Cout]
cudaError_t fold_up2_weights(const float* w, const float* inv_sigma, int Cout, int Cin, bf16* dst, cudaStream_t st,
                             int layout = 0);
// every G conv1 of a forward at once (same values): job j covers tiles [tile0, tile0 + ceil(Cout/32)*ceil(Cin/32));
// dst0 = the layout-0 operand, dst1 = the layout-1 operand (written when dgrad)
struct FoldJob {
  const float* w;
  const float* inv_sigma;
  bf16* dst0;
  bf16* dst1;
  int Cout, Cin, tile0;
  int tf;   // 1: fold the input-gradient kernel of w (w is [Cin][9][Cout]; tap t reads w[c][8 - t][o])
};
cudaError_t fold_up2_grouped(const FoldJob* jobs_d, int njobs, int tiles, bool dgrad, cudaStream_t st);

// ---------------- generic fp32 SIMT kernels of the SN-DCGAN path (config 1; SURVEY Appendix B "K7")
// strided k x k conv, NHWC, zero padding p; w OHWI [Cout][k][k][ldw] (first Cin of ldw used)
cudaError_t gconv_fwd(const float* x, int N, int H, int W, int Cin, const float* w, int ldw, int Cout, int k, int s,
                      int p, int Ho, int Wo, const float* bias, float* y, cudaStream_t st);
// dx[n,iy,ix,ci] = bias[ci] + sum_{co,ky,kx: iy = oy*s - p + ky} dy[n,oy,ox,co] w[co][ky][kx][ci]  (the conv's
// adjoint; with bias it is the transposed conv / deconv forward)
cudaError_t gconv_dgrad(const float* dy, int N, int Ho, int Wo, int Cout, const float* w, int ldw, int Cin, int k,
                        int s, int p, int H, int W, const float* bias, float* dx, cudaStream_t st);
// dw[co][ky][kx][ci] (ldw = Cin) = sum_{n,oy,ox} dy[n,oy,ox,co] x[n, oy*s-p+ky, ox*s-p+kx, ci]  (fp64 sums)
cudaError_t gconv_wgrad(const float* x, int N, int H, int W, int Cin, const float* dy, int Ho, int Wo, int Cout,
                        int k, int s, int p, float* dw, cudaStream_t st);
// y = x > 0 ? x : slope * x ;  dx = dy * (pre > 0 ? 1 : slope)
cudaError_t lrelu_fwd(const float* x, float* y, long long n, float slope, cudaStream_t st);
cudaError_t lrelu_bwd(const float* dy, const float* pre, float* dx, long long n, float slope, cudaStream_t st);
// per-channel BN over [M][C] fp32 (any C): local sums[2C] = (sum x, sum x^2) in fp64
cudaError_t bn_sums_generic(const float* x, long long M, int C, double* sums, cudaStream_t st);
// y = (relu?) ((x - mean) * rstd * gamma + beta)
cudaError_t bn_apply_generic(const float* x, long long M, int C, const float* mean, const float* rstd,
                             const float* gamma, const float* beta, int relu, float* y, cudaStream_t st);
// tot[0:C] = sum g, tot[C:2C] = sum g * xhat over the local rows, g = dy masked by the output ReLU; also
// written (fp32) to dbeta / dgamma (local parameter gradients)
cudaError_t bn_bwd_sums_generic(const float* x, const float* dy, long long M, int C, const float* mean,
                                const float* rstd, const float* gamma, const float* beta, int relu, double* tot,
                                float* dgamma, float* dbeta, cudaStream_t st);
// dx = gamma * rstd * (g - tot[c] / count - xhat * tot[C + c] / count)   (tot all-reduced over ranks)
cudaError_t bn_bwd_apply_generic(const float* x, const float* dy, long long M, int C, const float* mean,
                                 const float* rstd, const float* gamma, const float* beta, int relu, const double* tot,
                                 double count, float* dx, cudaStream_t st);

// ---------------- thin fp32 conv (C_out = 3): G's fp32 output layer, 3x3 pad 1
cudaError_t thin_conv_fwd(const float* x, int N, int H, int W, int C, const float* w, int CO, const float* bias,
                          float* y, cudaStream_t st);
// dx[m][c] = transposed conv of dy[m][CO] with w[CO][9][C]
cudaError_t thin_conv_dgrad(const float* dy, int N, int H, int W, int C, const float* w, int CO, float* dx,
                            cudaStream_t st);
// dw[CO][9][C] = sum_m dy[m][o] x[m+tap][c]  (deterministic: per-block partials in scratch, fixed-order sum)
// split = true: x is the two-term bf16 split [m][2C] = [x1 | x2] of the activation (R36), read as x1 + x2
cudaError_t thin_conv_wgrad(const void* x, const float* dy, int N, int H, int W, int C, int CO, float* dw,
                            float* scratch, size_t scratch_floats, cudaStream_t st, bool split = false);
// G's output layer on the tensor cores (R36; tc_outconv.cu): y2[p] = [bf16(x) | bf16(x - bf16(x))]
// ([P][2C]), and the three-term bf16 split of w[3][9][C] as the B operand [96][2C] (row layout: kernels.cu)
cudaError_t split_planes(const float* x, long long P, int C, bf16* y2, cudaStream_t st);
}  // namespace pg
#include "../../include/paragan.h"
namespace pg {
cudaError_t pack_stats(const float* ld, const float* lg, const long long* td, const long long* tg, const int* nf,
                       float inv, paragan_stats* out, cudaStream_t st);
cudaError_t split_out_weights(const float* w, int C, bf16* ws, cudaStream_t st);
// the dgrad operand [C16][128] over the output-gradient im2col [dy1 | dy2 | dy1 | dy1] (tc_outconv.cu)
cudaError_t split_out_weights_dgrad(const float* w, int C, int C16, bf16* wd, cudaStream_t st);
// output-BN apply + ReLU written as the split planes y2 [P][2C] (the fp32 result never stored)
cudaError_t bn_apply_relu_split(const bf16* x, int N, int H, int W, int C, const float* mean, const float* rstd,
                                const float* gamma, const float* beta, bf16* y2, cudaStream_t st);

// ---------------- discriminator head + hinge loss (A7, A8), fp32
template <typename T>
cudaError_t d_head_fwd(const T* h, int N, int HW, int C, const float* w_lin, const float* b_lin, const float* embed,
                       const int32_t* y, float* feat, float* logits, cudaStream_t st);
// mode 0: D loss over [fake(B); real(B)]; mode 1: G loss over B fakes.  Writes loss[0..3]
// (loss, mean real logit, mean fake logit, nonfinite) and dlogits (local-mean scaling 1/B).
cudaError_t hinge_loss(const float* logits, int B, int mode, float* dlogits, float* loss_out, cudaStream_t st);
// backward: dfeat = dl*(w + E[y]); dh = dfeat * [h > 0]; grads of w, b, E (if want_wgrad)
template <typename T>
cudaError_t d_head_bwd(const T* h, int N, int HW, int C, const float* w_lin, const float* embed, const int32_t* y,
                       const float* feat, const float* dlogits, T* dh, float* dw_lin, float* db_lin, float* dembed,
                       int n_classes, bool want_wgrad, cudaStream_t st);

// ---------------- attention (A6)
// pooled[n][hw/4][c] = max over 2x2 of x[n][.][c_off + c] (ld = ldx); also transposed copy pooledT[n][c][hw/4]
template <typename T>
cudaError_t maxpool2_split(const T* x, int N, int H, int W, int ldx, int c_off, int C, T* pooled, T* pooledT,
                           cudaStream_t st);
// dx[n][h][w][c_off+c] = dpooled at the argmax of each 2x2 block (others 0); dpooled given [n][hw/4][c] (fp32)
template <typename T>
cudaError_t maxpool2_split_bwd(const T* x, int N, int H, int W, int ldx, int c_off, int C, const float* dpooled,
                               T* dx, cudaStream_t st);
// P = softmax rows of S [rows][cols] fp32 -> T
template <typename T>
cudaError_t softmax_rows(const float* S, long long rows, int cols, T* P, cudaStream_t st);
// dS = P * (dP - rowsum(dP * P)) with P = softmax(S) recomputed in fp32 from the scores -> T
template <typename T>
cudaError_t softmax_bwd_rows(const float* S, const float* dP, long long rows, int cols, T* dS, cudaStream_t st);
// batched SIMT GEMM for the F32 path: C[b][m][n] = sum_k A[b](m,k) B[b](n,k)
// the attention GEMMs of the unfused (small-image) path in bf16: bf16 operands, fp32 accumulation, fp32 or bf16 C
cudaError_t gemm_bf16_batched(int batch, int M, int N, int K, const bf16* A, long long sab, long long sam,
                              long long sak, const bf16* B, long long sbb, long long sbn, long long sbk, void* C,
                              bool c_f32, long long scb, long long ldc, cudaStream_t st);
cudaError_t gemm_f32_batched(int batch, int M, int N, int K, const float* A, long long sab, long long sam,
                             long long sak, const float* B, long long sbb, long long sbn, long long sbk, float* C,
                             long long scb, long long ldc, float beta, cudaStream_t st);

// ---------------- spectral norm (A2) and Adam (A13)
struct SnJob {
  const float* w;   // [rows][K] fp32 master
  float* u;         // [rows] (updated in place)
  float* v;         // [K] out
  float* t;         // [K] scratch (W^T u)
  float* s;         // [rows] scratch (W v)
  float* sigma;     // [2]: sigma, 1/sigma
  float* part;      // [nrc][K] partial W^T u over row chunks of 128
  float* grad;      // [rows][K] gradient w.r.t. W/sigma (SN backward, in place)
  double* coef;     // [1] SN backward coefficient
  int rows, K, nrc;
  float eps;        // n(x) = x / max(||x||, eps)  (paragan_config.sn_eps, R4)
  long long bwd_blk0, bwd_nblk;   // SN-backward block range of this job
};
struct SnPack {     // one packed copy of W/sigma
  const float* w;
  const float* sigma;
  void* dst;        // bf16 or fp32
  int rows, taps, cin;  // W is [rows][taps][cin]
  int mode;         // 0: dst[o + row_off][t][c] (row stride taps*dst_cin); 1: dgrad dst[c][taps-1-t][o + row_off]
  int dst_bf16;
  int dst_row_offset;  // sub-block placement (qkv packing)
  int dst_rows;        // mode 1: total rows (row stride of the transposed layout)
  int dst_cin;         // mode 0: padded input channels (>= cin; pads left untouched = 0)
  int vec8;            // set by sn_pack_prepare: 8 channels per thread (mode 0, bf16, aligned);
                       // set by sn_pack_t_prepare: 64x64 tiles with 16-byte stores (mode 1)
};
// decides SnPack::vec8 and returns the number of 256-thread blocks the job needs in sn_pack
long long sn_pack_prepare(SnPack& j);
// the same for the dgrad-layout pack (sn_pack_t)
long long sn_pack_t_prepare(SnPack& j);
// columns of W one pass-1 block of the power iteration covers (1024 with float4 rows, else 256)
inline int sn_cols_per_block(long long K) { return (K % 4 == 0) ? 1024 : 256; }
// power step over all SN weights of a net: pass 1a blocks = (job, 256 columns, 128-row chunk),
// pass 1b blocks = (job, 256 columns), pass 2 blocks = (job, 8 rows), pass 3 = one block per job
cudaError_t sn_power(const SnJob* jobs_dev, int n_jobs, const int* b1_job, const int* b1_k0, const int* b1_rc, int n_b1,
                     const int* b1b_job, const int* b1b_k0, int n_b1b, const int* b2_job, const int* b2_r0, int n_b2,
                     cudaStream_t st);
cudaError_t sn_pack(const SnPack* jobs_dev, const long long* blk_start_dev, int n_jobs, long long total_blocks,
                    cudaStream_t st);
// dgrad-layout (mode 1) packs through 32x32 smem tiles; blocks per job = taps * ceil(rows/32) * ceil(cin/32)
cudaError_t sn_pack_t(const SnPack* jobs_dev, const long long* blk_start_dev, int n_jobs, long long total_blocks,
                      cudaStream_t st);
// SN backward over all SN weights: g <- g / sigma - (<g, W> / sigma^2) u v^T; blocks of 4096 elements,
// deterministic (per-block fp64 partial dots reduced per job in block order)
cudaError_t sn_backward(const SnJob* jobs_dev, int n_jobs, const long long* blk_start_dev, long long total_blocks,
                        double* dot_partial, cudaStream_t st);

// flag[0] |= any non-finite in g
cudaError_t check_finite(const float* g, long long n, int* flag, cudaStream_t st);
cudaError_t check_finite_scalar(const float* loss, int* flag, cudaStream_t st);
// Adam over a flat buffer; g scaled by gscale (1/world); skipped when *flag != 0
cudaError_t adam_flat(float* w, const float* g, float* m, float* v, long long n, float lr, float b1, float b2,
                      float eps, const long long* t_dev, float gscale, const int* flag, cudaStream_t st);
cudaError_t adam_bookkeep(long long* t_dev, const int* flag, int* nonfinite_sticky, cudaStream_t st);

// seeded on-device init: counter-based Gaussian (Box-Muller over a 64-bit hash)
cudaError_t fill_normal(float* p, long long n, float std, uint64_t seed, uint64_t offset, cudaStream_t st);
cudaError_t fill_const(float* p, long long n, float v, cudaStream_t st);
cudaError_t normalize_vec(float* p, int n, cudaStream_t st);

// conversions between canonical OIHW and internal OHWI master layout
cudaError_t oihw_to_ohwi(const float* src, float* dst, int O, int I, int taps, cudaStream_t st);
cudaError_t ohwi_to_oihw(const float* src, float* dst, int O, int I, int taps, cudaStream_t st);
cudaError_t scale_f32(float* p, long long n, float s, cudaStream_t st);
// p[i] *= *s (device scalar)
cudaError_t scale_dev(float* p, long long n, const float* s, cudaStream_t st);
// out[0] (+)= sum_i a[i]*b[i]  (fp64 accumulation, single block)
cudaError_t dot_f32(const float* a, const float* b, long long n, float* out, int accumulate, cudaStream_t st);
cudaError_t dot_bf16_f32(const bf16* a, const float* b, long long n, float* out, int accumulate, cudaStream_t st);
// dst[r*ldd + j] (+)= src[r*lds + j] for j < cols
cudaError_t copy_rows_cols(const float* src, long long lds, long long rows, int cols, float* dst, long long ldd,
                           int accumulate, cudaStream_t st);

}  // namespace pg
