// Internal interface of the tcgen05 convolution kernels (tc_conv.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <cuda.h>

namespace pg {

struct TcEpilogue {
  const float* bias = nullptr;     // [Cout] fp32, added after scaling
  const float* alpha = nullptr;    // device scalar; acc is scaled by *alpha (attention gamma)
  const void* residual = nullptr;  // bf16, added last (same pixel or half-res nearest-upsampled)
  int res_mode = 0;                // 1 = same resolution, 2 = half resolution (x2 nearest)
  int ldr = 0;                     // residual row stride (elements), default Cout
  const void* relu_ref = nullptr;  // bf16 [M][ldo]: acc is zeroed where ref <= 0 (fused ReLU backward)
  void* out = nullptr;             // bf16 or fp32 [M][ldo]
  int out_f32 = 0;
  int ldo = 0;                     // default Cout
  int relu_out = 0;                // ReLU applied last, before the single rounding (D's conv1 -> conv2 input)
  // fused 2x2 average pooling (W <= 64, H and W even; tiles of whole row pairs): instead of `out` the kernel
  // writes pool_out = avgpool2(bf16(epilogue)) [M/4][ldo] and, when set, pool_relu = relu(pool_out)
  void* pool_out = nullptr;
  void* pool_relu = nullptr;
};

struct TcFpropArgs {
  long long M;
  int H, W, ksz, taps, c_chunks, last_ksteps, Cout, m_tiles, n_tiles;
  const float* bias;
  const float* alpha;
  const void* residual;
  int res_mode, ldr;
  const void* relu_ref;
  void* out;
  int out_f32, ldo;
  int tma_store;   // epilogue writes through SW128 staging tiles + TMA bulk stores
  int relu_out;
  // sub-pixel mode (phases = 4): the 3x3 conv of a x2-nearest-upsampled input computed as four 2x2
  // convs of the low-resolution input, one per output phase (a, b); H, W, M are low-resolution and
  // the output is [N][2H][2W][Cout] written through a 5-D map {C, 2, W, 2, N*H}
  int phases;
  void* pool_out;    // see TcEpilogue
  void* pool_relu;
  // phase dgrad (phase_dgrad = 1): the input gradient of conv3x3(up2(x)) at low resolution,
  // dX[i][j] = sum_{phase (a,b), tap (p,q)} dY[2(i+1-a-p)+a][2(j+1-b-q)+b] Wfold_ab[p][q]^T:
  // K = 16 taps, tap u = phase * 4 + p * 2 + q read through the phase's own dY tensor map
  int phase_dgrad;
};

struct TmaQuad {   // four tensor maps passed by value (64-byte aligned)
  CUtensorMap m[4];
};

struct TcWgradArgs {
  int H, W, ksz, taps, Cin, Cout, c_blocks, m_tiles, n_tiles, total_kb, kb_per_split, splits;
  float* out;   // [splits][Cout][taps][Cin] partials, or dW directly
  float* bias_out;   // [splits][Cout] partial bias gradients (sum of dY over pixels), or db directly; may be null
  // phase wgrad (phases = 4): weight gradient of conv3x3(up2(X)) as 16 folded taps (phase * 4 + tap) over
  // the low-resolution X and the phase views of dY; bias partials are [splits][4 phases][Cout]
  int phases;
};

// Y[N,H,W,Cout] = epilogue( conv(X[N,H,W,Cin] bf16, Wp[Cout][ksz*ksz][Cin] bf16) )
// Also used for dgrad with X = dY and Wp = the flipped, transposed weight.
cudaError_t tc_conv_fprop(const void* x, int N, int H, int W, int Cin, const void* wpack, int Cout, int ksz,
                          const TcEpilogue& epi, cudaStream_t st);

// dW[Cout][ksz*ksz][Cin] (+)= sum_p dY[p][o] X[p + tap][c]   (fp32; split-K with a
// deterministic reduction through ``scratch``)
// dbias (optional, fp32 [Cout]) = sum_p dY[p][o], computed by the same launch (written, not accumulated)
cudaError_t tc_conv_wgrad(const void* x, const void* dy, int N, int H, int W, int Cin, int Cout, int ksz,
                          float* dw, int accumulate, float* scratch, size_t scratch_floats, cudaStream_t st,
                          float* dbias = nullptr);

// Y[N,2H,2W,Cout] = epilogue( conv3x3( up2_nearest(X[N,H,W,Cin]) ) ) through the phase decomposition:
// wpack4 = [4 phases (a,b)][Cout][4 taps (p,q)][Cin], the 3x3 weight folded per phase (fold_up2_weights).
// 2.25x fewer MACs than the conv on the upsampled tensor; epilogue: bias (+alpha) only.
cudaError_t tc_conv_fprop_up2(const void* x, int N, int H, int W, int Cin, const void* wpack4, int Cout,
                              const TcEpilogue& epi, cudaStream_t st);
// dX[N,H,W,Cin] (+ epilogue) = input gradient of conv3x3(up2(X)) from dY[N,2H,2W,Cout]: wt4 =
// [Cin][16 = phase*4 + tap][Cout], the folded kernel transposed (fold_up2_weights, layout 1).
cudaError_t tc_conv_dgrad_up2(const void* dy, int N, int H, int W, int Cout, const void* wt4, int Cin,
                              const TcEpilogue& epi, cudaStream_t st);
// dW[Cout][9][Cin] (written) = weight gradient of conv3x3(up2(X)) from the low-resolution X[N,H,W,Cin] and
// dY[N,2H,2W,Cout]: 16 folded-tap sums (2.25x fewer MACs), unfolded onto the 3x3 taps by the reduction;
// dbias (optional) = sum of dY.  scratch >= 16*Cout*Cin + 4*Cout floats.
cudaError_t tc_conv_wgrad_up2(const void* x, const void* dy, int N, int H, int W, int Cin, int Cout, float* dw,
                              float* scratch, size_t scratch_floats, cudaStream_t st, float* dbias);
size_t tc_wgrad_workspace_floats(int N, int H, int W, int Cin, int Cout, int ksz);
int tc_fprop_bn(int cout);
// true when an H x W image tiles into 128-pixel TMA boxes (see tc_conv.cu)
bool tc_geometry_ok(int H, int W);

}  // namespace pg
