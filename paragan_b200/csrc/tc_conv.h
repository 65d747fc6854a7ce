// Internal interface of the tcgen05 convolution kernels (tc_conv.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

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
};

struct TcWgradArgs {
  int H, W, ksz, taps, Cin, Cout, c_blocks, m_tiles, n_tiles, total_kb, kb_per_split, splits;
  float* out;   // [splits][Cout][taps][Cin] partials, or dW directly
  float* bias_out;   // [splits][Cout] partial bias gradients (sum of dY over pixels), or db directly; may be null
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

size_t tc_wgrad_workspace_floats(int N, int H, int W, int Cin, int Cout, int ksz);
int tc_fprop_bn(int cout);
// true when an H x W image tiles into 128-pixel TMA boxes (see tc_conv.cu)
bool tc_geometry_ok(int H, int W);

}  // namespace pg
