// G's fp32 output layer on the tcgen05 tensor cores through bf16 splits (tc_outconv.cu; reading R36).
#pragma once
#include <cuda_runtime.h>

namespace pg {

// true when the tensor-core output layer applies: W = 128 (one image row per M tile), C % 8 == 0, C <= 128
bool out_conv_tc_ok(int H, int W, int C);

// y[N][H][W][3] (fp32) = bias + conv3x3(x, w) with x given as its two-term bf16 split xs = [x1 | x2]
// (bf16 [N][H][W][2C]; split_planes / bn_apply_relu_split) and w as the three-term split ws
// (bf16 [96][2C]; split_out_weights): Z = xs ws^T on the tensor cores, then the 3x3 spatial sum.
cudaError_t out_conv_fwd_tc(const void* xs, int N, int H, int W, int C, const void* ws, const float* bias, float* y,
                            cudaStream_t st);

// Both gradients of the same layer in one pass (R36): dx[N][H][W][C] (fp32) = conv^T(dy, w) and
// dw[3][9][C] (fp32, written) = sum_p dy[p][o] x[p + tap][c], from xs (the split activation above), dy
// (fp32 [N][H][W][3]) and wd (bf16 [C16][128], split_out_weights_dgrad: the dgrad operand over
// [dy1 | dy2 | dy1 | dy1]).  scratch >= out_conv_bwd_scratch_floats(C) (per-CTA dW partials).
size_t out_conv_bwd_scratch_floats(int C);
cudaError_t out_conv_bwd_tc(const void* xs, const float* dy, int N, int H, int W, int C, const void* wd, float* dx,
                            float* dw, float* scratch, size_t scratch_floats, cudaStream_t st);

}  // namespace pg
