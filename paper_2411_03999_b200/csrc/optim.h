// Asymmetric optimisation policy kernels (PAPER.md:285-307 [Sec. 5.2]):
// AdaBelief / RAdam / SGD-momentum / Adam rules, LARS trust-ratio scaling, Lookahead slow weights,
// global-norm gradient clipping and the warmup / schedule learning-rate ramp.  Memory-bound: one pass
// over (w, g, m, v) per update (plus one read of g for clipping and one of (w, u) for LARS).
// Every reduction is per 16K-element chunk of one parameter tensor, summed in chunk order
// (deterministic, identical on every replica).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pg {

constexpr int kOptChunk = 16384;

struct OptChunk {        // one chunk of one parameter tensor of the flat buffer
  long long start;
  int len;
  int first;             // index of the tensor's first chunk
  int count;             // chunks of the tensor
};

struct OptRule {         // per-network policy (paragan_policy + paragan_adam)
  int rule;              // 0 adam, 1 adabelief, 2 radam, 3 sgd (momentum beta1)
  int lars;
  int lookahead_k;
  int warmup;
  int schedule;          // 0 constant, 1 cosine, 2 linear
  int total;
  float lr, b1, b2, eps, trust, alpha, clip;
  float gscale;          // 1 / world size (the gradient buffer holds the sum over ranks)
};

// part[c] = sum over chunk c of (gscale * g)^2 (fp64)
cudaError_t opt_sumsq(const float* g, const OptChunk* chunks, int n_chunks, float gscale, double* part,
                      cudaStream_t st);
// clip_scale[0] = min(1, clip / sqrt(sum part)); flag |= sum part non-finite
cudaError_t opt_clip_finalize(const double* part, int n_chunks, float clip, float* clip_scale, int* flag,
                              cudaStream_t st);
// one update of the rule (t = *t_dev + 1); skipped when *flag.  Without LARS w is updated in place;
// with LARS the step direction is written to u and per-chunk |w|^2, |u|^2 to wpart / upart, and
// opt_lars_apply finishes the update.  clip_scale may be null (no clipping).
cudaError_t opt_update(float* w, const float* g, float* m, float* v, float* u, const OptChunk* chunks, int n_chunks,
                       const OptRule& r, const long long* t_dev, const float* clip_scale, const int* flag,
                       double* wpart, double* upart, cudaStream_t st);
cudaError_t opt_lars_apply(float* w, const float* u, const OptChunk* chunks, int n_chunks, const OptRule& r,
                           const long long* t_dev, const double* wpart, const double* upart, const int* flag,
                           cudaStream_t st);
// Lookahead (after the step counter advanced): when t % k == 0: slow += alpha (w - slow); w = slow
cudaError_t opt_lookahead(float* w, float* slow, long long n, int k, float alpha, const long long* t_dev,
                          const int* flag, cudaStream_t st);

}  // namespace pg
