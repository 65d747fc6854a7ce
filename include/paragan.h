/* libparagan — C-ABI of the B200-native ParaGAN hot path.
 *
 * The hot path is ParaGAN's replicated, data-parallel BigGAN training
 * iteration (arXiv 2411.03999): "the accelerators execute forward and backward
 * passes and then synchronize gradients among other accelerators"
 * (Sec. 3.2 Computation Model), with data parallelism as the
 * distribution strategy (Sec. 2), D and G updated one after the
 * other (Sec. 5.1), separate optimiser settings per network
 * (Sec. 5.2), bf16 storage with fp32 last layers
 * and the hardware-aware layout
 * transformation (Sec. 4.2).  BigGAN-specific
 * readings (hinge loss, spectral norm, cross-replica BN, topology) are listed
 * in DESIGN.md §3.
 *
 * Conventions
 *  - Every function returns a paragan_status.  Arguments are validated on the
 *    host before anything is enqueued; device work is stream-ordered on the
 *    caller's stream (cudaStream_t passed as void*), except the NCCL
 *    collectives, which run on the same stream.
 *  - "device" pointers must be CUDA device memory (16-byte aligned);
 *    "host" pointers are ordinary host memory.
 *  - The caller owns all buffers it passes, the workspace and the stream; the
 *    library owns the context, its NCCL communicator and its internal events.
 *  - One host thread per context.  After a CUDA/NCCL failure the context is
 *    poisoned: every call but paragan_last_error / paragan_destroy returns
 *    PARAGAN_ERR_ORDER.
 *  - There is no CPU fallback: without a usable sm_100 device, paragan_init
 *    returns PARAGAN_ERR_CUDA.
 */
#ifndef PARAGAN_H_
#define PARAGAN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARAGAN_ABI_VERSION 3

typedef struct paragan_ctx paragan_ctx; /* opaque, library-owned */

typedef enum {
  PARAGAN_OK = 0,
  PARAGAN_ERR_INVALID_ARG = 1, /* null / misaligned pointer, bad size */
  PARAGAN_ERR_CONFIG = 2,      /* inconsistent configuration (SPEC exit code 2) */
  PARAGAN_ERR_NONFINITE = 3,   /* non-finite loss or gradient: update skipped (SPEC exit code 3) */
  PARAGAN_ERR_IO = 4,
  PARAGAN_ERR_CUDA = 5,
  PARAGAN_ERR_NCCL = 6,
  PARAGAN_ERR_ORDER = 7,       /* call sequence violated, or context poisoned */
  PARAGAN_ERR_OOM = 8          /* workspace too small */
} paragan_status;

typedef enum { PARAGAN_F32 = 0, PARAGAN_BF16 = 1 } paragan_dtype;
/* BigGAN (configs 2-5, R1) or the tiny SN-DCGAN 32x32 (config 1, R25; fp32 SIMT path only). */
typedef enum { PARAGAN_ARCH_BIGGAN = 0, PARAGAN_ARCH_SNDCGAN = 1 } paragan_arch;
typedef enum { PARAGAN_NET_D = 0, PARAGAN_NET_G = 1 } paragan_net;

/* Adam hyper-parameters of one network (asymmetric policy, PAPER.md:285-307;
 * "a slightly larger epsilon" under bf16). */
typedef struct {
  float lr, beta1, beta2, eps;
} paragan_adam;

/* Per-network optimisation policy (asymmetric policy, PAPER.md:285-307 [Sec. 5.2]: "users can set the
 * optimization policy for the generator and discriminator respectively, which currently includes
 * optimizers, learning rate schedulers, warmup epochs, and gradient norms"; the optimizers of P:293:
 * AdaBelief, RAdam, Lookahead, LARS).  Hyper-parameters lr, beta1, beta2, eps come from the net's
 * paragan_adam.  The update of step t (1-based count of applied updates):
 *   g <- g * min(1, clip_norm / ||g||)           (global norm over the net; clip_norm 0 = off)
 *   u  = rule(g; m, v, t)                        (ADAM / ADABELIEF / RADAM / SGD with momentum beta1)
 *   u <- u * lars_trust * ||w_l|| / ||u_l||      (per parameter tensor l, when lars)
 *   w <- w - lr(t) u,  lr(t) = lr * min(1, t / warmup_steps) * schedule(t)
 *   every lookahead_k steps: phi <- phi + lookahead_alpha (w - phi); w <- phi
 * schedule(t): CONSTANT 1, COSINE 0.5 (1 + cos(pi min(t,T)/T)), LINEAR max(0, 1 - t/T), T = total_steps.
 * All-zero fields = plain Adam (the round-1 behaviour).  Exact rules: DESIGN.md R26-R30. */
typedef enum { PARAGAN_OPT_ADAM = 0, PARAGAN_OPT_ADABELIEF = 1, PARAGAN_OPT_RADAM = 2, PARAGAN_OPT_SGD = 3 } paragan_opt_rule;
typedef enum { PARAGAN_SCHED_CONSTANT = 0, PARAGAN_SCHED_COSINE = 1, PARAGAN_SCHED_LINEAR = 2 } paragan_schedule;
typedef struct {
  int32_t rule;          /* paragan_opt_rule */
  int32_t lars;          /* 1 = LARS trust-ratio scaling per parameter tensor */
  float lars_trust;      /* > 0 when lars */
  int32_t lookahead_k;   /* 0 = off, else the slow-weight sync period */
  float lookahead_alpha; /* (0, 1] */
  int32_t warmup_steps;  /* 0 = off; linear ramp from 0 */
  int32_t schedule;      /* paragan_schedule */
  int32_t total_steps;   /* T of the COSINE / LINEAR schedules */
  float clip_norm;       /* 0 = off */
} paragan_policy;

/* Model configuration.  BigGAN: the architecture is derived from (resolution, ch)
 * exactly as DESIGN.md §3 R1 states (BigGAN channel tables; 128/256/512 and the
 * small 16/32 test resolutions).  SN-DCGAN (arch = PARAGAN_ARCH_SNDCGAN): resolution 32,
 * widths x ch/64, dim_z 128, unconditional (labels ignored; n_classes only sizes
 * the label inputs), compute = F32 (R25). */
typedef struct {
  int32_t abi_version;   /* PARAGAN_ABI_VERSION */
  int32_t resolution;    /* 16, 32, 64, 128, 256, 512 */
  int32_t ch;            /* channel multiplier (96 for BigGAN) */
  int32_t n_classes;     /* 1000 for ImageNet */
  int32_t shared_dim;    /* shared class embedding (128) */
  int32_t z_chunk;       /* hierarchical latent chunk (20); dim_z = (blocks+1)*z_chunk */
  int32_t attn_res;      /* resolution of the non-local block (64), 0 = none */
  int32_t local_batch;   /* B per GPU, same for D and G */
  int32_t d_steps_per_g; /* n_d >= 1 (step ratio) */
  paragan_dtype compute; /* F32 = exact SIMT path; BF16 = bf16 storage + tcgen05 */
  int32_t c_pad_image;   /* channel padding of the packed image (>= 3; 8 for BF16) */
  paragan_adam adam_d, adam_g;
  float sn_eps, bn_eps;
  int32_t rank, world_size, device;
  uint64_t seed;         /* on-device weight init (paragan_init_params) */
  int32_t arch;          /* a paragan_arch value; field added in ABI 2 */
  paragan_policy policy_d, policy_g;   /* ABI 3 */
  int32_t grad_comm_bf16; /* 1 = gradient all-reduce in bf16 (half the NVLink bytes, "faster to ...
                           * communicate"); 0 = fp32 (default; exact integer sums, bit-identical replicas
                           * either way) */
} paragan_config;

typedef struct {
  float d_loss, g_loss, d_real_mean, d_fake_mean;
  int32_t nonfinite; /* a step of this iteration skipped its update */
  int64_t t_d, t_g;  /* Adam step counts */
} paragan_stats;

/* ------------------------------------------------------------------ setup */

/* 128-byte NCCL unique id; call on rank 0 and broadcast it (torch.distributed). */
paragan_status paragan_get_unique_id(uint8_t id[128]);

/* Bytes of device workspace paragan_init needs for this config (activations,
 * weights, optimiser state, scratch). */
paragan_status paragan_workspace_size(const paragan_config* cfg, size_t* bytes);

/* Length of the canonical flat fp32 state of one network: trainable tensors in
 * forward-layer order (conv weights OIHW, linears [out,in], embeddings
 * [classes,dim], each weight followed by its bias), then the spectral-norm u
 * vectors in the same layer order. */
paragan_status paragan_param_count(const paragan_config* cfg, paragan_net net, size_t* n_state,
                                   size_t* n_trainable);

/* Create a context on cfg->device.  id: the broadcast NCCL id (ignored when
 * world_size == 1).  workspace: device buffer of at least
 * paragan_workspace_size bytes, owned by the caller.  stream: cudaStream_t. */
paragan_status paragan_init(const paragan_config* cfg, const uint8_t id[128], void* workspace, size_t ws_bytes,
                            void* stream, paragan_ctx** out);

/* Seeded on-device initialisation: N(0, 0.02) weights, zero biases, unit BN
 * gains, attention gamma = attn_gamma, unit-norm Gaussian u vectors.  Every rank
 * with the same seed gets the identical replica. */
paragan_status paragan_init_params(paragan_ctx* ctx, float attn_gamma);

/* Canonical flat state (host, fp32, paragan_param_count n_state floats).
 * set resets Adam moments and step counts; get/get_grads synchronise the stream.
 * get_grads returns the all-reduced (mean) gradient of the last step of `net`
 * (n_trainable floats). */
paragan_status paragan_set_params(paragan_ctx* ctx, paragan_net net, const float* host, size_t n);
paragan_status paragan_get_params(paragan_ctx* ctx, paragan_net net, float* host, size_t n);
paragan_status paragan_get_grads(paragan_ctx* ctx, paragan_net net, float* host, size_t n);
/* Test hook: overwrite the net's local gradient buffer with a canonical-layout host array (n_trainable
 * floats), as if this rank's backward had produced it (the next paragan_allreduce_grads sums it). */
paragan_status paragan_set_grads(paragan_ctx* ctx, paragan_net net, const float* host, size_t n);

/* --------------------------------------------------------------- hot path */

/* Hardware-aware layout transformation: NCHW fp32 ->
 * NHWC with channels zero-padded to c_pad, stored as `dst` dtype (bf16 by
 * round-to-nearest-even).  src, dst: device.  Bit-exact.  Independent of any
 * context.  c_pad >= c; for BF16 c_pad % 8 == 0. */
paragan_status paragan_layout_pack(const float* src_nchw, void* dst_nhwc, paragan_dtype dst, int32_t n, int32_t c,
                                   int32_t h, int32_t w, int32_t c_pad, void* stream);
/* Exact inverse on the first c channels (NHWC -> NCHW fp32). */
paragan_status paragan_layout_unpack(const void* src_nhwc, paragan_dtype src, float* dst_nchw, int32_t n, int32_t c,
                                     int32_t h, int32_t w, int32_t c_pad, void* stream);

/* One discriminator step: SN(G) -> G(z, fake_y) with
 * cross-replica BN -> SN(D) -> D([fake; real]) (one pass over 2B images,
 * PAPER.md:243) -> hinge L_D -> backward through D -> gradient all-reduce
 * -> Adam(D).
 *   real_nhwc : device, [B, R, R, c_pad_image] in the compute dtype (output of
 *               paragan_layout_pack)
 *   real_y, fake_y : device int32 [B];  z : device fp32 [B, dim_z]
 *   flags     : PARAGAN_FLAG_* */
paragan_status paragan_d_step(paragan_ctx* ctx, const void* real_nhwc, const int32_t* real_y, const float* z,
                              const int32_t* fake_y, uint32_t flags);

/* One generator step: SN(G) -> G(z, y) -> SN(D) -> D(fake) -> L_G = -mean ->
 * backward through D (inputs only) and G -> all-reduce -> Adam(G).
 * Returns PARAGAN_ERR_ORDER unless d_steps_per_g D steps preceded it. */
paragan_status paragan_g_step(paragan_ctx* ctx, const float* z, const int32_t* y, uint32_t flags);

/* ---------------------------------------------- asynchronous update scheme (Sec. 5.1)
 * "instead of waiting on the other component, the generator/discriminator can write their intermediate
 * output to the buffer and proceed to update using the current state of the network.  For iteration t,
 * discriminators D_t receive a batch of real and generated samples from the image buffer (img_buff).
 * Similarly, the generators can use the snapshot of the current discriminator state ... breaking the data
 * dependency."  The library provides the per-side steps; the buffers and the placement of G and D on
 * disjoint GPU groups live in paper_2411_03999_b200/async_gan.py (R31-R33). */

/* D step on GIVEN fakes (an img_buff entry): no SN(G) / G forward.  fakes_nhwc: device, [B,R,R,c_pad] in
 * the compute dtype (as paragan_generate / paragan_export_fakes write them).  Otherwise as paragan_d_step. */
paragan_status paragan_d_step_fakes(paragan_ctx* ctx, const void* real_nhwc, const int32_t* real_y,
                                    const void* fakes_nhwc, const int32_t* fake_y, uint32_t flags);
/* G forward only (SN(G) power step + cross-replica BN, as in the D step): fakes for img_buff, written to
 * dst_nhwc (device, [B,R,R,c_pad], compute dtype). */
paragan_status paragan_generate(paragan_ctx* ctx, const float* z, const int32_t* y, void* dst_nhwc);
/* Copy the last generated images (the last G step's or D step's fakes) to dst_nhwc (device, as above). */
paragan_status paragan_export_fakes(paragan_ctx* ctx, void* dst_nhwc);
/* Device-to-device snapshot of a network's state (the D snapshot G uses): dst/src device fp32 buffers of
 * paragan_state_size floats in the library's INTERNAL layout (16-byte aligned tensors, then the u vectors;
 * only meaningful between contexts of the same config).  import resets nothing else (Adam state stays). */
paragan_status paragan_state_size(paragan_ctx* ctx, paragan_net net, size_t* n_floats);
paragan_status paragan_export_state(paragan_ctx* ctx, paragan_net net, float* dst_device);
paragan_status paragan_import_state(paragan_ctx* ctx, paragan_net net, const float* src_device);

/* In-place SUM of the net's gradient over all ranks (NCCL all-reduce over
 * NVLink); the mean's 1/world_size is folded into the update
 * (paragan_apply_update) and into paragan_get_grads, so no separate scaling pass
 * runs.  d_step/g_step call it themselves unless PARAGAN_FLAG_NO_ALLREDUCE is set. */
paragan_status paragan_allreduce_grads(paragan_ctx* ctx, paragan_net net);

/* The net's optimiser update with its own policy and hyper-parameters
 * (paragan_policy); skipped (state unchanged) when the gradient
 * is non-finite.  Pairs with PARAGAN_FLAG_NO_UPDATE. */
paragan_status paragan_apply_update(paragan_ctx* ctx, paragan_net net);

/* Losses of the last D and G steps; synchronises the stream.  Returns
 * PARAGAN_ERR_NONFINITE when an update was skipped since the last call. */
paragan_status paragan_sync_stats(paragan_ctx* ctx, paragan_stats* out);

/* The same values without a host synchronisation: enqueues, on the context's stream, device-to-host
 * copies of the last steps' statistics into `out` (caller-owned, page-locked host memory, valid once the
 * stream has reached this point — e.g. after an event recorded right after the call).  Losses are already
 * divided by world_size, as in paragan_sync_stats; `nonfinite` is the sticky flag, which only
 * paragan_sync_stats clears.  For pipelined host loops that read step i's losses while step i + 1 runs. */
paragan_status paragan_stats_async(paragan_ctx* ctx, paragan_stats* out);

/* Copy the last generated images (bf16/fp32 NHWC as D saw them) to host NCHW fp32 [B,3,R,R]. */
paragan_status paragan_get_fakes(paragan_ctx* ctx, float* host_nchw, size_t n);

/* Test hook: the gradient of the last G step's loss with respect to the generated images, as D's
 * backward produced it (the dgrad of D's first conv, in the compute dtype), unpacked to host NCHW fp32
 * [B,3,R,R].  Available only after a paragan_g_step called with PARAGAN_FLAG_KEEP_DFAKE (otherwise
 * PARAGAN_ERR_ORDER).  Lets tests compare G's backward and D's input gradient with the oracle
 * separately (each fed the other side's tensor).  Synchronises the stream. */
paragan_status paragan_get_dfake(paragan_ctx* ctx, float* host_nchw, size_t n);

/* Number of kernels this context launched since creation (bench accounting). */
paragan_status paragan_kernel_launches(const paragan_ctx* ctx, uint64_t* n);

/* Live kernel timing for the roofline report: while enabled, every tcgen05
 * convolution launch of the step is bracketed by CUDA events on the context's
 * stream.  profile_read (synchronises) returns, for kind 0 = implicit-GEMM
 * fprop/dgrad kernel, 1 = wgrad (incl. its split-K reduction), 2 = NCCL collectives
 * (gradient, cross-replica BN and loss all-reduces), the number of launches, their
 * summed device time (ms) and their ALGORITHMIC flops (2*M*N*K with unpadded channel
 * counts, G's conv1 counted over the upsampled tensor as BigGAN defines it; for kind 2:
 * bytes reduced).  Kinds 3 / 4: the launches of kinds 0 / 1 with the flops actually
 * issued to the tensor cores (the sub-pixel conv1 issues 1/2.25 of its algorithmic
 * work).  Kind 5: the fused attention kernels (forward + backward; flops = their MMA work); kind 6: G's fp32
 * output layer (thin fprop / dgrad / wgrad; 2*27*C flops per pixel each).  enable=1 also clears the record. */
paragan_status paragan_profile(paragan_ctx* ctx, int32_t enable);
paragan_status paragan_profile_read(paragan_ctx* ctx, int32_t kind, uint64_t* launches, double* ms, double* flops);

/* ------------------------------------------ host-side system features (PAPER.md:221-233 [Sec. 4.1]) */

/* Asynchronous checkpoint writer ("We use an asynchronous checkpoint writer to save model
 * checkpoints. The checkpoint will be streamed into the output buffer instead of having a blocking call to
 * pass it to the CPU host"): the full training state (both networks' weights and SN u vectors, optimiser
 * moments and step counts, Lookahead slow weights) is snapshotted stream-ordered into a device staging
 * buffer on the caller's stream (a device-to-device copy), streamed to pinned host memory on a separate
 * copy stream, and written to `path` (via `path`.tmp + rename) by a host thread while training continues.
 * At most one checkpoint is in flight per context: a second save first waits for the first.  The file
 * holds a header (magic, ABI version, the config fields that fix the layout, array sizes) and a 64-bit
 * FNV-1a hash of the payload. */
paragan_status paragan_checkpoint_save_async(paragan_ctx* ctx, const char* path);
/* Blocks until the checkpoint in flight (if any) is on disk; PARAGAN_ERR_IO if writing it failed. */
paragan_status paragan_checkpoint_wait(paragan_ctx* ctx);
/* Synchronous restore into a context of the same configuration (PARAGAN_ERR_CONFIG on a layout mismatch,
 * PARAGAN_ERR_IO on a short or corrupt file); resumes training exactly where the checkpoint was taken. */
paragan_status paragan_checkpoint_load(paragan_ctx* ctx, const char* path);

/* Congestion-aware prefetcher: reader threads fill a bounded queue of batches read from
 * sample shards (paragan_shard_write format); a sliding window of per-batch read latencies (ms) adds a
 * reader and doubles the queue depth when the window mean exceeds latency_threshold_ms, and releases a
 * reader and halves the depth when it falls below half the threshold ("once the latency falls below the
 * threshold, it releases the resources").  Batches come out in order (batch i = samples [iB, (i+1)B),
 * cyclic over the shards).  Host only: no CUDA calls. */
typedef struct {
  int32_t batch, channels, height, width;  /* a sample: channels*height*width fp32 + one int32 label */
  int32_t min_workers, max_workers;        /* reader threads (resources the tuner scales) */
  int32_t min_depth, max_depth;            /* prefetched batches */
  int32_t window;                          /* latency samples per decision */
  float latency_threshold_ms;
  float inject_latency_ms;                 /* test hook: simulated storage/network delay per batch read */
} paragan_prefetch_config;
typedef struct {
  int32_t active_workers, depth, queued;
  float window_mean_ms;
  int64_t batches_read, scale_ups, scale_downs;
} paragan_prefetch_stats;
typedef struct paragan_prefetcher paragan_prefetcher;
/* Writes n samples (images fp32 NCHW [n,c,h,w], labels int32 [n]) as one shard file. */
paragan_status paragan_shard_write(const char* path, const float* images, const int32_t* labels, int32_t n,
                                   int32_t c, int32_t h, int32_t w);
paragan_status paragan_prefetch_create(const paragan_prefetch_config* cfg, const char* const* shard_paths,
                                       int32_t n_shards, paragan_prefetcher** out);
/* Copies the next batch (in order) into caller-owned host buffers ([batch,c,h,w] fp32, [batch] int32;
 * pinned memory makes the following host-to-device copy asynchronous); blocks until it is read. */
paragan_status paragan_prefetch_next(paragan_prefetcher* p, float* host_images, int32_t* host_labels);
paragan_status paragan_prefetch_get_stats(paragan_prefetcher* p, paragan_prefetch_stats* out);
paragan_status paragan_prefetch_set_latency(paragan_prefetcher* p, float inject_latency_ms);
paragan_status paragan_prefetch_destroy(paragan_prefetcher* p);

const char* paragan_last_error(const paragan_ctx* ctx);
paragan_status paragan_destroy(paragan_ctx* ctx);

#define PARAGAN_FLAG_NO_ALLREDUCE 1u /* keep the local gradient (test hook) */
#define PARAGAN_FLAG_NO_UPDATE 2u    /* skip Adam (test hook) */
#define PARAGAN_FLAG_KEEP_DFAKE 4u   /* g_step keeps dL_G/d(fake images) for paragan_get_dfake (test hook) */
#define PARAGAN_FLAG_ASYNC 8u        /* g_step in the asynchronous scheme: no D steps precede it in this
                                      * context (it trains through an imported D snapshot) */

/* ------------------------------------------------------- op-level test hooks
 * Single kernels of the path, exposed so tests can compare each with the
 * oracle.  All pointers are device pointers; shapes as stated. */

/* y[N,H,W,Cout] = conv(x[N,H,W,Cin], w[Cout][k*k][Cin]) + bias[Cout]; 3x3 pad 1 or 1x1.
 * BF16: x, w, y bf16 (tcgen05 path, Cin % 8 == 0); F32: fp32 SIMT path. */
paragan_status paragan_op_conv_fwd(paragan_dtype dt, const void* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                                   const void* wgt, const float* bias, int32_t cout, int32_t ksz, void* y,
                                   void* stream);
/* The same BF16 tcgen05 convolution with the fused epilogues the training step uses (tc_conv.cu):
 *   y = bf16( relu_out ? max(0, acc + bias + r) : acc + bias + r ),  acc zeroed where relu_ref <= 0,
 * r = residual[pixel] (res_mode 1, bf16 [N,H,W,Cout]) or residual at the half-resolution pixel
 * (res_mode 2, bf16 [N,H/2,W/2,Cout]: the x2-nearest-upsampled skip of G's blocks), or 0 (residual
 * NULL).  relu_ref: bf16 [N,H,W,Cout] or NULL (the dgrad's fused ReLU-backward mask).  All device
 * pointers 16-byte aligned; shapes as op_conv_fwd. */
paragan_status paragan_op_conv_fwd_ex(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const void* wgt,
                                      const float* bias, int32_t cout, int32_t ksz, const void* residual,
                                      int32_t res_mode, const void* relu_ref, int32_t relu_out, void* y,
                                      void* stream);
/* D's block output with the 2x2 average pooling fused into the conv epilogue (the engine's path for blocks with
 * a downsample at W <= 64): t = bf16(conv(x, wgt) + bias + residual) as op_conv_fwd_ex (res_mode 1), then
 *   y_pool[n][h/2][w/2][Cout] = bf16(((t00 + t01) + (t10 + t11)) * 0.25),  y_relu = relu(y_pool) (optional)
 * without t reaching memory.  BF16; W <= 64, H and W even, the 128-pixel tiling of op_conv_fwd, Cout % 16 == 0,
 * 16-byte aligned device pointers. */
paragan_status paragan_op_conv_fwd_pool(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const void* wgt,
                                        const float* bias, int32_t cout, int32_t ksz, const void* residual,
                                        void* y_pool, void* y_relu, void* stream);
/* dw[Cout][k*k][Cin] (fp32) = sum_p dy[p][o] * x[p + tap][c]; db[Cout] (fp32, optional, NULL to skip) =
 * sum_p dy[p][o], the bias gradient (BF16: computed by the same tcgen05 launch).
 * F32 with Cout = 3, 3x3 (G's fp32 output layer) runs the thin kernels, also in op_conv_fwd. */
paragan_status paragan_op_conv_wgrad(paragan_dtype dt, const void* x, const void* dy, int32_t n, int32_t h,
                                     int32_t w, int32_t cin, int32_t cout, int32_t ksz, float* dw, float* db,
                                     void* stream);
/* y[N,2H,2W,Cout] = conv3x3(up2_nearest(x[N,H,W,Cin])) + bias — G's conv1 (SURVEY §8(f) NEXT-1,
 * sub-pixel phase decomposition): BF16 only; w fp32 [Cout][9][Cin] (OHWI), folded on the device into
 * four 2x2 phase kernels (rounded to bf16 after the fold), x / y bf16 NHWC, Cin and Cout % 8 == 0. */
paragan_status paragan_op_conv_up2_fwd(const void* x, int32_t n, int32_t h, int32_t w, int32_t cin, const float* wgt,
                                       const float* bias, int32_t cout, void* y, void* stream);

/* dx[N,H,W,Cin] = the input gradient of conv3x3(up2_nearest(x)) at LOW resolution from dy[N,2H,2W,Cout]
 * (the up2 adjoint included), through the same phase decomposition; BF16; w fp32 [Cout][9][Cin]. */
paragan_status paragan_op_conv_up2_dgrad(const void* dy, int32_t n, int32_t h, int32_t w, int32_t cout,
                                         const float* wgt, int32_t cin, void* dx, void* stream);

/* dw[Cout][9][Cin] (fp32) = weight gradient of conv3x3(up2_nearest(x)) from the LOW-resolution
 * x[N,H,W,Cin] and dy[N,2H,2W,Cout] through the phase decomposition (16 folded taps, unfolded onto the
 * 3x3 taps); db[Cout] (optional) = sum of dy.  BF16. */
paragan_status paragan_op_conv_up2_wgrad(const void* x, const void* dy, int32_t n, int32_t h, int32_t w, int32_t cin,
                                         int32_t cout, float* dw, float* db, void* stream);

/* dx[N,H,W,Cin] = sum_{o,tap} dy[p - delta_tap][o] w[o][tap][c]: the input gradient of the 3x3 conv.
 * F32 only, Cout = 3 (G's fp32 output layer), Cin % 4 == 0; dx 16-byte aligned. */
paragan_status paragan_op_conv_dgrad(paragan_dtype dt, const void* dy, int32_t n, int32_t h, int32_t w, int32_t cout,
                                     const void* wgt, int32_t cin, int32_t ksz, void* dx, void* stream);

/* G's fp32 output layer as the BF16 engine runs it on the tensor cores (reading R36 in DESIGN.md):
 * x fp32 [N,H,W,Cin] is split into two bf16 planes x1 = bf16(x), x2 = bf16(x - x1), w fp32 [3][9][Cin]
 * (OHWI) into three bf16 terms w1 = bf16(w), w2 = bf16(w - w1), w3 = bf16(w - w1 - w2), and
 *   y[p][o] = bias[o] + sum_{tap,c} (x1 + x2)[p + tap][c] (w1 + w2)[o][tap][c] + x1[p + tap][c] w3[o][tap][c]
 * with fp32 tensor-core accumulation (y fp32 [N,H,W,3]; bias may be NULL).  When dy (fp32 [N,H,W,3]) and
 * dw (fp32 [3][9][Cin]) are both non-NULL, also the backward pass the engine runs (one kernel): with
 * dy1 = bf16(dy), dy2 = bf16(dy - dy1),
 *   dw[o][tap][c] = sum_p (dy1 + dy2)[p][o] (x1 + x2)[p + tap][c]                      (written)
 *   dx[p][c]      = sum_{o,tap} (dy1 + dy2)[p - tap][o] w1[o][tap][c] + dy1[p - tap][o] (w2 + w3)[o][tap][c]
 * (dx fp32 [N,H,W,Cin], optional; requires dw).  3x3 pad 1;
 * W = 128 (one image row per tensor-core tile), Cin % 8 == 0, Cin <= 128; device pointers, 16-byte
 * aligned; the split planes and partials are stream-ordered temporaries.  PARAGAN_ERR_INVALID_ARG on a
 * shape or alignment violation. */
paragan_status paragan_op_out_conv_split(const float* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                                         const float* wgt, const float* bias, float* y, const float* dy, float* dw,
                                         float* dx, void* stream);

/* Fused attention core of the non-local block (BigGAN's self-attention,
 * reading R8 — beta = softmax_rows(theta^T phi) without a 1/sqrt(d) scale, o = beta g).
 * BF16 only (tcgen05).  Per image of hw pixels and q = hw/4 pooled keys:
 *   qkv  bf16 [n][hw][ct]  theta = channels [0, cq)   (cq = 16 or 32; channels beyond C/8 zero)
 *   phi  bf16 [n][q][cq]   max-pooled phi;  gp bf16 [n][q][c2] max-pooled g (c2 % 16 == 0, <= 128)
 *   o    bf16 [n][hw][c2]  = beta gp with beta rounded to bf16 (R14);  o32 fp32 the same before the
 *        final rounding (may be NULL);  lse fp32 [n][hw] = log sum_j exp(s_ij)
 * hw and q must be multiples of 128; all pointers device, 16-byte aligned, caller-owned.
 * Returns PARAGAN_ERR_INVALID_ARG for shapes outside that set. */
paragan_status paragan_op_attn_fwd(const void* qkv, const void* phi, const void* gp, int32_t n, int32_t hw,
                                   int32_t cq, int32_t c2, int32_t ct, void* o, float* o32, float* lse,
                                   void* stream);
/* Backward of the same: from dO bf16 [n][hw][c2], o32 and lse of the forward,
 *   dS = beta (dP - rowsum(dO o32)),  dP = dO gp^T (fp32, beta recomputed in fp32),
 *   dtheta = bf16(dS) phi -> bf16 into dqkv [n][hw][ct] channels [0, cq) (other channels untouched),
 *   dphi fp32 [n][q][cq] = bf16(dS)^T theta,  dgp fp32 [n][q][c2] = bf16(beta)^T dO.
 * Sums are taken in a fixed order (bit-reproducible). */
paragan_status paragan_op_attn_bwd(const void* qkv, const void* phi, const void* gp, const void* dO,
                                   const float* o32, const float* lse, int32_t n, int32_t hw, int32_t cq,
                                   int32_t c2, int32_t ct, void* dqkv, float* dphi, float* dgp, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PARAGAN_H_ */
