// BigGAN step engine.
//
// One Engine<T> per rank; T = float (F32 mode: exact SIMT path) or bf16 (BF16
// mode: bf16 storage, tcgen05 convolutions, fp32 last layers as PAPER.md:202
// prescribes).  Everything the step touches lives in the caller's workspace,
// carved once at init by a bump arena; the step itself allocates nothing.
//
// Parameter storage: one flat fp32 buffer per network in canonical order
// (include/paragan.h), except that conv weights are held OHWI ([C_out][taps]
// [C_in], the K-major GEMM B operand) instead of OIHW; set/get convert.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "engine.h"
#include "host_io.h"
#include "tc_attn.h"
#include "kernels.h"
#include "optim.h"
#include "tc_conv.h"
#include "tc_outconv.h"

namespace pg {

namespace {

constexpr int kMaxPartialBlocks = 1184;  // 8 waves of 148 SMs
constexpr int kDcondK = 256;              // K slice of the split-K CBN dcond GEMMs

struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <class X>
  X* get(size_t count) {
    off = (off + 255) & ~size_t(255);
    X* p = reinterpret_cast<X*>((base ? base : reinterpret_cast<char*>(0x100000)) + off);
    off += count * sizeof(X);
    return p;
  }
};

struct PEntry {
  std::string name;
  std::vector<int> shape;
  bool conv4d = false;
  bool sn = false;
  long long off = 0, n = 0;   // internal offset (16-byte aligned) and size
  long long coff = 0;         // offset in the canonical (unpadded) flat layout of the C-ABI
  long long u_off = -1, v_off = -1;
  int job = -1;
};

struct Net {
  std::vector<PEntry> E;
  long long n = 0, nu = 0, nv = 0;   // n: internal flat size (every tensor starts 16-byte aligned)
  long long nc = 0;                  // canonical flat size (paragan_param_count n_trainable)
  float *p = nullptr, *g = nullptr, *m = nullptr, *v = nullptr, *u = nullptr;
  float *sn_v = nullptr, *sn_t = nullptr, *sn_s = nullptr, *sigma = nullptr;
  std::vector<int> sn_entries;                // entry index per SN job
  SnJob* jobs_d = nullptr;
  int *b1_job = nullptr, *b1_k0 = nullptr, *b1_rc = nullptr, *b1b_job = nullptr, *b1b_k0 = nullptr;
  int *b2_job = nullptr, *b2_r0 = nullptr;
  int nb1 = 0, nb1b = 0, nb2 = 0;
  float* sn_part = nullptr;
  long long npart = 0;
  double *sn_coef = nullptr, *sn_dotp = nullptr;
  long long* snb_start = nullptr;
  long long snb_blocks = 0;
  std::vector<SnPack> pf_h, pb_h;             // fwd packs, dgrad packs
  SnPack *pf_d = nullptr, *pb_d = nullptr;
  long long *pf_start = nullptr, *pb_start = nullptr;
  long long pf_blocks = 0, pb_blocks = 0;
  int* snb_idx = nullptr;
  float** snb_grad = nullptr;
  long long* t_dev = nullptr;
  int* flag = nullptr;
  float* loss = nullptr;   // [4]
  // optimiser policy (NEXT-3): chunk table over the parameter tensors, reduction partials, slow weights
  std::vector<OptChunk> chunks_h;
  OptChunk* chunks_d = nullptr;
  double *opt_wpart = nullptr, *opt_upart = nullptr;
  float* clip_scale = nullptr;
  float* slow = nullptr;   // Lookahead phi (only when enabled)
  float gsum = 1.0f;       // ranks summed into g by the last all-reduce (1/gsum = the mean's factor)
  bf16* g16 = nullptr;     // bf16 wire copy of g (grad_comm_bf16 with world_size > 1)
  int add(const std::string& name, std::vector<int> shape, bool conv4d, bool sn) {
    PEntry e;
    e.name = name;
    e.shape = shape;
    e.conv4d = conv4d;
    e.sn = sn;
    e.n = 1;
    for (int s : shape) e.n *= s;
    e.coff = nc;
    nc += e.n;
    e.off = (n + 3) & ~3LL;   // 16-byte aligned tensors: float4 / 8 x bf16 vector paths everywhere
    n = (e.off + e.n + 3) & ~3LL;
    E.push_back(e);
    return (int)E.size() - 1;
  }
  float* P(int e) const { return p + E[e].off; }
  float* G(int e) const { return g + E[e].off; }
};

struct ConvL {
  int w = -1, b = -1;              // entries (b = -1: no bias)
  int cin = 0, cin_x = 0, cout = 0, ksz = 3;
  void* wp = nullptr;              // fprop operand [cout][taps][cin_x]
  void* wt = nullptr;              // dgrad operand [cin_x][taps][cout]
  void* wp4 = nullptr;             // sub-pixel fprop operand [4 phases][cout][4 taps][cin] (G conv1, BF16)
  void* wt4 = nullptr;             // sub-pixel dgrad operand [cin][4 phases x 4 taps][cout]
  bool f32 = false;                // SIMT fp32 layer (G output conv)
};
struct LinL {
  int w = -1, b = -1;
  int in = 0, out = 0;
  float* what = nullptr;           // W / sigma (fp32) [out][in]
};
struct AttnL {
  int C = 0, C8 = 0, C2 = 0, Cq = 0, Ct = 0, H = 0;
  int th = -1, ph = -1, gg = -1, o = -1, gamma = -1;
  void* qkv_wp = nullptr;          // [Ct][1][C]
  void* qkv_wt = nullptr;          // [C][1][Ct]
  ConvL oc;                        // o-conv (C2 -> C), no bias
  // activations
  void *qkv, *phi_p, *g_p, *P, *ov;
  float* S;
  // fused tcgen05 path (BF16, tc_attn_ok): S / P never materialised
  bool fused = false;
  void* gT = nullptr;              // pooled g transposed [n][C2][Q]
  float *o32 = nullptr, *lse = nullptr, *Dr = nullptr;
  float* phimax = nullptr;         // [n] max_j |phi_j| (enables the single-pass fused forward)
  float* thetamax = nullptr;       // [n] max_i |theta_i| (with phimax: the flat schedule)
};
struct GBlock {
  int cin, cout, hin;
  LinL g1, b1, g2, b2;
  ConvL c1, c2, sc;
  bool attn = false;
  // activations (batch B)
  void *x, *u1, *h1, *a2, *s, *out;
  void* u1lo = nullptr;            // CBN1-ReLU output before the upsample (sub-pixel conv1 input)
  float *gain1, *bias1, *gain2, *bias2, *cond, *dcond;
  float* dcond_part;   // [slices][B][cond_dim] split-K partials of dcond
  int dcond_nslot;
  float *ab1 = nullptr, *ab2 = nullptr;   // CBN backward per-sample [dbias | dgain] rows [B][2C]
  float *mean1, *rstd1, *mean2, *rstd2;
  double *sums1, *sums2;
};
struct DBlock {
  int cin, cin_x, cout, hin, hout;
  bool down, learn_sc, attn;
  bool im2col = false;   // first layer as a K = 27 (-> 32) GEMM over an im2col of the image
  ConvL c1, c2, sc, c1x;
  void *x, *rx, *c1o, *r1, *t, *xp, *s, *out, *xi;
  void* wp4dg = nullptr;   // conv2's input-gradient kernel folded into the four phases (pooled blocks)
  void* wp4f = nullptr;    // conv2 + 2x2 pool as a 16-tap stride-2 conv, phase-major (R38; pooled blocks)
  bool dg_phase = false;   // conv2's input gradient through wp4dg (R37); else wp4dg is only the fold's scratch
};

int round8(int x) { return (x + 7) / 8 * 8; }
int round_up(int x, int m) { return (x + m - 1) / m * m; }

struct Arch {
  std::vector<int> gin, gout;
  std::vector<int> din, dout, ddown;   // din[0] = -1 -> RGB
};
bool arch_for(int res, Arch& a) {
  switch (res) {
    case 16: a.gin = {4, 4}; a.gout = {4, 4}; a.din = {-1, 4, 4}; a.dout = {4, 4, 4}; a.ddown = {1, 1, 0}; return true;
    case 32:
      a.gin = {4, 4, 4}; a.gout = {4, 4, 4}; a.din = {-1, 4, 4, 4}; a.dout = {4, 4, 4, 4}; a.ddown = {1, 1, 0, 0};
      return true;
    case 64:
      a.gin = {16, 16, 8, 4}; a.gout = {16, 8, 4, 2}; a.din = {-1, 1, 2, 4, 8}; a.dout = {1, 2, 4, 8, 16};
      a.ddown = {1, 1, 1, 1, 0};
      return true;
    case 128:
      a.gin = {16, 16, 8, 4, 2}; a.gout = {16, 8, 4, 2, 1}; a.din = {-1, 1, 2, 4, 8, 16};
      a.dout = {1, 2, 4, 8, 16, 16}; a.ddown = {1, 1, 1, 1, 1, 0};
      return true;
    case 256:
      a.gin = {16, 16, 8, 8, 4, 2}; a.gout = {16, 8, 8, 4, 2, 1}; a.din = {-1, 1, 2, 4, 8, 8, 16};
      a.dout = {1, 2, 4, 8, 8, 16, 16}; a.ddown = {1, 1, 1, 1, 1, 1, 0};
      return true;
    case 512:
      a.gin = {16, 16, 8, 8, 4, 2, 1}; a.gout = {16, 8, 8, 4, 2, 1, 1}; a.din = {-1, 1, 1, 2, 4, 8, 8, 16};
      a.dout = {1, 1, 2, 4, 8, 8, 16, 16}; a.ddown = {1, 1, 1, 1, 1, 1, 1, 0};
      return true;
  }
  return false;
}

}  // namespace

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e_ = (x);                                       \
    ++launches_;                                                \
    if (e_ != cudaSuccess) return fail_cuda(e_, #x);            \
  } while (0)
#define CKS(x)                                                  \
  do {                                                          \
    paragan_status s_ = (x);                                    \
    if (s_ != PARAGAN_OK) return s_;                            \
  } while (0)


// ============================================================================
template <typename T>
class Engine final : public EngineBase {
  static constexpr bool kBF = std::is_same<T, bf16>::value;

 public:
  Engine(const paragan_config& c, cudaStream_t st) : cfg_(c), st_(st) {
    const char* as = std::getenv("PARAGAN_ATTN_SINGLE");
    attn_single_ = as == nullptr || std::atoi(as) != 0;
    const char* pf = std::getenv("PARAGAN_POOL_FUSE");
    pool_fuse_ = pf == nullptr || std::atoi(pf) != 0;
    const char* af = std::getenv("PARAGAN_ATTN_FLAT");
    attn_flat_ = af == nullptr || std::atoi(af) != 0;
    const char* sp = std::getenv("PARAGAN_SUBPIXEL");
    subpix_ = kBF && (sp == nullptr || std::atoi(sp) != 0);
    const char* dgp = std::getenv("PARAGAN_DGRAD_UP2");
    dgrad_pool_ = subpix_ && (dgp == nullptr || std::atoi(dgp) != 0);
    const char* pfw = std::getenv("PARAGAN_POOL_FWD");
    pool_fwd_ = dgrad_pool_ && (pfw == nullptr || std::atoi(pfw) != 0);
    const char* pf0 = std::getenv("PARAGAN_POOL_FWD0");
    pool_fwd0_ = pool_fwd_ && (pf0 == nullptr || std::atoi(pf0) != 0);
    const char* gr = std::getenv("PARAGAN_GRAPHS");
    graphs_on_ = gr == nullptr || std::atoi(gr) != 0;
    const char* tt = std::getenv("PARAGAN_THIN_TC");
    thin_tc_ = kBF && (tt == nullptr || std::atoi(tt) != 0);
    dcgan_ = c.arch == PARAGAN_ARCH_SNDCGAN;
  }
  ~Engine() override {
    for (auto& g : graphs_)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (ck_thread_.joinable()) ck_thread_.join();
    if (ck_dev_) cudaFree(ck_dev_);
    if (ck_host_) cudaFreeHost(ck_host_);
    if (ck_stream_) cudaStreamDestroy(ck_stream_);
    if (ck_ev_snap_) cudaEventDestroy(ck_ev_snap_);
    if (ck_ev_done_) cudaEventDestroy(ck_ev_done_);
    if (dfake_keep_) cudaFree(dfake_keep_);
    if (pending_d_) cudaStreamSynchronize(cs_);
    if (gcomm_) ncclCommDestroy(gcomm_);
    if (bncomm_) ncclCommDestroy(bncomm_);
    if (cs_) cudaStreamDestroy(cs_);
    if (ev_grad_) cudaEventDestroy(ev_grad_);
    if (ev_ar_) cudaEventDestroy(ev_ar_);
    if (comm_) ncclCommDestroy(comm_);
  }

  // ------------------------------------------------------------------ plan
  size_t workspace_bytes() override {
    Arena a;
    build(a);
    return a.off + 4096;
  }
  void counts(paragan_net net, size_t* ns, size_t* nt) override {
    if (!planned_) {
      Arena a;
      build(a);
    }
    const Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (ns) *ns = (size_t)(N.nc + N.nu);
    if (nt) *nt = (size_t)N.nc;
  }

  paragan_status init(const uint8_t* id, void* ws, size_t ws_bytes) override {
    const size_t need = workspace_bytes();
    if (ws_bytes < need) {
      err_ = "workspace too small: need " + std::to_string(need);
      return PARAGAN_ERR_OOM;
    }
    if (((uintptr_t)ws) & 255) return fail_arg("workspace must be 256-byte aligned");
    Arena a;
    a.base = static_cast<char*>(ws);
    build(a);
    if (cudaMemsetAsync(ws, 0, a.off, st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "memset ws");
    paragan_status s = upload_tables();
    if (s != PARAGAN_OK) return s;
    if (fill_const(ones_buf_, maxc_, 1.0f, st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "ones");
    if (quarter_ && fill_const(quarter_, 1, 0.25f, st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "quarter");
    if (cfg_.world_size > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof(uid));
      ncclResult_t r = ncclCommInitRank(&comm_, cfg_.world_size, uid, cfg_.rank);
      if (r != ncclSuccess) return fail_msg(PARAGAN_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      // A12 overlap: D's gradient all-reduce runs on its own stream and communicator (at most
      // kOverlapCTAs CTAs) while G's forward runs with kOverlapSMs SMs left free; the batch-norm / loss
      // all-reduces get a 2-CTA communicator so the two never compete for more SMs than are reserved
      // (default: off when the CUDA-graph step cache is on — measured at 2 GPUs, graphs without the overlap
      // 5,257-5,270 img/s vs the overlap without graphs 5,217-5,229; PARAGAN_OVERLAP=1 forces it)
      const char* ov = std::getenv("PARAGAN_OVERLAP");
      overlap_ = (ov == nullptr ? !graphs_on_ : std::atoi(ov) != 0) && !cfg_.grad_comm_bf16;
      if (const char* e = std::getenv("PARAGAN_OVERLAP_SMS")) overlap_sms_ = std::atoi(e);
      if (const char* e = std::getenv("PARAGAN_OVERLAP_BLOCKS")) overlap_blocks_ = std::atoi(e);
      if (overlap_) {
        ncclConfig_t gc = NCCL_CONFIG_INITIALIZER, bc = NCCL_CONFIG_INITIALIZER;
        gc.maxCTAs = kOverlapCTAs;
        bc.maxCTAs = 2;
        r = ncclCommSplit(comm_, 0, cfg_.rank, &gcomm_, &gc);
        if (r == ncclSuccess) r = ncclCommSplit(comm_, 0, cfg_.rank, &bncomm_, &bc);
        if (r != ncclSuccess) return fail_msg(PARAGAN_ERR_NCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(r));
        if (cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_grad_, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_ar_, cudaEventDisableTiming) != cudaSuccess)
          return fail_cuda(cudaGetLastError(), "overlap stream");
      }
    }
    if (cudaStreamSynchronize(st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "init sync");
    ready_ = true;
    return PARAGAN_OK;
  }

  // ------------------------------------------------------------------ params
  paragan_status init_params(float attn_gamma) override {
    if (!ready_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    uint64_t salt = 0;
    for (Net* N : {&G_, &D_}) {
      ++salt;
      for (auto& e : N->E) {
        float* p = N->P((int)(&e - N->E.data()));
        const std::string& nm = e.name;
        auto ends = [&](const char* suf) {
          const size_t l = std::strlen(suf);
          return nm.size() >= l && nm.compare(nm.size() - l, l, suf) == 0;
        };
        const bool is_bias = ends(".b") || ends(".beta");
        if (nm.find("gamma") != std::string::npos && nm.find("attn") != std::string::npos) {
          CK(fill_const(p, e.n, attn_gamma, st_));
        } else if (ends(".gamma")) {   // BN gains
          CK(fill_const(p, e.n, 1.0f, st_));
        } else if (is_bias) {
          CK(fill_const(p, e.n, 0.0f, st_));
        } else {
          CK(fill_normal(p, e.n, 0.02f, cfg_.seed * 1000003ull + salt, (uint64_t)e.coff, st_));
        }
        if (e.sn) {
          float* u = N->u + e.u_off;
          CK(fill_normal(u, e.shape[0], 1.0f, cfg_.seed * 7919ull + salt, (uint64_t)(1ull << 40) + e.u_off, st_));
          CK(normalize_vec(u, e.shape[0], st_));
        }
      }
      reset_opt(*N);
    }
    return sync_ok();
  }

  paragan_status set_params(paragan_net net, const float* host, size_t n) override {
    if (!ready_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (!host || n != (size_t)(N.nc + N.nu)) return fail_arg("set_params: size mismatch");
    // canonical -> staging (g buffer, canonical offsets) -> internal (conv OIHW -> OHWI, aligned offsets)
    if (cudaMemcpyAsync(N.g, host, sizeof(float) * N.nc, cudaMemcpyHostToDevice, st_) != cudaSuccess ||
        cudaMemcpyAsync(N.u, host + N.nc, sizeof(float) * N.nu, cudaMemcpyHostToDevice, st_) != cudaSuccess)
      return fail_cuda(cudaGetLastError(), "set_params copy");
    for (size_t i = 0; i < N.E.size(); ++i) {
      const PEntry& e = N.E[i];
      if (e.conv4d) {
        CK(oihw_to_ohwi(N.g + e.coff, N.p + e.off, e.shape[0], e.shape[1], e.shape[2] * e.shape[3], st_));
      } else {
        if (cudaMemcpyAsync(N.p + e.off, N.g + e.coff, sizeof(float) * e.n, cudaMemcpyDeviceToDevice, st_))
          return fail_cuda(cudaGetLastError(), "set_params d2d");
      }
    }
    CK(cudaMemsetAsync(N.g, 0, sizeof(float) * N.n, st_));
    reset_opt(N);
    return sync_ok();
  }
  paragan_status get_params(paragan_net net, float* host, size_t n) override {
    if (!ready_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (!host || n != (size_t)(N.nc + N.nu)) return fail_arg("get_params: size mismatch");
    return export_flat(N, N.p, host, true);
  }
  paragan_status get_grads(paragan_net net, float* host, size_t n) override {
    if (!ready_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (!host || n != (size_t)N.nc) return fail_arg("get_grads: size mismatch");
    return export_flat(N, N.g, host, false, 1.0f / N.gsum);
  }
  paragan_status set_grads(paragan_net net, const float* host, size_t n) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (!host || n != (size_t)N.nc) return fail_arg("set_grads: size mismatch");
    // canonical -> staging -> internal layout (conv OIHW -> OHWI), as set_params
    if (cudaMemcpyAsync(scratch_f_, host, sizeof(float) * N.nc, cudaMemcpyHostToDevice, st_) != cudaSuccess)
      return fail_cuda(cudaGetLastError(), "set_grads copy");
    CK(cudaMemsetAsync(N.g, 0, sizeof(float) * N.n, st_));
    for (const PEntry& e : N.E) {
      if (e.conv4d) CK(oihw_to_ohwi(scratch_f_ + e.coff, N.g + e.off, e.shape[0], e.shape[1], e.shape[2] * e.shape[3], st_));
      else CK(cudaMemcpyAsync(N.g + e.off, scratch_f_ + e.coff, sizeof(float) * e.n, cudaMemcpyDeviceToDevice, st_));
    }
    N.gsum = 1.0f;
    return sync_ok();
  }
  paragan_status get_fakes(float* host, size_t n) override {
    if (!ready_) return PARAGAN_ERR_ORDER;
    const size_t need = (size_t)B_ * 3 * R_ * R_;
    if (!host || n != need) return fail_arg("get_fakes: size mismatch");
    CK(layout_unpack<T>(static_cast<const T*>(dimg_), scratch_f_, B_, 3, R_, R_, cpad_, st_));
    if (cudaMemcpyAsync(host, scratch_f_, need * sizeof(float), cudaMemcpyDeviceToHost, st_))
      return fail_cuda(cudaGetLastError(), "get_fakes");
    return sync_ok();
  }

  paragan_status get_dfake(float* host, size_t n) override {
    if (!ready_ || !dfake_valid_) return PARAGAN_ERR_ORDER;
    const size_t need = (size_t)B_ * 3 * R_ * R_;
    if (!host || n != need) return fail_arg("get_dfake: size mismatch");
    if (cudaMemcpyAsync(host, dfake_keep_, need * sizeof(float), cudaMemcpyDeviceToHost, st_))
      return fail_cuda(cudaGetLastError(), "get_dfake");
    return sync_ok();
  }
  // test hook (PARAGAN_FLAG_KEEP_DFAKE): keep dL_G/d(fake) before G's backward reuses the buffers
  paragan_status keep_dfake() {
    const size_t need = (size_t)B_ * 3 * R_ * R_;
    if (!dfake_keep_ && cudaMalloc(&dfake_keep_, need * sizeof(float)) != cudaSuccess)
      return fail_cuda(cudaGetLastError(), "keep_dfake alloc");
    CK(layout_unpack<T>(static_cast<const T*>(dimg_grad_), dfake_keep_, B_, 3, R_, R_, cpad_, st_));
    dfake_valid_ = true;
    return PARAGAN_OK;
  }

  // ------------------------------------------------------------------ asynchronous checkpoint writer
  // (P:233).  Payload: per net (D then G) p[n], u[nu], m[n], v[n], slow[n] (Lookahead only), then the two
  // int64 step counters; internal (16-byte aligned) layout, so only a context of the same config reads it.
  struct CkHeader {
    char magic[8];
    int32_t abi, arch, resolution, ch, n_classes, shared_dim, z_chunk, attn_res, compute, la_d, la_g, pad;
    int64_t nD, nuD, nG, nuG, payload_bytes;
    uint64_t hash;
  };
  CkHeader ck_header() const {
    CkHeader h{};
    std::memcpy(h.magic, "PGCKPT01", 8);
    h.abi = PARAGAN_ABI_VERSION;
    h.arch = cfg_.arch;
    h.resolution = cfg_.resolution;
    h.ch = cfg_.ch;
    h.n_classes = cfg_.n_classes;
    h.shared_dim = cfg_.shared_dim;
    h.z_chunk = cfg_.z_chunk;
    h.attn_res = cfg_.attn_res;
    h.compute = cfg_.compute;
    h.la_d = D_.slow != nullptr;
    h.la_g = G_.slow != nullptr;
    h.nD = D_.n;
    h.nuD = D_.nu;
    h.nG = G_.n;
    h.nuG = G_.nu;
    h.payload_bytes = (int64_t)ck_bytes();
    return h;
  }
  size_t ck_bytes() const {
    size_t f = 0;
    for (const Net* N : {&D_, &G_}) f += (size_t)(3 * N->n + N->nu + (N->slow ? N->n : 0));
    return f * sizeof(float) + 2 * sizeof(long long);
  }
  // visits the payload sections in order: fn(device pointer, bytes)
  template <class F>
  void ck_sections(F&& fn) {
    for (Net* N : {&D_, &G_}) {
      fn((void*)N->p, sizeof(float) * N->n);
      fn((void*)N->u, sizeof(float) * N->nu);
      fn((void*)N->m, sizeof(float) * N->n);
      fn((void*)N->v, sizeof(float) * N->n);
      if (N->slow) fn((void*)N->slow, sizeof(float) * N->n);
    }
    fn((void*)D_.t_dev, sizeof(long long));
    fn((void*)G_.t_dev, sizeof(long long));
  }
  paragan_status checkpoint_save_async(const char* path) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    if (!path) return fail_arg("checkpoint: null path");
    paragan_status ws = checkpoint_wait();
    if (ws != PARAGAN_OK) return ws;
    const size_t bytes = ck_bytes();
    if (!ck_dev_) {
      if (cudaMalloc(&ck_dev_, bytes) != cudaSuccess || cudaMallocHost(&ck_host_, bytes) != cudaSuccess ||
          cudaStreamCreateWithFlags(&ck_stream_, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ck_ev_snap_, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ck_ev_done_, cudaEventDisableTiming) != cudaSuccess)
        return fail_cuda(cudaGetLastError(), "checkpoint buffers");
    }
    // 1) stream-ordered snapshot on the compute stream (the next update cannot race it)
    size_t off = 0;
    cudaError_t e = cudaSuccess;
    ck_sections([&](void* src, size_t b) {
      if (e == cudaSuccess) e = cudaMemcpyAsync(static_cast<char*>(ck_dev_) + off, src, b, cudaMemcpyDeviceToDevice, st_);
      off += b;
    });
    if (e != cudaSuccess) return fail_cuda(e, "checkpoint snapshot");
    // 2) device -> pinned host on the copy stream, overlapping the following steps
    if (cudaEventRecord(ck_ev_snap_, st_) || cudaStreamWaitEvent(ck_stream_, ck_ev_snap_, 0) ||
        cudaMemcpyAsync(ck_host_, ck_dev_, bytes, cudaMemcpyDeviceToHost, ck_stream_) ||
        cudaEventRecord(ck_ev_done_, ck_stream_))
      return fail_cuda(cudaGetLastError(), "checkpoint stream");
    // 3) a host thread writes the file once the copy has landed
    CkHeader h = ck_header();
    const std::string p(path);
    const int dev = cfg_.device;
    ck_status_ = PARAGAN_OK;
    ck_thread_ = std::thread([this, h, p, bytes, dev]() mutable {
      cudaSetDevice(dev);
      if (cudaEventSynchronize(ck_ev_done_) != cudaSuccess) {
        ck_status_ = PARAGAN_ERR_CUDA;
        return;
      }
      h.hash = fnv1a64(ck_host_, bytes);
      const std::string tmp = p + ".tmp";
      FILE* f = std::fopen(tmp.c_str(), "wb");
      bool ok = f && std::fwrite(&h, sizeof(h), 1, f) == 1 && std::fwrite(ck_host_, 1, bytes, f) == bytes;
      if (f) ok = (std::fclose(f) == 0) && ok;
      ok = ok && std::rename(tmp.c_str(), p.c_str()) == 0;
      ck_status_ = ok ? PARAGAN_OK : PARAGAN_ERR_IO;
    });
    return PARAGAN_OK;
  }
  paragan_status checkpoint_wait() override {
    if (ck_thread_.joinable()) ck_thread_.join();
    const paragan_status s = ck_status_;
    if (s == PARAGAN_ERR_IO) err_ = "checkpoint: writing the file failed";
    ck_status_ = PARAGAN_OK;
    return s;
  }
  paragan_status checkpoint_load(const char* path) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    if (!path) return fail_arg("checkpoint: null path");
    paragan_status ws = checkpoint_wait();
    if (ws != PARAGAN_OK) return ws;
    FILE* f = std::fopen(path, "rb");
    if (!f) {
      err_ = std::string("checkpoint: cannot open ") + path;
      return PARAGAN_ERR_IO;
    }
    CkHeader h{}, want = ck_header();
    std::vector<char> buf;
    bool ok = std::fread(&h, sizeof(h), 1, f) == 1;
    if (ok) {
      want.hash = h.hash;
      if (std::memcmp(&h, &want, sizeof(h)) != 0) {
        std::fclose(f);
        err_ = "checkpoint: configuration / layout mismatch";
        return PARAGAN_ERR_CONFIG;
      }
      buf.resize((size_t)h.payload_bytes);
      ok = std::fread(buf.data(), 1, buf.size(), f) == buf.size();
    }
    std::fclose(f);
    if (!ok || fnv1a64(buf.data(), buf.size()) != h.hash) {
      err_ = "checkpoint: short or corrupt file";
      return PARAGAN_ERR_IO;
    }
    size_t off = 0;
    cudaError_t e = cudaSuccess;
    ck_sections([&](void* dst, size_t b) {
      if (e == cudaSuccess) e = cudaMemcpyAsync(dst, buf.data() + off, b, cudaMemcpyHostToDevice, st_);
      off += b;
    });
    if (e != cudaSuccess) return fail_cuda(e, "checkpoint restore");
    return sync_ok();   // buf is released after the copies completed
  }

  // ------------------------------------------------------------------ steps
  paragan_status d_step(const void* real, const int32_t* real_y, const float* z, const int32_t* fake_y,
                        uint32_t flags) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    if (!real || !real_y || !z || !fake_y || ((uintptr_t)real & 15)) return fail_arg("d_step: bad pointer");
    return run_graphed(GraphKey{0, flags, {real, real_y, z, fake_y}}, [&]() -> paragan_status {
      // SN(G) + G forward (no grad) writes fakes into D-input rows [0, B)
      CKS(sn_forward(G_, false));
      CKS(fold_subpixel(false));
      if (dcgan_) CKS(g_forward_dc(z));
      else CKS(g_forward(z, fake_y, false));
      return d_step_body(real, real_y, fake_y, flags);
    });
  }

  // ------------------------------------------------------------------ CUDA-graph step cache
  // A D or G step issues ~250 launches.  Each distinct (step kind, flags, input pointers) is captured once into
  // a CUDA graph (NCCL collectives included at world_size > 1) and replayed afterwards: the step's device state (weights,
  // u vectors, optimiser moments, the step counter t) lives on the device, so a replay is the same computation as
  // the eager call; the host-side bookkeeping of the step is re-applied by hand.  Disabled while profiling, with
  // the overlapped D all-reduce (it spans two steps) and with PARAGAN_GRAPHS=0.  A capture that fails falls back
  // to eager execution for good.
  struct GraphKey {
    int kind;
    uint32_t flags;
    const void* p[4];
    bool operator==(const GraphKey& o) const {
      return kind == o.kind && flags == o.flags && p[0] == o.p[0] && p[1] == o.p[1] && p[2] == o.p[2] && p[3] == o.p[3];
    }
  };
  struct HostState {   // what a step changes on the host
    int d_since_g;
    bool dfake_valid;
    float dgsum, ggsum;
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
    HostState after{};
  };
  HostState host_state() const { return HostState{d_since_g_, dfake_valid_, D_.gsum, G_.gsum}; }
  void set_host_state(const HostState& h) {
    d_since_g_ = h.d_since_g;
    dfake_valid_ = h.dfake_valid;
    D_.gsum = h.dgsum;
    G_.gsum = h.ggsum;
  }
  static constexpr size_t kMaxGraphs = 16;
  template <class F>
  paragan_status run_graphed(const GraphKey& k, F&& body) {
    if (!graphs_on_ || prof_ || pending_d_ || overlap_) return body();
    for (auto& g : graphs_) {
      if (g.key == k) {
        // a D step's host effect depends on the count before it (++), a G step's does not (= 0)
        HostState h = g.after;
        if (k.kind == 0) h.d_since_g = d_since_g_ + 1;
        if (cudaGraphLaunch(g.exec, st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "graph launch");
        set_host_state(h);
        launches_ += g.launches;
        return PARAGAN_OK;
      }
    }
    if (graphs_.size() >= kMaxGraphs) return body();
    const HostState before = host_state();
    const uint64_t l0 = launches_;
    if (cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      graphs_on_ = false;
      return body();
    }
    const paragan_status s = body();
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(st_, &graph);
    cudaGraphExec_t exec = nullptr;
    if (s == PARAGAN_OK && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (s != PARAGAN_OK || e != cudaSuccess) {   // nothing ran: undo the host effects, run eagerly from now on
      cudaGetLastError();
      if (exec) cudaGraphExecDestroy(exec);
      graphs_on_ = false;
      set_host_state(before);
      launches_ = l0;
      if (s != PARAGAN_OK) poisoned_ = false, err_.clear();
      return body();
    }
    GraphEntry g;
    g.key = k;
    g.exec = exec;
    g.launches = launches_ - l0;
    g.after = host_state();
    graphs_.push_back(g);
    if (cudaGraphLaunch(exec, st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "graph launch");
    return PARAGAN_OK;
  }
  // asynchronous scheme: D on an img_buff entry instead of a fresh G forward
  paragan_status d_step_fakes(const void* real, const int32_t* real_y, const void* fakes, const int32_t* fake_y,
                              uint32_t flags) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    if (!real || !real_y || !fakes || !fake_y || ((uintptr_t)real & 15) || ((uintptr_t)fakes & 15))
      return fail_arg("d_step_fakes: bad pointer");
    const size_t img_bytes = (size_t)B_ * R_ * R_ * cpad_ * sizeof(T);
    if (cudaMemcpyAsync(dimg_, fakes, img_bytes, cudaMemcpyDeviceToDevice, st_))
      return fail_cuda(cudaGetLastError(), "copy fakes");
    return d_step_body(real, real_y, fake_y, flags);
  }
  paragan_status generate(const float* z, const int32_t* y, void* dst) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    if (!z || !y) return fail_arg("generate: bad pointer");
    CKS(sn_forward(G_, false));
    CKS(fold_subpixel(false));
    if (dcgan_) CKS(g_forward_dc(z));
    else CKS(g_forward(z, y, false));
    return export_fakes(dst);
  }
  paragan_status export_fakes(void* dst) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    const size_t img_bytes = (size_t)B_ * R_ * R_ * cpad_ * sizeof(T);
    if (cudaMemcpyAsync(dst, dimg_, img_bytes, cudaMemcpyDeviceToDevice, st_))
      return fail_cuda(cudaGetLastError(), "export fakes");
    return PARAGAN_OK;
  }
  size_t state_floats(paragan_net net) override {
    const Net& N = net == PARAGAN_NET_D ? D_ : G_;
    return (size_t)(N.n + N.nu);
  }
  paragan_status export_state(paragan_net net, float* dst) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (cudaMemcpyAsync(dst, N.p, sizeof(float) * N.n, cudaMemcpyDeviceToDevice, st_) ||
        cudaMemcpyAsync(dst + N.n, N.u, sizeof(float) * N.nu, cudaMemcpyDeviceToDevice, st_))
      return fail_cuda(cudaGetLastError(), "export_state");
    return PARAGAN_OK;
  }
  paragan_status import_state(paragan_net net, const float* src) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (cudaMemcpyAsync(N.p, src, sizeof(float) * N.n, cudaMemcpyDeviceToDevice, st_) ||
        cudaMemcpyAsync(N.u, src + N.n, sizeof(float) * N.nu, cudaMemcpyDeviceToDevice, st_))
      return fail_cuda(cudaGetLastError(), "import_state");
    return PARAGAN_OK;
  }
  // D's deferred update: wait for the overlapped all-reduce, then the optimiser step (before D is read again)
  paragan_status flush_d() {
    g_sm_cap = kNumSMs;
    if (!pending_d_) return PARAGAN_OK;
    pending_d_ = false;
    if (cudaStreamWaitEvent(st_, ev_ar_, 0) != cudaSuccess) return fail_cuda(cudaGetLastError(), "overlap wait");
    return update_net(PARAGAN_NET_D);
  }
  paragan_status d_step_body(const void* real, const int32_t* real_y, const int32_t* fake_y, uint32_t flags) {
    CKS(flush_d());
    // reals into rows [B, 2B) (one D pass over the concatenated batch)
    const size_t img_bytes = (size_t)B_ * R_ * R_ * cpad_ * sizeof(T);
    if (cudaMemcpyAsync(static_cast<char*>(dimg_) + img_bytes, real, img_bytes, cudaMemcpyDeviceToDevice, st_))
      return fail_cuda(cudaGetLastError(), "copy reals");
    CK(cudaMemcpyAsync(ylab_, fake_y, sizeof(int32_t) * B_, cudaMemcpyDeviceToDevice, st_));
    CK(cudaMemcpyAsync(ylab_ + B_, real_y, sizeof(int32_t) * B_, cudaMemcpyDeviceToDevice, st_));
    CKS(sn_forward(D_, true));
    if (dcgan_) CKS(d_forward_dc(2 * B_));
    else CKS(d_forward(2 * B_));
    CK(hinge_loss(logits_, B_, 0, dlogits_, D_.loss, st_));
    CKS(allreduce_loss(D_.loss));
    CK(cudaMemsetAsync(D_.g, 0, sizeof(float) * D_.n, st_));
    D_.gsum = 1.0f;
    if (dcgan_) CKS(d_backward_dc(2 * B_, true, false));
    else CKS(d_backward(2 * B_, true, false));
    CKS(sn_backward_net(D_));
    if (overlap_ && !(flags & (PARAGAN_FLAG_NO_ALLREDUCE | PARAGAN_FLAG_NO_UPDATE))) {
      // A12: the all-reduce overlaps the next G forward; the update is applied before D is used again
      if (cudaEventRecord(ev_grad_, st_) != cudaSuccess || cudaStreamWaitEvent(cs_, ev_grad_, 0) != cudaSuccess)
        return fail_cuda(cudaGetLastError(), "overlap record");
      const ncclResult_t r = ncclAllReduce(D_.g, D_.g, (size_t)D_.n, ncclFloat32, ncclSum, gcomm_, cs_);
      if (r != ncclSuccess) return fail_msg(PARAGAN_ERR_NCCL, std::string("grad allreduce: ") + ncclGetErrorString(r));
      ++launches_;
      if (cudaEventRecord(ev_ar_, cs_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "overlap record");
      D_.gsum = (float)cfg_.world_size;
      pending_d_ = true;
    } else {
      if (!(flags & PARAGAN_FLAG_NO_ALLREDUCE)) CKS(allreduce(PARAGAN_NET_D));
      if (!(flags & PARAGAN_FLAG_NO_UPDATE)) CKS(update_net(PARAGAN_NET_D));
    }
    ++d_since_g_;
    return PARAGAN_OK;
  }

  paragan_status g_step(const float* z, const int32_t* y, uint32_t flags) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    if (d_since_g_ < cfg_.d_steps_per_g && !(flags & PARAGAN_FLAG_ASYNC)) {
      err_ = "g_step before d_steps_per_g D steps";
      return PARAGAN_ERR_ORDER;
    }
    if (!z || !y) return fail_arg("g_step: bad pointer");
    return run_graphed(GraphKey{1, flags, {z, y, nullptr, nullptr}}, [&]() { return g_step_body(z, y, flags); });
  }
  paragan_status g_step_body(const float* z, const int32_t* y, uint32_t flags) {
    dfake_valid_ = false;
    CKS(sn_forward(G_, true));
    CKS(fold_subpixel(true));
    if (dcgan_) CKS(g_forward_dc(z));
    else CKS(g_forward(z, y, true));
    CK(cudaMemcpyAsync(ylab_, y, sizeof(int32_t) * B_, cudaMemcpyDeviceToDevice, st_));
    CKS(flush_d());   // D's update (its all-reduce overlapped the G forward above)
    CKS(sn_forward(D_, true));
    if (dcgan_) CKS(d_forward_dc(B_));
    else CKS(d_forward(B_));
    CK(hinge_loss(logits_, B_, 1, dlogits_, G_.loss, st_));
    CKS(allreduce_loss(G_.loss));
    CK(cudaMemsetAsync(G_.g, 0, sizeof(float) * G_.n, st_));
    G_.gsum = 1.0f;
    if (dcgan_) {
      CKS(d_backward_dc(B_, false, true));   // dgrad only, down to the image
      if (flags & PARAGAN_FLAG_KEEP_DFAKE) CKS(keep_dfake());
      CKS(g_backward_dc());
    } else {
      CKS(d_backward(B_, false, true));   // dgrad only, down to the image
      if (flags & PARAGAN_FLAG_KEEP_DFAKE) CKS(keep_dfake());
      CKS(g_backward());
    }
    CKS(sn_backward_net(G_));
    if (!(flags & PARAGAN_FLAG_NO_ALLREDUCE)) CKS(allreduce(PARAGAN_NET_G));
    if (!(flags & PARAGAN_FLAG_NO_UPDATE)) CKS(update(PARAGAN_NET_G));
    d_since_g_ = 0;
    return PARAGAN_OK;
  }

  paragan_status allreduce(paragan_net net) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    if (cfg_.world_size > 1 && N.gsum == 1.0f) {
      // sum over ranks; the mean's 1/W (R15) is folded into the update and into get_grads
      if (N.g16) {   // bf16 on the wire: round, sum in bf16, widen back
        CK(convert_f32<bf16>(N.g, N.g16, N.n, st_));
        CKS(nccl_sum(N.g16, (size_t)N.n, ncclBfloat16, "grad allreduce (bf16)"));
        CK(to_f32<bf16>(N.g16, N.g, N.n, st_));
      } else {
        CKS(nccl_sum(N.g, (size_t)N.n, ncclFloat32, "grad allreduce"));
      }
      N.gsum = (float)cfg_.world_size;
    }
    return PARAGAN_OK;
  }

  paragan_status update(paragan_net net) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    return update_net(net);
  }
  paragan_status update_net(paragan_net net) {
    Net& N = net == PARAGAN_NET_D ? D_ : G_;
    const paragan_adam& h = net == PARAGAN_NET_D ? cfg_.adam_d : cfg_.adam_g;
    const float gscale = 1.0f / N.gsum;
    CK(cudaMemsetAsync(N.flag, 0, sizeof(int), st_));
    CK(check_finite_scalar(N.loss, N.flag, st_));
    if (plain_adam(N)) {
      CK(check_finite(N.g, N.n, N.flag, st_));
      CK(adam_flat(N.p, N.g, N.m, N.v, N.n, h.lr, h.beta1, h.beta2, h.eps, N.t_dev, gscale, N.flag, st_));
    } else {
      // asymmetric optimisation policy (NEXT-3)
      const paragan_policy& p = policy(N);
      const int nc = (int)N.chunks_h.size();
      OptRule r{p.rule, p.lars, p.lookahead_k, p.warmup_steps, p.schedule, p.total_steps,
                h.lr, h.beta1, h.beta2, h.eps, p.lars_trust, p.lookahead_alpha, p.clip_norm, gscale};
      const float* cs = nullptr;
      if (p.clip_norm > 0.0f) {   // one pass gives the global norm and the finiteness of g
        CK(opt_sumsq(N.g, N.chunks_d, nc, gscale, N.opt_wpart, st_));
        CK(opt_clip_finalize(N.opt_wpart, nc, p.clip_norm, N.clip_scale, N.flag, st_));
        cs = N.clip_scale;
      } else {
        CK(check_finite(N.g, N.n, N.flag, st_));
      }
      CK(opt_update(N.p, N.g, N.m, N.v, scratch_f_, N.chunks_d, nc, r, N.t_dev, cs, N.flag, N.opt_wpart, N.opt_upart,
                    st_));
      if (p.lars) {
        CK(opt_lars_apply(N.p, scratch_f_, N.chunks_d, nc, r, N.t_dev, N.opt_wpart, N.opt_upart, N.flag, st_));
      }
    }
    CK(adam_bookkeep(N.t_dev, N.flag, nonfinite_sticky_, st_));
    if (N.slow) {
      const paragan_policy& p = policy(N);
      CK(opt_lookahead(N.p, N.slow, N.n, p.lookahead_k, p.lookahead_alpha, N.t_dev, N.flag, st_));
    }
    return PARAGAN_OK;
  }

  // device-side copy of the stats struct (losses scaled by 1/world_size on the device), copied out by
  // stats_async without a host synchronisation
  paragan_status stats_async(paragan_stats* out) override {
    if (!ready_ || poisoned_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    CK(pack_stats(D_.loss, G_.loss, D_.t_dev, G_.t_dev, nonfinite_sticky_, 1.0f / cfg_.world_size, stats_dev_, st_));
    if (cudaMemcpyAsync(out, stats_dev_, sizeof(paragan_stats), cudaMemcpyDeviceToHost, st_) != cudaSuccess)
      return fail_cuda(cudaGetLastError(), "stats_async copy");
    return PARAGAN_OK;
  }
  paragan_status sync_stats(paragan_stats* out) override {
    if (!ready_) return PARAGAN_ERR_ORDER;
    CKS(flush_d());
    float ld[4], lg[4];
    long long td, tg;
    int nf;
    if (cudaMemcpyAsync(ld, D_.loss, sizeof(ld), cudaMemcpyDeviceToHost, st_) ||
        cudaMemcpyAsync(lg, G_.loss, sizeof(lg), cudaMemcpyDeviceToHost, st_) ||
        cudaMemcpyAsync(&td, D_.t_dev, sizeof(td), cudaMemcpyDeviceToHost, st_) ||
        cudaMemcpyAsync(&tg, G_.t_dev, sizeof(tg), cudaMemcpyDeviceToHost, st_) ||
        cudaMemcpyAsync(&nf, nonfinite_sticky_, sizeof(nf), cudaMemcpyDeviceToHost, st_))
      return fail_cuda(cudaGetLastError(), "sync_stats copy");
    paragan_status s = sync_ok();
    if (s != PARAGAN_OK) return s;
    if (out) {
      const float inv = 1.0f / cfg_.world_size;
      out->d_loss = ld[0] * inv;
      out->d_real_mean = ld[1] * inv;
      out->d_fake_mean = ld[2] * inv;
      out->g_loss = lg[0] * inv;
      out->nonfinite = nf;
      out->t_d = td;
      out->t_g = tg;
    }
    if (nf) {
      cudaMemsetAsync(nonfinite_sticky_, 0, sizeof(int), st_);
      return PARAGAN_ERR_NONFINITE;
    }
    return PARAGAN_OK;
  }
  uint64_t launches() const override { return launches_; }

  // ---------------------------------------------------------------- live kernel timing (bench roofline)
  paragan_status profile(int enable) override {
    if (enable) {
      for (auto& r : recs_) { ev_free_.push_back(r.a); ev_free_.push_back(r.b); }
      recs_.clear();
    }
    prof_ = enable != 0;
    return PARAGAN_OK;
  }
  paragan_status profile_read(int kind, uint64_t* n, double* ms, double* flops) override {
    if (cudaStreamSynchronize(st_) != cudaSuccess) return fail_cuda(cudaGetLastError(), "profile sync");
    uint64_t c = 0;
    double t = 0, f = 0;
    const bool verbose = std::getenv("PARAGAN_PROFILE_VERBOSE") != nullptr;
    // kinds 3 / 4: the launches of kinds 0 / 1 with their executed instead of algorithmic flops
    const int k = (kind == 3 || kind == 4) ? kind - 3 : kind;
    for (auto& r : recs_) {
      if (r.kind != k) continue;
      float e = 0;
      if (cudaEventElapsedTime(&e, r.a, r.b) != cudaSuccess) return fail_cuda(cudaGetLastError(), "event time");
      ++c;
      t += e;
      f += (kind == 3 || kind == 4) ? r.exec_flops : r.flops;
      if (verbose)
        std::fprintf(stderr, "PROF kind=%d ms=%.4f tflops=%.1f exec_tflops=%.1f %s\n", k, e, r.flops / (e * 1e9),
                     r.exec_flops / (e * 1e9), r.what);
    }
    if (n) *n = c;
    if (ms) *ms = t;
    if (flops) *flops = f;
    return PARAGAN_OK;
  }

 private:
  // ================================================================== helpers
  paragan_status fail_cuda(cudaError_t e, const char* what) {
    err_ = std::string(what) + ": " + cudaGetErrorString(e);
    poisoned_ = true;
    return PARAGAN_ERR_CUDA;
  }
  paragan_status fail_msg(paragan_status s, const std::string& m) {
    err_ = m;
    if (s == PARAGAN_ERR_CUDA || s == PARAGAN_ERR_NCCL) poisoned_ = true;
    return s;
  }
  paragan_status fail_arg(const std::string& m) {
    err_ = m;
    return PARAGAN_ERR_INVALID_ARG;
  }
  paragan_status sync_ok() {
    cudaError_t e = cudaStreamSynchronize(st_);
    if (e != cudaSuccess) return fail_cuda(e, "stream sync");
    return PARAGAN_OK;
  }
  void reset_opt(Net& N) {
    cudaMemsetAsync(N.m, 0, sizeof(float) * N.n, st_);
    cudaMemsetAsync(N.v, 0, sizeof(float) * N.n, st_);
    cudaMemsetAsync(N.t_dev, 0, sizeof(long long), st_);
    if (N.slow) cudaMemcpyAsync(N.slow, N.p, sizeof(float) * N.n, cudaMemcpyDeviceToDevice, st_);   // phi_0 = w_0
  }
  paragan_status export_flat(Net& N, const float* src, float* host, bool with_u, float scale = 1.0f) {
    float* stage = scratch_f_;
    for (const PEntry& e : N.E) {
      if (e.conv4d) {
        CK(ohwi_to_oihw(src + e.off, stage + e.coff, e.shape[0], e.shape[1], e.shape[2] * e.shape[3], st_));
      } else {
        CK(cudaMemcpyAsync(stage + e.coff, src + e.off, sizeof(float) * e.n, cudaMemcpyDeviceToDevice, st_));
      }
    }
    if (scale != 1.0f) CK(scale_f32(stage, N.nc, scale, st_));   // sum over ranks -> mean (R15)
    if (cudaMemcpyAsync(host, stage, sizeof(float) * N.nc, cudaMemcpyDeviceToHost, st_))
      return fail_cuda(cudaGetLastError(), "export copy");
    if (with_u && cudaMemcpyAsync(host + N.nc, N.u, sizeof(float) * N.nu, cudaMemcpyDeviceToHost, st_))
      return fail_cuda(cudaGetLastError(), "export u");
    return sync_ok();
  }

  // ------------------------------------------------------------------ building the plan
  ConvL conv(Net& N, const std::string& nm, int cin, int cin_x, int cout, int ksz, bool bias, bool f32 = false) {
    ConvL c;
    c.cin = cin;
    c.cin_x = cin_x;
    c.cout = cout;
    c.ksz = ksz;
    c.f32 = f32;
    c.w = N.add(nm + ".w", {cout, cin, ksz, ksz}, true, true);
    if (bias) c.b = N.add(nm + ".b", {cout}, false, false);
    return c;
  }
  LinL lin(Net& N, const std::string& nm, int in, int out, bool bias, bool sn, bool wsuffix = true) {
    LinL l;
    l.in = in;
    l.out = out;
    l.w = N.add(wsuffix ? nm + ".w" : nm, {out, in}, false, sn);
    if (bias) l.b = N.add(nm + ".b", {out}, false, false);
    return l;
  }
  AttnL attn(Net& N, int C, int H) {
    AttnL a;
    a.C = C;
    a.H = H;
    a.C8 = C / 8;
    a.C2 = C / 2;
    a.Cq = round_up(a.C8, 16);   // K steps of the tensor-core MMA are 16 wide
    a.Ct = 2 * a.Cq + round8(a.C2);
    a.th = N.add("attn.theta", {a.C8, C, 1, 1}, true, true);
    a.ph = N.add("attn.phi", {a.C8, C, 1, 1}, true, true);
    a.gg = N.add("attn.g", {a.C2, C, 1, 1}, true, true);
    a.oc.w = N.add("attn.o", {C, a.C2, 1, 1}, true, true);
    a.oc.cin = a.C2;
    a.oc.cin_x = a.C2;
    a.oc.cout = C;
    a.oc.ksz = 1;
    a.o = a.oc.w;
    a.gamma = N.add("attn.gamma", {1}, false, false);
    return a;
  }

  // SN bookkeeping (u / v offsets, job ids) and the flat parameter / optimiser buffers of both nets
  void finalize_nets(Arena& A) {
    // u / v offsets
    for (Net* N : {&G_, &D_}) {
      N->nu = 0;
      N->nv = 0;
      N->sn_entries.clear();
      for (auto& e : N->E)
        if (e.sn) {
          e.u_off = N->nu;
          N->nu += e.shape[0];
          e.v_off = N->nv;
          N->nv += ((e.n / e.shape[0]) + 3) & ~3LL;   // 16-byte aligned v / t slices (float4 passes)
          e.job = (int)N->sn_entries.size();
          N->sn_entries.push_back((int)(&e - N->E.data()));
        }
    }
    // ---------------- device memory
    for (Net* N : {&G_, &D_}) {
      N->p = A.get<float>(N->n);
      N->g = A.get<float>(N->n);
      N->m = A.get<float>(N->n);
      N->v = A.get<float>(N->n);
      N->u = A.get<float>(N->nu);
      N->sn_s = A.get<float>(N->nu);
      N->sn_v = A.get<float>(N->nv);
      N->sn_t = A.get<float>(N->nv);
      N->sigma = A.get<float>(2 * N->sn_entries.size());
      N->t_dev = A.get<long long>(1);
      N->flag = A.get<int>(1);
      N->loss = A.get<float>(4);
    }
    nonfinite_sticky_ = A.get<int>(1);
  }
  const paragan_policy& policy(const Net& N) const { return &N == &D_ ? cfg_.policy_d : cfg_.policy_g; }
  bool plain_adam(const Net& N) const {
    const paragan_policy& p = policy(N);
    return p.rule == PARAGAN_OPT_ADAM && !p.lars && p.lookahead_k == 0 && p.warmup_steps == 0 &&
           (p.schedule == PARAGAN_SCHED_CONSTANT || p.total_steps == 0) && p.clip_norm == 0.0f;
  }
  // chunk table of the optimiser kernels: every parameter tensor split into kOptChunk pieces
  void alloc_opt_tables(Arena& A) {
    for (Net* N : {&G_, &D_}) {
      N->chunks_h.clear();
      for (const PEntry& e : N->E) {
        const int first = (int)N->chunks_h.size(), cnt = ceil_div(e.n, kOptChunk);
        for (int c = 0; c < cnt; ++c) {
          const long long a = (long long)c * kOptChunk;
          N->chunks_h.push_back(OptChunk{e.off + a, (int)std::min<long long>(kOptChunk, e.n - a), first, cnt});
        }
      }
      const size_t nc = N->chunks_h.size();
      N->chunks_d = A.get<OptChunk>(nc);
      N->opt_wpart = A.get<double>(nc);
      N->opt_upart = A.get<double>(nc);
      N->clip_scale = A.get<float>(1);
      N->slow = policy(*N).lookahead_k > 0 ? A.get<float>(N->n) : nullptr;
      N->g16 = (cfg_.grad_comm_bf16 && cfg_.world_size > 1) ? A.get<bf16>(N->n) : nullptr;
    }
  }
  paragan_status upload_opt_tables() {
    for (Net* N : {&G_, &D_})
      CK(cudaMemcpyAsync(N->chunks_d, N->chunks_h.data(), N->chunks_h.size() * sizeof(OptChunk),
                         cudaMemcpyHostToDevice, st_));
    return PARAGAN_OK;
  }
  // device tables of the grouped SN power iteration / backward and the SN pack lists
  void alloc_sn_tables(Arena& A) {
    // tables
    for (Net* N : {&G_, &D_}) {
      N->jobs_d = A.get<SnJob>(N->sn_entries.size());
      long long nb1 = 0, nb1b = 0, nb2 = 0, npart = 0, nbw = 0;
      for (int ei : N->sn_entries) {
        const PEntry& e = N->E[ei];
        const long long K = e.n / e.shape[0];
        const int nrc = ceil_div(e.shape[0], 128);
        nb1 += ceil_div(K, sn_cols_per_block(K)) * nrc;
        nb1b += ceil_div(K, sn_cols_per_block(K));
        nb2 += ceil_div(e.shape[0], 8);
        npart += ((long long)nrc * K + 3) & ~3LL;
        nbw += ceil_div(e.n, 4096);
      }
      N->nb1 = (int)nb1;
      N->nb1b = (int)nb1b;
      N->nb2 = (int)nb2;
      N->npart = npart;
      N->snb_blocks = nbw;
      N->b1_job = A.get<int>(nb1);
      N->b1_k0 = A.get<int>(nb1);
      N->b1_rc = A.get<int>(nb1);
      N->b1b_job = A.get<int>(nb1b);
      N->b1b_k0 = A.get<int>(nb1b);
      N->b2_job = A.get<int>(nb2);
      N->b2_r0 = A.get<int>(nb2);
      N->sn_part = A.get<float>(npart);
      N->sn_coef = A.get<double>(N->sn_entries.size());
      N->sn_dotp = A.get<double>(nbw);
      N->snb_start = A.get<long long>(N->sn_entries.size());
      N->snb_idx = A.get<int>(N->sn_entries.size());
      N->snb_grad = A.get<float*>(N->sn_entries.size());
      N->pf_d = A.get<SnPack>(64 + N->sn_entries.size() * 2);
      N->pb_d = A.get<SnPack>(64 + N->sn_entries.size() * 2);
      N->pf_start = A.get<long long>(64 + N->sn_entries.size() * 2);
      N->pb_start = A.get<long long>(64 + N->sn_entries.size() * 2);
    }
  }

  void build(Arena& A) {
    G_ = Net();
    D_ = Net();
    gb_.clear();
    db_.clear();
    if (dcgan_) {
      build_dcgan(A);
      return;
    }
    const int ch = cfg_.ch;
    B_ = cfg_.local_batch;
    R_ = cfg_.resolution;
    cpad_ = cfg_.c_pad_image;
    Arch ar;
    arch_for(R_, ar);
    const int nbg = (int)ar.gin.size();
    zc_ = cfg_.z_chunk;
    dimz_ = (nbg + 1) * zc_;
    cd_ = cfg_.shared_dim + zc_;
    // ---------------- G parameters, canonical order
    shared_ = G_.add("shared", {cfg_.n_classes, cfg_.shared_dim}, false, false);
    c0_ = ar.gin[0] * ch;
    glin_ = lin(G_, "linear", zc_, 16 * c0_, true, true);
    int h = 4;
    for (int i = 0; i < nbg; ++i) {
      GBlock b{};
      b.cin = ar.gin[i] * ch;
      b.cout = ar.gout[i] * ch;
      b.hin = h;
      const std::string p = "b" + std::to_string(i) + ".";
      b.g1 = lin(G_, p + "cbn1.gain", cd_, b.cin, false, true, false);
      b.b1 = lin(G_, p + "cbn1.bias", cd_, b.cin, false, true, false);
      b.c1 = conv(G_, p + "conv1", b.cin, b.cin, b.cout, 3, true);
      b.g2 = lin(G_, p + "cbn2.gain", cd_, b.cout, false, true, false);
      b.b2 = lin(G_, p + "cbn2.bias", cd_, b.cout, false, true, false);
      b.c2 = conv(G_, p + "conv2", b.cout, b.cout, b.cout, 3, true);
      b.sc = conv(G_, p + "sc", b.cin, b.cin, b.cout, 1, true);
      b.attn = (cfg_.attn_res == 2 * h);
      if (b.attn) gattn_ = attn(G_, b.cout, 2 * h);
      gb_.push_back(b);
      h *= 2;
    }
    cl_ = ar.gout.back() * ch;
    obn_g_ = G_.add("out_bn.gamma", {cl_}, false, false);
    obn_b_ = G_.add("out_bn.beta", {cl_}, false, false);
    oconv_ = conv(G_, "out_conv", cl_, cl_, 3, 3, true, true);
    // ---------------- D parameters
    h = R_;
    bool placed = false;
    for (size_t j = 0; j < ar.din.size(); ++j) {
      DBlock b{};
      b.cin = ar.din[j] < 0 ? 3 : ar.din[j] * ch;
      b.cin_x = ar.din[j] < 0 ? cpad_ : b.cin;
      b.cout = ar.dout[j] * ch;
      b.down = ar.ddown[j] != 0;
      b.hin = h;
      b.hout = b.down ? h / 2 : h;
      b.learn_sc = (b.cin != b.cout) || b.down;
      const std::string p = "b" + std::to_string(j) + ".";
      b.c1 = conv(D_, p + "conv1", b.cin, b.cin_x, b.cout, 3, true);
      static const bool im2col_on = [] {
        const char* e = std::getenv("PARAGAN_IM2COL");
        return e == nullptr || std::atoi(e) != 0;
      }();
      if (kBF && ar.din[j] < 0 && im2col_on) {
        b.im2col = true;
        b.c1x = b.c1;
        b.c1x.cin = 27;
        b.c1x.cin_x = 32;
        b.c1x.ksz = 1;
      }
      b.c2 = conv(D_, p + "conv2", b.cout, b.cout, b.cout, 3, true);
      if (b.learn_sc) b.sc = conv(D_, p + "sc", b.cin, b.cin_x, b.cout, 1, true);
      b.attn = !placed && cfg_.attn_res == b.hout;
      placed = placed || b.attn;
      if (b.attn) dattn_ = attn(D_, b.cout, b.hout);
      db_.push_back(b);
      h = b.hout;
    }
    cdl_ = ar.dout.back() * ch;
    hl_ = h;
    dlin_ = lin(D_, "linear", cdl_, 1, true, true);
    demb_ = D_.add("embed", {cfg_.n_classes, cdl_}, false, true);
    finalize_nets(A);
    const size_t wsz = kBF ? 2 : 4;
    auto alloc_conv = [&](ConvL& c) {
      const size_t nw = (size_t)c.cout * c.ksz * c.ksz * c.cin_x;
      const size_t es = c.f32 ? 4 : wsz;
      c.wp = A.get<char>(nw * es);
      c.wt = A.get<char>(nw * es);
    };
    auto alloc_lin = [&](LinL& l) { l.what = A.get<float>((size_t)l.in * l.out); };
    alloc_lin(glin_);
    for (auto& b : gb_) {
      alloc_lin(b.g1); alloc_lin(b.b1); alloc_lin(b.g2); alloc_lin(b.b2);
      alloc_conv(b.c1); alloc_conv(b.c2); alloc_conv(b.sc);
      if (kBF && subpix_) {
        b.c1.wp4 = A.get<char>((size_t)16 * b.c1.cout * b.c1.cin * 2);
        b.c1.wt4 = A.get<char>((size_t)16 * b.c1.cout * b.c1.cin * 2);
      }
    }
    if (kBF && subpix_ && !gb_.empty()) fold_jobs_d_ = A.get<FoldJob>(gb_.size());
    stats_dev_ = A.get<paragan_stats>(1);
    alloc_conv(oconv_);
    int ndg = 0;
    for (size_t j = 0; j < db_.size(); ++j) {
      DBlock& b = db_[j];
      if (b.im2col) alloc_conv(b.c1x); else alloc_conv(b.c1);
      alloc_conv(b.c2);
      if (b.learn_sc) alloc_conv(b.sc);
      b.wp4dg = nullptr;
      // (not D's first block: its 96-channel phase conv at 128^2 measured slower than the plain dgrad,
      // 1.47 vs 1.37 ms at n = 512)
      if (dgrad_pool_ && j > 0 && b.down && b.c2.ksz == 3 && tc_geometry_ok(b.hout, b.hout) && b.learn_sc &&
          b.sc.ksz == 1) {
        b.wp4dg = A.get<char>((size_t)16 * b.cout * b.cout * 2);
        b.wp4f = pool_fwd_ ? A.get<char>((size_t)16 * b.cout * b.cout * 2) : nullptr;
        b.dg_phase = true;
        ++ndg;
      } else if (pool_fwd0_ && j == 0 && b.down && b.c2.ksz == 3 && tc_geometry_ok(b.hout, b.hout)) {
        b.wp4dg = A.get<char>((size_t)16 * b.cout * b.cout * 2);
        b.wp4f = A.get<char>((size_t)16 * b.cout * b.cout * 2);
        ++ndg;
      }
    }
    fold_jobs_dd_ = ndg ? A.get<FoldJob>(ndg) : nullptr;
    alloc_lin(dlin_);
    demb_hat_ = A.get<float>((size_t)cfg_.n_classes * cdl_);
    for (AttnL* at : {&gattn_, &dattn_}) {
      if (!at->C) continue;
      at->qkv_wp = A.get<char>((size_t)at->Ct * at->C * wsz);
      at->qkv_wt = A.get<char>((size_t)at->Ct * at->C * wsz);
      alloc_conv(at->oc);
    }
    // ---------------- activations
    const int B = B_, B2 = 2 * B_;
    big_ = 0;
    auto act = [&](long long n, int h_, int w_, int c_) -> void* {
      const long long e = n * h_ * w_ * c_;
      big_ = std::max(big_, e);
      return A.get<char>((size_t)e * sizeof(T));
    };
    zin_ = A.get<float>((size_t)B * dimz_);
    yg_ = A.get<int32_t>(B);
    emb_ = A.get<float>((size_t)B * cfg_.shared_dim);
    demb_g_ = A.get<float>((size_t)B * cfg_.shared_dim);
    h0f_ = A.get<float>((size_t)B * 16 * c0_);
    for (auto& b : gb_) {
      const int H = b.hin;
      b.x = (&b == &gb_[0]) ? act(B, H, H, b.cin) : nullptr;   // later blocks read the previous output in place
      b.u1 = (kBF && subpix_) ? nullptr : act(B, 2 * H, 2 * H, b.cin);
      b.u1lo = (kBF && subpix_) ? act(B, H, H, b.cin) : nullptr;
      b.h1 = act(B, 2 * H, 2 * H, b.cout);
      b.a2 = act(B, 2 * H, 2 * H, b.cout);
      b.s = act(B, H, H, b.cout);
      b.out = act(B, 2 * H, 2 * H, b.cout);
      b.gain1 = A.get<float>((size_t)B * b.cin);
      b.bias1 = A.get<float>((size_t)B * b.cin);
      b.gain2 = A.get<float>((size_t)B * b.cout);
      b.bias2 = A.get<float>((size_t)B * b.cout);
      b.cond = A.get<float>((size_t)B * cd_);
      b.dcond = A.get<float>((size_t)B * cd_);
      b.dcond_part = A.get<float>((size_t)B * cd_ * (2 * ceil_div(b.cin, kDcondK) + 2 * ceil_div(b.cout, kDcondK)));
      b.ab1 = A.get<float>((size_t)B * 2 * b.cin);
      b.ab2 = A.get<float>((size_t)B * 2 * b.cout);
      b.mean1 = A.get<float>(b.cin);
      b.rstd1 = A.get<float>(b.cin);
      b.mean2 = A.get<float>(b.cout);
      b.rstd2 = A.get<float>(b.cout);
      b.sums1 = A.get<double>(2 * b.cin);
      b.sums2 = A.get<double>(2 * b.cout);
    }
    // fp32 output-BN activation, or — tensor-core output layer (R36) — its two-term bf16 split
    // [x1 | x2], the same bytes
    aout_ = A.get<float>((size_t)B * R_ * R_ * cl_);
    thin_tc_ = thin_tc_ && out_conv_tc_ok(R_, R_, cl_);
    if (thin_tc_) {
      oconv_ws_ = A.get<bf16>((size_t)96 * 2 * cl_);
      oconv_wd_ = A.get<bf16>((size_t)round_up(cl_, 16) * 128);
    }
    omean_ = A.get<float>(cl_);
    orstd_ = A.get<float>(cl_);
    osums_ = A.get<double>(2 * cl_);
    pre_ = A.get<float>((size_t)B * R_ * R_ * 3);
    img_ = A.get<float>((size_t)B * R_ * R_ * 3);
    dimg_ = act(B2, R_, R_, cpad_);
    ylab_ = A.get<int32_t>(B2);
    for (auto& b : db_) {
      const int H = b.hin;
      b.x = (&b == &db_[0]) ? dimg_ : nullptr;   // set below to previous output
      b.rx = act(B2, H, H, b.cin_x);
      b.c1o = kBF ? nullptr : act(B2, H, H, b.cout);   // bf16: conv1 writes relu(.) straight into r1
      b.r1 = act(B2, H, H, b.cout);
      b.t = act(B2, H, H, b.cout);
      b.xp = b.down ? act(B2, H / 2, H / 2, b.cin_x) : nullptr;
      b.s = b.learn_sc ? act(B2, H, H, b.cout) : nullptr;
      b.out = act(B2, b.hout, b.hout, b.cout);
      b.xi = b.im2col ? act(B2, H, H, 32) : nullptr;
    }
    for (AttnL* at : {&gattn_, &dattn_}) {
      if (!at->C) continue;
      const int n = (at == &gattn_) ? B : B2;
      const long long HW = (long long)at->H * at->H, Q = HW / 4;
      at->qkv = act(n, at->H, at->H, at->Ct);
      at->phi_p = A.get<char>((size_t)n * Q * at->Cq * sizeof(T));
      at->g_p = A.get<char>((size_t)n * Q * at->C2 * sizeof(T));
      at->ov = act(n, at->H, at->H, at->C2);
      attn_out_[at == &gattn_ ? 0 : 1] = act(n, at->H, at->H, at->C);
      at->fused = kBF && std::getenv("PARAGAN_ATTN_UNFUSED") == nullptr &&
                  tc_attn_ok((int)HW, (int)Q, at->Cq, at->C2);
      if (at->fused) {
        at->gT = A.get<char>((size_t)n * Q * at->C2 * sizeof(T));
        at->o32 = A.get<float>((size_t)n * HW * at->C2);
        at->lse = A.get<float>((size_t)n * HW);
        at->phimax = A.get<float>((size_t)n);
        at->thetamax = A.get<float>((size_t)n);
        at->Dr = A.get<float>((size_t)n * HW);
        dth_part_floats_ = std::max(dth_part_floats_, (size_t)((Q / 128) * n * HW * at->Cq));
      } else {
        at->S = A.get<float>((size_t)n * HW * Q);
        at->P = A.get<char>((size_t)n * HW * Q * sizeof(T));
        big_ = std::max(big_, (long long)n * HW * Q);
        unfused_dp_ = std::max(unfused_dp_, (long long)n * HW * Q);
      }
      dpool_floats_ = std::max(dpool_floats_, (size_t)(n * Q * (at->C2 + at->Cq)));
    }
    if (dth_part_floats_) dth_part_ = A.get<float>(dth_part_floats_);
    {
      long long mdo = 0, mdq = 0;
      for (AttnL* at : {&gattn_, &dattn_}) {
        if (!at->C) continue;
        const long long n = (at == &gattn_) ? B : B2;
        mdo = std::max(mdo, n * at->H * at->H * at->C2);
        mdq = std::max(mdq, n * at->H * at->H * at->Ct);
      }
      tmp_attn_dO_ = A.get<char>((size_t)std::max(mdo, 1LL) * sizeof(T));
      tmp_attn_dqkv_ = A.get<char>((size_t)std::max(mdq, 1LL) * sizeof(T));
      dP_ = A.get<float>((size_t)std::max(unfused_dp_, 1LL));
      dxp_ = A.get<char>((size_t)B2 * (R_ / 2) * (R_ / 2) * cpad_ * sizeof(T));
    }
    maxc_ = 8;
    for (auto& b : gb_) maxc_ = std::max(maxc_, std::max(b.cin, b.cout));
    for (auto& b : db_) maxc_ = std::max(maxc_, std::max(b.cin_x, b.cout));
    ones_buf_ = A.get<float>(maxc_);
    quarter_ = A.get<float>(1);
    feat_ = A.get<float>((size_t)B2 * cdl_);
    logits_ = A.get<float>(B2);
    dlogits_ = A.get<float>(B2);
    // temps: 4 gradient buffers of the largest activation, fp32 scratch
    for (int i = 0; i < 4; ++i) tmp_[i] = A.get<char>((size_t)big_ * sizeof(T));
    dpre_ = A.get<float>((size_t)B * R_ * R_ * 3);
    daout_ = A.get<float>((size_t)B * R_ * R_ * cl_);
    dh0f_ = A.get<float>((size_t)B * 16 * c0_);
    ab_ = A.get<float>((size_t)B * 2 * maxc_);
    // grouped CBN-linear GEMM tables (A4): forward (4 per block + the G linear), dW (4 per block), dcond (1 per block)
    {
      const size_t nb = gb_.size();
      cbn_fwd_d_ = A.get<GemmProblem>(4 * nb + 1);
      cbn_dw_d_ = A.get<GemmProblem>(4 * nb);
      size_t nslots = 0;
      for (auto& b : gb_) nslots += 2 * ceil_div(b.cin, kDcondK) + 2 * ceil_div(b.cout, kDcondK);
      cbn_dcond_d_ = A.get<GemmProblem>(std::max<size_t>(nslots, 1));
    }
    bn_part_ = A.get<float>((size_t)B * 64 * 2 * maxc_);
    dpart_ = A.get<double>((size_t)kMaxPartialBlocks * 2 * std::max(maxc_, 16 * c0_));
    tot_ = A.get<double>(4 * maxc_);   // fp64 channel sums + fp32 means (bn_bwd_apply)
    size_t sf = std::max<size_t>((size_t)std::max(G_.n, D_.n), (size_t)B * 3 * R_ * R_);
    sf = std::max<size_t>(sf, (size_t)64 << 20);
    scratch_floats_ = sf;
    scratch_f_ = A.get<float>(sf);
    wg_scratch_ = A.get<float>((size_t)16 << 20);   // padded / qkv weight-gradient staging
    dpool_ = A.get<float>(std::max<size_t>(dpool_floats_, 1));
    alloc_sn_tables(A);
    alloc_opt_tables(A);
    // chain G block inputs (block i+1 reads block i's output, or the attention output, in place)
    for (size_t i = 1; i < gb_.size(); ++i) gb_[i].x = gb_[i - 1].attn ? attn_out_[0] : gb_[i - 1].out;
    gout_in_ = gb_.back().attn ? attn_out_[0] : gb_.back().out;
    // chain D block inputs
    void* prev = dimg_;
    for (auto& b : db_) {
      b.x = prev;
      prev = b.out;
      if (b.attn) prev = attn_out_[1];
    }
    planned_ = true;
  }

  // SN job tables and pack lists (host -> device once)
  paragan_status upload_cbn_tables() {
    const int B = B_;
    auto seg = [](const float* A, long long sam, long long sak, const float* Bm, long long sbn, long long sbk, int K) {
      GemmSeg g{};
      g.A = A;
      g.sam = sam;
      g.sak = sak;
      g.B = Bm;
      g.sbn = sbn;
      g.sbk = sbk;
      g.K = K;
      return g;
    };
    std::vector<GemmProblem> fw, dw, dc;
    {
      // G linear: h0f = z0 W^T + b
      GemmProblem p{};
      p.M = B;
      p.N = 16 * c0_;
      p.nseg = 1;
      p.seg[0] = seg(zin_, dimz_, 1, glin_.what, zc_, 1, zc_);
      p.C = h0f_;
      p.ldc = 16 * c0_;
      p.bias = G_.P(glin_.b);
      fw.push_back(p);
    }
    for (GBlock& b : gb_) {
      const LinL* L[4] = {&b.g1, &b.b1, &b.g2, &b.b2};
      float* outs[4] = {b.gain1, b.bias1, b.gain2, b.bias2};
      float* abs_[4] = {b.ab1 + b.cin, b.ab1, b.ab2 + b.cout, b.ab2};   // dgain = AB[:, C:2C], dbias = AB[:, 0:C]
      const int Cs[4] = {b.cin, b.cin, b.cout, b.cout};
      b.dcond_nslot = 0;
      for (int k = 0; k < 4; ++k) {
        GemmProblem p{};
        p.M = B;
        p.N = Cs[k];
        p.nseg = 1;
        p.seg[0] = seg(b.cond, cd_, 1, L[k]->what, cd_, 1, cd_);
        p.C = outs[k];
        p.ldc = Cs[k];
        fw.push_back(p);
        // dW[c][k] = sum_n dX[n][c] cond[n][k]
        GemmProblem q{};
        q.M = Cs[k];
        q.N = cd_;
        q.nseg = 1;
        q.seg[0] = seg(abs_[k], 1, 2 * Cs[k], b.cond, 1, cd_, B);
        q.C = G_.G(L[k]->w);
        q.ldc = cd_;
        dw.push_back(q);
        // dcond[n][k] = sum over the four linears of sum_c dX[n][c] What[c][k]: M x N = B x cond_dim
        // is small and K = C long, so split K into kDcondK-channel slices (one partial each, summed
        // in slice order afterwards) — as one tile row per block it ran on 60 SMs for 0.7 ms
        for (int c0 = 0; c0 < Cs[k]; c0 += kDcondK) {
          GemmProblem pc{};
          pc.M = B;
          pc.N = cd_;
          pc.nseg = 1;
          pc.seg[0] = seg(abs_[k] + c0, 2 * Cs[k], 1, L[k]->what + (size_t)c0 * cd_, 1, cd_,
                          std::min(kDcondK, Cs[k] - c0));
          pc.C = b.dcond_part + (size_t)b.dcond_nslot++ * B * cd_;
          pc.ldc = cd_;
          dc.push_back(pc);
        }
      }
    }
    cbn_fwd_n_ = (int)fw.size();
    cbn_fwd_tiles_ = gemm_grouped_plan(fw.data(), cbn_fwd_n_);
    cbn_dw_n_ = (int)dw.size();
    cbn_dw_tiles_ = gemm_grouped_plan(dw.data(), cbn_dw_n_);
    cbn_dcond_n_ = (int)dc.size();
    cbn_dcond_tiles_ = gemm_grouped_plan(dc.data(), cbn_dcond_n_);
    CK(cudaMemcpyAsync(cbn_fwd_d_, fw.data(), sizeof(GemmProblem) * fw.size(), cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(cbn_dw_d_, dw.data(), sizeof(GemmProblem) * dw.size(), cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(cbn_dcond_d_, dc.data(), sizeof(GemmProblem) * dc.size(), cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));   // the host vectors die here
    return PARAGAN_OK;
  }

  paragan_status upload_tables() {
    CKS(upload_opt_tables());
    if (!dcgan_) CKS(upload_cbn_tables());
    for (Net* N : {&G_, &D_}) {
      std::vector<SnJob> jobs;
      std::vector<int> b1j, b1k, b1r, b1bj, b1bk, b2j, b2r;
      std::vector<long long> bstart;
      long long part_off = 0, bw = 0;
      for (int ei : N->sn_entries) {
        const PEntry& e = N->E[ei];
        SnJob j{};
        j.w = N->p + e.off;
        j.u = N->u + e.u_off;
        j.v = N->sn_v + e.v_off;
        j.t = N->sn_t + e.v_off;
        j.s = N->sn_s + e.u_off;
        j.sigma = N->sigma + 2 * e.job;
        j.rows = e.shape[0];
        j.K = (int)(e.n / e.shape[0]);
        j.nrc = ceil_div(j.rows, 128);
        j.eps = cfg_.sn_eps;
        j.part = N->sn_part + part_off;
        part_off += ((long long)j.nrc * j.K + 3) & ~3LL;
        j.grad = N->g + e.off;
        const int ji = (int)jobs.size();
        j.coef = N->sn_coef + ji;
        j.bwd_blk0 = bw;
        j.bwd_nblk = ceil_div(e.n, 4096);
        bstart.push_back(bw);
        bw += j.bwd_nblk;
        const int cpb = sn_cols_per_block(j.K);
        for (int rc = 0; rc < j.nrc; ++rc)
          for (int k = 0; k < j.K; k += cpb) { b1j.push_back(ji); b1k.push_back(k); b1r.push_back(rc); }
        for (int k = 0; k < j.K; k += cpb) { b1bj.push_back(ji); b1bk.push_back(k); }
        for (int r = 0; r < j.rows; r += 8) { b2j.push_back(ji); b2r.push_back(r); }
        jobs.push_back(j);
      }
      auto up = [&](void* dst, const void* src, size_t bytes) {
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st_);
      };
      CK(up(N->jobs_d, jobs.data(), jobs.size() * sizeof(SnJob)));
      CK(up(N->b1_job, b1j.data(), b1j.size() * sizeof(int)));
      CK(up(N->b1_k0, b1k.data(), b1k.size() * sizeof(int)));
      CK(up(N->b1_rc, b1r.data(), b1r.size() * sizeof(int)));
      CK(up(N->b1b_job, b1bj.data(), b1bj.size() * sizeof(int)));
      CK(up(N->b1b_k0, b1bk.data(), b1bk.size() * sizeof(int)));
      CK(up(N->b2_job, b2j.data(), b2j.size() * sizeof(int)));
      CK(up(N->b2_r0, b2r.data(), b2r.size() * sizeof(int)));
      CK(up(N->snb_start, bstart.data(), bstart.size() * sizeof(long long)));
      CK(cudaStreamSynchronize(st_));   // host vectors go out of scope
      jobs_h_[N == &G_ ? 0 : 1] = jobs;
    }
    // pack lists
    auto sig = [&](Net& N, int e) { return N.sigma + 2 * N.E[e].job; };
    auto add_conv = [&](Net& N, const ConvL& c) {
      SnPack f{};
      f.w = N.P(c.w);
      f.sigma = sig(N, c.w);
      f.dst = c.wp;
      f.rows = c.cout;
      f.taps = c.ksz * c.ksz;
      f.cin = c.cin;
      f.mode = 0;
      f.dst_bf16 = (kBF && !c.f32) ? 1 : 0;
      f.dst_row_offset = 0;
      f.dst_rows = c.cout;
      f.dst_cin = c.cin_x;
      N.pf_h.push_back(f);
      SnPack b = f;
      b.dst = c.wt;
      b.mode = 1;
      N.pb_h.push_back(b);
    };
    auto add_lin = [&](Net& N, const LinL& l) {
      SnPack f{};
      f.w = N.P(l.w);
      f.sigma = sig(N, l.w);
      f.dst = l.what;
      f.rows = l.out;
      f.taps = 1;
      f.cin = l.in;
      f.mode = 0;
      f.dst_bf16 = 0;
      f.dst_rows = l.out;
      f.dst_cin = l.in;
      N.pf_h.push_back(f);
    };
    auto add_attn = [&](Net& N, AttnL& a) {
      const int rows[3] = {a.C8, a.C8, a.C2}, offs[3] = {0, a.Cq, 2 * a.Cq}, es[3] = {a.th, a.ph, a.gg};
      for (int k = 0; k < 3; ++k) {
        SnPack f{};
        f.w = N.P(es[k]);
        f.sigma = sig(N, es[k]);
        f.dst = a.qkv_wp;
        f.rows = rows[k];
        f.taps = 1;
        f.cin = a.C;
        f.mode = 0;
        f.dst_bf16 = kBF ? 1 : 0;
        f.dst_row_offset = offs[k];
        f.dst_rows = a.Ct;
        f.dst_cin = a.C;
        N.pf_h.push_back(f);
        SnPack b = f;
        b.dst = a.qkv_wt;
        b.mode = 1;
        N.pb_h.push_back(b);
      }
      add_conv(N, a.oc);
    };
    G_.pf_h.clear(); G_.pb_h.clear(); D_.pf_h.clear(); D_.pb_h.clear();
    if (dcgan_) {
      for (auto& L : dcd_) add_conv(D_, L.c);
      add_lin(D_, dlin_);
    } else {
    add_lin(G_, glin_);
    for (auto& b : gb_) {
      add_lin(G_, b.g1); add_lin(G_, b.b1); add_lin(G_, b.g2); add_lin(G_, b.b2);
      add_conv(G_, b.c1); add_conv(G_, b.c2); add_conv(G_, b.sc);
    }
    if (gattn_.C) add_attn(G_, gattn_);
    add_conv(G_, oconv_);
    for (auto& b : db_) {
      add_conv(D_, b.im2col ? b.c1x : b.c1);
      add_conv(D_, b.c2);
      if (b.learn_sc) add_conv(D_, b.sc);
    }
    if (dattn_.C) add_attn(D_, dattn_);
    add_lin(D_, dlin_);
    {
      LinL e;
      e.w = demb_;
      e.in = cdl_;
      e.out = cfg_.n_classes;
      e.what = demb_hat_;
      add_lin(D_, e);
    }
    }
    for (Net* N : {&G_, &D_}) {
      for (int pass = 0; pass < 2; ++pass) {
        auto& lst = pass == 0 ? N->pf_h : N->pb_h;
        std::vector<long long> st;
        long long acc = 0;
        for (auto& j : lst) {
          st.push_back(acc);
          acc += pass == 0 ? sn_pack_prepare(j) : sn_pack_t_prepare(j);
        }
        (pass == 0 ? N->pf_blocks : N->pb_blocks) = acc;
        CK(cudaMemcpyAsync(pass == 0 ? N->pf_d : N->pb_d, lst.data(), lst.size() * sizeof(SnPack),
                           cudaMemcpyHostToDevice, st_));
        CK(cudaMemcpyAsync(pass == 0 ? N->pf_start : N->pb_start, st.data(), st.size() * sizeof(long long),
                           cudaMemcpyHostToDevice, st_));
      }
    }
    // G's conv1 fold table (sub-pixel mode): one grouped launch per G forward
    std::vector<FoldJob> fj;
    if (fold_jobs_d_) {
      int tiles = 0;
      for (GBlock& b : gb_) {
        const PEntry& e = G_.E[b.c1.w];
        FoldJob j{};
        j.w = G_.p + e.off;
        j.inv_sigma = G_.sigma + 2 * e.job + 1;
        j.dst0 = static_cast<bf16*>(b.c1.wp4);
        j.dst1 = static_cast<bf16*>(b.c1.wt4);
        j.Cout = b.c1.cout;
        j.Cin = b.c1.cin;
        j.tile0 = tiles;
        tiles += ceil_div(b.c1.cout, 32) * ceil_div(b.c1.cin, 32);
        fj.push_back(j);
      }
      fold_tiles_ = tiles;
      CK(cudaMemcpyAsync(fold_jobs_d_, fj.data(), fj.size() * sizeof(FoldJob), cudaMemcpyHostToDevice, st_));
    }
    // D's pooled-block conv2 input-gradient kernels (transposed, flipped, folded)
    std::vector<FoldJob> fd;
    if (fold_jobs_dd_) {
      int tiles = 0;
      for (DBlock& b : db_) {
        if (!b.wp4dg) continue;
        const PEntry& e = D_.E[b.c2.w];
        FoldJob j{};
        j.w = D_.p + e.off;
        j.inv_sigma = D_.sigma + 2 * e.job + 1;
        j.dst0 = static_cast<bf16*>(b.wp4dg);
        j.dst1 = static_cast<bf16*>(b.wp4f);   // same fold, [Cin][16][Cout] for the pooled forward (R38)
        j.Cout = b.cout;   // output channels of the input-gradient conv = conv2's input channels
        j.Cin = b.cout;
        j.tile0 = tiles;
        j.tf = 1;
        tiles += ceil_div(b.cout, 32) * ceil_div(b.cout, 32);
        fd.push_back(j);
      }
      fold_tiles_dd_ = tiles;
      fold_njobs_dd_ = (int)fd.size();
      CK(cudaMemcpyAsync(fold_jobs_dd_, fd.data(), fd.size() * sizeof(FoldJob), cudaMemcpyHostToDevice, st_));
    }
    return sync_ok();
  }

  // ------------------------------------------------------------------ SN forward (A2)
  paragan_status sn_forward(Net& N, bool need_dgrad) {
    if (N.sn_entries.empty()) return PARAGAN_OK;
    CK(sn_power(N.jobs_d, (int)N.sn_entries.size(), N.b1_job, N.b1_k0, N.b1_rc, N.nb1, N.b1b_job, N.b1b_k0, N.nb1b,
                N.b2_job, N.b2_r0, N.nb2, st_));
    launches_ += 3;
    CK(sn_pack(N.pf_d, N.pf_start, (int)N.pf_h.size(), N.pf_blocks, st_));
    if (need_dgrad) CK(sn_pack_t(N.pb_d, N.pb_start, (int)N.pb_h.size(), N.pb_blocks, st_));
    return PARAGAN_OK;
  }
  // W/sigma of every G conv1 folded into the four phase kernels of the sub-pixel conv
  paragan_status fold_subpixel(bool need_dgrad) {
    if (!subpix_) return PARAGAN_OK;
    CK(fold_up2_grouped(fold_jobs_d_, (int)gb_.size(), fold_tiles_, need_dgrad, st_));
    return PARAGAN_OK;
  }
  paragan_status sn_backward_net(Net& N) {
    if (N.sn_entries.empty()) return PARAGAN_OK;
    CK(sn_backward(N.jobs_d, (int)N.sn_entries.size(), N.snb_start, N.snb_blocks, N.sn_dotp, st_));
    launches_ += 2;
    return PARAGAN_OK;
  }

  struct ProfRec {
    int kind;
    double flops;        // algorithmic (the BigGAN-defined work of the launch)
    cudaEvent_t a, b;
    char what[48];
    double exec_flops;   // what the tensor cores were issued (differs for the sub-pixel G conv1)
  };
  cudaEvent_t ev_get() {
    if (!ev_free_.empty()) {
      cudaEvent_t e = ev_free_.back();
      ev_free_.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  // brackets one launch with events when profiling; kind 0 = tcgen05 fprop/dgrad, 1 = tcgen05 wgrad
  template <class F>
  cudaError_t timed(int kind, double flops, F&& f, const char* what = "", double exec_flops = -1.0) {
    if (!prof_) return f();
    ProfRec r{kind, flops, ev_get(), ev_get(), {0}, exec_flops < 0 ? flops : exec_flops};
    std::snprintf(r.what, sizeof(r.what), "%s", what);
    cudaEventRecord(r.a, st_);
    cudaError_t e = f();
    cudaEventRecord(r.b, st_);
    recs_.push_back(r);
    return e;
  }

  // ------------------------------------------------------------------ conv dispatch
  // pool_out (BF16 engine): y is not written; the epilogue writes avgpool2(y) there (and relu of it to pool_relu)
  paragan_status conv_fwd(const void* x, int n, int H, const ConvL& c, void* y, const float* bias,
                          const void* res, int res_mode, const float* alpha = nullptr, bool relu_out = false,
                          void* pool_out = nullptr, void* pool_relu = nullptr) {
    if constexpr (kBF) {
      if (!c.f32) {
        TcEpilogue e;
        e.relu_out = relu_out ? 1 : 0;
        e.bias = bias;
        e.alpha = alpha;
        e.residual = res;
        e.res_mode = res ? res_mode : 0;
        e.out = pool_out ? nullptr : y;
        e.pool_out = pool_out;
        e.pool_relu = pool_relu;
        const double fl = 2.0 * n * H * H * (double)c.cout * c.ksz * c.ksz * c.cin;
        char what[48];
        std::snprintf(what, sizeof(what), "fprop n%d %dx%d %d->%d k%d", n, H, H, c.cin, c.cout, c.ksz);
        CK(timed(0, fl, [&] { return tc_conv_fprop(x, n, H, H, c.cin_x, c.wp, c.cout, c.ksz, e, st_); }, what));
        return PARAGAN_OK;
      }
    }
    CK((simt_conv_fwd<float, float, float>(static_cast<const float*>(x), n, H, H, c.cin_x,
                                           static_cast<const float*>(c.wp), c.cout, c.ksz, bias, alpha,
                                           static_cast<const float*>(res), res_mode, static_cast<float*>(y), st_)));
    return PARAGAN_OK;
  }
  // y[n,2H,2H,cout] = conv3x3(up2(x[n,H,H,cin])) + bias via the phase decomposition (BF16 only)
  paragan_status conv_fwd_up2(const void* x, int n, int H, const ConvL& c, void* y, const float* bias) {
    if constexpr (kBF) {
      TcEpilogue e;
      e.bias = bias;
      e.out = y;
      // algorithmic work: the 3x3 conv over the upsampled tensor; executed: 4 phases x 4 taps
      // per low-resolution pixel, 1/2.25 of it
      const double fl = 2.0 * n * (4.0 * H * H) * 9.0 * c.cout * c.cin;
      const double fx = 2.0 * n * H * H * 16.0 * c.cout * c.cin;
      char what[48];
      std::snprintf(what, sizeof(what), "fprop-up2 n%d %dx%d %d->%d", n, H, H, c.cin, c.cout);
      CK(timed(0, fl, [&] { return tc_conv_fprop_up2(x, n, H, H, c.cin, c.wp4, c.cout, e, st_); }, what, fx));
      return PARAGAN_OK;
    }
    return fail_msg(PARAGAN_ERR_CONFIG, "sub-pixel conv needs the BF16 engine");
  }
  // conv3x3(up2(x)) backward through the phase decomposition (BF16 only): dW + db into the grad slots
  paragan_status conv_wgrad_up2(const void* x_lo, const void* dy, int n, int H, const ConvL& c) {
    if constexpr (kBF) {
      const double fl = 2.0 * n * (4.0 * H * H) * 9.0 * c.cout * c.cin;
      const double fx = 2.0 * n * H * H * 16.0 * c.cout * c.cin;
      char what[48];
      std::snprintf(what, sizeof(what), "wgrad-up2 n%d %dx%d %d->%d", n, H, H, c.cin, c.cout);
      float* db = c.b >= 0 ? G_.G(c.b) : nullptr;
      CK(timed(1, fl, [&] {
        return tc_conv_wgrad_up2(x_lo, dy, n, H, H, c.cin, c.cout, G_.G(c.w), scratch_f_, scratch_floats_, st_, db);
      }, what, fx));
      return PARAGAN_OK;
    }
    return fail_msg(PARAGAN_ERR_CONFIG, "sub-pixel conv needs the BF16 engine");
  }
  paragan_status conv_dgrad_up2(const void* dy, int n, int H, const ConvL& c, void* dx_lo) {
    if constexpr (kBF) {
      TcEpilogue e;
      e.out = dx_lo;
      const double fl = 2.0 * n * (4.0 * H * H) * 9.0 * c.cout * c.cin;
      const double fx = 2.0 * n * H * H * 16.0 * c.cout * c.cin;
      char what[48];
      std::snprintf(what, sizeof(what), "dgrad-up2 n%d %dx%d %d->%d", n, H, H, c.cout, c.cin);
      CK(timed(0, fl, [&] { return tc_conv_dgrad_up2(dy, n, H, H, c.cout, c.wt4, c.cin, e, st_); }, what, fx));
      return PARAGAN_OK;
    }
    return fail_msg(PARAGAN_ERR_CONFIG, "sub-pixel conv needs the BF16 engine");
  }
  // dx[n,H,H,cin_x] = alpha * dgrad(dy) (+ add)
  paragan_status conv_dgrad(const void* dy, int n, int H, const ConvL& c, void* dx, const void* add,
                            const float* alpha = nullptr, const void* relu_ref = nullptr, int add_mode = 1) {
    if constexpr (kBF) {
      if (!c.f32) {
        TcEpilogue e;
        e.alpha = alpha;
        e.relu_ref = relu_ref;
        e.residual = add;
        e.res_mode = add ? add_mode : 0;
        e.out = dx;
        const double fl = 2.0 * n * H * H * (double)c.cout * c.ksz * c.ksz * c.cin;
        char what[48];
        std::snprintf(what, sizeof(what), "dgrad n%d %dx%d %d->%d k%d", n, H, H, c.cout, c.cin, c.ksz);
        CK(timed(0, fl, [&] { return tc_conv_fprop(dy, n, H, H, c.cout, c.wt, c.cin_x, c.ksz, e, st_); }, what));
        return PARAGAN_OK;
      }
    }
    CK((simt_conv_fwd<float, float, float>(static_cast<const float*>(dy), n, H, H, c.cout,
                                           static_cast<const float*>(c.wt), c.cin_x, c.ksz, nullptr, alpha,
                                           static_cast<const float*>(add), add ? 1 : 0, static_cast<float*>(dx),
                                           st_, static_cast<const float*>(relu_ref))));
    return PARAGAN_OK;
  }
  // dW (into the net's grad slot, OHWI) = wgrad(x, dy); db = column sums of dy when bias_entry >= 0
  // (fused into the tcgen05 wgrad launch in BF16 mode)
  paragan_status conv_wgrad(Net& N, const void* x, const void* dy, int n, int H, const ConvL& c, int bias_entry = -1) {
    float* dst = N.G(c.w);
    const bool pad = c.cin_x != c.cin;
    float* out = pad ? wg_scratch_ : dst;
    if constexpr (kBF) {
      if (!c.f32) {
        const double fl = 2.0 * n * H * H * (double)c.cout * c.ksz * c.ksz * c.cin;
        char what[48];
        std::snprintf(what, sizeof(what), "wgrad n%d %dx%d %d->%d k%d", n, H, H, c.cin, c.cout, c.ksz);
        float* db = bias_entry >= 0 ? N.G(bias_entry) : nullptr;
        CK(timed(1, fl, [&] {
          return tc_conv_wgrad(x, dy, n, H, H, c.cin_x, c.cout, c.ksz, out, 0, scratch_f_, scratch_floats_, st_, db);
        }, what));
        if (pad) CK(copy_rows_cols(out, c.cin_x, (long long)c.cout * c.ksz * c.ksz, c.cin, dst, c.cin, 0, st_));
        return PARAGAN_OK;
      }
    }
    CK((simt_conv_wgrad<float, float>(static_cast<const float*>(x), static_cast<const float*>(dy), n, H, H, c.cin_x,
                                      c.cout, c.ksz, out, 0, st_, scratch_f_, scratch_floats_)));
    if (pad) CK(copy_rows_cols(out, c.cin_x, (long long)c.cout * c.ksz * c.ksz, c.cin, dst, c.cin, 0, st_));
    if (bias_entry >= 0)
      CK(col_sum<T>(static_cast<const T*>(dy), (long long)n * H * H, c.cout, dpart_, kMaxPartialBlocks,
                    N.G(bias_entry), 0, st_));
    return PARAGAN_OK;
  }
  paragan_status bgemm(int batch, int M, int N, int K, const void* A, long long sab, long long sam, long long sak,
                       const void* Bm, long long sbb, long long sbn, long long sbk, void* C, bool c_f32, long long scb,
                       long long ldc) {
    if constexpr (kBF) {
      CK(gemm_bf16_batched(batch, M, N, K, static_cast<const bf16*>(A), sab, sam, sak, static_cast<const bf16*>(Bm), sbb,
                           sbn, sbk, C, c_f32, scb, ldc, st_));
      return PARAGAN_OK;
    } else {
      (void)c_f32;
      CK(gemm_f32_batched(batch, M, N, K, static_cast<const float*>(A), sab, sam, sak, static_cast<const float*>(Bm),
                          sbb, sbn, sbk, static_cast<float*>(C), scb, ldc, 0.0f, st_));
      return PARAGAN_OK;
    }
  }
  // cross-replica BN statistics (A4): local sums -> NCCL all-reduce -> mean / rstd
  paragan_status bn_forward_stats(const void* x, long long M, int C, double* sums, float* mean, float* rstd) {
    CK(bn_stats<T>(static_cast<const T*>(x), M, C, dpart_, kMaxPartialBlocks, sums, st_));
    ++launches_;
    if (cfg_.world_size > 1) {
      CKS(nccl_sum(sums, (size_t)2 * C, ncclFloat64, "bn allreduce", bncomm_));
    }
    CK(bn_finalize(sums, C, (double)M * cfg_.world_size, cfg_.bn_eps, mean, rstd, st_));
    return PARAGAN_OK;
  }
  // losses / logit means are local means: sum over ranks here, / world_size in sync_stats (R15);
  // the non-finite flag (loss[3]) becomes the number of ranks that saw one
  // in-place sum over ranks on the compute stream; timed as profile kind 2 (collectives)
  paragan_status nccl_sum(void* buf, size_t count, ncclDataType_t dt, const char* what, ncclComm_t comm = nullptr) {
    ncclResult_t r = ncclSuccess;
    const size_t bytes = count * (dt == ncclFloat64 ? 8 : dt == ncclBfloat16 ? 2 : 4);
    char label[48];
    std::snprintf(label, sizeof(label), "%s %zu B", what, bytes);
    cudaError_t e = timed(2, (double)bytes, [&] {
      r = ncclAllReduce(buf, buf, count, dt, ncclSum, comm ? comm : comm_, st_);
      return r == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
    }, label);
    if (r != ncclSuccess) return fail_msg(PARAGAN_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
    CK(e);
    return PARAGAN_OK;
  }
  paragan_status allreduce_loss(float* loss4) {
    if (cfg_.world_size > 1) {
      CKS(nccl_sum(loss4, 4, ncclFloat32, "loss allreduce", bncomm_));
    }
    return PARAGAN_OK;
  }
  paragan_status allreduce_small(double* p, int n) {
    if (cfg_.world_size > 1) {
      CKS(nccl_sum(p, (size_t)n, ncclFloat64, "allreduce", bncomm_));
    }
    return PARAGAN_OK;
  }
  void* tmp(int i) { return tmp_[i]; }

  // ------------------------------------------------------------------ G forward (A3, A4, A5, A6)
  paragan_status g_forward(const float* z, const int32_t* y, bool train) {
    (void)train;
    const int B = B_;
    CK(cudaMemcpyAsync(zin_, z, sizeof(float) * B * dimz_, cudaMemcpyDeviceToDevice, st_));
    CK(cudaMemcpyAsync(yg_, y, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st_));
    CK(gather_rows(G_.P(shared_), yg_, B, cfg_.shared_dim, emb_, cfg_.shared_dim, st_));
    for (size_t i = 0; i < gb_.size(); ++i) {
      // cond_i = [shared[y] | z_{i+1}]  (R11)
      CK(copy_cols(emb_, cfg_.shared_dim, B, cfg_.shared_dim, gb_[i].cond, cd_, st_));
      CK(copy_cols(zin_ + (i + 1) * zc_, dimz_, B, zc_, gb_[i].cond + cfg_.shared_dim, cd_, st_));
    }
    // the G linear z0 -> [B, 4, 4, C0] (R10: NHWC view of the 16*C0 vector) and every CBN gain / bias
    // linear of every block, one grouped launch
    CK(gemm_f32_grouped(cbn_fwd_d_, cbn_fwd_n_, cbn_fwd_tiles_, st_));
    CK(convert_f32<T>(h0f_, static_cast<T*>(gb_[0].x), (long long)B * 16 * c0_, st_));
    for (size_t i = 0; i < gb_.size(); ++i) {
      // while D's gradient all-reduce is in flight, the first blocks' persistent grids leave SMs free for it
      g_sm_cap = (pending_d_ && (int)i < overlap_blocks_) ? kNumSMs - overlap_sms_ : kNumSMs;
      GBlock& b = gb_[i];
      const int H = b.hin, H2 = 2 * H;
      // CBN1 -> ReLU -> up x2 (fused)
      CKS(bn_forward_stats(b.x, (long long)B * H * H, b.cin, b.sums1, b.mean1, b.rstd1));
      if (subpix_) {
        // conv3x3(up2(u)) as four 2x2 phase convs of the low-resolution u (2.25x fewer MACs); the
        // upsampled tensor is materialised only when G's backward (conv1 wgrad) will read it
        CK((bn_apply_relu<T, T>(static_cast<const T*>(b.x), B, H, H, b.cin, b.mean1, b.rstd1, b.gain1, b.bias1,
                                nullptr, nullptr, static_cast<T*>(b.u1lo), false, st_)));
        CKS(conv_fwd_up2(b.u1lo, B, H, b.c1, b.h1, G_.P(b.c1.b)));
      } else {
        CK((bn_apply_relu<T, T>(static_cast<const T*>(b.x), B, H, H, b.cin, b.mean1, b.rstd1, b.gain1, b.bias1,
                                nullptr, nullptr, static_cast<T*>(b.u1), true, st_)));
        CKS(conv_fwd(b.u1, B, H2, b.c1, b.h1, G_.P(b.c1.b), nullptr, 0));
      }
      CKS(bn_forward_stats(b.h1, (long long)B * H2 * H2, b.cout, b.sums2, b.mean2, b.rstd2));
      CK((bn_apply_relu<T, T>(static_cast<const T*>(b.h1), B, H2, H2, b.cout, b.mean2, b.rstd2, b.gain2, b.bias2,
                              nullptr, nullptr, static_cast<T*>(b.a2), false, st_)));
      // skip 1x1 before the upsample (commutes), added by conv2's epilogue with x2 nearest indexing
      CKS(conv_fwd(b.x, B, H, b.sc, b.s, G_.P(b.sc.b), nullptr, 0));
      void* out = b.out;
      CKS(conv_fwd(b.a2, B, H2, b.c2, out, G_.P(b.c2.b), b.s, 2));
      if (b.attn) {
        CKS(attn_forward(G_, gattn_, out, B, attn_out_[0]));
        out = attn_out_[0];
      }
    }
    // output layer in fp32: BN -> ReLU -> conv3x3 (96 -> 3) -> tanh
    const long long M = (long long)B * R_ * R_;
    CKS(bn_forward_stats(gout_in_, M, cl_, osums_, omean_, orstd_));
    if constexpr (kBF) {
      if (thin_tc_) {   // on the tensor cores through the bf16 splits of activation and weight (R36)
        CK(bn_apply_relu_split(static_cast<const bf16*>(gout_in_), B, R_, R_, cl_, omean_, orstd_, G_.P(obn_g_),
                               G_.P(obn_b_), reinterpret_cast<bf16*>(aout_), st_));
        CK(timed(6, 2.0 * B * R_ * R_ * 27.0 * cl_, [&] {
          PG_CUDA(split_out_weights(static_cast<const float*>(oconv_.wp), cl_, oconv_ws_, st_));
          return out_conv_fwd_tc(aout_, B, R_, R_, cl_, oconv_ws_, G_.P(oconv_.b), pre_, st_);
        }, "thin fwd"));
        ++launches_;   // two launches in the timed region above
      }
    }
    if (!thin_tc_) {
      CK((bn_apply_relu<T, float>(static_cast<const T*>(gout_in_), B, R_, R_, cl_, omean_, orstd_, nullptr, nullptr,
                                  G_.P(obn_g_), G_.P(obn_b_), aout_, false, st_)));
      CK(timed(6, 2.0 * B * R_ * R_ * 27.0 * cl_, [&] {
        return thin_conv_fwd(aout_, B, R_, R_, cl_, static_cast<const float*>(oconv_.wp), 3, G_.P(oconv_.b), pre_,
                             st_);
      }, "thin fwd"));
    }
    CK(tanh_to_image<T>(pre_, img_, static_cast<T*>(dimg_), M, cpad_, st_));
    return PARAGAN_OK;
  }


  // ================================================================== SN-DCGAN (config 1; R25; fp32 SIMT)
  struct DcD {          // D conv: SN'd, bias, LeakyReLU 0.1
    ConvL c;
    int k = 3, s = 1, hin = 0, hout = 0;
    float *pre = nullptr, *act = nullptr;
  };
  struct DcG {          // G deconv 4x4 s2 p1 (no SN) + BN (learned gamma/beta, cross-replica) + ReLU
    int w = -1, b = -1, g = -1, be = -1;
    int cin = 0, cout = 0, hin = 0, hout = 0;
    float *pre = nullptr, *act = nullptr, *mean = nullptr, *rstd = nullptr;
    double* sums = nullptr;
  };
  std::vector<DcD> dcd_;
  std::vector<DcG> dcg_;
  int dc_lin_w_ = -1, dc_lin_b_ = -1, dc_bn0_g_ = -1, dc_bn0_b_ = -1, dc_out_w_ = -1, dc_out_b_ = -1, dc_f0_ = 0;
  float *dc_h0_ = nullptr, *dc_a0_ = nullptr, *dc_mean0_ = nullptr, *dc_rstd0_ = nullptr, *dc_tmpw_ = nullptr;
  float* dc_g_[2] = {nullptr, nullptr};
  double* dc_sums0_ = nullptr;
  float* dc_z_ = nullptr;
  static constexpr float kLrelu = 0.1f;

  void build_dcgan(Arena& A) {
    const int ch = cfg_.ch;
    B_ = cfg_.local_batch;
    R_ = 32;
    cpad_ = cfg_.c_pad_image;
    dimz_ = 128;
    const int gw[4] = {8 * ch, 4 * ch, 2 * ch, ch};
    const int dw[7] = {ch, ch, 2 * ch, 2 * ch, 4 * ch, 4 * ch, 8 * ch};
    const int dk[7] = {3, 4, 3, 4, 3, 4, 3}, dst[7] = {1, 2, 1, 2, 1, 2, 1};
    dc_f0_ = 16 * gw[0];
    // G, canonical order (no SN); the deconv weight [C_in, C_out, 4, 4] is stored OHWI = [C_in][4][4][C_out],
    // i.e. exactly the conv weight whose adjoint the deconv is
    dc_lin_w_ = G_.add("linear.w", {dc_f0_, dimz_}, false, false);
    dc_lin_b_ = G_.add("linear.b", {dc_f0_}, false, false);
    dc_bn0_g_ = G_.add("bn0.gamma", {dc_f0_}, false, false);
    dc_bn0_b_ = G_.add("bn0.beta", {dc_f0_}, false, false);
    dcg_.clear();
    int h = 4;
    for (int i = 0; i < 3; ++i) {
      DcG L;
      L.cin = gw[i];
      L.cout = gw[i + 1];
      L.hin = h;
      L.hout = 2 * h;
      const std::string k = std::to_string(i + 1);
      L.w = G_.add("deconv" + k + ".w", {L.cin, L.cout, 4, 4}, true, false);
      L.b = G_.add("deconv" + k + ".b", {L.cout}, false, false);
      L.g = G_.add("bn" + k + ".gamma", {L.cout}, false, false);
      L.be = G_.add("bn" + k + ".beta", {L.cout}, false, false);
      dcg_.push_back(L);
      h *= 2;
    }
    dc_out_w_ = G_.add("out_conv.w", {3, gw[3], 3, 3}, true, false);
    dc_out_b_ = G_.add("out_conv.b", {3}, false, false);
    cl_ = gw[3];
    // D, canonical order (SN on every layer)
    dcd_.clear();
    h = R_;
    int cin = 3;
    for (int i = 0; i < 7; ++i) {
      DcD L;
      L.k = dk[i];
      L.s = dst[i];
      L.hin = h;
      L.hout = h / dst[i];
      L.c = conv(D_, "conv" + std::to_string(i + 1), cin, i == 0 ? cpad_ : cin, dw[i], dk[i], true, true);
      dcd_.push_back(L);
      cin = dw[i];
      h = L.hout;
    }
    cdl_ = 16 * dw[6];
    dlin_ = lin(D_, "linear", cdl_, 1, true, true);
    finalize_nets(A);
    size_t maxw = 0;
    for (auto& L : dcd_) {
      const size_t nw = (size_t)L.c.cout * L.c.ksz * L.c.ksz * L.c.cin_x;
      L.c.wp = A.get<float>(nw);
      L.c.wt = A.get<float>(nw);
      maxw = std::max(maxw, nw);
    }
    dlin_.what = A.get<float>((size_t)dlin_.in * dlin_.out);
    dc_tmpw_ = A.get<float>(maxw);
    // activations (fp32)
    const int B = B_, B2 = 2 * B_;
    dimg_ = A.get<float>((size_t)B2 * R_ * R_ * cpad_);
    ylab_ = A.get<int32_t>(B2);
    long long big = (long long)B2 * R_ * R_ * cpad_;
    for (auto& L : dcd_) {
      const long long e = (long long)B2 * L.hout * L.hout * L.c.cout;
      L.pre = A.get<float>(e);
      L.act = A.get<float>(e);
      big = std::max(big, e);
    }
    dc_z_ = A.get<float>((size_t)B * dimz_);
    dc_h0_ = A.get<float>((size_t)B * dc_f0_);
    dc_a0_ = A.get<float>((size_t)B * dc_f0_);
    dc_mean0_ = A.get<float>(dc_f0_);
    dc_rstd0_ = A.get<float>(dc_f0_);
    dc_sums0_ = A.get<double>(2 * dc_f0_);
    for (auto& L : dcg_) {
      const long long e = (long long)B * L.hout * L.hout * L.cout;
      L.pre = A.get<float>(e);
      L.act = A.get<float>(e);
      L.mean = A.get<float>(L.cout);
      L.rstd = A.get<float>(L.cout);
      L.sums = A.get<double>(2 * L.cout);
      big = std::max(big, e);
    }
    big = std::max(big, (long long)B * dc_f0_);
    aout_ = dcg_.back().act;
    pre_ = A.get<float>((size_t)B * R_ * R_ * 3);
    img_ = A.get<float>((size_t)B * R_ * R_ * 3);
    dpre_ = A.get<float>((size_t)B * R_ * R_ * 3);
    for (int i = 0; i < 2; ++i) dc_g_[i] = A.get<float>((size_t)big);
    feat_ = dcd_.back().act;
    logits_ = A.get<float>(B2);
    dlogits_ = A.get<float>(B2);
    maxc_ = dc_f0_;
    ones_buf_ = A.get<float>(maxc_);
    tot_ = A.get<double>(4 * maxc_);
    dpart_ = A.get<double>((size_t)kMaxPartialBlocks * 2 * maxc_);
    scratch_floats_ = std::max<size_t>((size_t)std::max(G_.n, D_.n), (size_t)B * 3 * R_ * R_);
    scratch_floats_ = std::max<size_t>(scratch_floats_, (size_t)4 * 148 * 27 * cl_);
    scratch_f_ = A.get<float>(scratch_floats_);
    alloc_sn_tables(A);
    alloc_opt_tables(A);
  }

  // cross-replica BN (learned gamma/beta) over [M][C] rows, then ReLU
  paragan_status dc_bn_forward(const float* x, long long M, int C, double* sums, float* mean, float* rstd,
                               const float* gamma, const float* beta, float* y) {
    CK(bn_sums_generic(x, M, C, sums, st_));
    CKS(allreduce_small(sums, 2 * C));
    CK(bn_finalize(sums, C, (double)M * cfg_.world_size, cfg_.bn_eps, mean, rstd, st_));
    CK(bn_apply_generic(x, M, C, mean, rstd, gamma, beta, 1, y, st_));
    launches_ += 3;
    return PARAGAN_OK;
  }
  // its backward: dy is the gradient of the ReLU output; writes dgamma / dbeta (local sums) and dx
  paragan_status dc_bn_backward(const float* x, const float* dy, long long M, int C, const float* mean,
                                const float* rstd, int g_entry, int b_entry, float* dx) {
    CK(bn_bwd_sums_generic(x, dy, M, C, mean, rstd, G_.P(g_entry), G_.P(b_entry), 1, tot_, G_.G(g_entry),
                           G_.G(b_entry), st_));
    CKS(allreduce_small(tot_, 2 * C));
    CK(bn_bwd_apply_generic(x, dy, M, C, mean, rstd, G_.P(g_entry), G_.P(b_entry), 1, tot_,
                            (double)M * cfg_.world_size, dx, st_));
    launches_ += 2;
    return PARAGAN_OK;
  }

  paragan_status g_forward_dc(const float* z) {
    const int B = B_;
    CK(cudaMemcpyAsync(zin_dc(), z, sizeof(float) * B * dimz_, cudaMemcpyDeviceToDevice, st_));
    // linear 128 -> 16*8ch, per-feature BN (the [B,1,1,F] view), ReLU; the F vector is NHWC [4,4,8ch] (R10)
    CK(gemm_f32(B, dc_f0_, dimz_, zin_dc(), dimz_, 1, G_.P(dc_lin_w_), dimz_, 1, dc_h0_, dc_f0_, 0.0f,
                G_.P(dc_lin_b_), st_));
    CKS(dc_bn_forward(dc_h0_, B, dc_f0_, dc_sums0_, dc_mean0_, dc_rstd0_, G_.P(dc_bn0_g_), G_.P(dc_bn0_b_),
                      dc_a0_));
    const float* x = dc_a0_;
    for (auto& L : dcg_) {
      // deconv = adjoint of the stride-2 conv with the same weight (OHWI [cin][4][4][cout]), plus bias
      CK(gconv_dgrad(x, B, L.hin, L.hin, L.cin, G_.P(L.w), L.cout, L.cout, 4, 2, 1, L.hout, L.hout, G_.P(L.b),
                     L.pre, st_));
      CKS(dc_bn_forward(L.pre, (long long)B * L.hout * L.hout, L.cout, L.sums, L.mean, L.rstd, G_.P(L.g),
                        G_.P(L.be), L.act));
      x = L.act;
      launches_ += 1;
    }
    CK(thin_conv_fwd(x, B, R_, R_, cl_, G_.P(dc_out_w_), 3, G_.P(dc_out_b_), pre_, st_));
    CK(tanh_to_image<T>(pre_, img_, static_cast<T*>(dimg_), (long long)B * R_ * R_, cpad_, st_));
    launches_ += 3;
    return PARAGAN_OK;
  }
  float* zin_dc() { return dc_z_; }

  paragan_status d_forward_dc(int n) {
    const float* x = static_cast<const float*>(dimg_);
    for (auto& L : dcd_) {
      CK(gconv_fwd(x, n, L.hin, L.hin, L.c.cin_x, static_cast<const float*>(L.c.wp), L.c.cin_x, L.c.cout, L.k, L.s,
                   1, L.hout, L.hout, D_.P(L.c.b), L.pre, st_));
      CK(lrelu_fwd(L.pre, L.act, (long long)n * L.hout * L.hout * L.c.cout, kLrelu, st_));
      x = L.act;
      launches_ += 2;
    }
    // logits = SN-linear(flatten NHWC) + b
    CK(gemm_f32(n, 1, cdl_, feat_, cdl_, 1, dlin_.what, cdl_, 1, logits_, 1, 0.0f, D_.P(dlin_.b), st_));
    ++launches_;
    return PARAGAN_OK;
  }

  paragan_status d_backward_dc(int n, bool want_w, bool want_dimg) {
    float* g = dc_g_[0];
    float* other = dc_g_[1];
    if (want_w) {   // head: dW = dlogit^T feat, db = sum dlogit
      CK(gemm_f32(1, cdl_, n, dlogits_, 1, 1, feat_, 1, cdl_, D_.G(dlin_.w), cdl_, 0.0f, nullptr, st_));
      CK(col_sum<float>(dlogits_, n, 1, dpart_, kMaxPartialBlocks, D_.G(dlin_.b), 0, st_));
    }
    // dfeat[n][k] = dlogit[n] * W_hat[0][k]
    CK(gemm_f32(n, cdl_, 1, dlogits_, 1, 1, dlin_.what, 1, 1, g, cdl_, 0.0f, nullptr, st_));
    for (int i = (int)dcd_.size() - 1; i >= 0; --i) {
      DcD& L = dcd_[i];
      const long long no = (long long)n * L.hout * L.hout * L.c.cout;
      CK(lrelu_bwd(g, L.pre, other, no, kLrelu, st_));
      std::swap(g, other);   // g = d pre
      const float* xin = i == 0 ? static_cast<const float*>(dimg_) : dcd_[i - 1].act;
      if (want_w) {
        const bool pad = L.c.cin_x != L.c.cin;
        float* dst = pad ? dc_tmpw_ : D_.G(L.c.w);
        CK(gconv_wgrad(xin, n, L.hin, L.hin, L.c.cin_x, g, L.hout, L.hout, L.c.cout, L.k, L.s, 1, dst, st_));
        if (pad)
          CK(copy_rows_cols(dst, L.c.cin_x, (long long)L.c.cout * L.k * L.k, L.c.cin, D_.G(L.c.w), L.c.cin, 0, st_));
        CK(col_sum<float>(g, (long long)n * L.hout * L.hout, L.c.cout, dpart_, kMaxPartialBlocks, D_.G(L.c.b), 0, st_));
        launches_ += 3;
      }
      if (i > 0 || want_dimg) {
        CK(gconv_dgrad(g, n, L.hout, L.hout, L.c.cout, static_cast<const float*>(L.c.wp), L.c.cin_x, L.c.cin_x, L.k,
                       L.s, 1, L.hin, L.hin, nullptr, other, st_));
        std::swap(g, other);
        ++launches_;
      }
    }
    dimg_grad_ = want_dimg ? g : nullptr;   // [n][32][32][c_pad] gradient of the D input
    return PARAGAN_OK;
  }

  paragan_status g_backward_dc() {
    const int B = B_;
    const long long M = (long long)B * R_ * R_;
    CK(tanh_bwd<T>(static_cast<const T*>(dimg_grad_), cpad_, img_, dpre_, M, st_));
    CK(thin_conv_wgrad(aout_, dpre_, B, R_, R_, cl_, 3, G_.G(dc_out_w_), scratch_f_, scratch_floats_, st_));
    CK(col_sum<float>(dpre_, M, 3, dpart_, kMaxPartialBlocks, G_.G(dc_out_b_), 0, st_));
    float* g = (dimg_grad_ == dc_g_[0]) ? dc_g_[1] : dc_g_[0];
    float* other = (g == dc_g_[0]) ? dc_g_[1] : dc_g_[0];
    CK(thin_conv_dgrad(dpre_, B, R_, R_, cl_, G_.P(dc_out_w_), 3, g, st_));
    launches_ += 4;
    for (int i = (int)dcg_.size() - 1; i >= 0; --i) {
      DcG& L = dcg_[i];
      const long long Mo = (long long)B * L.hout * L.hout;
      CKS(dc_bn_backward(L.pre, g, Mo, L.cout, L.mean, L.rstd, L.g, L.be, other));
      std::swap(g, other);   // g = d(deconv output)
      const float* xin = i == 0 ? dc_a0_ : dcg_[i - 1].act;
      // deconv wgrad: the conv wgrad with the roles of input and output exchanged
      CK(gconv_wgrad(g, B, L.hout, L.hout, L.cout, xin, L.hin, L.hin, L.cin, 4, 2, 1, G_.G(L.w), st_));
      CK(col_sum<float>(g, Mo, L.cout, dpart_, kMaxPartialBlocks, G_.G(L.b), 0, st_));
      // deconv input gradient = the strided conv of g with the same weight
      CK(gconv_fwd(g, B, L.hout, L.hout, L.cout, G_.P(L.w), L.cout, L.cin, 4, 2, 1, L.hin, L.hin, nullptr, other, st_));
      std::swap(g, other);
      launches_ += 3;
    }
    CKS(dc_bn_backward(dc_h0_, g, B, dc_f0_, dc_mean0_, dc_rstd0_, dc_bn0_g_, dc_bn0_b_, other));
    // linear: dW = dh0^T z, db = sum dh0
    CK(gemm_f32(dc_f0_, dimz_, B, other, 1, dc_f0_, zin_dc(), 1, dimz_, G_.G(dc_lin_w_), dimz_, 0.0f, nullptr, st_));
    CK(col_sum<float>(other, B, dc_f0_, dpart_, kMaxPartialBlocks, G_.G(dc_lin_b_), 0, st_));
    launches_ += 2;
    return PARAGAN_OK;
  }
  // ------------------------------------------------------------------ attention (A6)
  TcAttnArgs attn_args(const AttnL& a, int n) {
    TcAttnArgs t{};
    t.n = n;
    t.HW = a.H * a.H;
    t.Q = t.HW / 4;
    t.Cq = a.Cq;
    t.C2 = a.C2;
    t.Ct = a.Ct;
    t.qkv = a.qkv;
    t.phi = a.phi_p;
    t.gp = a.g_p;
    t.gT = a.gT;
    t.o = a.ov;
    t.o32 = a.o32;
    t.lse = a.lse;
    t.Dr = a.Dr;
    t.phimax = attn_single_ ? a.phimax : nullptr;
    t.thetamax = attn_single_ && attn_flat_ ? a.thetamax : nullptr;
    return t;
  }
  paragan_status attn_forward(Net& N, AttnL& a, const void* x, int n, void* out) {
    const int H = a.H;
    const long long HW = (long long)H * H, Q = HW / 4;
    {
      TcEpilogue e;
      e.out = a.qkv;
      if constexpr (kBF) {
        CK(tc_conv_fprop(x, n, H, H, a.C, a.qkv_wp, a.Ct, 1, e, st_));
      } else {
        CK((simt_conv_fwd<float, float, float>(static_cast<const float*>(x), n, H, H, a.C,
                                               static_cast<const float*>(a.qkv_wp), a.Ct, 1, nullptr, nullptr, nullptr,
                                               0, static_cast<float*>(a.qkv), st_)));
      }
    }
    const T* qkv = static_cast<const T*>(a.qkv);
    // pooled phi keeps the zero channels C/8..Cq (the theta / phi rows of the packed weight beyond C/8 are zero)
    CK(maxpool2_split<T>(qkv, n, H, H, a.Ct, a.Cq, a.Cq, static_cast<T*>(a.phi_p), nullptr, st_));
    CK(maxpool2_split<T>(qkv, n, H, H, a.Ct, 2 * a.Cq, a.C2, static_cast<T*>(a.g_p), nullptr, st_));
    if (a.fused) {
      CK(attn_transpose(a.g_p, n, (int)Q, a.C2, a.gT, st_));
      CK(attn_phimax(a.phi_p, n, (int)Q, a.Cq, a.phimax, st_));
      ++launches_;   // two kernels (max, square root)
      if (attn_flat_) {
        CK(attn_thetamax(a.qkv, n, (int)HW, a.Cq, a.Ct, a.thetamax, st_));
        ++launches_;
      }
      TcAttnArgs t = attn_args(a, n);
      CK(timed(5, 2.0 * n * HW * Q * (double)(a.Cq + a.C2), [&] { return tc_attn_fwd(t, st_); }, "attn fwd"));
    } else {
      // S = theta phi^T  [n][HW][Q] fp32
      CKS(bgemm(n, (int)HW, (int)Q, a.Cq, qkv, HW * a.Ct, a.Ct, 1, a.phi_p, Q * a.Cq, a.Cq, 1, a.S, true, HW * Q, Q));
      CK(softmax_rows<T>(a.S, n * HW, (int)Q, static_cast<T*>(a.P), st_));
      // o = beta g  [n][HW][C2]
      CKS(bgemm(n, (int)HW, a.C2, (int)Q, a.P, HW * Q, Q, 1, a.g_p, Q * a.C2, 1, a.C2, a.ov, !kBF, HW * a.C2, a.C2));
    }
    // out = x + gamma * conv1x1(o)
    CKS(conv_fwd(a.ov, n, H, a.oc, out, nullptr, x, 1, N.P(a.gamma)));
    return PARAGAN_OK;
  }
  // dout -> dx (= dout + attention path), weight grads when want_w
  paragan_status attn_backward(Net& N, AttnL& a, const void* x, int n, const void* dout, void* dx, bool want_w) {
    const int H = a.H;
    const long long HW = (long long)H * H, Q = HW / 4;
    const long long M = n * HW;
    void* dO = tmp_attn_dO_;
    void* dqkv = tmp_attn_dqkv_;
    if (want_w) {
      // G_o = wgrad(o, dout) unscaled; dgamma = <W_o/sigma, G_o>; dW_o_hat = gamma * G_o
      float* go = N.G(a.oc.w);
      CKS(conv_wgrad(N, a.ov, dout, n, H, a.oc));
      // dgamma against the very operand the forward used (W_o/sigma as packed, bf16 in BF16 mode)
      if constexpr (kBF) {
        CK(dot_bf16_f32(static_cast<const bf16*>(a.oc.wp), go, (long long)a.C * a.C2, N.G(a.gamma), 0, st_));
      } else {
        CK(dot_f32(static_cast<const float*>(a.oc.wp), go, (long long)a.C * a.C2, N.G(a.gamma), 0, st_));
      }
      CK(scale_dev(go, (long long)a.C * a.C2, N.P(a.gamma), st_));
    }
    CKS(conv_dgrad(dout, n, H, a.oc, dO, nullptr, N.P(a.gamma)));   // dO = gamma * W_o^T dout
    if (a.fused) {
      float* dgp = dpool_;
      float* dph = dpool_ + (size_t)n * Q * a.C2;
      CK(attn_rowdot(dO, a.o32, M, a.C2, a.Dr, st_));
      TcAttnArgs t = attn_args(a, n);
      t.dO = dO;
      t.dgp = dgp;
      t.dphi = dph;
      t.dth_part = dth_part_;
      CK(timed(5, 2.0 * n * HW * Q * (double)(3 * a.Cq + 2 * a.C2), [&] { return tc_attn_bwd(t, st_); }, "attn bwd"));
      // every channel of dqkv is written below: theta [0,Cq), phi [Cq,2Cq), g [2Cq,2Cq+C2)
      CK(attn_dtheta_reduce(dth_part_, (int)(Q / 128), M, a.Cq, dqkv, a.Ct, st_));
      CK(maxpool2_split_bwd<T>(static_cast<const T*>(a.qkv), n, H, H, a.Ct, a.Cq, a.Cq, dph, static_cast<T*>(dqkv),
                               st_));
      CK(maxpool2_split_bwd<T>(static_cast<const T*>(a.qkv), n, H, H, a.Ct, 2 * a.Cq, a.C2, dgp,
                               static_cast<T*>(dqkv), st_));
      return attn_qkv_backward(N, a, x, n, dout, dx, dqkv, want_w);
    }
    float* dP = dP_;
    // dgp = P^T dO  [n][Q][C2] fp32 ; dP = dO gp^T [n][HW][Q] fp32
    float* dgp = dpool_;
    CKS(bgemm(n, (int)Q, a.C2, (int)HW, a.P, HW * Q, 1, Q, dO, HW * a.C2, 1, a.C2, dgp, true, Q * a.C2, a.C2));
    CKS(bgemm(n, (int)HW, (int)Q, a.C2, dO, HW * a.C2, a.C2, 1, a.g_p, Q * a.C2, a.C2, 1, dP, true, HW * Q, Q));
    // dS with P recomputed in fp32 from the kept scores (gradients kept in higher precision)
    CK(softmax_bwd_rows<T>(a.S, dP, M, (int)Q, static_cast<T*>(a.P), st_));  // P <- dS
    const void* dS = a.P;
    CK(cudaMemsetAsync(dqkv, 0, sizeof(T) * (size_t)M * a.Ct, st_));
    // dtheta = dS phi_p -> dqkv[:, 0:Cq]
    CKS(bgemm(n, (int)HW, a.Cq, (int)Q, dS, HW * Q, Q, 1, a.phi_p, Q * a.Cq, 1, a.Cq, dqkv, false, HW * a.Ct, a.Ct));
    // dphi_p = dS^T theta [n][Q][Cq] fp32
    float* dph = dpool_ + (size_t)n * Q * a.C2;
    CKS(bgemm(n, (int)Q, a.Cq, (int)HW, dS, HW * Q, 1, Q, a.qkv, HW * a.Ct, 1, a.Ct, dph, true, Q * a.Cq, a.Cq));
    CK(maxpool2_split_bwd<T>(static_cast<const T*>(a.qkv), n, H, H, a.Ct, a.Cq, a.Cq, dph, static_cast<T*>(dqkv), st_));
    CK(maxpool2_split_bwd<T>(static_cast<const T*>(a.qkv), n, H, H, a.Ct, 2 * a.Cq, a.C2, dgp, static_cast<T*>(dqkv),
                             st_));
    return attn_qkv_backward(N, a, x, n, dout, dx, dqkv, want_w);
  }
  // dx = dout + W_qkv^T dqkv; the theta / phi / g weight gradients
  paragan_status attn_qkv_backward(Net& N, AttnL& a, const void* x, int n, const void* dout, void* dx, void* dqkv,
                                   bool want_w) {
    const int H = a.H;
    ConvL q;
    q.cin = a.C;
    q.cin_x = a.C;
    q.cout = a.Ct;
    q.ksz = 1;
    q.wp = a.qkv_wp;
    q.wt = a.qkv_wt;
    CKS(conv_dgrad(dqkv, n, H, q, dx, dout));
    if (want_w) {
      // wgrad of the packed qkv conv, then scatter the real rows to theta / phi / g
      if constexpr (kBF) {
        CK(tc_conv_wgrad(x, dqkv, n, H, H, a.C, a.Ct, 1, wg_scratch_, 0, scratch_f_, scratch_floats_, st_));
      } else {
        CK((simt_conv_wgrad<float, float>(static_cast<const float*>(x), static_cast<const float*>(dqkv), n, H, H, a.C,
                                          a.Ct, 1, wg_scratch_, 0, st_, scratch_f_, scratch_floats_)));
      }
      CK(copy_rows_cols(wg_scratch_, a.C, a.C8, a.C, N.G(a.th), a.C, 0, st_));
      CK(copy_rows_cols(wg_scratch_ + (size_t)a.Cq * a.C, a.C, a.C8, a.C, N.G(a.ph), a.C, 0, st_));
      CK(copy_rows_cols(wg_scratch_ + (size_t)2 * a.Cq * a.C, a.C, a.C2, a.C, N.G(a.gg), a.C, 0, st_));
    }
    return PARAGAN_OK;
  }

  // ------------------------------------------------------------------ D forward (A7)
  // R38: out = 0.25 * up2^T(conv3x3^T_K(r1)) + b + skip at half resolution (K = conv2's flipped, transposed kernel
  // folded per phase): conv2 + 2x2 average pool as a 16-tap stride-2 conv over the four input phases of r1
  paragan_status pool_fwd_conv(DBlock& b, int n, const void* skip) {
    const int H = b.hin, Ho = b.hout;
    TcEpilogue e;
    e.alpha = quarter_;
    e.bias = D_.P(b.c2.b);
    e.residual = skip;
    e.res_mode = 1;
    e.out = b.out;
    const double fl = 2.0 * n * H * H * 9.0 * b.cout * b.cout;
    const double fx = 2.0 * n * Ho * Ho * 16.0 * b.cout * b.cout;
    char what[48];
    std::snprintf(what, sizeof(what), "fwd-pool n%d %dx%d %d->%d", n, H, H, b.cout, b.cout);
    CK(timed(0, fl, [&] { return tc_conv_dgrad_up2(b.r1, n, Ho, Ho, b.cout, b.wp4f, b.cout, e, st_); }, what, fx));
    return PARAGAN_OK;
  }
  paragan_status d_forward(int n) {
    // D's W/sigma of this step folded for the pooled blocks: conv2's input gradient (R37, used by d_backward
    // with the same weights) and the pooled forward (R38)
    if (fold_njobs_dd_) CK(fold_up2_grouped(fold_jobs_dd_, fold_njobs_dd_, fold_tiles_dd_, pool_fwd_, st_));
    bool rx_ready = false;   // the previous block's pooling already wrote relu(x) into this block's rx
    for (size_t j = 0; j < db_.size(); ++j) {
      DBlock& b = db_[j];
      const int H = b.hin, Ho = b.hout;
      const long long Mi = (long long)n * H * H;
      const void* cin = b.x;
      // the next block's pre-activation relu(x) comes out of this block's pooling when nothing sits in between
      T* next_rx = (j + 1 < db_.size() && !b.attn) ? static_cast<T*>(db_[j + 1].rx) : nullptr;
      bool xp_ready = false;   // R38 blocks: avgpool2(x) for the half-resolution shortcut
      if (j > 0) {
        if (!rx_ready && b.wp4f && b.cin_x % 8 == 0) {
          // relu(x) for conv1 and avgpool2(x) for the shortcut from one read of x (bit-identical to the two passes)
          CK(avgpool2<T>(static_cast<const T*>(b.x), n, H, H, b.cin_x, b.cin_x, nullptr, static_cast<T*>(b.xp), st_,
                         nullptr, static_cast<T*>(b.rx)));
          xp_ready = true;
        } else if (!rx_ready) {
          CK(relu_copy<T>(static_cast<const T*>(b.x), static_cast<T*>(b.rx), Mi * b.cin_x, st_));
        }
        cin = b.rx;
      }
      rx_ready = false;
      // conv1 with the ReLU that feeds conv2 fused into its epilogue (kBF); the fp32 path keeps a separate pass
      if (b.im2col) {
        CK(im2col3<T>(static_cast<const T*>(b.x), n, H, H, b.cin_x, static_cast<T*>(b.xi), st_));
        CKS(conv_fwd(b.xi, n, H, b.c1x, kBF ? b.r1 : b.c1o, D_.P(b.c1.b), nullptr, 0, nullptr, kBF));
      } else {
        CKS(conv_fwd(cin, n, H, b.c1, kBF ? b.r1 : b.c1o, D_.P(b.c1.b), nullptr, 0, nullptr, kBF));
      }
      if (!kBF) CK(relu_copy<T>(static_cast<const T*>(b.c1o), static_cast<T*>(b.r1), Mi * b.cout, st_));
      if (j == 0 && b.down) {
        // skip: avgpool the image, then 1x1 conv (block 0 has no pre-activation)
        CK(avgpool2<T>(static_cast<const T*>(b.x), n, H, H, b.cin_x, b.cin_x, nullptr, static_cast<T*>(b.xp), st_));
        CKS(conv_fwd(b.xp, n, Ho, b.sc, b.s, D_.P(b.sc.b), nullptr, 0));
        if (b.wp4f) {
          if constexpr (kBF) CKS(pool_fwd_conv(b, n, b.s));   // R38
        } else {
          CKS(conv_fwd(b.r1, n, H, b.c2, b.t, D_.P(b.c2.b), nullptr, 0));
          CK(avgpool2<T>(static_cast<const T*>(b.t), n, H, H, b.cout, b.cout, static_cast<const T*>(b.s),
                         static_cast<T*>(b.out), st_, next_rx));
          rx_ready = next_rx != nullptr;
        }
      } else if (b.wp4f) {
        // R38: avgpool(conv2(r1) + sc(x) + b) = conv2 at stride 2 folded into 16 taps over the four input phases
        // (x 0.25 in the epilogue) + sc(avgpool(x)) + b, all at half resolution: 16 / 4 = 4 full-resolution taps
        // of MACs instead of 9, and the 1x1 shortcut on a quarter of the pixels
        if (!xp_ready)
          CK(avgpool2<T>(static_cast<const T*>(b.x), n, H, H, b.cin_x, b.cin_x, nullptr, static_cast<T*>(b.xp), st_));
        CKS(conv_fwd(b.xp, n, Ho, b.sc, b.s, D_.P(b.sc.b), nullptr, 0));
        if constexpr (kBF) CKS(pool_fwd_conv(b, n, b.s));
      } else {
        const void* skip = b.x;
        if (b.learn_sc) {
          CKS(conv_fwd(b.x, n, H, b.sc, b.s, D_.P(b.sc.b), nullptr, 0));
          skip = b.s;
        }
        if (b.down && kBF && pool_fuse_ && H <= 64 && b.cout % 16 == 0) {
          // conv2 + skip + 2x2 average pooling (+ the next block's relu) in one epilogue: the full-resolution
          // sum never reaches HBM (bit-identical to conv2 -> avgpool2)
          CKS(conv_fwd(b.r1, n, H, b.c2, nullptr, D_.P(b.c2.b), skip, 1, nullptr, false, b.out, next_rx));
          rx_ready = next_rx != nullptr;
        } else if (b.down) {
          CKS(conv_fwd(b.r1, n, H, b.c2, b.t, D_.P(b.c2.b), skip, 1));
          CK(avgpool2<T>(static_cast<const T*>(b.t), n, H, H, b.cout, b.cout, nullptr, static_cast<T*>(b.out), st_,
                         next_rx));
          rx_ready = next_rx != nullptr;
        } else {
          CKS(conv_fwd(b.r1, n, H, b.c2, b.out, D_.P(b.c2.b), skip, 1));
        }
      }
      if (b.attn) CKS(attn_forward(D_, dattn_, b.out, n, attn_out_[1]));
    }
    const DBlock& last = db_.back();
    const void* hlast = last.attn ? attn_out_[1] : last.out;
    CK(d_head_fwd<T>(static_cast<const T*>(hlast), n, hl_ * hl_, cdl_, dlin_.what, D_.P(dlin_.b), demb_hat_, ylab_,
                     feat_, logits_, st_));
    return PARAGAN_OK;
  }

  // ------------------------------------------------------------------ D backward (A8-A11)
  // want_w: weight grads (D step); want_dimg: gradient down to the image (G step)
  paragan_status d_backward(int n, bool want_w, bool want_dimg) {
    const DBlock& last = db_.back();
    const void* hlast = last.attn ? attn_out_[1] : last.out;
    void* cur = tmp(0);   // gradient w.r.t. the current block output
    CK(d_head_bwd<T>(static_cast<const T*>(hlast), n, hl_ * hl_, cdl_, dlin_.what, demb_hat_, ylab_, feat_, dlogits_,
                     static_cast<T*>(cur), D_.G(dlin_.w), D_.G(dlin_.b), D_.G(demb_), cfg_.n_classes, want_w, st_));
    int ic = 0;   // index of cur in tmp_
    auto other = [&](int a_, int b_ = -1, int c_ = -1) {
      for (int k = 0; k < 4; ++k)
        if (k != a_ && k != b_ && k != c_) return k;
      return -1;
    };
    for (int j = (int)db_.size() - 1; j >= 0; --j) {
      DBlock& b = db_[j];
      const int H = b.hin, Ho = b.hout;
      if (b.attn) {
        const int k = other(ic);
        CKS(attn_backward(D_, dattn_, b.out, n, cur, tmp(k), want_w));
        ic = k;
        cur = tmp(k);
      }
      // dt: gradient at the conv2 output (full res) = up2(cur) / 4 behind the pool.  With the phase kernel
      // (R37) conv2's input gradient is conv3x3^T(up2(cur)) / 4 straight from the pooled gradient, and dt is
      // only materialised for the weight gradients
      const bool pool_dg = b.down && b.wp4dg != nullptr && b.dg_phase;
      int it;
      void* dt;
      if (b.down) {
        it = other(ic);
        dt = tmp(it);
        if (!pool_dg || want_w)
          CK(avgpool2_bwd<T>(static_cast<const T*>(cur), n, H, H, b.cout, nullptr, static_cast<T*>(dt), b.cout, st_));
      } else {
        it = ic;
        dt = cur;
      }
      // conv2 backward
      const int ir1 = other(ic, it);
      void* dr1 = tmp(ir1);
      // gradient at the conv1 output: dgrad(conv2) masked by relu'(c1) in the epilogue
      if (pool_dg) {
        if constexpr (kBF) {
          TcEpilogue e;
          e.alpha = quarter_;
          e.relu_ref = b.r1;
          e.out = dr1;
          const double fl = 2.0 * n * H * H * 9.0 * b.cout * b.cout;
          const double fx = 2.0 * n * Ho * Ho * 16.0 * b.cout * b.cout;
          char what[48];
          std::snprintf(what, sizeof(what), "dgrad-pool n%d %dx%d %d->%d", n, H, H, b.cout, b.cout);
          CK(timed(0, fl, [&] { return tc_conv_fprop_up2(cur, n, Ho, Ho, b.cout, b.wp4dg, b.cout, e, st_); }, what,
                   fx));
        }
      } else {
        CKS(conv_dgrad(dt, n, H, b.c2, dr1, nullptr, nullptr, b.r1));
      }
      if (want_w) {
        CKS(conv_wgrad(D_, b.r1, dt, n, H, b.c2, b.c2.b));
      }
      // skip branch
      const bool need_dx = (j > 0) || want_dimg;
      int isk = -1;
      void* dskip = nullptr;
      bool dskip_half = false;   // dskip at half resolution (nearest-upsampled by the consumer's epilogue)
      if (j == 0 && b.down) {
        // s = sc(avgpool(x)) at half res; its gradient is cur (half res)
        if (want_w) {
          CKS(conv_wgrad(D_, b.xp, cur, n, Ho, b.sc, b.sc.b));
        }
        if (need_dx) {
          isk = other(ic, it, ir1);
          // dxp (half res) into the tail of tmp(isk), then avgpool adjoint into tmp(isk) head
          void* dxp = dxp_;
          CKS(conv_dgrad(cur, n, Ho, b.sc, dxp, nullptr));
          CK(avgpool2_bwd<T>(static_cast<const T*>(dxp), n, H, H, b.cin_x, nullptr, static_cast<T*>(tmp(isk)),
                             b.cin_x, st_));
          dskip = tmp(isk);
        }
      } else if (b.learn_sc) {
        if (want_w) {
          // with the pooled forward (R38) avgpool(x) is resident: sum_full (up2(cur)/4) x = sum_half cur avgpool(x),
          // the 1x1 weight gradient on a quarter of the pixels
          if (b.wp4f) CKS(conv_wgrad(D_, b.xp, cur, n, Ho, b.sc, b.sc.b));
          else CKS(conv_wgrad(D_, b.x, dt, n, H, b.sc, b.sc.b));
        }
        if (need_dx) {
          isk = other(ic, it, ir1);
          if (kBF && b.down && b.sc.ksz == 1) {
            // the 1x1 shortcut's input gradient commutes with the pool's adjoint: sc^T(up2(cur) / 4) =
            // up2(sc^T(cur)) / 4, computed at half resolution (x 0.25 in the epilogue, exact) and added by conv1's
            // dgrad epilogue through the half-resolution residual mode — bit-identical, 4x fewer bytes and MACs
            CKS(conv_dgrad(cur, n, Ho, b.sc, tmp(isk), nullptr, quarter_));
            dskip_half = true;
          } else {
            CKS(conv_dgrad(dt, n, H, b.sc, tmp(isk), nullptr));
          }
          dskip = tmp(isk);
        }
      } else {
        dskip = dt;   // identity skip
        isk = it;
      }
      const void* cin = (j > 0) ? b.rx : b.x;
      if (want_w) {
        if (b.im2col) CKS(conv_wgrad(D_, b.xi, dr1, n, H, b.c1x, b.c1.b));
        else CKS(conv_wgrad(D_, cin, dr1, n, H, b.c1, b.c1.b));
      }
      if (!need_dx) break;
      // dx = relu'(x) * dgrad(conv1) + dskip   (block 0: no pre-activation)
      int ix = -1;
      for (int k = 0; k < 4; ++k)
        if (k != ir1 && k != isk) { ix = k; break; }
      void* dx = tmp(ix);
      if (j > 0) {   // pre-activation block: relu'(x) mask and the skip gradient fused in the epilogue
        CKS(conv_dgrad(dr1, n, H, b.c1, dx, dskip, nullptr, b.x, dskip_half ? 2 : 1));
      } else if (b.im2col) {
        // dgrad into the im2col buffer (no longer needed), then its adjoint (col2im) + skip gradient
        CKS(conv_dgrad(dr1, n, H, b.c1x, b.xi, nullptr));
        CK(col2im3<T>(static_cast<const T*>(b.xi), n, H, H, b.cin_x, static_cast<const T*>(dskip), static_cast<T*>(dx),
                      st_));
      } else {
        CKS(conv_dgrad(dr1, n, H, b.c1, dx, dskip));
      }
      cur = dx;
      ic = ix;
    }
    dimg_grad_ = want_dimg ? cur : nullptr;
    dimg_idx_ = ic;
    return PARAGAN_OK;
  }

  // ------------------------------------------------------------------ G backward (A9-A11)
  paragan_status g_backward() {
    const int B = B_;
    const long long M = (long long)B * R_ * R_;
    // tanh' and the fp32 output conv
    CK(tanh_bwd<T>(static_cast<const T*>(dimg_grad_), cpad_, img_, dpre_, M, st_));
    if (thin_tc_) {   // both gradients in one tensor-core pass over the split activation (R36)
      CK(timed(6, 2 * 2.0 * B * R_ * R_ * 27.0 * cl_, [&] {
        PG_CUDA(split_out_weights_dgrad(static_cast<const float*>(oconv_.wp), cl_, round_up(cl_, 16), oconv_wd_,
                                        st_));
        return out_conv_bwd_tc(aout_, dpre_, B, R_, R_, cl_, oconv_wd_, daout_, G_.G(oconv_.w), scratch_f_,
                               scratch_floats_, st_);
      }, "thin bwd"));
      launches_ += 2;   // three launches in the timed region above
      CK(col_sum<float>(dpre_, M, 3, dpart_, kMaxPartialBlocks, G_.G(oconv_.b), 0, st_));
    } else {
      CK(timed(6, 2.0 * B * R_ * R_ * 27.0 * cl_, [&] {
        return thin_conv_wgrad(aout_, dpre_, B, R_, R_, cl_, 3, G_.G(oconv_.w), scratch_f_, scratch_floats_, st_);
      }, "thin wgrad"));
      CK(col_sum<float>(dpre_, M, 3, dpart_, kMaxPartialBlocks, G_.G(oconv_.b), 0, st_));
      CK(timed(6, 2.0 * B * R_ * R_ * 27.0 * cl_, [&] {
        return thin_conv_dgrad(dpre_, B, R_, R_, cl_, static_cast<const float*>(oconv_.wp), 3, daout_, st_);
      }, "thin dgrad"));
    }
    // output BN backward (plain BN, learned gamma/beta)
    int ic = (dimg_idx_ + 1) % 4;
    void* cur = tmp(ic);
    CK((bn_bwd_reduce<T, float>(static_cast<const T*>(gout_in_), daout_, B, R_, R_, cl_, omean_, orstd_, nullptr,
                                nullptr, G_.P(obn_g_), G_.P(obn_b_), false, bn_part_, bn_chunks(R_ * R_), ab_, st_)));
    // dgamma[c] = sum_n Bv[n][c], dbeta[c] = sum_n A[n][c]: channel totals with unit gain
    CK(bn_bwd_totals(ab_, B, cl_, nullptr, ones_(cl_), tot_, st_));
    CK(to_f32_from_d(tot_, G_.G(obn_b_), cl_));
    CK(to_f32_from_d(tot_ + cl_, G_.G(obn_g_), cl_));
    CK(bn_bwd_totals(ab_, B, cl_, nullptr, G_.P(obn_g_), tot_, st_));
    CKS(allreduce_small(tot_, 2 * cl_));
    CK((bn_bwd_apply<T, float, T>(static_cast<const T*>(gout_in_), daout_, B, R_, R_, cl_, omean_, orstd_, nullptr,
                                  nullptr, G_.P(obn_g_), G_.P(obn_b_), false, tot_, (double)M * cfg_.world_size,
                                  nullptr, static_cast<T*>(cur), st_)));
    for (int i = (int)gb_.size() - 1; i >= 0; --i) {
      GBlock& b = gb_[i];
      const int H = b.hin, H2 = 2 * H;
      if (b.attn) {
        const int k = (ic + 1) % 4;
        CKS(attn_backward(G_, gattn_, b.out, B, cur, tmp(k), true));
        ic = k;
        cur = tmp(k);
      }
      const int i_a2 = (ic + 1) % 4, i_ds = (ic + 2) % 4, i_dxs = (ic + 3) % 4;
      // conv2
      CKS(conv_dgrad(cur, B, H2, b.c2, tmp(i_a2), nullptr));
      CKS(conv_wgrad(G_, b.a2, cur, B, H2, b.c2, b.c2.b));
      // skip: out += up2(s) -> ds = 2x2 sum of dout
      CK(up2_bwd<T>(static_cast<const T*>(cur), B, H, H, b.cout, static_cast<T*>(tmp(i_ds)), st_));
      CKS(conv_wgrad(G_, b.x, tmp(i_ds), B, H, b.sc, b.sc.b));
      CKS(conv_dgrad(tmp(i_ds), B, H, b.sc, tmp(i_dxs), nullptr));
      // CBN2 backward: da2 -> dh1 (into cur's buffer)
      CKS(cbn_backward(b.h1, tmp(i_a2), B, H2, b.cout, b.mean2, b.rstd2, b.gain2, b.bias2, false, nullptr, cur,
                       b.ab2));
      if (subpix_) {
        // conv1 through the phase decomposition: dW from the low-resolution input, and the input
        // gradient at low resolution with the upsample's adjoint included
        CKS(conv_wgrad_up2(b.u1lo, cur, B, H, b.c1));
        CKS(conv_dgrad_up2(cur, B, H, b.c1, tmp(i_a2)));
        CKS(cbn_backward(b.x, tmp(i_a2), B, H, b.cin, b.mean1, b.rstd1, b.gain1, b.bias1, false, tmp(i_dxs),
                         tmp(i_ds), b.ab1));
      } else {
        // conv1 on the upsampled activation
        CKS(conv_wgrad(G_, b.u1, cur, B, H2, b.c1, b.c1.b));
        CKS(conv_dgrad(cur, B, H2, b.c1, tmp(i_a2), nullptr));
        // CBN1 backward through the upsample (2x2 sum), plus the skip gradient
        CKS(cbn_backward(b.x, tmp(i_a2), B, H, b.cin, b.mean1, b.rstd1, b.gain1, b.bias1, true, tmp(i_dxs),
                         tmp(i_ds), b.ab1));
      }
      ic = i_ds;
      cur = tmp(ic);
    }
    // CBN linears: every dW, then every block's dcond (sum over its four linears), one launch each
    CK(gemm_f32_grouped(cbn_dw_d_, cbn_dw_n_, cbn_dw_tiles_, st_));
    CK(gemm_f32_grouped(cbn_dcond_d_, cbn_dcond_n_, cbn_dcond_tiles_, st_));
    for (GBlock& b : gb_) CK(sum_slices(b.dcond_part, b.dcond_nslot, B * cd_, b.dcond, st_));
    // cond -> shared embedding gradient (first shared_dim columns), blocks in order
    for (size_t i0 = 0; i0 < gb_.size(); i0 += 8) {
      RowSrcs rs{};
      for (size_t i = i0; i < gb_.size() && i < i0 + 8; ++i) rs.p[rs.n++] = gb_[i].dcond;
      CK(scatter_add_rows_multi(rs, cd_, yg_, B, cfg_.shared_dim, cfg_.n_classes, G_.G(shared_), st_));
    }
    // G linear: h0 = z0 W^T + b
    CK(to_f32<T>(static_cast<const T*>(cur), dh0f_, (long long)B * 16 * c0_, st_));
    CK(gemm_f32(16 * c0_, zc_, B, dh0f_, 1, 16 * c0_, zin_, 1, dimz_, G_.G(glin_.w), zc_, 0.0f, nullptr, st_));
    CK(col_sum<float>(dh0f_, B, 16 * c0_, dpart_, kMaxPartialBlocks, G_.G(glin_.b), 0, st_));
    return PARAGAN_OK;
  }
  // conditional BN backward; writes dx (+ add), per-sample gain/bias grads into the CBN linears and dcond
  paragan_status cbn_backward(const void* x, const void* dy, int n, int H, int C, const float* mean, const float* rstd,
                              const float* gain, const float* bias, bool up2, const void* add, void* dx, float* ab) {
    CK((bn_bwd_reduce<T, T>(static_cast<const T*>(x), static_cast<const T*>(dy), n, H, H, C, mean, rstd, gain, bias,
                            nullptr, nullptr, up2, bn_part_, bn_chunks(H * H), ab, st_)));
    CK(bn_bwd_totals(ab, n, C, gain, nullptr, tot_, st_));
    CKS(allreduce_small(tot_, 2 * C));
    CK((bn_bwd_apply<T, T, T>(static_cast<const T*>(x), static_cast<const T*>(dy), n, H, H, C, mean, rstd, gain, bias,
                              nullptr, nullptr, up2, tot_, (double)n * H * H * cfg_.world_size,
                              static_cast<const T*>(add), static_cast<T*>(dx), st_)));
    // AB[n][0:C] = dbias (sum g0), AB[n][C:2C] = dgain (sum g0 * x_hat): consumed by the grouped
    // CBN-linear GEMMs at the end of g_backward
    return PARAGAN_OK;
  }
  int bn_chunks(long long hw) const {
    long long c = (hw + 1023) / 1024;
    if (c < 1) c = 1;
    if (c > 64) c = 64;
    return (int)c;
  }
  const float* ones_(int C) {
    (void)C;
    return ones_buf_;
  }
  cudaError_t to_f32_from_d(const double* s, float* d, int n) {
    // tiny: copy through host-free kernel path (reuse convert via scratch)
    return d2f(s, d, n, st_);
  }
  static cudaError_t d2f(const double* s, float* d, int n, cudaStream_t st);

  // ------------------------------------------------------------------ state
  paragan_config cfg_;
  cudaStream_t st_;
  ncclComm_t comm_ = nullptr;
  // A12 overlap: D's gradient all-reduce in flight on cs_ (gcomm_) while G's forward runs; applied by flush_d()
  static constexpr int kOverlapCTAs = 8;
  ncclComm_t gcomm_ = nullptr, bncomm_ = nullptr;
  cudaStream_t cs_ = nullptr;
  cudaEvent_t ev_grad_ = nullptr, ev_ar_ = nullptr;
  bool overlap_ = false, pending_d_ = false;
  int overlap_sms_ = 16, overlap_blocks_ = 3;
  bool ready_ = false, poisoned_ = false, planned_ = false, ones_ready_ = false;
  std::vector<GraphEntry> graphs_;   // CUDA-graph step cache (run_graphed)
  bool graphs_on_ = false;
  FoldJob* fold_jobs_d_ = nullptr;   // G conv1 fold table (sub-pixel mode)
  FoldJob* fold_jobs_dd_ = nullptr;  // D pooled-block conv2 input-gradient fold table
  int fold_tiles_dd_ = 0, fold_njobs_dd_ = 0;
  bool dgrad_pool_ = false;          // D conv2's input gradient behind the pool through the phase kernel (R37)
  bool pool_fwd_ = false;            // D conv2 + pool as a stride-2 phase conv at half resolution (R38)
  bool pool_fwd0_ = false;           // ... also for D's first block (96 channels at 128^2)
  paragan_stats* stats_dev_ = nullptr;   // stats_async staging
  int fold_tiles_ = 0;
  bool thin_tc_ = false;  // G's output layer on the tensor cores via bf16 splits (R36; BF16 mode)
  bf16* oconv_ws_ = nullptr;  // its split weight operand [96][2 cl]
  bf16* oconv_wd_ = nullptr;  // the dgrad operand [round_up(cl, 16)][128]
  bool pool_fuse_ = true;   // D blocks: 2x2 average pooling in conv2's epilogue (W <= 64)
  bool attn_flat_ = true;   // attention forward: image-wide offset when the score bound allows (tc_attn.cu)
  bool subpix_ = false;   // G conv1 as four phase 2x2 convs of the low-resolution input (NEXT-1)
  bool attn_single_ = true;   // single-pass fused attention forward when the score bound allows (R21)
  bool dcgan_ = false;    // SN-DCGAN (config 1) instead of BigGAN
  int d_since_g_ = 0;
  uint64_t launches_ = 0;
  Net G_, D_;
  std::vector<SnJob> jobs_h_[2];
  int B_ = 0, R_ = 0, cpad_ = 0, zc_ = 0, dimz_ = 0, cd_ = 0, c0_ = 0, cl_ = 0, cdl_ = 0, hl_ = 0;
  int shared_ = -1, obn_g_ = -1, obn_b_ = -1, demb_ = -1;
  LinL glin_, dlin_;
  ConvL oconv_;
  std::vector<GBlock> gb_;
  std::vector<DBlock> db_;
  AttnL gattn_, dattn_;
  void* attn_out_[2] = {nullptr, nullptr};
  long long big_ = 0;
  void* tmp_[4] = {};
  void* tmp_attn_dO_ = nullptr;
  void* dxp_ = nullptr;
  float* dP_ = nullptr;
  float* dth_part_ = nullptr;
  size_t dth_part_floats_ = 0, dpool_floats_ = 0;
  long long unfused_dp_ = 0;
  bool prof_ = false;
  std::vector<ProfRec> recs_;
  std::vector<cudaEvent_t> ev_free_;
  float* ones_buf_ = nullptr;
  float* quarter_ = nullptr;   // device 0.25 (the x2 average pool's adjoint scale as a conv epilogue alpha)
  int maxc_ = 8;
  void* tmp_attn_dqkv_ = nullptr;
  float *zin_ = nullptr, *emb_ = nullptr, *demb_g_ = nullptr, *h0f_ = nullptr, *dh0f_ = nullptr;
  int32_t *yg_ = nullptr, *ylab_ = nullptr;
  void* gout_in_ = nullptr;
  float *aout_ = nullptr, *daout_ = nullptr, *omean_ = nullptr, *orstd_ = nullptr, *pre_ = nullptr, *img_ = nullptr,
        *dpre_ = nullptr;
  double* osums_ = nullptr;
  void* dimg_ = nullptr;
  void* dimg_grad_ = nullptr;
  float* dfake_keep_ = nullptr;   // test hook buffer (PARAGAN_FLAG_KEEP_DFAKE), allocated on first use
  // asynchronous checkpoint writer (allocated on the first save)
  void* ck_dev_ = nullptr;
  void* ck_host_ = nullptr;
  cudaStream_t ck_stream_ = nullptr;
  cudaEvent_t ck_ev_snap_ = nullptr, ck_ev_done_ = nullptr;
  std::thread ck_thread_;
  volatile paragan_status ck_status_ = PARAGAN_OK;
  bool dfake_valid_ = false;
  int dimg_idx_ = 0;
  float* demb_hat_ = nullptr;
  float *feat_ = nullptr, *logits_ = nullptr, *dlogits_ = nullptr;
  float *ab_ = nullptr, *bn_part_ = nullptr;
  GemmProblem *cbn_fwd_d_ = nullptr, *cbn_dw_d_ = nullptr, *cbn_dcond_d_ = nullptr;
  int cbn_fwd_n_ = 0, cbn_fwd_tiles_ = 0, cbn_dw_n_ = 0, cbn_dw_tiles_ = 0, cbn_dcond_n_ = 0, cbn_dcond_tiles_ = 0;
  double *dpart_ = nullptr, *tot_ = nullptr;
  float *scratch_f_ = nullptr, *wg_scratch_ = nullptr, *dpool_ = nullptr;
  size_t scratch_floats_ = 0;
  int* nonfinite_sticky_ = nullptr;
#undef CK
#undef CKS
};

namespace {
__global__ void k_d2f(const double* s, float* d, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = (float)s[i];
}
}  // namespace
template <typename T>
cudaError_t Engine<T>::d2f(const double* s, float* d, int n, cudaStream_t st) {
  k_d2f<<<(n + 255) / 256, 256, 0, st>>>(s, d, n);
  return cudaGetLastError();
}

static bool policy_ok(const paragan_policy& p) {
  if (p.rule < PARAGAN_OPT_ADAM || p.rule > PARAGAN_OPT_SGD) return false;
  if (p.lars && !(p.lars_trust > 0.0f)) return false;
  if (p.lookahead_k < 0 || (p.lookahead_k > 0 && !(p.lookahead_alpha > 0.0f && p.lookahead_alpha <= 1.0f))) return false;
  if (p.warmup_steps < 0 || p.total_steps < 0 || !(p.clip_norm >= 0.0f)) return false;
  if (p.schedule < PARAGAN_SCHED_CONSTANT || p.schedule > PARAGAN_SCHED_LINEAR) return false;
  if (p.schedule != PARAGAN_SCHED_CONSTANT && p.total_steps == 0) return false;
  return true;
}

paragan_status validate_config(const paragan_config* c) {
  if (!c) return PARAGAN_ERR_INVALID_ARG;
  if (c->abi_version != PARAGAN_ABI_VERSION) return PARAGAN_ERR_CONFIG;
  if (!policy_ok(c->policy_d) || !policy_ok(c->policy_g)) return PARAGAN_ERR_CONFIG;
  for (const paragan_adam* a : {&c->adam_d, &c->adam_g})
    if (!(a->lr >= 0.0f) || !(a->beta1 >= 0.0f && a->beta1 < 1.0f) || !(a->beta2 >= 0.0f && a->beta2 < 1.0f) ||
        !(a->eps > 0.0f))
      return PARAGAN_ERR_CONFIG;
  if (c->arch == PARAGAN_ARCH_SNDCGAN) {   // config 1 (R25): 32x32, fp32 SIMT path
    if (c->resolution != 32 || c->compute != PARAGAN_F32 || c->ch < 1 || c->ch % 4 || c->local_batch < 1 ||
        c->d_steps_per_g < 1 || c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size || c->n_classes < 1 ||
        c->c_pad_image < 3 || !(c->sn_eps > 0) || !(c->bn_eps > 0))
      return PARAGAN_ERR_CONFIG;
    return PARAGAN_OK;
  }
  if (c->arch != PARAGAN_ARCH_BIGGAN) return PARAGAN_ERR_CONFIG;
  // D runs on [fake; real] = 2B rows; its projection-head gradient kernel handles at most 2048 rows per launch
  if (c->local_batch > 1024) return PARAGAN_ERR_CONFIG;
  Arch a;
  if (!arch_for(c->resolution, a)) return PARAGAN_ERR_CONFIG;
  if (c->ch < 1 || c->n_classes < 1 || c->shared_dim < 1 || c->z_chunk < 1 || c->local_batch < 1 ||
      c->d_steps_per_g < 1 || c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size)
    return PARAGAN_ERR_CONFIG;
  if (c->compute != PARAGAN_F32 && c->compute != PARAGAN_BF16) return PARAGAN_ERR_CONFIG;
  if (c->c_pad_image < 3 || c->c_pad_image % 8) return PARAGAN_ERR_CONFIG;
  // every BN / tensor-core channel count must be a multiple of 8 (16-byte NHWC pixel rows)
  for (int m : a.gin) if ((m * c->ch) % 8) return PARAGAN_ERR_CONFIG;
  for (int m : a.gout) if ((m * c->ch) % 8 || (m * c->ch) / 8 > 256) return PARAGAN_ERR_CONFIG;
  for (size_t j = 1; j < a.din.size(); ++j) if ((a.din[j] * c->ch) % 8) return PARAGAN_ERR_CONFIG;
  if (c->attn_res) {
    bool ok = false;
    for (int h = 8; h <= c->resolution; h *= 2) ok |= (h == c->attn_res);
    if (!ok) return PARAGAN_ERR_CONFIG;
    // attention channel C must give C/2 % 8 == 0
    for (size_t i = 0; i < a.gout.size(); ++i)
      if ((8 << i) == c->attn_res && ((a.gout[i] * c->ch) / 2) % 8) return PARAGAN_ERR_CONFIG;
  }
  if (!(c->sn_eps > 0) || !(c->bn_eps > 0)) return PARAGAN_ERR_CONFIG;
  return PARAGAN_OK;
}

EngineBase* make_engine(const paragan_config* cfg, void* stream, paragan_status* st) {
  *st = validate_config(cfg);
  if (*st != PARAGAN_OK) return nullptr;
  if (cfg->compute == PARAGAN_BF16) return new Engine<bf16>(*cfg, static_cast<cudaStream_t>(stream));
  return new Engine<float>(*cfg, static_cast<cudaStream_t>(stream));
}

}  // namespace pg
