// Step engine of libparagan: owns the BigGAN plan for one rank (parameters,
// optimiser state, activations carved from the caller's workspace, NCCL
// communicator) and sequences the kernels of one D or G step.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/paragan.h"

namespace pg {

class EngineBase {
 public:
  virtual ~EngineBase() = default;
  virtual paragan_status init(const uint8_t* nccl_id, void* ws, size_t ws_bytes) = 0;
  virtual size_t workspace_bytes() = 0;
  virtual void counts(paragan_net net, size_t* n_state, size_t* n_train) = 0;
  virtual paragan_status init_params(float attn_gamma) = 0;
  virtual paragan_status set_params(paragan_net net, const float* host, size_t n) = 0;
  virtual paragan_status get_params(paragan_net net, float* host, size_t n) = 0;
  virtual paragan_status get_grads(paragan_net net, float* host, size_t n) = 0;
  virtual paragan_status set_grads(paragan_net net, const float* host, size_t n) = 0;
  virtual paragan_status d_step(const void* real, const int32_t* real_y, const float* z, const int32_t* fake_y,
                                uint32_t flags) = 0;
  virtual paragan_status g_step(const float* z, const int32_t* y, uint32_t flags) = 0;
  virtual paragan_status allreduce(paragan_net net) = 0;
  virtual paragan_status update(paragan_net net) = 0;
  virtual paragan_status sync_stats(paragan_stats* out) = 0;
  virtual paragan_status stats_async(paragan_stats* out) = 0;
  virtual paragan_status get_fakes(float* host, size_t n) = 0;
  virtual paragan_status get_dfake(float* host, size_t n) = 0;
  virtual paragan_status d_step_fakes(const void* real, const int32_t* real_y, const void* fakes, const int32_t* fake_y,
                                      uint32_t flags) = 0;
  virtual paragan_status generate(const float* z, const int32_t* y, void* dst) = 0;
  virtual paragan_status export_fakes(void* dst) = 0;
  virtual paragan_status export_state(paragan_net net, float* dst) = 0;
  virtual size_t state_floats(paragan_net net) = 0;
  virtual paragan_status checkpoint_save_async(const char* path) = 0;
  virtual paragan_status checkpoint_wait() = 0;
  virtual paragan_status checkpoint_load(const char* path) = 0;
  virtual paragan_status import_state(paragan_net net, const float* src) = 0;
  virtual uint64_t launches() const = 0;
  virtual paragan_status profile(int enable) = 0;
  virtual paragan_status profile_read(int kind, uint64_t* n, double* ms, double* flops) = 0;
  const char* last_error() const { return err_.c_str(); }

 protected:
  std::string err_;
};

// validates cfg; returns nullptr with *st set on error
EngineBase* make_engine(const paragan_config* cfg, void* stream, paragan_status* st);
paragan_status validate_config(const paragan_config* cfg);

}  // namespace pg
