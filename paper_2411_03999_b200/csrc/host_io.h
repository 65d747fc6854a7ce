// Host-side helpers shared by the checkpoint writer (engine.cu) and host_io.cu.
#pragma once
#include <cstddef>
#include <cstdint>

namespace pg {

// FNV-1a 64-bit hash (checkpoint payload integrity)
uint64_t fnv1a64(const void* data, size_t n, uint64_t h = 1469598103934665603ull);

}  // namespace pg
