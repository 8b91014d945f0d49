// Per-device launch state. cudaFuncSetAttribute and occupancy are properties
// of a (device, kernel) pair, so they are tracked per device under a mutex:
// contexts on different GPUs in one process, and threads driving separate
// contexts, never see each other's settings (hpg.h: separate contexts are
// thread-safe).
#pragma once

#include <cuda_runtime.h>

namespace hpg {

// Raises kernel `fn`'s dynamic shared-memory limit on the current device to at
// least `bytes` (no-op when already there).
cudaError_t ensure_dyn_smem(const void* fn, int bytes);

// cudaOccupancyMaxActiveBlocksPerMultiprocessor, memoised per
// (device, kernel, threads, dynamic bytes).
cudaError_t occupancy_per_sm(const void* fn, int threads, int bytes, int* per_sm);

}  // namespace hpg
