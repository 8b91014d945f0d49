// Config-5 sweep tables and launch entry points.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace hpg {

// Device tables of the counter-based generator, built once per context.
struct SweepTablesDev {
  int32_t n_dev, n_tasks, n_tgs;
  const int8_t* tg_group;   // [n_tgs * 6] group of each task slot
  const int8_t* tg_ng;      // [n_tgs]
  const int32_t* opt_off;   // [T * (N + 1) + 1] layout options of (slot, count)
  const int16_t* opt;       // [n_opt * 3] (dp, pp, tp) in enumerate_layouts order
};

struct SweepPartial {
  double best;
  unsigned long long best_k;
  unsigned long long n_feasible;
  unsigned long long xor_bits;
};

cudaError_t launch_gen(const SweepTablesDev& tb, uint64_t seed, uint64_t k0, int64_t n,
                       uint8_t* d_recs, int64_t stride, unsigned long long* d_bytes,
                       cudaStream_t st);
cudaError_t launch_reduce(const EvalResult* d_res, int64_t n, uint64_t k0, SweepPartial* d_out,
                          int blocks, cudaStream_t st);

}  // namespace hpg
