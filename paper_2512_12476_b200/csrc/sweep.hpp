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
  int32_t train_mask;       // bit t: task slot t is a training task (DP rings)
  int32_t gen_slot, train6_slot;  // generation / actor-training slots (bridge), -1 if absent
};

// Work-class grouping of a chunk (sweep.cu): gen_kernel gives every plan a
// key of per-task work classes (kSweepKeyBits bits) and counts them; a
// counting sort orders the chunk by key, so the plan-warps of one CTA score
// plans of similar shape side by side (their per-task phase barriers then
// wait little; see sweep_kernel.cuh).
constexpr int kSweepKeyBits = 20;  // PPO: 2 x 4 (training) + 3 (bridge) + 3 (generation) + 3 x 2
struct SweepOrder {
  uint32_t* keys = nullptr;   // [chunk]
  uint32_t* hist = nullptr;   // [1 << kSweepKeyBits], bin offsets after the scan
  uint32_t* order = nullptr;  // [chunk] plan index in key order
};

struct SweepPartial {
  double best;
  unsigned long long best_k;
  unsigned long long n_feasible;
  unsigned long long xor_bits;
};

// the sweep scoring kernel (sweep_kernel.cuh): CTAs of `warps` plan-warps,
// each with a `slab_bytes` shared-memory slab for its plan's scratch, plus a
// CTA-shared copy of the link-class matrix when N*N <= kClsSweepMax
constexpr int kClsSweepMax = 16384;
struct SweepLaunch {
  int warps = 8;
  int blocks = 2;  // CTAs per SM
  int grid = 0;
  int slab_bytes = 0;
  int cls_bytes = 0;
  int64_t gslab_bytes = 0;       // per-warp global fallback slab (worst-case plan)
  uint8_t* gslab = nullptr;      // [grid * warps * gslab_bytes]
  SweepPartial* part = nullptr;  // [grid * warps], merged in place across chunks
  unsigned long long* n_global = nullptr;  // plans that used the global slab
  int sync = 0;  // CTA-wide barriers at plan and task boundaries (shared instruction fetch)
};
cudaError_t sweep_plan(int N, int T, int n_sm, int warps, int slab_req, SweepLaunch& L);
cudaError_t launch_sweep(const DevProblem& P, const DevCostConfig& cfg, const uint8_t* d_recs,
                         int64_t stride, int64_t n, uint64_t k0, SweepLaunch& L,
                         const uint32_t* d_order, EvalResult* d_res, cudaStream_t st);

cudaError_t launch_gen(const SweepTablesDev& tb, uint64_t seed, uint64_t k0, int64_t n,
                       uint8_t* d_recs, int64_t stride, unsigned long long* d_bytes,
                       const SweepOrder* ord, cudaStream_t st);
// counting sort of the chunk's plans by their gen_kernel keys (ord->order)
cudaError_t launch_order(const SweepOrder& ord, int64_t n, cudaStream_t st);
}  // namespace hpg
