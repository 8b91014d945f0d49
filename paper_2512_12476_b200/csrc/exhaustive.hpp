// exhaustive_search on the device (reference search.cpp:837-1031).
//
// The reference walks, per (task grouping, composition) "block": every
// distinct group labelling of the device list (std::next_permutation over the
// sorted label multiset), then per task in group order every layout option x
// every permutation of the group's devices, and evaluates a candidate only
// the first time its canonical key (device ids replaced by
// class * 4096 + first-appearance counter within the class) is seen.
//
// Here a block's raw candidates are indexed by a mixed radix in exactly that
// nesting order (labelling outermost, then per task: option, permutation),
// so the index order IS the reference's enumeration order:
//   exh_key_kernel     index -> candidate -> canonical key bytes
//   exh_insert_kernel  open-addressing table keyed by the exact key bytes,
//                      slot value = min index (the first occurrence)
//   exh_rep_kernel     first occurrences -> compact plan records at their
//                      index (mode e2e), the others -> mode skip
//   eval_kernel        end_to_end_cost + check_memory (mode e2e)
//   exh_reduce_kernel  argmin over memory-feasible representatives by
//                      (cost, index) = the reference's strict-< first minimum
// Keys never collide across blocks (the layouts pin the composition), so a
// block is deduplicated on its own. Blocks are queued back to back on one
// stream (buffers reused in stream order) with a single host sync at the end.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace hpg {

constexpr int kExhMaxDevices = 20;  // factorials in u64
constexpr int kExhMaxOpts = 64;     // layout options per (task, group size)

struct ExhBlock {
  int32_t n, T, k;                  // devices, tasks, groups
  int32_t order[kMaxTasks];         // task slot per position in group order
  int32_t grp[kMaxTasks];           // group of each position
  int32_t comp[kMaxTasks];          // devices per group
  int32_t nopt[kMaxTasks];          // layout options per position
  int16_t opt[kMaxTasks][kExhMaxOpts][3];  // (dp, pp, tp) in enumerate_layouts order
  uint64_t fact[kExhMaxDevices + 1];
  uint64_t perms[kMaxTasks];        // comp[grp[t]]! per position
  uint64_t multinom;                // distinct labellings
  uint64_t raw;                     // candidates in the block
  uint8_t cls[kExhMaxDevices];      // symmetry class per device
  int32_t key_bytes;                // padded to 8
  int32_t rec_stride;
};

// Decodes raw index `idx` of block B: per position t the option index and the
// devices in flat (i, j, k) order; devs[t * n .. + comp[grp[t]]).
HPG_HD void exh_decode(const ExhBlock& B, uint64_t idx, int* opt_idx, uint8_t* devs) {
  uint64_t rr[kMaxTasks];
  uint64_t x = idx;
  for (int t = B.T - 1; t >= 0; --t) {
    rr[t] = x % B.perms[t];
    x /= B.perms[t];
    opt_idx[t] = static_cast<int>(x % static_cast<uint64_t>(B.nopt[t]));
    x /= static_cast<uint64_t>(B.nopt[t]);
  }
  // labelling x: lexicographic rank among the permutations of the sorted
  // label multiset; count of completions = multinomial of the remaining labels
  int left[kMaxTasks];
  for (int g = 0; g < B.k; ++g) left[g] = B.comp[g];
  uint8_t gdev[kMaxTasks][kExhMaxDevices];
  int gn[kMaxTasks];
  for (int g = 0; g < kMaxTasks; ++g) gn[g] = 0;
  int rem = B.n;
  for (int i = 0; i < B.n; ++i) {
    --rem;
    for (int g = 0; g < B.k; ++g) {
      if (left[g] == 0) continue;
      // completions with label g at position i: rem! / prod(left') !
      uint64_t cnt = B.fact[rem];
      for (int h = 0; h < B.k; ++h) cnt /= B.fact[h == g ? left[h] - 1 : left[h]];
      if (x < cnt) {
        --left[g];
        gdev[g][gn[g]++] = static_cast<uint8_t>(i);
        break;
      }
      x -= cnt;
    }
  }
  // per position: lexicographic permutation rr[t] of the group's ascending devices
  for (int t = 0; t < B.T; ++t) {
    const int g = B.grp[t], m = B.comp[g];
    uint8_t pool[kExhMaxDevices];
    for (int i = 0; i < m; ++i) pool[i] = gdev[g][i];
    uint64_t r = rr[t];
    uint8_t* out = devs + t * B.n;
    for (int i = 0; i < m; ++i) {
      const uint64_t f = B.fact[m - 1 - i];
      const int q = static_cast<int>(r / f);
      r %= f;
      out[i] = pool[q];
      for (int j = q; j < m - 1 - i; ++j) pool[j] = pool[j + 1];
    }
  }
}

struct ExhPartial {
  double best;
  unsigned long long best_idx;
};

cudaError_t launch_exh_keys(const ExhBlock& B, uint64_t n, uint8_t* d_keys, cudaStream_t st);
cudaError_t launch_exh_insert(const ExhBlock& B, uint64_t n, const uint8_t* d_keys,
                              unsigned long long* d_table, uint64_t mask,
                              unsigned long long* d_slot, cudaStream_t st);
cudaError_t launch_exh_reps(const ExhBlock& B, uint64_t n, const unsigned long long* d_table,
                            const unsigned long long* d_slot, uint8_t* d_recs, int32_t* d_modes,
                            unsigned long long* d_count, cudaStream_t st);
cudaError_t launch_exh_reduce(const EvalResult* d_res, int64_t n, ExhPartial* d_out, int blocks,
                              cudaStream_t st);

}  // namespace hpg
