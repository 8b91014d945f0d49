// GA initial candidates on the device (gen_ga.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"
#include "rng.hpp"

namespace hpg {

constexpr int kGenFastModMax = 1024;

// Problem tables for random_medium_assignment / random_fine_assignment,
// built once per staged problem: regions (lexicographic) -> nodes
// (lexicographic) -> devices (insertion order), and each device's node rank.
struct GenTablesDev {
  int32_t n_dev, n_regions, n_nodes, max_nodes_per_region;
  int32_t smem_per_thread;    // scratch bytes per generating thread
  const int32_t* region_off;  // [n_regions + 1] into the node list
  const int32_t* node_off;    // [n_nodes + 1] into node_devs
  const uint8_t* node_devs;   // [n_dev]
  const int16_t* node_rank;   // [n_dev]
  const uint64_t* fastmod;    // [2 * (kGenFastModMax + 1)] 128-bit ceil(2^128 / d), lo/hi
};

// One arm run's init chunk: `count` candidates at batch positions first...
// (compact positions first_out...). Every candidate draws the same number of
// values from the stream (gen_draws_per_candidate), so the host steps the
// stream to each candidate's start state and the device makes all
// candidates of a wave in parallel, one thread each.
struct GenItem {
  double bias;  // locality_bias
  int32_t first, first_out, count;
  int32_t n_groups, n_order;
  int32_t counts[kMaxTasks];     // devices per group
  int8_t order_slot[kMaxTasks];  // task slots in group order
  int8_t order_group[kMaxTasks];
};

// Draws of one make_candidate (search.cpp:152-234, 318-334): shuffles of m
// items draw max(m - 1, 0) values, the locality scramble two per position,
// and a task's fine assignment over a group of n devices n - 1 in total
// (node-order shuffle plus one shuffle per node bucket).
inline int64_t gen_draws_per_candidate(int n_dev, const int* nodes_per_region, int n_regions,
                                       const GenItem& it) {
  int64_t d = n_regions > 1 ? n_regions - 1 : 0;
  for (int r = 0; r < n_regions; ++r) d += nodes_per_region[r] > 1 ? nodes_per_region[r] - 1 : 0;
  d += n_dev > 1 ? 2 * static_cast<int64_t>(n_dev - 1) : 0;
  for (int k = 0; k < it.n_order; ++k) d += it.counts[it.order_group[k]] - 1;
  return d;
}

// cand_item[j] = the item of compact candidate j, starts[j] its stream state
cudaError_t launch_gen_ga(const GenTablesDev& tb, const GenItem* d_items,
                          const int32_t* d_cand_item, const Rng* d_starts, int n_cands,
                          uint8_t* d_recs, const int64_t* d_off, const int64_t* d_dev_out_off,
                          uint8_t* d_dev_out, cudaStream_t st);

}  // namespace hpg
