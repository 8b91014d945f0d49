// Nested successive halving + per-arm genetic search (search.cpp:437-835 of
// the reference), re-organised for the GPU: every arm's GA is a C++20
// coroutine that suspends whenever it needs candidates scored; all live arms
// of a halving round run in lockstep and their requests are batched into one
// eval_kernel launch per wave. Speculation keeps the RNG stream exact: the
// GA's data-independent draws (mutation retries, swap trials) are generated
// up front with RNG snapshots, scored in one wave, and the stream is rewound
// to the snapshot after the trial the sequential algorithm would have stopped
// at.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "engine.hpp"

namespace hpg {

struct InfeasibleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Knobs {
  int64_t budget = 1000;
  uint64_t seed = 0;
  int population = 16;
  double locality_bias = 0.8;
  int quantize = 1;
  bool adjacent = false;
  int level1_cap = 0;
  int gg_arm_cap = 64;
  int swap_pair_sample = 8;
  bool balance_data = true;
  bool balance_layers = true;
  bool recompute = true;
  double reshard_override = -1.0;
  double sync_override = -1.0;
  double exhaustive_cap = 1e6;
  bool has_tg_override = false;
  std::vector<std::vector<std::vector<int>>> tg_override;  // groups of task slots
  DevCostConfig cost_config() const;  // SearchKnobs::cost_config (search.cpp:38-44)
};

Knobs knobs_from_c(const Problem& P, const hpg_knobs& k);

using Grouping = std::vector<std::vector<int>>;  // task slots per group

struct ArmRec {
  int64_t tg = 0, gg = 0;
  double best = kInf;
  int64_t evals = 0;
};
struct Halving {
  int level = 0;
  int64_t before = 0, after = 0;
  double survivor_worst = 0, eliminated_best = 0;
};

struct SearchOut {
  int64_t budget = 0, consumed = 0;
  uint64_t seed = 0;
  std::vector<int64_t> b_m;
  std::vector<std::pair<int64_t, double>> trace;
  std::vector<ArmRec> arms;
  std::vector<Halving> halvings;
  std::vector<std::vector<int64_t>> survivors;
  int64_t task_groupings = 0;
  bool has_plan = false;
  Cand plan;
  Grouping plan_groups;
  std::vector<int> plan_counts;
  double est_cost = -1.0;
  int64_t prov_budget = -1;      // plan provenance budget; -1 = consumed
  std::vector<double> per_task;  // T*7
  double reshard_s = 0, sync_s = 0, e2e = 0;
  bool feasible = true;
  double wall_s = 0, time_to_best_s = 0;
  int64_t launches = 0, waves = 0, plans_gpu = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0, eval_launches = 0, canonical_bytes = 0;
  double eval_ms = 0.0, host_ms = 0.0, batch_ms = 0.0;
};

SearchOut nested_sha_search(Ctx& ctx, const Knobs& k, Dist* dist);
SearchOut ga_search(Ctx& ctx, const Grouping& tg, const std::vector<int>& counts, int64_t slice,
                    uint64_t seed, const Knobs& k);
// exhaustive_search / exhaustive_space_estimate (search.cpp:837-1031) on the
// device; SearchOut.consumed = unique plans evaluated (ExhaustiveResult::
// explored), SearchOut.budget = raw candidates enumerated
SearchOut exhaustive_search(Ctx& ctx, const Knobs& k);
double exhaustive_space_estimate(const Problem& P, const Knobs& k);

// enumerations (search.cpp:97-150, combinatorics.cpp:10-146)
std::vector<Grouping> enumerate_task_groupings(const Problem& P, bool adjacent);
std::vector<std::vector<int>> compositions(int total, int parts, int quantum);
double composition_count(int total, int parts, int quantum);
std::vector<int> sample_composition(int total, int parts, int quantum, Rng& rng);

// NCCL plumbing (dist.cpp)
void dist_unique_id(uint8_t out[128]);
void dist_init(Dist& d, int rank, int world, const uint8_t id[128], int device);
void dist_allgather(Dist& d, const void* send, void* recv, size_t bytes, cudaStream_t st);
void dist_destroy(Dist& d);

}  // namespace hpg
