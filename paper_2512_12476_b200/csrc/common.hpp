// Shared host/device definitions of the B200 plan-search engine.
//
// The reference planner (hetplan, C++20, single-threaded) keeps plans as
// std::map<int, ...> keyed by task id with device-id strings
// (proj/include/hetplan/plan.hpp:59-70). The engine keeps them as packed
// byte records (PlanRec below): integer device indices, per-task layout
// triples, stage splits and replica weights, laid out so one warp can stage a
// whole plan into shared memory with coalesced loads.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define HPG_HD __host__ __device__ __forceinline__
#else
#define HPG_HD inline
#endif

// Device-side bounds checks of the checked build (libhpg_checked.so, make
// checked): a failed check prints the condition and traps the kernel, which
// surfaces as a CUDA error on the host. Compiled out of libhpg.so.
#if defined(HPG_CHECKED) && defined(__CUDA_ARCH__)
#include <cstdio>
#define HPG_DCHECK(cond)                                                              \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      printf("HPG_DCHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);         \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define HPG_DCHECK(cond) ((void)0)
#endif

namespace hpg {

constexpr int kMaxTasks = 6;        // PPO: tasks 1..6 (workflow.cpp:64-69)
constexpr int kMaxDevices = 256;    // device slots are u8 indices
constexpr int kMaxClasses = 64;     // distinct (latency, bandwidth) link classes
constexpr double kInf = __builtin_inf();

enum TaskKind : int32_t { kGeneration = 0, kInference = 1, kTraining = 2 };

// Task constants, workflow order (== task-id order, workflow.cpp:111-125).
struct DevTask {
  int32_t id;
  int32_t kind;
  int32_t precision_bytes;
  int32_t include_embedding;
  int64_t h1, h2, nl, vocab;
  int64_t layer_params;  // ModelSpec::layer_params (workflow.hpp:27-30), int64
  int64_t param_count;   // ModelSpec::param_count (workflow.hpp:34-36), int64
};

// Cost-model configuration (cost_model.hpp:13-28 + plan.hpp:83-89).
struct DevCostConfig {
  int32_t recompute;
  int32_t dbs_cap;
  double reshard_override;
  double sync_override;
  double dbs_override;
  double train_bytes_per_param;
  double infer_bytes_per_param;
  double kv_bytes_per_elem;
  double act_factor;
};

// Device-wide ring memo (open addressing in HBM). A ring's bottleneck is a
// pure function of (ordered device list, volume bits) for a fixed topology,
// so concurrent inserts can only duplicate work, never change a result.
// Key: k1/k3 = two independent 64-bit hashes of the ordered device list
// (exact packing when n <= 7), k2 = volume bits; state 1 = value published.
struct RingSlot {
  unsigned long long k1, k2, k3;
  double value;
  unsigned long long state;
  unsigned long long seq;  // n > 8: arena byte offset << 16 | n of the stored device sequence
};
static_assert(sizeof(RingSlot) == 48, "ring slot layout");

// Problem header, passed by value to every kernel. Arrays live in one device
// allocation owned by the context.
struct DevProblem {
  int32_t n_dev;
  int32_t n_tasks;
  int32_t n_classes;
  int32_t mode;       // 0 sync, 1 async
  int32_t algorithm;  // 0 ppo, 1 grpo
  int32_t gen_slot;   // slot of task id 1 or -1
  int32_t train6_slot;  // slot of task id 6 or -1
  int32_t max_tp;     // DeviceTopology::max_devices_per_node
  double eta;
  int64_t global_batch, rpp, seq_in, seq_out, mbs, total_seq;
  DevTask task[kMaxTasks];
  const double* comp;  // [n_dev] FLOP/s   (Device::comp, topology.hpp:33)
  const double* mem;   // [n_dev] bytes    (Device::mem)
  const double* hbm;   // [n_dev] bytes/s  (Device::hbm)
  const uint8_t* cls;  // [n_dev * n_dev] link class of (a, b)
  const double* lat;   // [n_classes] seconds
  const double* bw;    // [n_classes] bytes/s (inf for self)
  RingSlot* ring_cache;       // nullptr = disabled
  unsigned long long ring_mask;  // slots - 1 (power of two)
  // device sequences of the memoised rings with n > 8 (their keys are
  // hashes: a hit is confirmed byte for byte); word 0 = bytes used
  uint8_t* ring_arena;
  unsigned long long ring_arena_cap;
};

// ---- packed plan record ----
//
//   int32 bytes, int32 n_tasks, int32 dp[6], pp[6], tp[6]     (80 bytes)
//   double  weights[sum dp]       replica_batch_weights per task
//   int32   stage_layers[sum pp]
//   uint8   devices[sum dp*pp*tp] flat (replica, stage, shard) order
//   padding to 8 bytes
struct RecHeader {
  int32_t bytes;
  int32_t n_tasks;
  int32_t dp[kMaxTasks];
  int32_t pp[kMaxTasks];
  int32_t tp[kMaxTasks];
};
static_assert(sizeof(RecHeader) == 80, "record header layout");

struct RecOffsets {
  int32_t w[kMaxTasks + 1];    // index into weights (doubles)
  int32_t sl[kMaxTasks + 1];   // index into stage layers (int32)
  int32_t dev[kMaxTasks + 1];  // index into devices (bytes)
  int32_t cell[kMaxTasks + 1];  // prefix of dp*pp
  int32_t dpk[kMaxTasks + 1];   // prefix of pp*tp (dp-ring slots)
  int32_t w_byte, sl_byte, dev_byte, bytes;
};

// n_tasks bit 16: compact record (no weight / stage-layer sections; unit
// weights and make_layout's uniform split are implied, plan.cpp:89-100).
constexpr int32_t kRecCompact = 1 << 16;

HPG_HD void rec_offsets(const RecHeader& h, RecOffsets& o) {
  o.w[0] = o.sl[0] = o.dev[0] = o.cell[0] = o.dpk[0] = 0;
  const int nt = h.n_tasks & 0xffff;
  for (int t = 0; t < nt; ++t) {
    o.w[t + 1] = o.w[t] + h.dp[t];
    o.sl[t + 1] = o.sl[t] + h.pp[t];
    o.dev[t + 1] = o.dev[t] + h.dp[t] * h.pp[t] * h.tp[t];
    o.cell[t + 1] = o.cell[t] + h.dp[t] * h.pp[t];
    o.dpk[t + 1] = o.dpk[t] + h.pp[t] * h.tp[t];
  }
  const bool compact = (h.n_tasks & kRecCompact) != 0;
  o.w_byte = static_cast<int32_t>(sizeof(RecHeader));
  o.sl_byte = o.w_byte + (compact ? 0 : 8 * o.w[nt]);
  o.dev_byte = o.sl_byte + (compact ? 0 : 4 * o.sl[nt]);
  o.bytes = (o.dev_byte + o.dev[nt] + 7) & ~7;
}

// Per-plan request modes of the evaluation kernel.
enum EvalMode : int32_t {
  kModeMemcheck = 0,     // check_memory only (plan.cpp:351-380)
  kModeE2E = 1,          // end_to_end_cost (cost_model.cpp:431-487), no balancing
  kModeEvaluate = 2,     // EvalContext::evaluate (search.cpp:259-279) if memory-feasible
  kModeBalanceData = 3,  // balance_data (balance.cpp:37-56) only
  kModeBalanceLayers = 4,  // balance_layers (balance.cpp:81-167) only
  kModeChain = 5,        // balance_data -> balance_layers -> e2e, no C3 gate
  kModeSkip = 6,         // no plan in this slot: result {cost -1, flags 0}
};

// Per-plan result slot.
struct EvalResult {
  double cost;       // end_to_end_s of the (balanced) plan, or -1 when not evaluated
  double reshard_s;
  double sync_s;
  int32_t flags;     // bit0: input memory-feasible; bit1: output memory-feasible;
                     // bit2: weights changed; bit3: stage layers changed
  int32_t pad;
};
static_assert(sizeof(EvalResult) == 32, "result layout");

constexpr int kResFeasIn = 1;
constexpr int kResFeasOut = 2;
constexpr int kResWeights = 4;
constexpr int kResLayers = 8;

// Per-batch shared-memory carve sizes of the evaluation kernel (the host
// computes the batch maxima while packing).
struct Carve {
  int32_t n_dev;      // N
  int32_t n_tasks;    // T
  int32_t max_w;      // max over plans of sum dp
  int32_t max_sl;     // max sum pp
  int32_t max_slots;  // max sum dp*pp*tp
  int32_t max_cells;  // max sum dp*pp
  int32_t max_dpk;    // max sum pp*tp
  int32_t bytes;      // total dynamic smem per CTA
  int32_t cls_smem;   // stage the link-class matrix in shared memory (small N, small waves)
  int32_t n_warps;    // warps per CTA: warp 0 evaluates, the others help with task costs
};

HPG_HD int carve_round(int b) { return (b + 15) & ~15; }

HPG_HD int carve_bytes(const Carve& c) {
  const int N = c.n_dev, T = c.n_tasks;
  int b = 0;
  b += 2 * carve_round(8 * c.max_w) + 2 * carve_round(8 * c.max_cells) + carve_round(8 * c.max_dpk);
  b += 7 * carve_round(8 * N) + carve_round(8 * kMaxClasses) + carve_round(8 * 64) +
       carve_round(8 * T * 7);
  b += 2 * carve_round(4 * c.max_sl) + carve_round(4 * c.max_dpk) + carve_round(4 * N);
  b += carve_round(c.max_slots) + carve_round(T * N) + 2 * carve_round(N);
  return b;
}

// warps per CTA when a plan's task costs are spread over a team (eval_kernel)
constexpr int kMaxTeamWarps = 4;

// the link-class matrix may be staged in shared memory when it is this small
// (latency-bound small waves: every SM starts with a cold L1)
constexpr int kClsSmemMax = 16384;

// per-warp scratch of a helper warp (cell pieces, ring scratch, class costs)
HPG_HD int team_scratch_bytes(const Carve& c) {
  const int N = c.n_dev;
  return 5 * carve_round(8 * N) + carve_round(8 * kMaxClasses) + carve_round(8 * 64) +
         2 * carve_round(N);
}

HPG_HD int carve2_bytes(const Carve& c) {
  return carve_bytes(c) + carve_round(8 * c.max_cells) + 2 * carve_round(8 * c.max_sl) +
         carve_round(8 * c.n_dev) + carve_round(4 * c.max_sl) +
         (c.cls_smem ? carve_round(c.n_dev * c.n_dev) : 0) +
         (c.n_warps > 1 ? (c.n_warps - 1) * team_scratch_bytes(c) : 0);
}

// ---- end_to_end-only scratch sized per plan (the config-5 sweep kernel) ----
//
// end_to_end_cost of one plan touches: weights/micro-batches per replica,
// the geometry memo per (task, replica, stage) cell, the DP-ring memo per
// (task, stage, shard), cell pieces of the task in flight, ring scratch of the
// largest ring, per-device residency and stage maps, and the memory tables per
// (task, stage). The balancers' arrays are not needed. Exact sizes of one plan:
struct E2ESizes {
  int32_t w, sl, slots, cells, dpk;  // sums over tasks of dp, pp, dp*pp*tp, dp*pp, pp*tp
  int32_t cell_max, ring_max;        // max over tasks of dp*pp, max(dp, tp)
};

HPG_HD E2ESizes e2e_sizes(const RecOffsets& o, const RecHeader& h, int n_tasks) {
  E2ESizes z;
  z.w = o.w[n_tasks];
  z.sl = o.sl[n_tasks];
  z.slots = o.dev[n_tasks];
  z.cells = o.cell[n_tasks];
  z.dpk = o.dpk[n_tasks];
  z.cell_max = 1;
  z.ring_max = 8;  // ring_small's 8-vertex scratch
  for (int t = 0; t < n_tasks; ++t) {
    const int c = h.dp[t] * h.pp[t];
    z.cell_max = z.cell_max > c ? z.cell_max : c;
    z.ring_max = z.ring_max > h.dp[t] ? z.ring_max : h.dp[t];
    z.ring_max = z.ring_max > h.tp[t] ? z.ring_max : h.tp[t];
  }
  return z;
}

// worst case over every plan of a problem (N devices, T tasks)
HPG_HD E2ESizes e2e_sizes_max(int N, int T) {
  E2ESizes z;
  z.w = z.slots = z.cells = z.dpk = T * N;
  z.sl = T * N;
  z.cell_max = N;
  z.ring_max = N > 8 ? N : 8;
  return z;
}

HPG_HD int e2e_carve_bytes(const E2ESizes& z, int N, int T) {
  return 2 * carve_round(8 * z.w) + 3 * carve_round(8 * z.cells) + carve_round(8 * z.dpk) +
         carve_round(4 * z.dpk) + carve_round(8 * N) + 4 * carve_round(8 * z.cell_max) +
         carve_round(8 * z.ring_max) + carve_round(8 * kMaxClasses) + carve_round(8 * 64) +
         carve_round(8 * T * 7) + carve_round(4 * z.sl) + 2 * carve_round(8 * z.sl) +
         carve_round(z.slots) + carve_round(T * N) + 2 * carve_round(z.ring_max);
}

}  // namespace hpg
