// Host side of the engine: problem staging, device buffers, plan records and
// the batched evaluation call used by the C ABI and by the search driver.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hpg.h"
#include "common.hpp"
#include "gen_ga.hpp"
#include "rng.hpp"
#include "sweep.hpp"

namespace hpg {

// Status-carrying errors, mapped to HPG_* codes at the C boundary
// (InputError / UsageError of proj/include/hetplan/errors.hpp:11-18).
struct InputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InternalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

struct HostTask {
  int id = 0;
  int kind = 0;
  int64_t h1 = 0, h2 = 0, nl = 0, vocab = 0;
  bool emb = false;
  int prec = 2;
  int64_t layer_params = 0, param_count = 0;
};

// Workflow + topology, flattened to integers (SURVEY.md §7 step 1 "problem
// flattener"): devices as indices, link classes, lexicographic orders of the
// id/node/region strings that drive the reference's std::map iteration.
struct Problem {
  int N = 0, T = 0;
  int algorithm = 0, mode = 0;
  double eta = 0.5;
  int64_t global_batch = 1, rpp = 1, seq_in = 1, seq_out = 0, mbs = 1;
  std::vector<HostTask> tasks;  // workflow order = task-id order
  int slot_of_id[8];            // task id -> slot, -1 absent
  std::set<std::pair<int, int>> dep_edges;
  // devices
  std::vector<std::string> dev_id, dev_node, dev_region, dev_model;
  std::vector<double> comp_tflops, mem_gb, hbm_gbps, intra_gbps;
  std::vector<double> comp, mem, hbm;  // SI
  int max_node_size = 0;
  // links
  std::vector<uint8_t> cls;  // N*N
  std::vector<double> lat, bw;
  // orders
  std::vector<int> id_rank;    // lexicographic rank of the device id
  std::vector<int> by_id_rank; // device index at each id rank
  std::vector<int> node_rank;  // lexicographic rank of the node name (global)
  int n_nodes = 0;
  // random_medium_assignment locality structure (search.cpp:163-186):
  // regions (lex) -> nodes (lex) -> devices (index order)
  std::vector<std::vector<std::vector<int>>> region_nodes;
  std::vector<int> region_node_count;
  // region links as given (for error messages and re-serialisation)
  std::vector<std::string> rl_src, rl_dst;
  std::vector<double> rl_lat_ms, rl_bw_gbps;
  double def_lat_ms = 0.1, def_bw_gbps = 100.0;
};

Problem build_problem(const hpg_problem& p);

DevCostConfig to_dev_cfg(const hpg_cost_config& c);
hpg_cost_config default_cost_config();

// One candidate in record form (common.hpp PlanRec) plus its host metadata.
struct Cand {
  std::vector<uint8_t> rec;
  RecOffsets o;
  int ng = 1;   // number of task groups (canonical-bytes accounting)
  RecHeader& hdr() { return *reinterpret_cast<RecHeader*>(rec.data()); }
  const RecHeader& hdr() const { return *reinterpret_cast<const RecHeader*>(rec.data()); }
  double* w() { return reinterpret_cast<double*>(rec.data() + o.w_byte); }
  int32_t* sl() { return reinterpret_cast<int32_t*>(rec.data() + o.sl_byte); }
  uint8_t* dev() { return rec.data() + o.dev_byte; }
  const double* w() const { return reinterpret_cast<const double*>(rec.data() + o.w_byte); }
  const int32_t* sl() const { return reinterpret_cast<const int32_t*>(rec.data() + o.sl_byte); }
  const uint8_t* dev() const { return rec.data() + o.dev_byte; }
  int size(int t) const { return o.dev[t + 1] - o.dev[t]; }
};

// Allocates a record for the given layouts; weights 1.0, uniform stage split
// (make_layout, plan.cpp:89-100), devices zeroed.
void init_cand(Cand& c, int T, const int* dp, const int* pp, const int* tp, const Problem& P);

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  void reserve(size_t n) {
    if (n <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    size_t c = n > cap * 2 ? n : cap * 2;
    if (c * sizeof(T) < (size_t{4} << 20)) c = (size_t{4} << 20) / sizeof(T);
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), c * sizeof(T)), "cudaMalloc");
    cap = c;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
template <typename T>
struct HostBuf {  // pinned
  T* p = nullptr;
  size_t cap = 0;
  void reserve(size_t n) {
    if (n <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    // geometric growth from 4 MiB: pinned allocations are slow, keep them rare
    size_t c = n > cap * 2 ? n : cap * 2;
    if (c * sizeof(T) < (size_t{4} << 20)) c = (size_t{4} << 20) / sizeof(T);
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&p), c * sizeof(T), cudaHostAllocDefault),
               "cudaHostAlloc");
    cap = c;
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

struct Batch {
  std::vector<const Cand*> cands;
  std::vector<int32_t> modes;
  // candidates whose devices the device generates (gen_ga.cu) before the
  // evaluation; GenItem.first / first_out index cands / the compact outputs
  std::vector<GenItem> gen;
  int n_gen = 0;                   // candidates covered by gen
  std::vector<int32_t> gen_item;   // [n_gen] item of each generated candidate
  std::vector<Rng> gen_starts;     // [n_gen] its stream state
};

// Multi-GPU: NCCL communicator of a context (created once, reused by every
// sharded search on it).
struct Dist {
  int rank = 0, world = 1;
  void* comm = nullptr;  // ncclComm_t
};
void dist_destroy(Dist& d);

struct BatchOut {
  std::vector<EvalResult> res;
  // what balancing changed in plan i, at out_ws + ws_off[i]: [generation
  // task weights | all stage layers] (apply_ws writes it into the record)
  const uint8_t* out_ws = nullptr;
  int64_t ws_bytes = 0;
  std::vector<int64_t> off, ws_off;
  std::vector<uint8_t> ws_store;  // chunked waves: the sections of every chunk
  // device-generated candidates (Batch::gen), by compact index j: their
  // device slots at gen_devs + gen_dev_off[j]
  const uint8_t* gen_devs = nullptr;
  std::vector<int64_t> gen_dev_off;
  std::vector<double> per_task;          // if requested
  std::vector<double> required;          // if requested
};

// Makes a context's GPU current for the duration of one C-ABI call and
// restores the caller's device afterwards (every entry point taking a context).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) cudaSetDevice(device);
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

struct Ctx {
  Problem prob;
  int device = 0;
  int n_sm = 0;
  cudaStream_t stream = nullptr;
  DevProblem dprob{};
  void* d_blob = nullptr;
  size_t blob_bytes = 0;
  HostBuf<uint8_t> h_blob;  // pinned staging of the problem tables
  // batch staging
  HostBuf<uint8_t> h_recs, h_out, h_recs2, h_out2;  // wave staging, two sets
  HostBuf<int64_t> h_off;
  HostBuf<int32_t> h_modes;
  HostBuf<EvalResult> h_res;
  DevBuf<uint8_t> d_recs, d_out, d_recs2, d_out2;
  DevBuf<int64_t> d_off;
  DevBuf<int32_t> d_modes;
  DevBuf<EvalResult> d_res;
  DevBuf<double> d_per_task, d_required;
  DevBuf<double> d_scratch;  // per-CTA global scratch of eval_kernel
  DevBuf<uint8_t> d_ring;    // device-wide ring memo (RingSlot table)
  DevBuf<uint8_t> d_xch_send, d_xch_recv;  // multi-GPU record exchange
  // device GA (ga_kernel.cuh): runs, record pools, results, queue, control
  DevBuf<uint8_t> d_ga;
  HostBuf<uint8_t> h_ga;
  // exhaustive_search block buffers (keys, dedup table, slots, records, ...)
  DevBuf<uint8_t> d_exh_keys, d_exh_recs;
  DevBuf<unsigned long long> d_exh_table, d_exh_slot, d_exh_count;
  DevBuf<EvalResult> d_exh_res;
  DevBuf<uint8_t> d_exh_part;
  Dist dist;                               // world 1 until hpg_search_dist attaches
  int64_t max_nl = 1;
  // sweep
  void* d_sweep_tables = nullptr;  // owns sweep_tb's arrays
  SweepTablesDev sweep_tb{};
  void* d_gen_tables = nullptr;  // owns gen_tb's arrays (GA candidates on the device)
  GenTablesDev gen_tb{};
  DevBuf<double> d_costs;
  DevBuf<uint8_t> d_feas;
  DevBuf<unsigned long long> d_best;
  DevBuf<uint8_t> d_sweep_gslab, d_sweep_part, d_sweep_order;
  DevBuf<uint8_t> d_prim;  // cost-model primitive calls (capi_prim.cpp)  // sweep_kernel fallback slabs, per-warp partials
  // best-half
  DevBuf<double> d_scores, d_events;
  DevBuf<int32_t> d_seg_off, d_arm_idx, d_keep;
  int64_t launches = 0;
  int64_t plans_evaluated = 0;
  // instrumentation for the bench contract
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  int64_t eval_launches = 0, canonical_bytes = 0;
  double eval_ms = 0.0;
  double host_ms = 0.0;   // GA coroutine time (candidate generation, bookkeeping)
  double batch_ms = 0.0;  // run_batch wall time (pack, copies, kernel, sync)
  double best_half_ms = 0.0;  // diagnostics: best_half_batch wall time
  int64_t best_half_calls = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // kernel timing, buffer set 0
  cudaEvent_t ev2 = nullptr, ev3 = nullptr;  // kernel timing, buffer set 1
  cudaEvent_t ev_done[2] = {nullptr, nullptr};  // wave results landed, per set
  cudaEvent_t ev_x[6] = {};  // diagnostics: copy timing
  ~Ctx();
};

Ctx* create_ctx(const hpg_problem& p, int device);
void stage_problem(Ctx& ctx, Problem&& P);
void restage(Ctx& ctx, const hpg_problem& p);
void reset_ring_memo(Ctx& ctx);

// Packs `b`, runs eval_kernel, returns per-plan results (and balanced records).
// writes a wave's [generation weights | stage layers] section into the record
void apply_ws(const Problem& P, Cand& c, const uint8_t* ws);
// problem tables of the device candidate generator (built on first use)
const GenTablesDev& gen_tables(Ctx& ctx);

void run_batch(Ctx& ctx, const Batch& b, const DevCostConfig& cfg, int kb_flags,
               bool want_out, bool want_per_task, bool want_required, BatchOut& out);

// Plan-table validation + packing (resolve_plan semantics, plan.cpp:257-349).
struct TablePlan {
  std::vector<std::vector<int>> groups;  // task slots per group
  std::vector<int> counts;
  Cand cand;
};
std::vector<TablePlan> unpack_table(const Problem& P, const hpg_plan_table& t);

}  // namespace hpg
