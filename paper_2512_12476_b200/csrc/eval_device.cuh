// Device side of the per-plan cost model: one warp evaluates one plan.
//
// Every formula restates the reference expression by expression, in the same
// association order, compiled with -fmad=false, so
// results are bit-identical to proj/src/cost_model.cpp and proj/src/plan.cpp.
// Only max/min folds are tree-reduced across lanes; every sum keeps the
// reference's sequential order.
//
// Geometry memo: inside one plan evaluation the tasklet->device assignment
// never changes (balancing only moves replica weights and stage splits), so
// TP rings, PP pairs and the gen->train bridge are computed once per plan and
// DP rings once per (stage, shard, stage-layer count). Same doubles as
// recomputing them, far fewer gathers.
#pragma once

#include <cstdint>

#include "common.hpp"

namespace hpg {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

// std::max / std::min semantics (NaN behaviour of the reference included)
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

__device__ __noinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = smax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __noinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = smin(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

struct Ws {
  // plan
  RecHeader h;
  RecOffsets o;
  double* w;
  int64_t* nm;
  int32_t* sl;
  uint8_t* dev;
  uint8_t* dstage;   // [T*N] stage of device d inside task t, 0xff = none
  // memo
  double* rtp;       // [cells] TP ring bottleneck per (task, replica, stage)
  double* ppp;       // [cells] cheapest cross-stage pair per (task, replica, stage)
  double* cmin;      // [cells] min over the cell's shards of Device::comp
  double* dpr;       // [dpk]   DP ring per (task, stage, shard)
  int32_t* dpr_sl;   // [dpk]   stage layers the DP memo was computed for
  // scratch
  double* resident;  // [N]
  double* c_comp;    // [N] per cell of the task in flight
  double* c_tp;
  double* c_pp;
  double* c_hbm;
  double* edge;      // [N]
  double* wnew;      // [N]
  double* cc;        // [kMaxClasses] class costs at the volume in flight
  double* rm;        // [64] small-ring cost matrix
  double* agg;       // [T*7]
  int32_t* sl_save;  // [sum pp]
  int32_t* split_best;   // [N]
  uint8_t* tour;     // [N]
  uint8_t* peers;    // [N]
  double* mmt;       // [sum pp] model_memory_bytes per (task, stage) at the current split
  double* wmt;       // [sum pp] working_memory_bytes per (task, stage)
  double* wsave;     // [N]
  int32_t* sl_save2;   // [sum pp]
  double* dtab;      // global scratch: DP ring maxima per (stage, layer count), -1 = unknown
  int32_t* cflag;    // global scratch after dtab: balance_layers column verdicts
  double* ccell;     // global scratch: balance_layers column cell pieces
  int32_t dtab_stride;
  int64_t nm_base[kMaxTasks];
  int32_t memo_tp_ok;   // bit t
  int32_t memo_pp_ok;
  int32_t memo_cm_ok;
  int32_t agg_ok;       // bit t: agg row t is end_to_end's task_cost for the current plan
  int32_t resident_ok;
  int32_t memv_ok, memv;  // cached check_memory of the current plan
  double bridge;
  int32_t bridge_ok;
  unsigned long long cc_sig;  // class-cost order signature of the staged volume
  int32_t cc_sig_ok;
  double cc_vol;              // staged volume
  int32_t cta_sync;           // sweep: CTA-wide barrier (threads) before each task's cost, 0 = none
  long long* prof;            // diagnostics: this plan's profile slots
  const uint8_t* cls;         // link class matrix [N*N]: shared-memory copy or P.cls
  // helper-warp team (one plan per CTA, warp 0 leads)
  Ws* team;                   // the CTA's Ws array (team[0] = lead)
  int32_t n_warps;
  volatile int32_t* job;      // [2]: kind, task mask (in team[0])
  int32_t job_words[2];
};

constexpr int kMaxTeam = kMaxTeamWarps;
constexpr int kJobTasks = 1, kJobExit = 2, kJobGeometry = 3, kJobStage = 4;

// diagnostics only (HPG_PLAN_PROFILE): per-plan clock64 phase stamps and
// per-phase cycle accumulators (sub-phase k < 27 also lands in the plan's
// slot 5 + k)
__device__ long long* g_plan_prof = nullptr;
__device__ unsigned long long g_phase_acc[32];
#define HPG_PH_BEGIN(k) const long long ph_##k = g_plan_prof ? clock64() : 0
#define HPG_PH_END(k)                                                         \
  do {                                                                        \
    if (g_plan_prof && s.prof && (threadIdx.x & 31) == 0) {                   \
      const long long dt_ = clock64() - ph_##k;                               \
      atomicAdd(&g_phase_acc[k], static_cast<unsigned long long>(dt_));       \
      if (k < 27) s.prof[5 + k] += dt_;                                       \
    }                                                                         \
  } while (0)
#define HPG_PH_COUNT(k, v)                                                    \
  do {                                                                        \
    if (g_plan_prof && (threadIdx.x & 31) == 0)                               \
      atomicAdd(&g_phase_acc[k], static_cast<unsigned long long>(v));         \
  } while (0)

// The current plan changed: task t's stage split (affects t, the generation
// task's decoding batch via residency, and memory feasibility) ...
__device__ __forceinline__ void invalidate_split(const DevProblem& P, Ws& s, int t) {
  if ((threadIdx.x & 31) == 0) {
    s.agg_ok &= ~(1 << t);
    if (P.gen_slot >= 0) s.agg_ok &= ~(1 << P.gen_slot);
    s.resident_ok = 0;
    s.memv_ok = 0;
  }
  __syncwarp();
}
// ... or task t's replica weights (only t's micro-batch counts move).
__device__ __forceinline__ void invalidate_weights(Ws& s, int t) {
  if ((threadIdx.x & 31) == 0) s.agg_ok &= ~(1 << t);
  __syncwarp();
}

__device__ __forceinline__ uint8_t* carve_ptr(uint8_t*& p, int bytes) {
  uint8_t* r = p;
  p += (bytes + 15) & ~15;
  return r;
}

__device__ inline uint8_t* carve(Ws& s, uint8_t* base, const Carve& c) {
  uint8_t* p = base;
  const int N = c.n_dev, T = c.n_tasks;
  s.w = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_w));
  s.nm = reinterpret_cast<int64_t*>(carve_ptr(p, 8 * c.max_w));
  s.rtp = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_cells));
  s.ppp = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_cells));
  s.dpr = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_dpk));
  s.resident = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_comp = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_tp = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_pp = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_hbm = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.edge = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.wnew = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.cc = reinterpret_cast<double*>(carve_ptr(p, 8 * kMaxClasses));
  s.rm = reinterpret_cast<double*>(carve_ptr(p, 8 * 64));
  s.agg = reinterpret_cast<double*>(carve_ptr(p, 8 * T * 7));
  s.sl = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.max_sl));
  s.sl_save = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.max_sl));
  s.dpr_sl = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.max_dpk));
  s.split_best = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * N));
  s.dev = carve_ptr(p, c.max_slots);
  s.dstage = carve_ptr(p, T * N);
  s.tour = carve_ptr(p, N);
  s.peers = carve_ptr(p, N);
  s.cmin = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_cells));
  s.mmt = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_sl));
  s.wmt = reinterpret_cast<double*>(carve_ptr(p, 8 * c.max_sl));
  s.wsave = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.sl_save2 = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.max_sl));
  s.cls = c.cls_smem ? carve_ptr(p, N * N) : nullptr;  // else P.cls (stage_link_classes)
  return p;
}

// a helper warp's private scratch (team_scratch_bytes); everything else in its
// Ws aliases the lead's plan state
__device__ inline uint8_t* carve_team_scratch(Ws& s, uint8_t* p, const Carve& c) {
  const int N = c.n_dev;
  s.c_comp = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_tp = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_pp = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_hbm = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.edge = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.cc = reinterpret_cast<double*>(carve_ptr(p, 8 * kMaxClasses));
  s.rm = reinterpret_cast<double*>(carve_ptr(p, 8 * 64));
  s.tour = carve_ptr(p, N);
  s.peers = carve_ptr(p, N);
  return p;
}

__device__ __forceinline__ void bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Stages the N x N link-class matrix in shared memory (once per CTA): every
// ring, pair and bridge edge cost is a lookup into it. Warp-collective.
__device__ inline void stage_link_classes(const DevProblem& P, Ws& s) {
  const int lane = threadIdx.x & 31;
  const int nn = P.n_dev * P.n_dev;
  uint8_t* dst = const_cast<uint8_t*>(s.cls);
  if ((nn & 7) == 0 && (reinterpret_cast<uintptr_t>(P.cls) & 7) == 0) {
    const uint2* src = reinterpret_cast<const uint2*>(P.cls);
    uint2* d2 = reinterpret_cast<uint2*>(dst);
    for (int i = lane; i < nn / 8; i += 32) d2[i] = src[i];
  } else {
    for (int i = lane; i < nn; i += 32) dst[i] = P.cls[i];
  }
  __syncwarp();
}

// ---- memory model (plan.cpp:160-220) ----

__device__ __forceinline__ double params_on_device(const DevTask& t, int sl_j, int tp,
                                                   int stage, int pp) {
  double p = static_cast<double>(sl_j) * static_cast<double>(t.layer_params) / tp;
  if (t.include_embedding) {
    const double emb = static_cast<double>(t.vocab) * static_cast<double>(t.h1) / tp;
    if (stage == 0) p += emb;
    if (stage == pp - 1) p += emb;
  }
  return p;
}

__device__ __forceinline__ double kv_bytes_per_sequence(const DevProblem& P, const DevTask& t,
                                                        int sl_j, int tp,
                                                        const DevCostConfig& cfg) {
  return static_cast<double>(P.seq_in + P.seq_out) * 2.0 * static_cast<double>(t.h1) *
         static_cast<double>(sl_j) * cfg.kv_bytes_per_elem / tp;
}

__device__ __forceinline__ double model_memory_bytes(const DevProblem& P, const DevTask& t,
                                                     int sl_j, int tp, int stage, int pp,
                                                     const DevCostConfig& cfg) {
  const double params = params_on_device(t, sl_j, tp, stage, pp);
  if (t.kind == kTraining) return params * cfg.train_bytes_per_param;
  if (t.kind == kInference) return params * cfg.infer_bytes_per_param;
  return params * cfg.infer_bytes_per_param +
         static_cast<double>(P.mbs) * cfg.dbs_cap * kv_bytes_per_sequence(P, t, sl_j, tp, cfg);
}

__device__ __forceinline__ double weights_memory_bytes(const DevTask& t, int sl_j, int tp,
                                                       int stage, int pp,
                                                       const DevCostConfig& cfg) {
  const double params = params_on_device(t, sl_j, tp, stage, pp);
  return t.kind == kTraining ? params * cfg.train_bytes_per_param
                             : params * cfg.infer_bytes_per_param;
}

__device__ __forceinline__ double working_memory_bytes(const DevProblem& P, const DevTask& t,
                                                       int sl_j, int tp,
                                                       const DevCostConfig& cfg) {
  return static_cast<double>(P.mbs) * static_cast<double>(P.seq_in + P.seq_out) *
         static_cast<double>(t.h1) * static_cast<double>(sl_j) * 2.0 * cfg.act_factor / tp;
}

// ---- formula helpers (cost_model.cpp:129-177, 220-241) ----

__device__ __forceinline__ double tp_comm_volume(int prec, int64_t mbs, int64_t seq_total,
                                                 int64_t h1, int tp) {
  return static_cast<double>(prec) * static_cast<double>(mbs) *
         static_cast<double>(seq_total) * static_cast<double>(h1) * (2.0 * (tp - 1) / tp);
}
__device__ __forceinline__ double pp_comm_volume(int prec, int64_t mbs, int64_t seq_total,
                                                 int64_t h1) {
  return static_cast<double>(prec) * static_cast<double>(mbs) *
         static_cast<double>(seq_total) * static_cast<double>(h1);
}
__device__ __forceinline__ double dp_comm_volume(int prec, int64_t nl_j, int64_t h1, int64_t h2,
                                                 int dp, int tp) {
  return static_cast<double>(prec) * static_cast<double>(nl_j) *
         (4.0 * static_cast<double>(h1) * static_cast<double>(h1) +
          3.0 * static_cast<double>(h1) * static_cast<double>(h2)) *
         (2.0 * (dp - 1) / (static_cast<double>(dp) * tp));
}
__device__ __forceinline__ double layer_flops(int64_t s, int64_t h1, int64_t h2) {
  const double sd = static_cast<double>(s);
  const double h1d = static_cast<double>(h1);
  const double h2d = static_cast<double>(h2);
  return 2.0 * 4.0 * sd * h1d * h1d + 2.0 * 2.0 * sd * sd * h1d + 2.0 * 3.0 * sd * h1d * h2d;
}
__device__ __forceinline__ double tp_pass_factor(int kind, bool recompute) {
  if (kind != kTraining) return 2.0;
  return recompute ? 6.0 : 4.0;
}
__device__ __forceinline__ double pp_pass_factor(int kind) { return kind == kTraining ? 2.0 : 1.0; }
__device__ __forceinline__ double comp_pass_factor(int kind) {
  return kind == kTraining ? 3.0 : 1.0;
}
__device__ __forceinline__ int64_t comp_seq(const DevProblem& P, int kind) {
  return kind == kGeneration ? P.seq_in : P.seq_in + P.seq_out;
}
__device__ __forceinline__ double compute_cost(int kind, int64_t nm, int64_t mbs, int64_t nl_j,
                                               double flops, double comp_d, int tp) {
  return comp_pass_factor(kind) * static_cast<double>(nm) * static_cast<double>(mbs) *
         static_cast<double>(nl_j) * flops / (comp_d * tp);
}
__device__ __forceinline__ double hbm_decode_cost(int64_t seq_out, int64_t nm, int64_t mbs,
                                                  int prec, int64_t nl_j, int64_t h1,
                                                  int64_t h2, double dbs, double hbm_d, int tp) {
  const double weight_bytes =
      static_cast<double>(prec) * static_cast<double>(nl_j) *
      (4.0 * static_cast<double>(h1) * static_cast<double>(h1) +
       3.0 * static_cast<double>(h1) * static_cast<double>(h2));
  return static_cast<double>(seq_out) * static_cast<double>(nm) * static_cast<double>(mbs) *
         weight_bytes / (dbs * hbm_d * tp);
}

// ---- plan staging ----

__device__ __forceinline__ int flat(int i, int j, int k, int pp, int tp) {
  return (i * pp + j) * tp + k;
}

// nm_base (workflow.cpp:148-157) and apportion_microbatches (plan.cpp:222-255)
__device__ __noinline__ void apportion(const DevProblem& P, Ws& s, int t) {
  const int lane = threadIdx.x & 31;
  const int dp = s.h.dp[t];
  const int64_t denom = static_cast<int64_t>(dp) * P.mbs;
  const int64_t nm_base = (P.total_seq + denom - 1) / denom;
  const double* w = s.w + s.o.w[t];
  int64_t* out = s.nm + s.o.w[t];
  if (lane == 0) s.nm_base[t] = nm_base;
  const int64_t total = nm_base * dp;
  // unit weights: wsum == dp exactly, every quota is exactly nm_base, no
  // remainder to hand out
  bool unit = true;
  for (int i = lane; i < dp; i += 32) unit &= w[i] == 1.0;
  if (__all_sync(kFull, unit)) {
    for (int i = lane; i < dp; i += 32) out[i] = nm_base;
    __syncwarp();
    return;
  }
  double wsum = 0.0;  // std::accumulate, sequential (all lanes redundantly)
  for (int i = 0; i < dp; ++i) wsum += w[i];
  // floor of quotas + remainders (remainders staged in s.edge, free here)
  double* rem = s.edge;
  int64_t assigned_part = 0;
  for (int i = lane; i < dp; i += 32) {
    const double quota = static_cast<double>(total) * w[i] / wsum;
    const int64_t f = static_cast<int64_t>(floor(quota));
    out[i] = f;
    rem[i] = quota - static_cast<double>(f);
    assigned_part += f;
  }
  for (int o = 16; o > 0; o >>= 1) assigned_part += __shfl_xor_sync(kFull, assigned_part, o);
  const int64_t deficit = total - assigned_part;
  __syncwarp();
  if (deficit > 0) {
    // rank of replica i in (remainder desc, index asc); deficit hands out one
    // micro-batch per rank position, cycling (plan.cpp:236-244)
    for (int i = lane; i < dp; i += 32) {
      const double ri = rem[i];
      int rank = 0;
      for (int k = 0; k < dp; ++k) {
        const double rk = rem[k];
        if (rk > ri || (rk == ri && k < i)) ++rank;
      }
      const int64_t extra = deficit / dp + (rank < deficit % dp ? 1 : 0);
      out[i] += extra;
    }
    __syncwarp();
  }
  // every replica processes at least one micro-batch (plan.cpp:246-253)
  bool any_zero = false;
  for (int i = lane; i < dp; i += 32) any_zero |= out[i] == 0;
  if (__any_sync(kFull, any_zero)) {
    if (lane == 0) {
      for (int i = 0; i < dp; ++i) {
        while (out[i] == 0) {
          int donor = 0;
          for (int k = 1; k < dp; ++k)
            if (out[donor] < out[k]) donor = k;  // std::max_element: first max
          --out[donor];
          ++out[i];
        }
      }
    }
    __syncwarp();
  }
}

__device__ inline void build_dstage(const DevProblem& P, Ws& s) {
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev;
  for (int e = lane; e < P.n_tasks * N; e += 32) s.dstage[e] = 0xff;
  __syncwarp();
  for (int t = 0; t < P.n_tasks; ++t) {
    const int pp = s.h.pp[t], tp = s.h.tp[t], size = s.h.dp[t] * pp * tp;
    const uint8_t* dv = s.dev + s.o.dev[t];
    for (int e = lane; e < size; e += 32) s.dstage[t * N + dv[e]] = static_cast<uint8_t>((e / tp) % pp);
  }
  __syncwarp();
}

// check_memory (plan.cpp:351-380): sum of model memory in task order plus the
// max working set, per device. Returns true when every device fits.
// model_memory_bytes / working_memory_bytes of every stage of task t at the
// current split (the per-device sums below only look these up).
__device__ __forceinline__ void mem_tables(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                           int t) {
  const int lane = threadIdx.x & 31;
  const int pp = s.h.pp[t], tp = s.h.tp[t], o = s.o.sl[t];
  __syncwarp();
  for (int j = lane; j < pp; j += 32) {
    s.mmt[o + j] = model_memory_bytes(P, P.task[t], s.sl[o + j], tp, j, pp, cfg);
    s.wmt[o + j] = working_memory_bytes(P, P.task[t], s.sl[o + j], tp, cfg);
  }
  __syncwarp();
}

__device__ __noinline__ bool check_memory(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                          double* required_out = nullptr) {
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev;
  if (!required_out && s.memv_ok) return s.memv != 0;
  bool viol = false;
  for (int d = lane; d < N; d += 32) {
    double ms = 0.0, wm = 0.0;
    for (int t = 0; t < P.n_tasks; ++t) {
      const int j = s.dstage[t * N + d];
      if (j == 0xff) continue;
      ms += s.mmt[s.o.sl[t] + j];
      wm = smax(wm, s.wmt[s.o.sl[t] + j]);
    }
    const double req = ms + wm;
    if (required_out) required_out[d] = req;
    if (req > P.mem[d]) viol = true;
  }
  const bool ok = !__any_sync(kFull, viol);
  __syncwarp();
  if (lane == 0) {
    s.memv = ok ? 1 : 0;
    s.memv_ok = 1;
  }
  __syncwarp();
  return ok;
}

// ---- communication primitives (cost_model.cpp:18-125, 179-218) ----

__device__ __forceinline__ void class_costs(const DevProblem& P, Ws& s, double volume) {
  const int lane = threadIdx.x & 31;
  HPG_PH_BEGIN(20);
  __syncwarp();
  for (int c = lane; c < P.n_classes; c += 32) s.cc[c] = P.lat[c] + volume / P.bw[c];
  if (lane == 0) {
    s.cc_sig_ok = 0;
    s.cc_vol = volume;
  }
  __syncwarp();
  HPG_PH_END(20);
}

// order signature of the staged class costs (computed on first use): rank of
// every class cost among all classes (ties share a rank), 4 bits per class.
// Every ring algorithm below decides only by comparing class costs, so equal
// signatures mean identical decisions. Warp-collective.
__device__ __noinline__ unsigned long long cc_signature(const DevProblem& P, Ws& s) {
  const int lane = threadIdx.x & 31;
  if (s.cc_sig_ok) return s.cc_sig;
  unsigned long long sig = 0;
  if (P.n_classes <= 16 && lane < P.n_classes) {
    int rank = 0;
    for (int c = 0; c < P.n_classes; ++c) rank += s.cc[c] < s.cc[lane] ? 1 : 0;
    sig = static_cast<unsigned long long>(rank) << (4 * lane);
  }
  for (int o = 16; o > 0; o >>= 1) sig |= __shfl_xor_sync(kFull, sig, o);
  __syncwarp();
  if (lane == 0) {
    s.cc_sig = sig;
    s.cc_sig_ok = 1;
  }
  __syncwarp();
  return sig;
}

__device__ __forceinline__ double ecost(const DevProblem& P, const Ws& s, int a, int b) {
  return s.cc[s.cls[a * P.n_dev + b]];
}

// ---- device-wide ring memo (common.hpp RingSlot) ----

__device__ __forceinline__ unsigned long long mix64d(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct RingKey {
  unsigned long long k1, k2, k3;
};

// Exact key for n <= 8 (packed device bytes + n); two independent 64-bit
// position-aware hashes otherwise (collision odds ~2^-128). k2 is the
// class-cost order signature (<= 16 classes; the slot then stores the
// bottleneck's link class, valid at every volume with the same order) or the
// volume bits (the slot stores the value). Warp-collective.
constexpr unsigned long long kSigMode = 1ull << 63;

__device__ __noinline__ RingKey ring_key(const DevProblem& P, Ws& s,
                                            const uint8_t* devs, int n) {
  const int lane = threadIdx.x & 31;
  RingKey k;
  const bool sig = P.n_classes <= 16;
  k.k2 = sig ? cc_signature(P, s) : static_cast<unsigned long long>(__double_as_longlong(s.cc_vol));
  const unsigned long long mode = sig ? kSigMode : 0ull;
  if (n <= 8) {
    unsigned long long p = 0;
    for (int i = 0; i < n; ++i) p |= static_cast<unsigned long long>(devs[i]) << (8 * i);
    k.k1 = p == 0 ? 1 : p;
    k.k3 = static_cast<unsigned long long>(n) | mode;
    return k;
  }
  unsigned long long a = 0, b = 0;
  for (int i = lane; i < n; i += 32) {
    const unsigned long long x = (static_cast<unsigned long long>(i) << 8) | devs[i];
    a += mix64d(x ^ 0x5851f42d4c957f2dULL);
    b += mix64d(x ^ 0x14057b7ef767814fULL);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(kFull, a, o);
    b += __shfl_xor_sync(kFull, b, o);
  }
  k.k1 = a == 0 ? 1 : a;
  k.k3 = ((b + static_cast<unsigned long long>(n)) & ~kSigMode) | mode;
  return k;
}

// cached payload -> ring value at the staged volume
__device__ __forceinline__ double ring_payload_value(const Ws& s, const RingKey& k, double stored) {
  if (k.k3 & kSigMode) return s.cc[__double_as_longlong(stored)];
  return stored;
}

// ring value -> payload: the class whose cost equals the bottleneck (any of
// equal-cost classes: they stay equal under the same order signature)
__device__ __forceinline__ bool ring_payload_of(const DevProblem& P, const Ws& s, const RingKey& k,
                                                double v, double& stored) {
  if (!(k.k3 & kSigMode)) {
    stored = v;
    return true;
  }
  const int lane = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(kFull, lane < P.n_classes && s.cc[lane] == v);
  if (!bal) return false;
  stored = __longlong_as_double(static_cast<long long>(__ffs(bal) - 1));
  return true;
}

// lane 0 probes; result broadcast. Returns true and sets v on a hit. Keys of
// rings with n > 8 are hashes: a hit is confirmed against the device
// sequence stored with the slot, byte for byte (warp-collective), so a hash
// collision reads as a miss and never changes a ring's value.
__device__ __noinline__ bool ring_lookup(const DevProblem& P, const RingKey& k, double& v,
                                         const uint8_t* devs, int n) {
  const int lane = threadIdx.x & 31;
  int hit = 0;
  double val = 0.0;
  unsigned long long seq = 0;
  if (lane == 0 && P.ring_cache) {
    const unsigned long long h = (k.k1 ^ mix64d(k.k2 ^ k.k3)) & P.ring_mask;
    for (int pr = 0; pr < 8; ++pr) {
      volatile RingSlot* sl = P.ring_cache + ((h + pr) & P.ring_mask);
      const unsigned long long a = sl->k1;
      if (a == 0) break;
      if (a != k.k1) continue;
      if (sl->state != 1) break;  // being published: treat as a miss
      __threadfence();
      if (sl->k2 == k.k2 && sl->k3 == k.k3) {
        val = sl->value;
        seq = sl->seq;
        hit = 1;
        break;
      }
    }
  }
  hit = __shfl_sync(kFull, hit, 0);
  if (hit && n > 8) {
    seq = __shfl_sync(kFull, seq, 0);
    const uint8_t* stored = P.ring_arena + (seq >> 16);
    bool diff = static_cast<int>(seq & 0xffffull) != n;
    if (!diff)
      for (int i = lane; i < n; i += 32) diff |= __ldcg(stored + i) != devs[i];
    if (__any_sync(kFull, diff)) hit = 0;
  }
  v = __shfl_sync(kFull, val, 0);
  return hit != 0;
}

__device__ __noinline__ void ring_insert(const DevProblem& P, const RingKey& k, double v,
                                         const uint8_t* devs, int n) {
  if (!P.ring_cache) return;
  const int lane = threadIdx.x & 31;
  // n > 8: the sequence goes to the arena first (no room: not memoised)
  unsigned long long off = 0;
  if (n > 8) {
    if (lane == 0) {
      off = atomicAdd(reinterpret_cast<unsigned long long*>(P.ring_arena),
                      static_cast<unsigned long long>(n));
      if (off + n > P.ring_arena_cap) off = 0;
    }
    off = __shfl_sync(kFull, off, 0);
    if (off == 0) return;
    for (int i = lane; i < n; i += 32) P.ring_arena[off + i] = devs[i];
    __threadfence();
    __syncwarp();
  }
  if (lane != 0) return;
  const unsigned long long h = (k.k1 ^ mix64d(k.k2 ^ k.k3)) & P.ring_mask;
  for (int pr = 0; pr < 8; ++pr) {
    RingSlot* sl = P.ring_cache + ((h + pr) & P.ring_mask);
    const unsigned long long prev = atomicCAS(&sl->k1, 0ULL, k.k1);
    if (prev == 0) {
      volatile RingSlot* vs = sl;
      vs->k2 = k.k2;
      vs->k3 = k.k3;
      vs->value = v;
      vs->seq = (off << 16) | static_cast<unsigned long long>(n);
      __threadfence();
      vs->state = 1;
      return;
    }
    if (prev == k.k1) return;  // someone else owns this key's slot
  }
}

// Exact min-bottleneck Hamiltonian cycle, 3 <= n <= 8 (the reference's
// RingSearch::dfs regime, cost_model.cpp:94-125, 196-206). The answer is a min
// of maxes of the same doubles, so any exact method returns identical bits:
// bounds first (LB = max over vertices of the 2nd-cheapest incident edge,
// UB = identity tour), then a lane-parallel DFS over 2-vertex prefixes.
// ub_known >= 0: the caller already has UB (and knows LB < UB).
__device__ __noinline__ double ring_small(const DevProblem& P, Ws& s, const uint8_t* devs, int n,
                                          double ub_known) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int e = lane; e < n * n; e += 32) s.rm[e] = ecost(P, s, devs[e / n], devs[e % n]);
  __syncwarp();
  const double* rm = s.rm;
  // lane v: its identity-tour edge (UB) and its 2nd-cheapest incident edge (LB)
  double ub = ub_known, lb = 0.0;
  if (ub_known < 0.0) {
    ub = 0.0;
    if (lane < n) {
      ub = rm[lane * n + (lane + 1) % n];
      double m1 = kInf, m2 = kInf;
      for (int u = 0; u < n; ++u) {
        if (u == lane) continue;
        const double c = rm[lane * n + u];
        if (c < m1) {
          m2 = m1;
          m1 = c;
        } else if (c < m2) {
          m2 = c;
        }
      }
      lb = m2;
    }
    ub = warp_max(ub);
    lb = warp_max(lb);
    if (ub == lb) return ub;
  }
  RingKey key;
  if (P.ring_cache) {
    key = ring_key(P, s, devs, n);
    double cached;
    if (ring_lookup(P, key, cached, devs, n)) return ring_payload_value(s, key, cached);
  }
  double best = ub;
  const int m = n - 1;
  const int nprefix = m * (m - 1);
  for (int p = lane; p < nprefix; p += 32) {
    const int a = 1 + p / (m - 1);
    const int bi = p % (m - 1);
    const int b = 1 + bi + ((1 + bi) >= a ? 1 : 0);
    const double c2 = smax(rm[a], rm[a * n + b]);
    if (c2 >= best) continue;
    if (n == 3) {
      best = smin(best, smax(c2, rm[b * n]));
      continue;
    }
    int path[8];
    double cmx[8];
    int nxt[9];
    path[0] = 0;
    path[1] = a;
    path[2] = b;
    cmx[2] = c2;
    unsigned used = 1u | (1u << a) | (1u << b);
    int d = 3;
    nxt[3] = 1;
    while (d >= 3) {
      if (d == n) {
        best = smin(best, smax(cmx[n - 1], rm[path[n - 1] * n]));
        --d;
        used &= ~(1u << path[d]);
        continue;
      }
      int v = nxt[d];
      while (v < n && ((used >> v) & 1u)) ++v;
      if (v >= n) {
        --d;
        if (d >= 3) used &= ~(1u << path[d]);
        continue;
      }
      nxt[d] = v + 1;
      const double c = smax(cmx[d - 1], rm[path[d - 1] * n + v]);
      if (c >= best) continue;
      path[d] = v;
      cmx[d] = c;
      used |= 1u << v;
      ++d;
      nxt[d] = 1;
    }
  }
  best = warp_min(best);
  double stored;
  if (P.ring_cache && ring_payload_of(P, s, key, best, stored)) ring_insert(P, key, stored, devs, n);
  return best;
}

// Open TP cells of one 32-cell block (LB < UB after the bounds pass), rings
// of 3 <= n <= 8 devices, batched over the warp instead of one ring_small per
// cell: memo probes and inserts one lane per cell (the n <= 8 keys are
// exact), then the exact DFS over (cell, 2-vertex prefix) items dealt
// round-robin to the lanes. Each cell's incumbent (its identity-tour UB to
// start) is shared through a 64-bit atomicMin on its bit pattern in ubb
// (costs >= 0 order like their bits), so a cycle found by any lane prunes the
// others. The result is the min over all cycles of the max edge, the same
// double ring_small returns.
__device__ __forceinline__ int nth_set_bit(unsigned m, int k) {
  for (int i = 0; i < k; ++i) m &= m - 1;
  return __ffs(m) - 1;
}

__device__ __noinline__ void open_rings(const DevProblem& P, Ws& s, const uint8_t* dv, int n,
                                        int c0, unsigned open, unsigned long long* ubb,
                                        double* out) {
  const int lane = threadIdx.x & 31;
  const bool memo = P.ring_cache != nullptr;
  const bool sig = P.n_classes <= 16;
  unsigned long long k2 = 0;
  if (memo) k2 = sig ? cc_signature(P, s) : static_cast<unsigned long long>(__double_as_longlong(s.cc_vol));
  const unsigned long long k3 = static_cast<unsigned long long>(n) | (sig ? kSigMode : 0ull);
  const int nopen = __popc(open);
  int my_c = -1;
  unsigned long long my_k1 = 0, h = 0;
  bool hit = false;
  if (lane < nopen) {
    my_c = c0 + nth_set_bit(open, lane);
    const uint8_t* r = dv + my_c * n;
    unsigned long long pk = 0;
    for (int i = 0; i < n; ++i) pk |= static_cast<unsigned long long>(r[i]) << (8 * i);
    my_k1 = pk == 0 ? 1 : pk;
    if (memo) {
      // ring_lookup's probe (n <= 8: the key is the ring itself)
      h = (my_k1 ^ mix64d(k2 ^ k3)) & P.ring_mask;
      for (int pr = 0; pr < 8; ++pr) {
        volatile RingSlot* sl = P.ring_cache + ((h + pr) & P.ring_mask);
        const unsigned long long a = sl->k1;
        if (a == 0) break;
        if (a != my_k1) continue;
        if (sl->state != 1) break;
        __threadfence();
        if (sl->k2 == k2 && sl->k3 == k3) {
          const double val = sl->value;
          out[my_c] = sig ? s.cc[__double_as_longlong(val)] : val;
          hit = true;
          break;
        }
      }
    }
  }
  const unsigned miss = __ballot_sync(kFull, lane < nopen && !hit);
  if (miss) {
    const int N = P.n_dev;
    const int m = n - 1, npre = m * (m - 1);
    const int items = __popc(miss) * npre;
    for (int it = lane; it < items; it += 32) {
      const int k = it / npre, p = it - k * npre;
      const int c = c0 + nth_set_bit(open, nth_set_bit(miss, k));
      const uint8_t* r = dv + c * n;
      unsigned long long dw = 0;
      for (int i = 0; i < n; ++i) dw |= static_cast<unsigned long long>(r[i]) << (8 * i);
      // rm[i * n + j] of ring_small = ecost(devs[i], devs[j])
      auto E = [&](int i, int j) {
        return s.cc[s.cls[static_cast<int>((dw >> (8 * i)) & 255u) * N +
                          static_cast<int>((dw >> (8 * j)) & 255u)]];
      };
      const int a = 1 + p / (m - 1);
      const int bi = p % (m - 1);
      const int b = 1 + bi + ((1 + bi) >= a ? 1 : 0);
      double best = __longlong_as_double(static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&ubb[c - c0])));
      const double start = best;
      const double c2 = smax(E(0, a), E(a, b));
      if (c2 >= best) continue;
      if (n == 3) {
        best = smin(best, smax(c2, E(b, 0)));
      } else {
        int path[8];
        double cmx[8];
        int nxt[9];
        path[0] = 0;
        path[1] = a;
        path[2] = b;
        cmx[2] = c2;
        unsigned used = 1u | (1u << a) | (1u << b);
        int d = 3;
        nxt[3] = 1;
        while (d >= 3) {
          if (d == n) {
            best = smin(best, smax(cmx[n - 1], E(path[n - 1], 0)));
            --d;
            used &= ~(1u << path[d]);
            continue;
          }
          int v = nxt[d];
          while (v < n && ((used >> v) & 1u)) ++v;
          if (v >= n) {
            --d;
            if (d >= 3) used &= ~(1u << path[d]);
            continue;
          }
          nxt[d] = v + 1;
          const double cc = smax(cmx[d - 1], E(path[d - 1], v));
          if (cc >= best) continue;
          path[d] = v;
          cmx[d] = cc;
          used |= 1u << v;
          ++d;
          nxt[d] = 1;
        }
      }
      if (best < start)
        atomicMin(&ubb[c - c0], static_cast<unsigned long long>(__double_as_longlong(best)));
    }
    __syncwarp();
    if ((miss >> lane) & 1u) {
      const double v = __longlong_as_double(
          static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&ubb[my_c - c0])));
      out[my_c] = v;
      if (memo) {
        // ring_payload_of + ring_insert (n <= 8: no arena), one lane per cell
        double stored = v;
        bool ok = true;
        if (sig) {
          ok = false;
          for (int j = 0; j < P.n_classes; ++j)
            if (s.cc[j] == v) {
              stored = __longlong_as_double(static_cast<long long>(j));
              ok = true;
              break;
            }
        }
        if (ok) {
          for (int pr = 0; pr < 8; ++pr) {
            RingSlot* sl = P.ring_cache + ((h + pr) & P.ring_mask);
            const unsigned long long prev = atomicCAS(&sl->k1, 0ULL, my_k1);
            if (prev == 0) {
              volatile RingSlot* vs = sl;
              vs->k2 = k2;
              vs->k3 = k3;
              vs->value = stored;
              vs->seq = static_cast<unsigned long long>(n);
              __threadfence();
              vs->state = 1;
              break;
            }
            if (prev == my_k1) break;
          }
        }
      }
    }
  }
  __syncwarp();
}

// Top-2 (value, position) among edges, excluding positions ex0/ex1.
__device__ __forceinline__ void top2_merge(double& v1, int& p1, double& v2, int& p2, double ov1,
                                           int op1, double ov2, int op2) {
  // merge two top-2 lists (values only matter; positions distinct by construction)
  double a[4] = {v1, v2, ov1, ov2};
  int b[4] = {p1, p2, op1, op2};
  double bv1 = -kInf, bv2 = -kInf;
  int bp1 = -1, bp2 = -1;
  for (int i = 0; i < 4; ++i) {
    if (b[i] < 0) continue;
    if (b[i] == bp1 || b[i] == bp2) continue;
    if (bp1 < 0 || a[i] > bv1) {
      bv2 = bv1;
      bp2 = bp1;
      bv1 = a[i];
      bp1 = b[i];
    } else if (bp2 < 0 || a[i] > bv2) {
      bv2 = a[i];
      bp2 = b[i];
    }
  }
  v1 = bv1;
  p1 = bp1;
  v2 = bv2;
  p2 = bp2;
}

// Nearest neighbour from devs[0] + bottleneck 2-opt, replicated exactly
// (heuristic_ring, cost_model.cpp:27-90): NN picks the earliest span position
// among the minima; 2-opt scans (i, j) lexicographically, continues after an
// acceptance, at most 8 passes, stops after a pass without improvement.
// A swap can only be accepted when every max-valued edge is one of the two
// removed edges, so each scan only visits the O(n) pairs that can succeed;
// the rejected pairs the reference visits change nothing.
__device__ __noinline__ double ring_heuristic(const DevProblem& P, Ws& s, const uint8_t* devs, int n) {
  const int lane = threadIdx.x & 31;
  uint8_t* tour = s.tour;
  double* edge = s.edge;
  bool used[8] = {false, false, false, false, false, false, false, false};
  if (lane == 0) used[0] = true;
  int last = devs[0];
  if (lane == 0) tour[0] = devs[0];
  for (int step = 1; step < n; ++step) {
    double bc = kInf;
    int bi = 0x7fffffff;
    for (int r = 0; r < 8; ++r) {
      const int i = lane + 32 * r;
      if (i >= n) break;
      if (!used[r]) {
        const double c = ecost(P, s, last, devs[i]);
        if (c < bc) {
          bc = c;
          bi = i;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double oc = __shfl_xor_sync(kFull, bc, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (oc < bc || (oc == bc && oi < bi)) {
        bc = oc;
        bi = oi;
      }
    }
    if ((bi & 31) == lane) used[bi >> 5] = true;
    last = devs[bi];
    if (lane == 0) tour[step] = static_cast<uint8_t>(last);
  }
  __syncwarp();
  double bott = 0.0;
  for (int i = lane; i < n; i += 32) {
    edge[i] = ecost(P, s, tour[i], tour[(i + 1) % n]);
    bott = smax(bott, edge[i]);
  }
  bott = warp_max(bott);
  __syncwarp();
  for (int pass = 0; pass < 8 && bott > 0; ++pass) {
    bool improved = false;
    int ci = 1, cj = 2;  // lexicographic resume point of the scan
    while (ci <= n - 2) {
      // positions holding the bottleneck value
      int cnt = 0, p = 0x7fffffff, q = 0x7fffffff;
      for (int i = lane; i < n; i += 32) {
        if (edge[i] == bott) {
          ++cnt;
          if (i < p) {
            q = p;
            p = i;
          } else if (i < q) {
            q = i;
          }
        }
      }
      cnt = warp_sum_i(cnt);
      if (cnt >= 3) break;
      for (int o = 16; o > 0; o >>= 1) {
        const int op = __shfl_xor_sync(kFull, p, o);
        const int oq = __shfl_xor_sync(kFull, q, o);
        int np, nq;
        if (op < p) {
          np = op;
          nq = min(p, oq);
        } else {
          np = p;
          nq = min(q, op);
        }
        p = np;
        q = nq;
      }
      // top-2 among non-bottleneck positions (for "rest")
      double v1 = -kInf, v2 = -kInf;
      int p1 = -1, p2 = -1;
      for (int i = lane; i < n; i += 32) {
        if (i == p || (cnt == 2 && i == q)) continue;
        top2_merge(v1, p1, v2, p2, edge[i], i, -kInf, -1);
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov1 = __shfl_xor_sync(kFull, v1, o);
        const int op1 = __shfl_xor_sync(kFull, p1, o);
        const double ov2 = __shfl_xor_sync(kFull, v2, o);
        const int op2 = __shfl_xor_sync(kFull, p2, o);
        top2_merge(v1, p1, v2, p2, ov1, op1, ov2, op2);
      }
      // candidate list in lexicographic order
      int na = 0, nb = 0;
      int a_lo = 1, b_lo = 0;
      if (cnt == 2) {
        // single candidate (p+1, q)
        na = 0;
        if (p + 1 <= n - 2 && q >= p + 2) {
          nb = 1;
        }
        b_lo = q;
      } else {
        if (p >= 2) na = p - 1;  // (i, p), i = 1..p-1
        if (p + 1 <= n - 2) nb = n - 1 - (p + 1);  // (p+1, j), j = p+2..n-1
        b_lo = p + 2;
      }
      const int total = na + nb;
      bool found = false;
      int fi = 0, fj = 0;
      double fn1 = 0, fn2 = 0, fcand = 0;
      for (int base = 0; base < total && !found; base += 32) {
        const int c = base + lane;
        bool acc = false;
        int i = 0, j = 0;
        double n1 = 0, n2 = 0, cd = 0;
        if (c < total) {
          if (c < na) {
            i = a_lo + c;
            j = p;
          } else if (cnt == 2) {
            i = p + 1;
            j = q;
          } else {
            i = p + 1;
            j = b_lo + (c - na);
          }
          const bool after = (i > ci) || (i == ci && j >= cj);
          if (after) {
            n1 = ecost(P, s, tour[i - 1], tour[j]);
            n2 = ecost(P, s, tour[i], tour[(j + 1) % n]);
            double rest;
            if (cnt == 2) {
              rest = v1;
            } else {
              const int x = (i - 1 == p) ? j : i - 1;
              rest = (p1 != x) ? v1 : v2;
            }
            cd = smax(smax(n1, n2), rest);
            acc = cd < bott;
          }
        }
        const unsigned bal = __ballot_sync(kFull, acc);
        if (bal) {
          const int src = __ffs(bal) - 1;
          fi = __shfl_sync(kFull, i, src);
          fj = __shfl_sync(kFull, j, src);
          fn1 = __shfl_sync(kFull, n1, src);
          fn2 = __shfl_sync(kFull, n2, src);
          fcand = __shfl_sync(kFull, cd, src);
          found = true;
        }
      }
      if (!found) break;
      // std::reverse(tour+i, tour+j+1); std::reverse(edge+i, edge+j)
      __syncwarp();
      const int len_t = fj - fi + 1;
      for (int k = lane; k < len_t / 2; k += 32) {
        const uint8_t tmp = tour[fi + k];
        tour[fi + k] = tour[fj - k];
        tour[fj - k] = tmp;
      }
      const int len_e = fj - fi;
      for (int k = lane; k < len_e / 2; k += 32) {
        const double tmp = edge[fi + k];
        edge[fi + k] = edge[fj - 1 - k];
        edge[fj - 1 - k] = tmp;
      }
      __syncwarp();
      if (lane == 0) {
        edge[fi - 1] = fn1;
        edge[fj] = fn2;
      }
      __syncwarp();
      bott = fcand;
      improved = true;
      ci = fi;
      cj = fj + 1;
      if (cj > n - 1) {
        ci = fi + 1;
        cj = ci + 1;
      }
    }
    if (!improved) break;
  }
  __syncwarp();
  return bott;
}

// min_ring_bottleneck (cost_model.cpp:179-207); class costs must be staged.
__device__ inline double ring_bottleneck_impl(const DevProblem& P, Ws& s, const uint8_t* devs,
                                              int n, double volume) {
  if (n <= 1) return 0.0;
  if (n == 2) return ecost(P, s, devs[0], devs[1]);
  if (n <= 8) return ring_small(P, s, devs, n, -1.0);
  if (!P.ring_cache) return ring_heuristic(P, s, devs, n);
  const RingKey key = ring_key(P, s, devs, n);
  double v;
  if (ring_lookup(P, key, v, devs, n)) return ring_payload_value(s, key, v);
  v = ring_heuristic(P, s, devs, n);
  double stored;
  if (ring_payload_of(P, s, key, v, stored)) ring_insert(P, key, stored, devs, n);
  return v;
}

__device__ inline double ring_bottleneck(const DevProblem& P, Ws& s, const uint8_t* devs, int n,
                                         double volume) {
  HPG_PH_BEGIN(21);
  const double v = ring_bottleneck_impl(P, s, devs, n, volume);
  HPG_PH_END(21);
  return v;
}

// ---- task_cost_detail (cost_model.cpp:270-396) ----
//
// Leaves per-cell comp/tp/pp/hbm in s.c_* for the balancers and writes the
// aggregate TaskCost (comp, tp, pp, dp, bubble, hbm, total) to agg[0..6].
// HBM decode cost of one generation cell (cost_model.cpp:315-337): max over
// the cell's shards of hbm_decode_cost. The shards share the numerator, so
// the max is the numerator over the smallest denominator (dbs*hbm_d)*tp
// (IEEE division is monotone); dbs per shard from the free memory after the
// resident weights (whole-plan residency, or the task's own weights).
__device__ __forceinline__ double hbm_cell(const DevProblem& P, const DevCostConfig& cfg,
                                           const Ws& s, const DevTask& tk, const uint8_t* shards,
                                           int tp, int j, int pp, int64_t nmi, int nl_j,
                                           bool use_resident) {
  const double weight_bytes =
      static_cast<double>(tk.precision_bytes) * static_cast<double>(nl_j) *
      (4.0 * static_cast<double>(tk.h1) * static_cast<double>(tk.h1) +
       3.0 * static_cast<double>(tk.h1) * static_cast<double>(tk.h2));
  const double num = static_cast<double>(P.seq_out) * static_cast<double>(nmi) *
                     static_cast<double>(P.mbs) * weight_bytes;
  double den = kInf;
  if (cfg.dbs_override > 0) {
    for (int k = 0; k < tp; ++k) den = smin(den, cfg.dbs_override * P.hbm[shards[k]] * tp);
  } else {
    const double kv_seq = kv_bytes_per_sequence(P, tk, nl_j, tp, cfg);
    const double own = use_resident ? 0.0 : weights_memory_bytes(tk, nl_j, tp, j, pp, cfg);
    const double hi = static_cast<double>(nmi * P.mbs);
    for (int k = 0; k < tp; ++k) {
      const int d = shards[k];
      const double res = use_resident ? s.resident[d] : own;
      const double free_bytes = P.mem[d] - res;
      double dbs = floor(free_bytes / kv_seq);
      dbs = (dbs < 1.0) ? 1.0 : ((hi < dbs) ? hi : dbs);  // std::clamp
      den = smin(den, dbs * P.hbm[d] * tp);
    }
  }
  return num / den;
}

// Geometry memo of task t (independent of splits and weights): TP ring
// bottleneck per (replica, stage) cell and cheapest cross-stage pair.
__device__ __noinline__ void ensure_geometry(const DevProblem& P, Ws& s, int t) {
  const int lane = threadIdx.x & 31;
  HPG_PH_BEGIN(12);
  const DevTask& tk = P.task[t];
  const int dp = s.h.dp[t], pp = s.h.pp[t], tp = s.h.tp[t];
  const int64_t seq_total = P.seq_in + P.seq_out;
  const uint8_t* dv = s.dev + s.o.dev[t];
  const int cell0 = s.o.cell[t];
  const int ncell = dp * pp;
  if (!((s.memo_cm_ok >> t) & 1)) {
    // compute_cost is x / (comp_d * tp) with x >= 0: IEEE multiplication and
    // division are monotone, so the max over a cell's shards
    // (cost_model.cpp:310-314) is attained at the slowest device
    for (int c = lane; c < ncell; c += 32) {
      double m = P.comp[dv[c * tp]];
      for (int k = 1; k < tp; ++k) m = smin(m, P.comp[dv[c * tp + k]]);
      s.cmin[cell0 + c] = m;
    }
    __syncwarp();
    if (lane == 0) s.memo_cm_ok |= 1 << t;
    __syncwarp();
  }
  if (tp > 1 && !((s.memo_tp_ok >> t) & 1)) {
    HPG_PH_BEGIN(13);
    const double cv_tp = tp_comm_volume(tk.precision_bytes, P.mbs, seq_total, tk.h1, tp);
    class_costs(P, s, cv_tp);
    if (tp == 2) {
      for (int c = lane; c < ncell; c += 32) s.rtp[cell0 + c] = ecost(P, s, dv[c * 2], dv[c * 2 + 1]);
    } else if (tp <= 8) {
      // all cells' ring bounds at once, one lane per (cell, vertex): UB = the
      // identity tour's largest edge, LB = the largest 2nd-cheapest incident
      // edge; LB == UB settles the exact ring (ring_small's fast path). Costs
      // are >= 0, so their bit patterns order like the values (64-bit
      // atomicMax in the c_comp/c_tp scratch, free until task_cost's cells).
      unsigned long long* ubb = reinterpret_cast<unsigned long long*>(s.c_comp);
      unsigned long long* lbb = reinterpret_cast<unsigned long long*>(s.c_tp);
      for (int c = lane; c < ncell; c += 32) ubb[c] = lbb[c] = 0ull;
      __syncwarp();
      for (int it = lane; it < ncell * tp; it += 32) {
        const int c = it / tp, v = it - (it / tp) * tp;
        const uint8_t* r = dv + c * tp;
        const double ub = ecost(P, s, r[v], r[v + 1 < tp ? v + 1 : 0]);
        double m1 = kInf, m2 = kInf;
        for (int u = 0; u < tp; ++u) {
          if (u == v) continue;
          const double x = ecost(P, s, r[v], r[u]);
          if (x < m1) {
            m2 = m1;
            m1 = x;
          } else if (x < m2) {
            m2 = x;
          }
        }
        atomicMax(&ubb[c], static_cast<unsigned long long>(__double_as_longlong(ub)));
        atomicMax(&lbb[c], static_cast<unsigned long long>(__double_as_longlong(m2)));
      }
      __syncwarp();
      HPG_PH_COUNT(30, ncell);
      unsigned open = 0;  // cells left to the exact search (rare)
      for (int c0 = 0; c0 < ncell; c0 += 32) {
        const int c = c0 + lane;
        bool o = false;
        if (c < ncell) {
          if (ubb[c] == lbb[c]) {
            s.rtp[cell0 + c] = __longlong_as_double(static_cast<long long>(ubb[c]));
          } else {
            o = true;
          }
        }
        open = __ballot_sync(kFull, o);
        if (open) {
          HPG_PH_BEGIN(28);
          open_rings(P, s, dv, tp, c0, open, ubb + c0, s.rtp + cell0);
          HPG_PH_END(28);
          HPG_PH_COUNT(29, __popc(open));
        }
      }
    } else {
      for (int c = 0; c < ncell; ++c) {
        const double r = ring_bottleneck(P, s, dv + c * tp, tp, cv_tp);
        if (lane == 0) s.rtp[cell0 + c] = r;
      }
    }
    __syncwarp();
    if (lane == 0) s.memo_tp_ok |= 1 << t;
    HPG_PH_END(13);
  }
  if (pp > 1 && !((s.memo_pp_ok >> t) & 1)) {
    HPG_PH_BEGIN(14);
    const double cv_pp = pp_comm_volume(tk.precision_bytes, P.mbs, seq_total, tk.h1);
    class_costs(P, s, cv_pp);
    const int tt = tp * tp;
    if (tt <= 4) {
      for (int c = lane; c < ncell; c += 32) {
        if (c % pp + 1 >= pp) continue;
        double best = kInf;
        for (int xy = 0; xy < tt; ++xy)
          best = smin(best, ecost(P, s, dv[c * tp + xy / tp], dv[(c + 1) * tp + xy % tp]));
        s.ppp[cell0 + c] = best;
      }
    } else {
      // cheapest pair per (cell, next stage): groups of g lanes per cell, g
      // the largest power of two that keeps every lane on one pass over the
      // cells (g = 1: a lane per cell), each group over the tp x tp pairs and
      // a min across the group (a min of the same doubles in any order)
      const int nq = dp * (pp - 1);
      int g = 1;
      while (2 * g <= 32 && 2 * g <= tt && 2 * g * nq <= 32) g *= 2;
      const int per = 32 / g, sub = lane & (g - 1), grp = lane / g;
      for (int q0 = 0; q0 < nq; q0 += per) {
        const int q = q0 + grp;
        const int c = q < nq ? (q / (pp - 1)) * pp + q % (pp - 1) : 0;
        double best = kInf;
        if (q < nq)
          for (int xy = sub; xy < tt; xy += g)
            best = smin(best, ecost(P, s, dv[c * tp + xy / tp], dv[(c + 1) * tp + xy % tp]));
        for (int o = g >> 1; o > 0; o >>= 1) best = smin(best, __shfl_xor_sync(kFull, best, o));
        if (q < nq && sub == 0) s.ppp[cell0 + c] = best;
      }
    }
    __syncwarp();
    if (lane == 0) s.memo_pp_ok |= 1 << t;
    HPG_PH_END(14);
  }
  __syncwarp();
  HPG_PH_END(12);
}

__device__ __noinline__ void task_cost(const DevProblem& P, const DevCostConfig& cfg, Ws& s, int t,
                                       bool use_resident, double* agg) {
  const int lane = threadIdx.x & 31;
  const DevTask& tk = P.task[t];
  const int dp = s.h.dp[t], pp = s.h.pp[t], tp = s.h.tp[t];
  const uint8_t* dv = s.dev + s.o.dev[t];
  const int32_t* sl = s.sl + s.o.sl[t];
  const int64_t* nm = s.nm + s.o.w[t];
  const int cell0 = s.o.cell[t];
  const int ncell = dp * pp;
  HPG_PH_BEGIN(16);
  ensure_geometry(P, s, t);

  const double tpf = tp_pass_factor(tk.kind, cfg.recompute != 0);
  const double ppf = pp_pass_factor(tk.kind);
  const double flops = layer_flops(comp_seq(P, tk.kind), tk.h1, tk.h2);
  const bool do_hbm = tk.kind == kGeneration && P.seq_out > 0;

  // phase 1: one lane per (replica, stage) cell
  for (int c = lane; c < ncell; c += 32) {
    const int i = c / pp, j = c % pp;
    const int64_t nmi = nm[i];
    const int64_t nl_j = sl[j];
    const double comp =
        smax(0.0, compute_cost(tk.kind, nmi, P.mbs, nl_j, flops, s.cmin[cell0 + c], tp));
    double hbm = 0.0;
    if (do_hbm) {
      hbm = smax(0.0, hbm_cell(P, cfg, s, tk, dv + c * tp, tp, j, pp, nmi,
                                static_cast<int>(nl_j), use_resident));
    }
    s.c_comp[c] = comp;
    s.c_hbm[c] = hbm;
    s.c_tp[c] = tp > 1 ? tpf * static_cast<double>(nmi) * static_cast<double>(nl_j) *
                             s.rtp[cell0 + c]
                       : 0.0;
    s.c_pp[c] = (j + 1 < pp) ? ppf * static_cast<double>(nmi) * s.ppp[cell0 + c] : 0.0;
  }
  __syncwarp();

  // phase 2: one lane per replica (sequential stage sums, bubble_cost :243-249)
  const bool training = tk.kind == kTraining;
  double m_comp = 0.0, m_tp = 0.0, m_pp = 0.0, m_hbm = 0.0, m_bub = 0.0, m_tot = 0.0;
  for (int i = lane; i < dp; i += 32) {
    double stage_max = 0.0;
    for (int j = 0; j < pp; ++j) {
      const int c = i * pp + j;
      m_comp = smax(m_comp, s.c_comp[c]);
      m_tp = smax(m_tp, s.c_tp[c]);
      m_pp = smax(m_pp, s.c_pp[c]);
      m_hbm = smax(m_hbm, s.c_hbm[c]);
      stage_max = smax(stage_max, s.c_comp[c] + s.c_tp[c] + s.c_pp[c] + s.c_hbm[c]);
    }
    double bub = 0.0;
    if (training && pp > 1) {
      double sum = 0.0;
      for (int j = 1; j < pp; ++j) {
        const int c = i * pp + j;
        sum += s.c_comp[c] + s.c_tp[c] + s.c_pp[c];
      }
      bub = sum / static_cast<double>(nm[i]);
    }
    m_bub = smax(m_bub, bub);
    m_tot = smax(m_tot, training ? stage_max + bub : stage_max);
  }
  for (int o = 16; o > 0; o >>= 1) {  // six independent butterflies, interleaved
    const double a = __shfl_xor_sync(kFull, m_comp, o), b = __shfl_xor_sync(kFull, m_tp, o),
                 c = __shfl_xor_sync(kFull, m_pp, o), d = __shfl_xor_sync(kFull, m_hbm, o),
                 e = __shfl_xor_sync(kFull, m_bub, o), f = __shfl_xor_sync(kFull, m_tot, o);
    m_comp = smax(m_comp, a);
    m_tp = smax(m_tp, b);
    m_pp = smax(m_pp, c);
    m_hbm = smax(m_hbm, d);
    m_bub = smax(m_bub, e);
    m_tot = smax(m_tot, f);
  }

  // phase 3: DP gradient rings over replica peers (training, dp > 1)
  double a_dp = 0.0;
  HPG_PH_BEGIN(15);
  if (training && dp > 1) {
    const int k0 = s.o.dpk[t];
    for (int j = 0; j < pp; ++j) {
      const int nl_j = sl[j];
      bool need = false;
      for (int k = 0; k < tp; ++k) need |= s.dpr_sl[k0 + j * tp + k] != nl_j;
      if (need) {
        const double cv_dp = dp_comm_volume(tk.precision_bytes, nl_j, tk.h1, tk.h2, dp, tp);
        class_costs(P, s, cv_dp);
        if (dp == 2) {
          for (int k = lane; k < tp; k += 32) {
            s.dpr[k0 + j * tp + k] = ecost(P, s, dv[flat(0, j, k, pp, tp)], dv[flat(1, j, k, pp, tp)]);
            s.dpr_sl[k0 + j * tp + k] = nl_j;
          }
        } else if (dp <= 8 && tp <= 32) {
          // the stage's tp exact rings at once: one lane per (ring k, vertex
          // v) computes v's identity-tour edge (UB) and 2nd-cheapest incident
          // edge (LB), folded per ring with 64-bit atomicMax on the bit
          // patterns (costs >= 0) in the ring scratch; LB == UB settles the
          // ring (ring_small's own fast path), the rest go to ring_small
          // with their UB. Same decisions, same bits, one pass for all rings.
          unsigned long long* ubb = reinterpret_cast<unsigned long long*>(s.rm);
          unsigned long long* lbb = ubb + 32;
          __syncwarp();
          for (int k = lane; k < tp; k += 32) ubb[k] = lbb[k] = 0ull;
          __syncwarp();
          for (int it = lane; it < tp * dp; it += 32) {
            const int k = it / dp, v = it - (it / dp) * dp;
            const int a = dv[flat(v, j, k, pp, tp)];
            const double ub = ecost(P, s, a, dv[flat(v + 1 < dp ? v + 1 : 0, j, k, pp, tp)]);
            double m1 = kInf, m2 = kInf;
            for (int u = 0; u < dp; ++u) {
              if (u == v) continue;
              const double x = ecost(P, s, a, dv[flat(u, j, k, pp, tp)]);
              if (x < m1) {
                m2 = m1;
                m1 = x;
              } else if (x < m2) {
                m2 = x;
              }
            }
            atomicMax(&ubb[k], static_cast<unsigned long long>(__double_as_longlong(ub)));
            atomicMax(&lbb[k], static_cast<unsigned long long>(__double_as_longlong(m2)));
          }
          __syncwarp();
          // lane k keeps ring k's bounds (the scratch is ring_small's matrix)
          const double my_ub = lane < tp ? __longlong_as_double(static_cast<long long>(ubb[lane])) : 0.0;
          const double my_lb = lane < tp ? __longlong_as_double(static_cast<long long>(lbb[lane])) : 0.0;
          const unsigned open = __ballot_sync(kFull, lane < tp && my_ub != my_lb);
          if (lane < tp) {
            s.dpr[k0 + j * tp + lane] = my_ub;
            s.dpr_sl[k0 + j * tp + lane] = nl_j;
          }
          for (unsigned rest = open; rest; rest &= rest - 1) {
            const int k = __ffs(rest) - 1;
            const double ub = __shfl_sync(kFull, my_ub, k);
            __syncwarp();
            for (int i = lane; i < dp; i += 32) s.peers[i] = dv[flat(i, j, k, pp, tp)];
            __syncwarp();
            const double r = ring_small(P, s, s.peers, dp, ub);
            if (lane == 0) s.dpr[k0 + j * tp + k] = r;
          }
        } else {
          for (int k = 0; k < tp; ++k) {
            __syncwarp();
            for (int i = lane; i < dp; i += 32) s.peers[i] = dv[flat(i, j, k, pp, tp)];
            __syncwarp();
            const double r = ring_bottleneck(P, s, s.peers, dp, cv_dp);
            if (lane == 0) {
              s.dpr[k0 + j * tp + k] = r;
              s.dpr_sl[k0 + j * tp + k] = nl_j;
            }
          }
        }
        __syncwarp();
      }
      for (int k = 0; k < tp; ++k) a_dp = smax(a_dp, s.dpr[k0 + j * tp + k]);
    }
  }
  HPG_PH_END(15);
  if (training) m_tot += a_dp;
  agg[0] = m_comp;
  agg[1] = m_tp;
  agg[2] = m_pp;
  agg[3] = a_dp;
  agg[4] = m_bub;
  agg[5] = m_hbm;
  agg[6] = m_tot;
  __syncwarp();
  HPG_PH_END(16);
}

// aggregate_phi (cost_model.cpp:251-262)
__device__ __forceinline__ double phi(const double* c, int n, double eta) {
  double mx = -kInf, sum = 0.0;
  for (int i = 0; i < n; ++i) {
    mx = smax(mx, c[i]);
    sum += c[i];
  }
  return mx + (1.0 - eta) * (sum - mx);
}

struct E2E {
  double e2e;
  double reshard;
  double sync;
  bool feasible;
};

// ---- helper-warp team: the independent per-task task_cost calls of one
// end_to_end are dealt round-robin over the CTA's warps (named barriers 1 =
// job posted, 2 = job done). Each warp keeps its own memo bits and scratch;
// the geometry memo arrays, aggregates and plan state are shared and every
// task's region is written by one warp only. The lead merges the memo bits.

__device__ __forceinline__ void team_share(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                           int kind, int mask, int w) {
  int rank = 0;
  for (int t = 0; t < P.n_tasks; ++t) {
    if (!((mask >> t) & 1)) continue;
    if (rank % s.n_warps == w) {
      if (kind == kJobTasks) {
        task_cost(P, cfg, s, t, true, s.agg + 7 * t);
      } else if (kind == kJobStage) {
        // micro-batches and memory tables only: the geometry memo waits for
        // the memory gate (evaluate skips infeasible candidates) and is then
        // spread over the team by team_geometry or built inside task_cost
        apportion(P, s, t);
        mem_tables(P, cfg, s, t);
      } else {
        ensure_geometry(P, s, t);
      }
    }
    ++rank;
  }
}

// lead side (warp 0): post a job, do the lead's share, wait, merge memo bits
__device__ __noinline__ void team_job(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                      int kind, int mask) {
  const int lane = threadIdx.x & 31;
  const int threads = 32 * s.n_warps;
  if (lane == 0) {
    s.job[0] = kind;
    s.job[1] = mask;
  }
  __syncwarp();
  bar_sync(1, threads);
  team_share(P, cfg, s, kind, mask, 0);
  bar_sync(2, threads);
  if (lane == 0) {
    for (int w = 1; w < s.n_warps; ++w) {
      s.memo_tp_ok |= s.team[w].memo_tp_ok;
      s.memo_pp_ok |= s.team[w].memo_pp_ok;
      s.memo_cm_ok |= s.team[w].memo_cm_ok;
    }
    if (kind == kJobTasks) s.agg_ok |= mask;
  }
  __syncwarp();
}

__device__ __forceinline__ void team_task_costs(const DevProblem& P, const DevCostConfig& cfg,
                                                Ws& s, int mask) {
  team_job(P, cfg, s, kJobTasks, mask);
}

// every task's geometry memo (TP rings, PP pairs, slowest device per cell),
// spread over the team; every evaluation needs all of it
__device__ __forceinline__ void team_geometry(const DevProblem& P, const DevCostConfig& cfg,
                                              Ws& s) {
  if (s.n_warps <= 1) return;
  int mask = 0;
  for (int t = 0; t < P.n_tasks; ++t) {
    const bool done = ((s.memo_cm_ok >> t) & 1) &&
                      (s.h.tp[t] <= 1 || ((s.memo_tp_ok >> t) & 1)) &&
                      (s.h.pp[t] <= 1 || ((s.memo_pp_ok >> t) & 1));
    if (!done) mask |= 1 << t;
  }
  if (__popc(mask) >= 2) team_job(P, cfg, s, kJobGeometry, mask);
}

__device__ __noinline__ void team_exit(Ws& s) {
  if (s.n_warps <= 1) return;
  if ((threadIdx.x & 31) == 0) s.job[0] = kJobExit;
  __syncwarp();
  bar_sync(1, 32 * s.n_warps);
}

// end_to_end_cost (cost_model.cpp:431-487). Per-task aggregates land in s.agg.
__device__ __noinline__ E2E end_to_end(const DevProblem& P, const DevCostConfig& cfg, Ws& s) {
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev;
  __syncwarp();
  HPG_PH_BEGIN(17);
  // weight residency per device, task order (cost_model.cpp:436-448); only the
  // generation task's decoding batch reads it
  const int g = P.gen_slot;
  if (!s.resident_ok && g >= 0 && !((s.agg_ok >> g) & 1)) {
    HPG_PH_BEGIN(22);
    for (int d = lane; d < N; d += 32) {
      double r = 0.0;
      for (int t = 0; t < P.n_tasks; ++t) {
        const int j = s.dstage[t * N + d];
        if (j == 0xff) continue;
        r += weights_memory_bytes(P.task[t], s.sl[s.o.sl[t] + j], s.h.tp[t], j, s.h.pp[t], cfg);
      }
      s.resident[d] = r;
    }
    __syncwarp();
    if (lane == 0) s.resident_ok = 1;
    __syncwarp();
    HPG_PH_END(22);
  }
  if (s.n_warps > 1) {
    int pending = 0;
    for (int t = 0; t < P.n_tasks; ++t)
      if (!((s.agg_ok >> t) & 1)) pending |= 1 << t;
    if (__popc(pending) >= 2) team_task_costs(P, cfg, s, pending);
  }
  double tot[kMaxTasks];
#pragma unroll
  for (int t = 0; t < kMaxTasks; ++t) {
    if (t >= P.n_tasks) break;
    // sweep kernel: the CTA's plan-warps enter every task's cost together, so
    // they fetch the same code at the same time (instruction-cache sharing)
    if (s.cta_sync) bar_sync(5, s.cta_sync);
    if (!((s.agg_ok >> t) & 1)) {
      task_cost(P, cfg, s, t, true, s.agg + 7 * t);
      if (lane == 0) s.agg_ok |= 1 << t;
      __syncwarp();
    }
    tot[t] = s.agg[7 * t + 6];
  }
  E2E r;
  r.reshard = 0.0;
  r.sync = 0.0;
  double transfer = 0.0;
  const double ov = P.mode == 0 ? cfg.reshard_override : cfg.sync_override;
  if (ov >= 0) {
    transfer = ov;
  } else if (P.gen_slot >= 0 && P.train6_slot >= 0) {
    if (!s.bridge_ok) {
      HPG_PH_BEGIN(23);
      const DevTask& g = P.task[P.gen_slot];
      const double bytes = static_cast<double>(g.param_count) * g.precision_bytes;
      class_costs(P, s, bytes);
      const int ga = P.gen_slot, tb = P.train6_slot;
      const int na = s.h.dp[ga] * s.h.pp[ga] * s.h.tp[ga];
      const int nb = s.h.dp[tb] * s.h.pp[tb] * s.h.tp[tb];
      const uint8_t* A = s.dev + s.o.dev[ga];
      const uint8_t* B = s.dev + s.o.dev[tb];
      double best = kInf;
      for (int e = lane; e < na * nb; e += 32) best = smin(best, ecost(P, s, A[e / nb], B[e % nb]));
      best = warp_min(best);
      if (lane == 0) {
        s.bridge = best;
        s.bridge_ok = 1;
      }
      __syncwarp();
      HPG_PH_END(23);
    }
    transfer = s.bridge;
  }
  if (P.mode == 0) {
    r.reshard = transfer;
  } else {
    r.sync = transfer;
  }
  // compose_end_to_end (cost_model.cpp:403-429): kinds staged, phi within a
  // kind. aggregate_phi's max and sequential sum are folded in task order as
  // the tasks come (the same operations as over the per-kind lists), so no
  // per-kind arrays live in local memory.
  double k_mx[3] = {-kInf, -kInf, -kInf}, k_sum[3] = {0.0, 0.0, 0.0};
  int k_n[3] = {0, 0, 0};
#pragma unroll
  for (int t = 0; t < kMaxTasks; ++t) {
    if (t >= P.n_tasks) break;
    const int kd = P.task[t].kind;  // kGeneration 0, kInference 1, kTraining 2
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q != kd) continue;
      k_mx[q] = smax(k_mx[q], tot[t]);
      k_sum[q] += tot[t];
      ++k_n[q];
    }
  }
  const double gen = k_n[0] == 0 ? 0.0 : k_mx[0] + (1.0 - P.eta) * (k_sum[0] - k_mx[0]);
  const double inf = k_n[1] == 0 ? 0.0 : k_mx[1] + (1.0 - P.eta) * (k_sum[1] - k_mx[1]);
  const double trn = k_n[2] == 0 ? 0.0 : k_mx[2] + (1.0 - P.eta) * (k_sum[2] - k_mx[2]);
  if (P.mode == 0) {
    r.e2e = gen + inf + trn + transfer;
  } else {
    r.e2e = smax(gen, inf + trn) + transfer;
  }
  r.feasible = check_memory(P, cfg, s);
  HPG_PH_END(17);
  return r;
}

}  // namespace dev
}  // namespace hpg
