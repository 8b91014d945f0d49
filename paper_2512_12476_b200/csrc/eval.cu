// eval_kernel: one warp per candidate plan, persistent grid-stride over the
// batch. Modes (common.hpp EvalMode):
//   memcheck       check_memory                       plan.cpp:351-380
//   e2e            end_to_end_cost                     cost_model.cpp:431-487
//   evaluate       EvalContext::evaluate minus the     search.cpp:259-279
//                  budget bookkeeping (balance_data -> balance_layers -> e2e),
//                  skipped when the input plan breaks C3 (the GA's memory_ok
//                  gate, search.cpp:458-460)
//   chain          the same chain without the C3 gate
//   balance_data   balance.cpp:37-56
//   balance_layers balance.cpp:81-167
// The balanced plan is written back as a record with the same layout.
//
// balance_layers' split trials (task_total_with_split, balance.cpp:61-77) are
// evaluated one trial per lane: a lane restates the whole-plan C3 check and
// the task's cost for its split serially from the per-plan geometry memo
// (TP rings, PP pairs) and a per-(stage, layer-count) DP-ring table, so the
// exact enumeration runs 32 trials per step instead of one.
#include <cuda_runtime.h>

#include <cstdio>

#include "eval_device.cuh"
#include "eval_launch.hpp"

namespace hpg {
namespace dev {

__device__ __forceinline__ void copy_i32(int32_t* dst, const int32_t* src, int n) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int i = lane; i < n; i += 32) dst[i] = src[i];
  __syncwarp();
}

// Sets task t's split (current plan) and refreshes what depends on it.
__device__ inline void set_split(const DevProblem& P, const DevCostConfig& cfg, Ws& s, int t,
                                 const int32_t* split) {
  copy_i32(s.sl + s.o.sl[t], split, s.h.pp[t]);
  mem_tables(P, cfg, s, t);
  invalidate_split(P, s, t);
}

__device__ inline void set_all_splits(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                      const int32_t* all) {
  copy_i32(s.sl, all, s.o.sl[P.n_tasks]);
  for (int t = 0; t < P.n_tasks; ++t) {
    mem_tables(P, cfg, s, t);
    invalidate_split(P, s, t);
  }
}

// ---- lane-serial pieces of task_cost_detail for one task and one split ----

struct TrialCtx {
  int t, dp, pp, tp, kind;
  bool training, do_hbm;
  double tpf, ppf, flops;
  int64_t nl;
};

__device__ __forceinline__ TrialCtx trial_ctx(const DevProblem& P, const DevCostConfig& cfg,
                                              const Ws& s, int t) {
  TrialCtx c;
  const DevTask& tk = P.task[t];
  c.t = t;
  c.dp = s.h.dp[t];
  c.pp = s.h.pp[t];
  c.tp = s.h.tp[t];
  c.kind = tk.kind;
  c.training = tk.kind == kTraining;
  c.do_hbm = tk.kind == kGeneration && P.seq_out > 0;
  c.tpf = tp_pass_factor(tk.kind, cfg.recompute != 0);
  c.ppf = pp_pass_factor(tk.kind);
  c.flops = layer_flops(comp_seq(P, tk.kind), tk.h1, tk.h2);
  c.nl = tk.nl;
  return c;
}

// One (replica, stage) cell at layer count nl_j with own-weights dbs
// (cost_model.cpp:297-346 with resident_weight_bytes empty).
__device__ __forceinline__ void cell_pieces(const DevProblem& P, const DevCostConfig& cfg,
                                            const Ws& s, const TrialCtx& c, int i, int j,
                                            int nl_j, double& s4, double& s3) {
  const DevTask& tk = P.task[c.t];
  const uint8_t* dv = s.dev + s.o.dev[c.t];
  const int64_t nmi = s.nm[s.o.w[c.t] + i];
  const int cell = i * c.pp + j;
  const double comp = smax(0.0, compute_cost(c.kind, nmi, P.mbs, nl_j, c.flops,
                                             s.cmin[s.o.cell[c.t] + cell], c.tp));
  const double hbm =
      c.do_hbm ? smax(0.0, hbm_cell(P, cfg, s, tk, dv + cell * c.tp, c.tp, j, c.pp, nmi, nl_j, false))
               : 0.0;
  const double tpc = c.tp > 1 ? c.tpf * static_cast<double>(nmi) * static_cast<double>(nl_j) *
                                    s.rtp[s.o.cell[c.t] + cell]
                              : 0.0;
  const double ppc =
      (j + 1 < c.pp) ? c.ppf * static_cast<double>(nmi) * s.ppp[s.o.cell[c.t] + cell] : 0.0;
  s3 = comp + tpc + ppc;
  s4 = s3 + hbm;
}

// split accessor: base[j] with up to two overridden stages
struct Split {
  const int32_t* base;
  int j1, v1, j2, v2;
  __device__ __forceinline__ int operator[](int j) const {
    return j == j1 ? v1 : (j == j2 ? v2 : base[j]);
  }
};

// task_total_with_split (balance.cpp:61-77) for one split, serially in the
// calling lane: whole-plan C3 check (only task t's devices can change; the
// other devices' verdict is `others_ok`), then task_cost(...).total with the
// task's own weights for dbs. DP rings come from dtab.
__device__ double trial_total(const DevProblem& P, const DevCostConfig& cfg, const Ws& s,
                              const TrialCtx& c, const Split& sp, bool others_ok) {
  if (!others_ok) return kInf;
  const int N = P.n_dev;
  const DevTask& tk = P.task[c.t];
  const uint8_t* dv = s.dev + s.o.dev[c.t];
  const int size = c.dp * c.pp * c.tp;
  // task t's per-stage memory at the trial split (stages are few in the exact
  // regime; large greedy pipelines fall back to per-device evaluation)
  double mmj[8], wmj[8];
  const bool tab = c.pp <= 8;
  if (tab) {
    for (int j = 0; j < c.pp; ++j) {
      mmj[j] = model_memory_bytes(P, tk, sp[j], c.tp, j, c.pp, cfg);
      wmj[j] = working_memory_bytes(P, tk, sp[j], c.tp, cfg);
    }
  }
  for (int e = 0; e < size; ++e) {
    const int d = dv[e];
    const int j = (e / c.tp) % c.pp;
    const int L = sp[j];
    double ms = 0.0, wm = 0.0;
    for (int u = 0; u < P.n_tasks; ++u) {
      double m, w;
      if (u == c.t) {
        m = tab ? mmj[j] : model_memory_bytes(P, tk, L, c.tp, j, c.pp, cfg);
        w = tab ? wmj[j] : working_memory_bytes(P, tk, L, c.tp, cfg);
      } else {
        const int jj = s.dstage[u * N + d];
        if (jj == 0xff) continue;
        m = s.mmt[s.o.sl[u] + jj];
        w = s.wmt[s.o.sl[u] + jj];
      }
      ms += m;
      wm = smax(wm, w);
    }
    if (ms + wm > P.mem[d]) return kInf;
  }
  double total = 0.0;
  for (int i = 0; i < c.dp; ++i) {
    double stage_max = 0.0, sum = 0.0;
    for (int j = 0; j < c.pp; ++j) {
      double s4, s3;
      cell_pieces(P, cfg, s, c, i, j, sp[j], s4, s3);
      stage_max = smax(stage_max, s4);
      if (j >= 1) sum += s3;
    }
    const double bub =
        (c.training && c.pp > 1) ? sum / static_cast<double>(s.nm[s.o.w[c.t] + i]) : 0.0;
    total = smax(total, c.training ? stage_max + bub : stage_max);
  }
  if (c.training) {
    double dpm = 0.0;
    if (c.dp > 1) {
      for (int j = 0; j < c.pp; ++j) dpm = smax(dpm, s.dtab[j * s.dtab_stride + sp[j]]);
    }
    total += dpm;
  }
  return total;
}

// dtab[j][L] = max_k min_ring_bottleneck(replica peers of (j, k), cv_dp(L))
__device__ __noinline__ void ensure_dtab(const DevProblem& P, Ws& s, int t, int j, int L) {
  const int lane = threadIdx.x & 31;
  double* slot = s.dtab + j * s.dtab_stride + L;
  if (*slot >= 0.0) return;
  const DevTask& tk = P.task[t];
  const int dp = s.h.dp[t], pp = s.h.pp[t], tp = s.h.tp[t];
  const uint8_t* dv = s.dev + s.o.dev[t];
  const double cv_dp = dp_comm_volume(tk.precision_bytes, L, tk.h1, tk.h2, dp, tp);
  class_costs(P, s, cv_dp);
  double m = 0.0;
  for (int k = 0; k < tp; ++k) {
    if (dp == 2) {
      m = smax(m, ecost(P, s, dv[flat(0, j, k, pp, tp)], dv[flat(1, j, k, pp, tp)]));
      continue;
    }
    __syncwarp();
    for (int i = lane; i < dp; i += 32) s.peers[i] = dv[flat(i, j, k, pp, tp)];
    __syncwarp();
    m = smax(m, ring_bottleneck(P, s, s.peers, dp, cv_dp));
  }
  __syncwarp();
  if (lane == 0) *slot = m;
  __syncwarp();
}

// memory verdict of every device that does not host task t (current plan)
__device__ __noinline__ bool others_fit(const DevProblem& P, const Ws& s, int t) {
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev;
  bool viol = false;
  for (int d = lane; d < N; d += 32) {
    if (s.dstage[t * N + d] != 0xff) continue;
    double ms = 0.0, wm = 0.0;
    for (int u = 0; u < P.n_tasks; ++u) {
      const int jj = s.dstage[u * N + d];
      if (jj == 0xff) continue;
      ms += s.mmt[s.o.sl[u] + jj];
      wm = smax(wm, s.wmt[s.o.sl[u] + jj]);
    }
    if (ms + wm > P.mem[d]) viol = true;
  }
  return !__any_sync(kFull, viol);
}

__device__ __forceinline__ uint64_t binom(int n, int k) {
  if (k < 0 || n < k) return 0;
  uint64_t r = 1;
  for (int i = 0; i < k; ++i) r = r * static_cast<uint64_t>(n - i) / static_cast<uint64_t>(i + 1);
  return r;
}

// r-th composition of nl into pp positive parts in lexicographic order (the
// order of compositions(), combinatorics.cpp:61-95)
__device__ __forceinline__ void unrank_composition(uint64_t r, int nl, int pp, int32_t* out) {
  int rem = nl;
  for (int pos = 0; pos < pp - 1; ++pos) {
    const int left = pp - pos;
    for (int v = 1; v <= rem - (left - 1); ++v) {
      const uint64_t cnt = binom(rem - v - 1, left - 2);
      if (r < cnt) {
        out[pos] = v;
        rem -= v;
        break;
      }
      r -= cnt;
    }
  }
  out[pp - 1] = rem;
}

// balance_data (balance.cpp:37-56) with rate_weights (:14-35). Returns true
// when it had work (a generation task with dp >= 2); then `cur` holds the
// end-to-end breakdown of the plan it returns.
__device__ __noinline__ bool balance_data_dev(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                              E2E& cur, bool& changed) {
  const int lane = threadIdx.x & 31;
  const int g = P.gen_slot;
  changed = false;
  if (g < 0 || s.h.dp[g] < 2) return false;
  const int dp = s.h.dp[g], pp = s.h.pp[g];
  double agg[7];
  task_cost(P, cfg, s, g, false, agg);
  const int64_t* nm = s.nm + s.o.w[g];
  for (int i = lane; i < dp; i += 32) {
    double bott = 0.0;
    for (int j = 0; j < pp; ++j) {
      const int c = i * pp + j;
      bott = smax(bott, s.c_comp[c] + s.c_tp[c] + s.c_pp[c] + s.c_hbm[c]);
    }
    const double per_mb = bott / static_cast<double>(nm[i]);
    s.wnew[i] = per_mb > 0 ? 1.0 / per_mb : 1.0;
  }
  __syncwarp();
  double sum = 0.0;
  for (int i = 0; i < dp; ++i) sum += s.wnew[i];
  __syncwarp();
  for (int i = lane; i < dp; i += 32) s.wnew[i] = static_cast<double>(dp) * s.wnew[i] / sum;
  __syncwarp();
  const E2E before = end_to_end(P, cfg, s);
  double keep_agg[7];
  for (int c = 0; c < 7; ++c) keep_agg[c] = s.agg[7 * g + c];
  double* w = s.w + s.o.w[g];
  for (int i = lane; i < dp; i += 32) {
    s.wsave[i] = w[i];
    w[i] = s.wnew[i];
  }
  __syncwarp();
  apportion(P, s, g);
  invalidate_weights(s, g);
  const E2E after = end_to_end(P, cfg, s);
  if (after.e2e < before.e2e) {
    cur = after;
    changed = true;
  } else {
    for (int i = lane; i < dp; i += 32) w[i] = s.wsave[i];
    __syncwarp();
    apportion(P, s, g);
    __syncwarp();
    for (int c = lane; c < 7; c += 32) s.agg[7 * g + c] = keep_agg[c];
    __syncwarp();
    cur = before;
  }
  return true;
}

// balance_layers (balance.cpp:81-167), including its aliasing quirk: the
// greedy branch updates the candidate in place (:150) so `touched` is only
// ever set by exact-mode tasks (:153); with no exact-mode task the input plan
// is returned unchanged, which is short-circuited here.
__device__ __noinline__ void balance_layers_dev(const DevProblem& P, const DevCostConfig& cfg,
                                                Ws& s, bool& have_cur, E2E& cur, bool& changed) {
  const int lane = threadIdx.x & 31;
  changed = false;
  bool exact_any = false;
  for (int t = 0; t < P.n_tasks; ++t) {
    const int pp = s.h.pp[t];
    const int64_t nl = P.task[t].nl;
    if (pp >= 2 && nl != pp && static_cast<int64_t>(pp) * nl <= 64) exact_any = true;
  }
  if (!exact_any) return;
  const int nsl = s.o.sl[P.n_tasks];
  copy_i32(s.sl_save, s.sl, nsl);
  bool touched = false;
  for (int t = 0; t < P.n_tasks; ++t) {
    const int pp = s.h.pp[t];
    const int64_t nl = P.task[t].nl;
    if (pp < 2 || nl == pp) continue;
    int32_t* sl_t = s.sl + s.o.sl[t];
    const TrialCtx tc = trial_ctx(P, cfg, s, t);
    ensure_geometry(P, s, t);
    // fresh DP-ring table for this task (devices fixed, volume follows L)
    if (lane == 0) s.dtab_stride = static_cast<int>(nl) + 1;
    __syncwarp();
    const bool need_dp = tc.training && tc.dp > 1;
    if (need_dp) {
      for (int e = lane; e < pp * s.dtab_stride; e += 32) s.dtab[e] = -1.0;
      __syncwarp();
    }
    const bool others = others_fit(P, s, t);
    copy_i32(s.split_best, sl_t, pp);
    if (static_cast<int64_t>(pp) * nl <= 64) {
      const int lmax = static_cast<int>(nl) - pp + 1;
      if (need_dp) {
        for (int j = 0; j < pp; ++j)
          for (int L = 1; L <= lmax; ++L) ensure_dtab(P, s, t, j, L);
      }
      // best = current split (lane 0), then every composition in parallel
      const uint64_t ntr = binom(static_cast<int>(nl) - 1, pp - 1);
      double best0 = 0.0;
      {
        double v = 0.0;
        if (lane == 0) v = trial_total(P, cfg, s, tc, Split{sl_t, -1, 0, -1, 0}, others);
        best0 = __shfl_sync(kFull, v, 0);
      }
      double bv = kInf;
      uint64_t br = ~0ull;
      int32_t comp[8];
      for (uint64_t base = 0; base < ntr; base += 32) {
        const uint64_t r = base + lane;
        if (r < ntr) {
          unrank_composition(r, static_cast<int>(nl), pp, comp);
          const double v = trial_total(P, cfg, s, tc, Split{comp, -1, 0, -1, 0}, others);
          if (v < bv) {  // first strict minimum within the lane's ranks
            bv = v;
            br = r;
          }
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, bv, o);
        const uint64_t orr = __shfl_xor_sync(kFull, br, o);
        if (ov < bv || (ov == bv && orr < br)) {
          bv = ov;
          br = orr;
        }
      }
      if (bv < best0) {  // strict improvement over the current split
        if (lane == 0) unrank_composition(br, static_cast<int>(nl), pp, s.split_best);
        __syncwarp();
      }
      bool diff = false;
      for (int j = lane; j < pp; j += 32) diff |= s.split_best[j] != sl_t[j];
      if (__any_sync(kFull, diff)) {
        set_split(P, cfg, s, t, s.split_best);
        touched = true;
      }
    } else {
      // greedy: shed one layer from the bottleneck stage to a neighbour; the
      // candidate is updated in place after every accepted step
      double best = 0.0;
      {
        if (need_dp)
          for (int j = 0; j < pp; ++j) ensure_dtab(P, s, t, j, sl_t[j]);
        double v = 0.0;
        if (lane == 0) v = trial_total(P, cfg, s, tc, Split{sl_t, -1, 0, -1, 0}, others);
        best = __shfl_sync(kFull, v, 0);
      }
      while (true) {
        // bottleneck stage: load_j = max_i stage sum, first j with the largest
        double worst = -1.0;
        int bn = 0;
        for (int j0 = 0; j0 < pp; j0 += 32) {
          const int j = j0 + lane;
          double load = -kInf;
          if (j < pp) {
            load = 0.0;
            for (int i = 0; i < tc.dp; ++i) {
              double s4, s3;
              cell_pieces(P, cfg, s, tc, i, j, sl_t[j], s4, s3);
              load = smax(load, s4);
            }
          }
          const double m = warp_max(load);
          if (m > worst) {
            const unsigned bal = __ballot_sync(kFull, j < pp && load == m);
            worst = m;
            bn = j0 + __ffs(bal) - 1;
          }
        }
        if (sl_t[bn] <= 1) break;
        const int nbs[2] = {bn - 1, bn + 1};
        if (need_dp) {
          ensure_dtab(P, s, t, bn, sl_t[bn] - 1);
          for (int side = 0; side < 2; ++side)
            if (nbs[side] >= 0 && nbs[side] < pp)
              ensure_dtab(P, s, t, nbs[side], sl_t[nbs[side]] + 1);
        }
        double v = kInf;
        if (lane < 2) {
          const int nb = nbs[lane];
          if (nb >= 0 && nb < pp) {
            v = trial_total(P, cfg, s, tc, Split{sl_t, bn, sl_t[bn] - 1, nb, sl_t[nb] + 1},
                            others);
          }
        }
        const double c0 = __shfl_sync(kFull, v, 0), c1 = __shfl_sync(kFull, v, 1);
        int pick = -1;
        double step_best = best;
        if (c0 < step_best) {
          step_best = c0;
          pick = 0;
        }
        if (c1 < step_best) {
          step_best = c1;
          pick = 1;
        }
        if (pick < 0) break;
        best = step_best;
        const int nb = nbs[pick];
        __syncwarp();
        if (lane == 0) {
          for (int j = 0; j < pp; ++j) s.split_step[j] = sl_t[j];
          --s.split_step[bn];
          ++s.split_step[nb];
        }
        __syncwarp();
        set_split(P, cfg, s, t, s.split_step);
      }
    }
  }
  if (!touched) {
    set_all_splits(P, cfg, s, s.sl_save);
    return;
  }
  if (!check_memory(P, cfg, s)) {
    set_all_splits(P, cfg, s, s.sl_save);
    return;
  }
  const E2E after = end_to_end(P, cfg, s);
  E2E before;
  if (have_cur) {
    before = cur;
  } else {
    copy_i32(s.sl_save2, s.sl, nsl);
    set_all_splits(P, cfg, s, s.sl_save);
    before = end_to_end(P, cfg, s);
    set_all_splits(P, cfg, s, s.sl_save2);
  }
  have_cur = true;
  if (after.e2e < before.e2e) {
    cur = after;
    changed = true;
  } else {
    set_all_splits(P, cfg, s, s.sl_save);
    cur = before;
  }
}

// diagnostics only (HPG_PLAN_PROFILE): per-plan clock64 phase stamps
__device__ long long* g_plan_prof = nullptr;

__global__ void __launch_bounds__(32)
eval_kernel(DevProblem P, DevCostConfig cfg, Carve cv, int32_t kb_flags,
            const uint8_t* __restrict__ recs, const int64_t* __restrict__ off,
            const int32_t* __restrict__ modes, int32_t uniform_mode, int n, int64_t stride,
            uint8_t* __restrict__ out_recs, EvalResult* __restrict__ res,
            double* __restrict__ per_task, double* __restrict__ required,
            double* __restrict__ gscratch, int64_t gscratch_doubles) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ws s;
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    carve(s, smem, cv);
    s.dtab = gscratch + static_cast<int64_t>(blockIdx.x) * gscratch_doubles;
    s.dtab_stride = 0;
  }
  __syncwarp();
  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    const int64_t rec_at = off ? off[p] : static_cast<int64_t>(p) * stride;
    const uint8_t* rec = recs + rec_at;
    const int mode = modes ? modes[p] : uniform_mode;
    long long* prof = g_plan_prof ? g_plan_prof + 5 * static_cast<int64_t>(p) : nullptr;
    if (prof && lane == 0) prof[0] = clock64();
    // ---- stage the plan ----
    if (lane < 20) reinterpret_cast<int32_t*>(&s.h)[lane] = reinterpret_cast<const int32_t*>(rec)[lane];
    __syncwarp();
    if (lane == 0) {
      rec_offsets(s.h, s.o);
      s.memo_tp_ok = 0;
      s.memo_pp_ok = 0;
      s.memo_cm_ok = 0;
      s.bridge_ok = 0;
      s.agg_ok = 0;
      s.resident_ok = 0;
      s.memv_ok = 0;
    }
    __syncwarp();
    const int nw = s.o.w[P.n_tasks], nsl = s.o.sl[P.n_tasks], nslot = s.o.dev[P.n_tasks];
    const double* rw = reinterpret_cast<const double*>(rec + s.o.w_byte);
    const int32_t* rsl = reinterpret_cast<const int32_t*>(rec + s.o.sl_byte);
    const uint8_t* rdev = rec + s.o.dev_byte;
    if (s.h.n_tasks & kRecCompact) {
      for (int i = lane; i < nw; i += 32) s.w[i] = 1.0;
      for (int t = 0; t < P.n_tasks; ++t) {
        const int pp = s.h.pp[t];
        const int64_t nl = P.task[t].nl;
        for (int j = lane; j < pp; j += 32)
          s.sl[s.o.sl[t] + j] = static_cast<int32_t>(nl / pp) + (j < nl % pp ? 1 : 0);
      }
    } else {
      for (int i = lane; i < nw; i += 32) s.w[i] = rw[i];
      for (int i = lane; i < nsl; i += 32) s.sl[i] = rsl[i];
    }
    for (int i = lane; i < nslot; i += 32) s.dev[i] = rdev[i];
    for (int i = lane; i < s.o.dpk[P.n_tasks]; i += 32) s.dpr_sl[i] = -1;
    __syncwarp();
    for (int t = 0; t < P.n_tasks; ++t) {
      apportion(P, s, t);
      mem_tables(P, cfg, s, t);
    }
    build_dstage(P, s);

    EvalResult r;
    r.cost = -1.0;
    r.reshard_s = 0.0;
    r.sync_s = 0.0;
    r.flags = 0;
    r.pad = 0;
    const bool feas_in =
        check_memory(P, cfg, s, required ? required + static_cast<int64_t>(p) * P.n_dev : nullptr);
    if (feas_in) r.flags |= kResFeasIn;
    if (mode == kModeE2E) {
      const E2E e = end_to_end(P, cfg, s);
      r.cost = e.e2e;
      r.reshard_s = e.reshard;
      r.sync_s = e.sync;
      if (e.feasible) r.flags |= kResFeasOut;
      if (per_task) {
        for (int i = lane; i < 7 * P.n_tasks; i += 32)
          per_task[static_cast<int64_t>(p) * 7 * P.n_tasks + i] = s.agg[i];
      }
    } else if (mode == kModeEvaluate || mode == kModeChain || mode == kModeBalanceData ||
               mode == kModeBalanceLayers) {
      const bool chain = mode == kModeEvaluate || mode == kModeChain;
      const bool go = mode != kModeEvaluate || feas_in;
      if (go) {
        bool have_cur = false, ch = false;
        E2E cur;
        if ((chain && (kb_flags & 1)) || mode == kModeBalanceData) {
          if (prof && lane == 0) prof[1] = clock64();
          have_cur = balance_data_dev(P, cfg, s, cur, ch);
          if (ch) r.flags |= kResWeights;
        }
        if (prof && lane == 0) prof[2] = clock64();
        if ((chain && (kb_flags & 2)) || mode == kModeBalanceLayers) {
          balance_layers_dev(P, cfg, s, have_cur, cur, ch);
          if (ch) r.flags |= kResLayers;
        }
        if (prof && lane == 0) prof[3] = clock64();
        if (!have_cur) cur = end_to_end(P, cfg, s);
        r.cost = cur.e2e;
        r.reshard_s = cur.reshard;
        r.sync_s = cur.sync;
        if (cur.feasible) r.flags |= kResFeasOut;
      }
    }
    // ---- write back ----
    if (out_recs) {
      uint8_t* orec = out_recs + rec_at;
      if (lane < 20) reinterpret_cast<int32_t*>(orec)[lane] = reinterpret_cast<const int32_t*>(&s.h)[lane];
      double* ow = reinterpret_cast<double*>(orec + s.o.w_byte);
      int32_t* osl = reinterpret_cast<int32_t*>(orec + s.o.sl_byte);
      uint8_t* odev = orec + s.o.dev_byte;
      for (int i = lane; i < nw; i += 32) ow[i] = s.w[i];
      for (int i = lane; i < nsl; i += 32) osl[i] = s.sl[i];
      for (int i = lane; i < nslot; i += 32) odev[i] = s.dev[i];
    }
    if (prof && lane == 0) prof[4] = clock64();
    if (lane == 0) res[p] = r;
    __syncwarp();
  }
}

}  // namespace dev

int eval_smem_bytes(const Carve& c) { return carve2_bytes(c); }

cudaError_t eval_set_plan_profile(long long* d_buf) {
  return cudaMemcpyToSymbol(dev::g_plan_prof, &d_buf, sizeof(d_buf));
}

int64_t eval_scratch_doubles(int n_dev, int64_t max_nl) {
  // per CTA: DP-ring table [pp <= N][nl + 1]
  return static_cast<int64_t>(n_dev) * (max_nl + 2);
}

cudaError_t eval_grid(Carve cv, int n, int n_sm, int& grid) {
  cv.bytes = carve2_bytes(cv);
  static int configured_bytes = 0;
  if (cv.bytes > 48 * 1024 && cv.bytes > configured_bytes) {
    cudaError_t e = cudaFuncSetAttribute(dev::eval_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, cv.bytes);
    if (e != cudaSuccess) return e;
    configured_bytes = cv.bytes;
  }
  static int cached_bytes = -1, cached_per_sm = 0;
  int per_sm = 0;
  if (cv.bytes == cached_bytes) {
    per_sm = cached_per_sm;
  } else {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::eval_kernel, 32,
                                                                  cv.bytes);
    if (e != cudaSuccess) return e;
    cached_bytes = cv.bytes;
    cached_per_sm = per_sm;
  }
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  grid = n < n_sm * per_sm ? n : n_sm * per_sm;
  return cudaSuccess;
}

cudaError_t launch_eval(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                        int32_t kb_flags, const uint8_t* d_recs, const int64_t* d_off,
                        const int32_t* d_modes, int32_t uniform_mode, int n, int64_t stride,
                        uint8_t* d_out, EvalResult* d_res, double* d_per_task,
                        double* d_required, double* d_scratch, int64_t scratch_doubles,
                        int grid, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cv.bytes = carve2_bytes(cv);
  dev::eval_kernel<<<grid, 32, cv.bytes, st>>>(P, cfg, cv, kb_flags, d_recs, d_off, d_modes,
                                               uniform_mode, n, stride, d_out, d_res, d_per_task,
                                               d_required, d_scratch, scratch_doubles);
  return cudaGetLastError();
}

}  // namespace hpg
