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

#include "devstate.hpp"

#include <cstdio>

#include "eval_device.cuh"
#include "eval_launch.hpp"
#include "sweep.hpp"

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

// task_total_with_split (balance.cpp:61-77) from per-(stage, layer-count)
// columns. With the devices, the other tasks' splits and the weights fixed,
// a trial's pieces depend on each stage's own layer count only:
//   cflag[j][L]  C3 verdict of stage j's devices at L layers (-1 = unknown;
//                whole-plan C3 = others_ok AND every stage's verdict)
//   ccell[j][L]  per replica i: (s4, s3) of cell (i, j) at L layers
//   dtab[j][L]   DP-ring maximum (training, dp > 1)
// A trial then reads pp columns; the replica maxima and the sequential bubble
// sum are evaluated in the reference's order (bit-exact).
__device__ __forceinline__ double* ccell_of(const Ws& s, int dp, int j, int L) {
  return s.ccell + static_cast<int64_t>(j * s.dtab_stride + L) * 2 * dp;
}

// Fills the missing columns among (js[q], Ls[q]), q < nq, with the whole warp.
__device__ __noinline__ void ensure_cols(const DevProblem& P, const DevCostConfig& cfg, Ws& s,
                                         const TrialCtx& c, const int* js, const int* Ls,
                                         int nq) {
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev;
  const DevTask& tk = P.task[c.t];
  const uint8_t* dv = s.dev + s.o.dev[c.t];
  const int per = c.dp + c.dp * c.tp;  // cells + devices of one column
  __syncwarp();
  int missing = 0;  // bit q: column q to fill (columns are distinct)
  for (int q = 0; q < nq; ++q)
    if (s.cflag[js[q] * s.dtab_stride + Ls[q]] < 0) missing |= 1 << q;
  if (!missing) return;
  __syncwarp();
  if (lane == 0)
    for (int q = 0; q < nq; ++q)
      if ((missing >> q) & 1) s.cflag[js[q] * s.dtab_stride + Ls[q]] = 1;
  __syncwarp();
  for (int it = lane; it < nq * per; it += 32) {
    const int q = it / per, r = it - q * per;
    if (!((missing >> q) & 1)) continue;
    const int j = js[q], L = Ls[q];
    if (r < c.dp) {
      double s4, s3;
      cell_pieces(P, cfg, s, c, r, j, L, s4, s3);
      double* col = ccell_of(s, c.dp, j, L);
      col[2 * r] = s4;
      col[2 * r + 1] = s3;
    } else {
      const int e = r - c.dp;  // (replica i, shard k) of stage j
      const int i = e / c.tp, k = e - (e / c.tp) * c.tp;
      const int d = dv[flat(i, j, k, c.pp, c.tp)];
      double ms = 0.0, wm = 0.0;
      for (int u = 0; u < P.n_tasks; ++u) {
        double m, w;
        if (u == c.t) {
          m = model_memory_bytes(P, tk, L, c.tp, j, c.pp, cfg);
          w = working_memory_bytes(P, tk, L, c.tp, cfg);
        } else {
          const int jj = s.dstage[u * N + d];
          if (jj == 0xff) continue;
          m = s.mmt[s.o.sl[u] + jj];
          w = s.wmt[s.o.sl[u] + jj];
        }
        ms += m;
        wm = smax(wm, w);
      }
      if (ms + wm > P.mem[d]) s.cflag[j * s.dtab_stride + L] = 0;
    }
  }
  __syncwarp();
}

// One trial from the columns, serially in the calling lane.
__device__ __forceinline__ double trial_cols(const Ws& s, const TrialCtx& c, const Split& sp,
                                             bool others_ok) {
  if (!others_ok) return kInf;
  for (int j = 0; j < c.pp; ++j)
    if (s.cflag[j * s.dtab_stride + sp[j]] == 0) return kInf;
  double total = 0.0;
  for (int i = 0; i < c.dp; ++i) {
    double stage_max = 0.0, sum = 0.0;
    for (int j = 0; j < c.pp; ++j) {
      const double* col = ccell_of(s, c.dp, j, sp[j]);
      stage_max = smax(stage_max, col[2 * i]);
      if (j >= 1) sum += col[2 * i + 1];
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

// One trial from the columns with the replicas spread over the lanes.
__device__ __forceinline__ double trial_cols_warp(const Ws& s, const TrialCtx& c,
                                                  const Split& sp, bool others_ok) {
  if (!others_ok) return kInf;
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < c.pp; ++j)
    if (s.cflag[j * s.dtab_stride + sp[j]] == 0) return kInf;
  double total = 0.0;
  for (int i = lane; i < c.dp; i += 32) {
    double stage_max = 0.0, sum = 0.0;
    for (int j = 0; j < c.pp; ++j) {
      const double* col = ccell_of(s, c.dp, j, sp[j]);
      stage_max = smax(stage_max, col[2 * i]);
      if (j >= 1) sum += col[2 * i + 1];
    }
    const double bub =
        (c.training && c.pp > 1) ? sum / static_cast<double>(s.nm[s.o.w[c.t] + i]) : 0.0;
    total = smax(total, c.training ? stage_max + bub : stage_max);
  }
  total = warp_max(total);
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

// binomials for the exact split regime (pp * nl <= 64 => n < 64, k <= 6)
struct BinomTab {
  uint64_t v[64][8];
};
constexpr BinomTab make_binom_tab() {
  BinomTab t{};
  for (int n = 0; n < 64; ++n)
    for (int k = 0; k < 8; ++k) {
      uint64_t r = k <= n ? 1 : 0;
      for (int i = 0; i < k && k <= n; ++i) r = r * static_cast<uint64_t>(n - i) / (i + 1);
      t.v[n][k] = r;
    }
  return t;
}
__constant__ BinomTab c_binom = make_binom_tab();

__device__ __forceinline__ uint64_t binom(int n, int k) {
  if (k < 0 || n < k) return 0;
  return c_binom.v[n & 63][k & 7];  // callers stay inside the table
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
    HPG_PH_BEGIN(0);
    ensure_geometry(P, s, t);
    HPG_PH_END(0);
    // fresh column tables for this task (devices, weights and the other
    // tasks' splits stay fixed while its split moves)
    const int stride = static_cast<int>(nl) + 1;
    if (lane == 0) {
      s.dtab_stride = stride;
      s.cflag = reinterpret_cast<int32_t*>(s.dtab + pp * stride);
      s.ccell = s.dtab + pp * stride + (pp * stride + 1) / 2;
    }
    __syncwarp();
    const bool need_dp = tc.training && tc.dp > 1;
    for (int e = lane; e < pp * stride; e += 32) {
      s.cflag[e] = -1;
      if (need_dp) s.dtab[e] = -1.0;
    }
    __syncwarp();
    HPG_PH_BEGIN(1);
    const bool others = others_fit(P, s, t);
    HPG_PH_END(1);
    copy_i32(s.split_best, sl_t, pp);
    if (static_cast<int64_t>(pp) * nl <= 64) {
      const int lmax = static_cast<int>(nl) - pp + 1;
      HPG_PH_BEGIN(2);
      if (need_dp) {
        for (int j = 0; j < pp; ++j)
          for (int L = 1; L <= lmax; ++L) ensure_dtab(P, s, t, j, L);
      }
      {
        int js[16], Ls[16], nq = 0;
        for (int j = 0; j < pp; ++j)
          for (int L = 1; L <= lmax; ++L) {
            js[nq] = j;
            Ls[nq] = L;
            if (++nq == 16) {
              ensure_cols(P, cfg, s, tc, js, Ls, nq);
              nq = 0;
            }
          }
        if (nq) ensure_cols(P, cfg, s, tc, js, Ls, nq);
      }
      HPG_PH_END(2);
      HPG_PH_BEGIN(3);
      // best = current split, then every composition, one per lane
      const uint64_t ntr = binom(static_cast<int>(nl) - 1, pp - 1);
      const double best0 = trial_cols_warp(s, tc, Split{sl_t, -1, 0, -1, 0}, others);
      double bv = kInf;
      uint64_t br = ~0ull;
      int32_t comp[8];
      for (uint64_t base = 0; base < ntr; base += 32) {
        const uint64_t r = base + lane;
        if (r < ntr) {
          unrank_composition(r, static_cast<int>(nl), pp, comp);
          const double v = trial_cols(s, tc, Split{comp, -1, 0, -1, 0}, others);
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
      HPG_PH_END(3);
      HPG_PH_COUNT(28, ntr);
      if (bv < best0) {  // strict improvement over the current split
        if (lane == 0) unrank_composition(br, static_cast<int>(nl), pp, s.split_best);
        __syncwarp();
      }
      bool diff = false;
      for (int j = lane; j < pp; j += 32) diff |= s.split_best[j] != sl_t[j];
      if (__any_sync(kFull, diff)) {
        HPG_PH_BEGIN(4);
        set_split(P, cfg, s, t, s.split_best);
        HPG_PH_END(4);
        touched = true;
      }
    } else {
      // greedy: shed one layer from the bottleneck stage to a neighbour; the
      // candidate is updated in place after every accepted step (its memory
      // tables and caches are refreshed once, after the walk: nothing in the
      // walk reads task t's own tables)
      double best = 0.0;
      bool moved = false;
      HPG_PH_COUNT(30, 1);
      {
        HPG_PH_BEGIN(5);
        if (need_dp)
          for (int j = 0; j < pp; ++j) ensure_dtab(P, s, t, j, sl_t[j]);
        int js[16], Ls[16];
        for (int j0 = 0; j0 < pp; j0 += 16) {
          const int nq = min(16, pp - j0);
          for (int q = 0; q < nq; ++q) {
            js[q] = j0 + q;
            Ls[q] = sl_t[j0 + q];
          }
          ensure_cols(P, cfg, s, tc, js, Ls, nq);
        }
        best = trial_cols_warp(s, tc, Split{sl_t, -1, 0, -1, 0}, others);
        HPG_PH_END(5);
      }
      while (true) {
        HPG_PH_COUNT(27, 1);
        HPG_PH_BEGIN(6);
        // bottleneck stage: load_j = max_i stage sum, first j with the largest
        double worst = -1.0;
        int bn = 0;
        for (int j0 = 0; j0 < pp; j0 += 32) {
          const int j = j0 + lane;
          double load = -kInf;
          if (j < pp) {
            load = 0.0;
            const double* col = ccell_of(s, tc.dp, j, sl_t[j]);
            for (int i = 0; i < tc.dp; ++i) load = smax(load, col[2 * i]);
          }
          const double m = warp_max(load);
          if (m > worst) {
            const unsigned bal = __ballot_sync(kFull, j < pp && load == m);
            worst = m;
            bn = j0 + __ffs(bal) - 1;
          }
        }
        HPG_PH_END(6);
        if (sl_t[bn] <= 1) break;
        const int nbs[2] = {bn - 1, bn + 1};
        HPG_PH_BEGIN(7);
        if (need_dp) {
          ensure_dtab(P, s, t, bn, sl_t[bn] - 1);
          for (int side = 0; side < 2; ++side)
            if (nbs[side] >= 0 && nbs[side] < pp)
              ensure_dtab(P, s, t, nbs[side], sl_t[nbs[side]] + 1);
        }
        {
          int js[3], Ls[3], nq = 0;
          js[nq] = bn;
          Ls[nq++] = sl_t[bn] - 1;
          for (int side = 0; side < 2; ++side)
            if (nbs[side] >= 0 && nbs[side] < pp) {
              js[nq] = nbs[side];
              Ls[nq++] = sl_t[nbs[side]] + 1;
            }
          ensure_cols(P, cfg, s, tc, js, Ls, nq);
        }
        HPG_PH_END(7);
        HPG_PH_BEGIN(8);
        double cv2[2];
        for (int side = 0; side < 2; ++side) {
          const int nb = nbs[side];
          cv2[side] = (nb >= 0 && nb < pp)
                          ? trial_cols_warp(s, tc, Split{sl_t, bn, sl_t[bn] - 1, nb, sl_t[nb] + 1},
                                            others)
                          : kInf;
        }
        const double c0 = cv2[0], c1 = cv2[1];
        HPG_PH_END(8);
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
          --sl_t[bn];
          ++sl_t[nb];
        }
        __syncwarp();
        moved = true;
      }
      if (moved) {
        HPG_PH_BEGIN(9);
        mem_tables(P, cfg, s, t);
        invalidate_split(P, s, t);
        HPG_PH_END(9);
      }
    }
  }
  HPG_PH_COUNT(29, 1);
  if (!touched) {
    set_all_splits(P, cfg, s, s.sl_save);
    return;
  }
  HPG_PH_BEGIN(10);
  const bool mem_ok = check_memory(P, cfg, s);
  HPG_PH_END(10);
  if (!mem_ok) {
    set_all_splits(P, cfg, s, s.sl_save);
    return;
  }
  HPG_PH_BEGIN(11);
  const E2E after = end_to_end(P, cfg, s);
  HPG_PH_END(11);
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

// helper warps (team_task_costs): wait for jobs from the lead until it exits
__device__ __noinline__ void team_helper(const DevProblem& P, const DevCostConfig& cfg, Ws* team,
                                         int w) {
  const int lane = threadIdx.x & 31;
  Ws& s = team[w];
  const Ws& s0 = team[0];
  const int threads = 32 * s.n_warps;
  while (true) {
    bar_sync(1, threads);
    const int kind = s0.job[0], mask = s0.job[1];
    if (kind == kJobExit) return;
    // the lead's current plan view
    {
      const int32_t* hs = reinterpret_cast<const int32_t*>(&s0.h);
      int32_t* hd = reinterpret_cast<int32_t*>(&s.h);
      for (int i = lane; i < static_cast<int>(sizeof(RecHeader) / 4); i += 32) hd[i] = hs[i];
      const int32_t* os = reinterpret_cast<const int32_t*>(&s0.o);
      int32_t* od = reinterpret_cast<int32_t*>(&s.o);
      for (int i = lane; i < static_cast<int>(sizeof(RecOffsets) / 4); i += 32) od[i] = os[i];
      if (lane == 0) {
        s.memo_tp_ok = s0.memo_tp_ok;
        s.memo_pp_ok = s0.memo_pp_ok;
        s.memo_cm_ok = s0.memo_cm_ok;
      }
      __syncwarp();
    }
    team_share(P, cfg, s, kind, mask, w);
    bar_sync(2, threads);
  }
}

// One plan evaluated by the warp of s (the lead of its team): stage the
// record, then the requested mode. Record bytes are read with ld.global.cg:
// the device GA writes records on other SMs within one launch (no stale L1
// lines). Balanced [generation weights | stage layers] are written to ows
// (packed, engine.cpp ws_bytes_of) or back into the record (rec_wb).
__device__ __forceinline__ EvalResult eval_one(const DevProblem& P, const DevCostConfig& cfg,
                                               Ws& s, int32_t kb_flags,
                                               const uint8_t* __restrict__ rec, int mode,
                                               long long* prof, double* per_task,
                                               double* required, uint8_t* ows, uint8_t* rec_wb) {
  const int lane = threadIdx.x & 31;
  if (prof && lane == 0) {
    s.prof = prof;
    prof[0] = clock64();
  }
  // ---- stage the plan ----
  if (lane < 20)
    reinterpret_cast<int32_t*>(&s.h)[lane] = __ldcg(reinterpret_cast<const int32_t*>(rec) + lane);
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
    for (int i = lane; i < nw; i += 32) s.w[i] = __ldcg(rw + i);
    for (int i = lane; i < nsl; i += 32) s.sl[i] = __ldcg(rsl + i);
  }
  for (int i = lane; i < nslot; i += 32) s.dev[i] = __ldcg(rdev + i);
  for (int i = lane; i < s.o.dpk[P.n_tasks]; i += 32) s.dpr_sl[i] = -1;
  __syncwarp();
  if (s.n_warps > 1 && P.n_tasks > 1 && mode != kModeMemcheck) {
    // per task, spread over the team: micro-batches and memory tables
    team_job(P, cfg, s, kJobStage, (1 << P.n_tasks) - 1);
  } else {
    for (int t = 0; t < P.n_tasks; ++t) {
      apportion(P, s, t);
      mem_tables(P, cfg, s, t);
    }
  }
  build_dstage(P, s);

  EvalResult r;
  r.cost = -1.0;
  r.reshard_s = 0.0;
  r.sync_s = 0.0;
  r.flags = 0;
  r.pad = 0;
  const bool feas_in = check_memory(P, cfg, s, required);
  if (feas_in) r.flags |= kResFeasIn;
  if (mode == kModeE2E) {
    const E2E e = end_to_end(P, cfg, s);
    r.cost = e.e2e;
    r.reshard_s = e.reshard;
    r.sync_s = e.sync;
    if (e.feasible) r.flags |= kResFeasOut;
    if (per_task) {
      for (int i = lane; i < 7 * P.n_tasks; i += 32) per_task[i] = s.agg[i];
    }
  } else if (mode == kModeEvaluate || mode == kModeChain || mode == kModeBalanceData ||
             mode == kModeBalanceLayers) {
    const bool chain = mode == kModeEvaluate || mode == kModeChain;
    const bool go = mode != kModeEvaluate || feas_in;
    if (go) {
      team_geometry(P, cfg, s);
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
  // ---- write back what balancing can change: [generation task weights |
  // all stage layers] (engine.cpp ws_bytes_of / apply_ws) ----
  if (!(s.h.n_tasks & kRecCompact)) {
    const int g = P.gen_slot;
    const int dpg = g >= 0 ? s.h.dp[g] : 0;
    if (ows) {
      double* ow = reinterpret_cast<double*>(ows);
      int32_t* osl = reinterpret_cast<int32_t*>(ows + 8 * dpg);
      for (int i = lane; i < dpg; i += 32) ow[i] = s.w[s.o.w[g] + i];
      for (int i = lane; i < nsl; i += 32) osl[i] = s.sl[i];
    } else if (rec_wb) {
      double* ow = reinterpret_cast<double*>(rec_wb + s.o.w_byte) + (g >= 0 ? s.o.w[g] : 0);
      int32_t* osl = reinterpret_cast<int32_t*>(rec_wb + s.o.sl_byte);
      for (int i = lane; i < dpg; i += 32) ow[i] = s.w[s.o.w[g] + i];
      for (int i = lane; i < nsl; i += 32) osl[i] = s.sl[i];
    }
  }
  __syncwarp();
  return r;
}

// kTeam = 1: one warp per CTA, register-capped for occupancy (big waves, the
// sweep); kTeam = 2: pairs at the same register cap (medium waves);
// kTeam = kMaxTeam: up to four warps per plan, uncapped (small waves)
template <int kTeam>
__global__ void __launch_bounds__(32 * kTeam, kTeam == 1 ? 16 : (kTeam == 2 ? 8 : 2))
eval_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ DevCostConfig cfg,
            const __grid_constant__ Carve cv, int32_t kb_flags,
            const uint8_t* __restrict__ recs, const int64_t* __restrict__ off,
            const int32_t* __restrict__ modes, int32_t uniform_mode, int n, int64_t stride,
            uint8_t* __restrict__ out_ws, const int64_t* __restrict__ out_off,
            EvalResult* __restrict__ res,
            double* __restrict__ per_task, double* __restrict__ required,
            double* __restrict__ gscratch, int64_t gscratch_doubles) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ws team[kTeam];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    Ws& l = team[0];
    uint8_t* p = carve(l, smem, cv);
    HPG_DCHECK(p - smem <= cv.bytes);
    l.dtab = gscratch + static_cast<int64_t>(blockIdx.x) * gscratch_doubles;
    l.dtab_stride = 0;
    l.prof = nullptr;
    l.team = team;
    l.n_warps = static_cast<int32_t>(blockDim.x >> 5);
    l.job_words[0] = l.job_words[1] = 0;
    l.job = l.job_words;
    l.cta_sync = 0;
    const bool smem_cls = l.cls != nullptr;
    if (!smem_cls) l.cls = P.cls;
    for (int w = 1; w < l.n_warps; ++w) {
      team[w] = l;
      p = carve_team_scratch(team[w], p, cv);
    }
  }
  __syncthreads();
  if (warp == 0 && cv.cls_smem) stage_link_classes(P, team[0]);
  __syncthreads();
  if (warp > 0) {
    team_helper(P, cfg, team, warp);
    return;
  }
  Ws& s = team[0];
  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    const int64_t rec_at = off ? off[p] : static_cast<int64_t>(p) * stride;
    const int mode = modes ? modes[p] : uniform_mode;
    if (mode == kModeSkip) {
      if (lane == 0) res[p] = EvalResult{-1.0, 0.0, 0.0, 0, 0};
      continue;
    }
    long long* prof = g_plan_prof ? g_plan_prof + kPlanProfSlots * static_cast<int64_t>(p) : nullptr;
    const EvalResult r =
        eval_one(P, cfg, s, kb_flags, recs + rec_at, mode, prof,
                 per_task ? per_task + static_cast<int64_t>(p) * 7 * P.n_tasks : nullptr,
                 required ? required + static_cast<int64_t>(p) * P.n_dev : nullptr,
                 out_ws ? out_ws + out_off[p] : nullptr, nullptr);
    if (prof && lane == 0) prof[4] = clock64();
    if (lane == 0) res[p] = r;
    __syncwarp();
  }
  team_exit(s);
}

}  // namespace dev

int eval_smem_bytes(const Carve& c) { return carve2_bytes(c); }

cudaError_t eval_set_plan_profile(long long* d_buf) {
  return cudaMemcpyToSymbol(dev::g_plan_prof, &d_buf, sizeof(d_buf));
}

cudaError_t eval_phase_acc(unsigned long long* out16) {
  return cudaMemcpyFromSymbol(out16, dev::g_phase_acc, 32 * sizeof(unsigned long long));
}

int64_t eval_scratch_doubles(int n_dev, int64_t max_nl) {
  // per CTA (pp * dp <= N): DP-ring table [pp][nl + 1], column verdicts
  // (int32) [pp][nl + 1] and column cell pieces [pp][nl + 1][dp][2]
  return 4 * static_cast<int64_t>(n_dev) * (max_nl + 2);
}

namespace {
template <int kTeam>
cudaError_t grid_for(Carve cv, int n, int n_sm, int& grid) {
  auto kern = dev::eval_kernel<kTeam>;
  // opt in to the dynamic size (static + dynamic may not exceed 48 KB without
  // it, and the kernel's own static shared memory counts); per device
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), cv.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = occupancy_per_sm(reinterpret_cast<const void*>(kern), 32 * cv.n_warps, cv.bytes, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  grid = n < n_sm * per_sm ? n : n_sm * per_sm;
  return cudaSuccess;
}
}  // namespace

cudaError_t eval_grid(Carve cv, int n, int n_sm, int& grid) {
  if (cv.n_warps < 1) cv.n_warps = 1;
  cv.bytes = carve2_bytes(cv);
  if (cv.n_warps == 1) return grid_for<1>(cv, n, n_sm, grid);
  if (cv.n_warps == 2) return grid_for<2>(cv, n, n_sm, grid);
  return grid_for<dev::kMaxTeam>(cv, n, n_sm, grid);
}

cudaError_t launch_eval(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                        int32_t kb_flags, const uint8_t* d_recs, const int64_t* d_off,
                        const int32_t* d_modes, int32_t uniform_mode, int n, int64_t stride,
                        uint8_t* d_out, const int64_t* d_out_off, EvalResult* d_res,
                        double* d_per_task,
                        double* d_required, double* d_scratch, int64_t scratch_doubles,
                        int grid, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (cv.n_warps < 1) cv.n_warps = 1;
  if (cv.n_warps > dev::kMaxTeam) return cudaErrorInvalidValue;
  cv.bytes = carve2_bytes(cv);
  if (cv.n_warps == 1) {
    dev::eval_kernel<1><<<grid, 32, cv.bytes, st>>>(P, cfg, cv, kb_flags, d_recs, d_off, d_modes,
                                                    uniform_mode, n, stride, d_out, d_out_off, d_res,
                                                    d_per_task, d_required, d_scratch,
                                                    scratch_doubles);
  } else if (cv.n_warps == 2) {
    dev::eval_kernel<2><<<grid, 64, cv.bytes, st>>>(P, cfg, cv, kb_flags, d_recs, d_off, d_modes,
                                                    uniform_mode, n, stride, d_out, d_out_off, d_res,
                                                    d_per_task, d_required, d_scratch,
                                                    scratch_doubles);
  } else {
    dev::eval_kernel<dev::kMaxTeam><<<grid, 32 * cv.n_warps, cv.bytes, st>>>(
        P, cfg, cv, kb_flags, d_recs, d_off, d_modes, uniform_mode, n, stride, d_out, d_out_off, d_res,
        d_per_task, d_required, d_scratch, scratch_doubles);
  }
  return cudaGetLastError();
}

}  // namespace hpg

#include "ga_kernel.cuh"
#include "sweep_kernel.cuh"
#include "prim_kernels.cuh"
