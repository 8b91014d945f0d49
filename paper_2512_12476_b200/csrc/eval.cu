// eval_kernel: one warp per candidate plan, persistent grid-stride over the
// batch. Modes (common.hpp EvalMode):
//   memcheck       check_memory                       plan.cpp:351-380
//   e2e            end_to_end_cost                     cost_model.cpp:431-487
//   evaluate       EvalContext::evaluate minus the     search.cpp:259-279
//                  budget bookkeeping (balance_data -> balance_layers -> e2e),
//                  skipped when the input plan breaks C3 (the GA's memory_ok
//                  gate, search.cpp:458-460)
//   balance_data   balance.cpp:37-56
//   balance_layers balance.cpp:81-167
// The balanced plan is written back as a record with the same layout.
#include <cuda_runtime.h>

#include <cstdio>

#include "eval_device.cuh"
#include "eval_launch.hpp"

namespace hpg {
namespace dev {

struct Ws2 : Ws {
  double* wsave;        // [N]
  int32_t* sl_save2;    // [max_sl]
  int32_t* split_step;  // [N]
  int32_t* sl_tsave;    // [N]
};

__device__ inline void carve2(Ws2& s, uint8_t* base, const Carve& c) {
  carve(s, base, c);
  uint8_t* p = base + carve_bytes(c);
  s.wsave = reinterpret_cast<double*>(carve_ptr(p, 8 * c.n_dev));
  s.sl_save2 = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.max_sl));
  s.split_step = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.n_dev));
  s.sl_tsave = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * c.n_dev));
}

__device__ __forceinline__ void copy_i32(int32_t* dst, const int32_t* src, int n) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int i = lane; i < n; i += 32) dst[i] = src[i];
  __syncwarp();
}

// task_total_with_split (balance.cpp:61-77): whole-plan C3 check with the
// trial split, then the task's own cost with own-weights dbs.
__device__ __noinline__ double total_with_split(const DevProblem& P, const DevCostConfig& cfg, Ws2& s,
                                          int t, const int32_t* split) {
  const int pp = s.h.pp[t];
  int32_t* sl_t = s.sl + s.o.sl[t];
  copy_i32(s.sl_tsave, sl_t, pp);
  copy_i32(sl_t, split, pp);
  double v = kInf;
  if (check_memory(P, cfg, s)) {
    double agg[7];
    task_cost(P, cfg, s, t, false, agg);
    v = agg[6];
  }
  copy_i32(sl_t, s.sl_tsave, pp);
  return v;
}

// balance_data (balance.cpp:37-56) with rate_weights (:14-35). Returns true
// when it had work (a generation task with dp >= 2); then `cur` holds the
// end-to-end breakdown of the plan it returns.
__device__ __noinline__ bool balance_data_dev(const DevProblem& P, const DevCostConfig& cfg, Ws2& s,
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
  double* w = s.w + s.o.w[g];
  for (int i = lane; i < dp; i += 32) {
    s.wsave[i] = w[i];
    w[i] = s.wnew[i];
  }
  __syncwarp();
  apportion(P, s, g);
  const E2E after = end_to_end(P, cfg, s);
  if (after.e2e < before.e2e) {
    cur = after;
    changed = true;
  } else {
    for (int i = lane; i < dp; i += 32) w[i] = s.wsave[i];
    __syncwarp();
    apportion(P, s, g);
    cur = before;
  }
  return true;
}

// next composition in lexicographic order (combinatorics.cpp:61-95 order)
__device__ __forceinline__ bool next_composition(int32_t* c, int parts) {
  int tail = c[parts - 1];
  for (int i = parts - 2; i >= 0; --i) {
    if (tail > parts - 1 - i) {
      ++c[i];
      for (int k = i + 1; k < parts - 1; ++k) c[k] = 1;
      c[parts - 1] = tail - 1 - (parts - 2 - i);
      return true;
    }
    tail += c[i];
  }
  return false;
}

// balance_layers (balance.cpp:81-167), including its aliasing quirk: the
// greedy branch updates the candidate in place (:150) so `touched` is only
// ever set by exact-mode tasks (:153); with no exact-mode task the input plan
// is returned unchanged, which is short-circuited here.
__device__ __noinline__ void balance_layers_dev(const DevProblem& P, const DevCostConfig& cfg, Ws2& s,
                                          bool& have_cur, E2E& cur, bool& changed) {
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
    copy_i32(s.split_best, sl_t, pp);
    double best = total_with_split(P, cfg, s, t, s.split_best);
    if (static_cast<int64_t>(pp) * nl <= 64) {
      if (lane == 0) {
        for (int k = 0; k < pp - 1; ++k) s.split_trial[k] = 1;
        s.split_trial[pp - 1] = static_cast<int32_t>(nl) - (pp - 1);
      }
      __syncwarp();
      while (true) {
        const double c = total_with_split(P, cfg, s, t, s.split_trial);
        if (c < best) {
          best = c;
          copy_i32(s.split_best, s.split_trial, pp);
        }
        bool more = false;
        if (lane == 0) more = next_composition(s.split_trial, pp);
        more = __shfl_sync(kFull, more, 0);
        __syncwarp();
        if (!more) break;
      }
      bool diff = false;
      for (int j = lane; j < pp; j += 32) diff |= s.split_best[j] != sl_t[j];
      if (__any_sync(kFull, diff)) {
        copy_i32(sl_t, s.split_best, pp);
        touched = true;
      }
    } else {
      // greedy: shed one layer from the bottleneck stage to a neighbour
      const int dp = s.h.dp[t];
      while (true) {
        double agg[7];
        task_cost(P, cfg, s, t, false, agg);
        double worst = -1.0;
        int bn = 0;
        // load_j = max_i stage sum; first j with the strictly largest load
        for (int j0 = 0; j0 < pp; j0 += 32) {
          const int j = j0 + lane;
          double load = 0.0;
          if (j < pp) {
            for (int i = 0; i < dp; ++i) {
              const int c = i * pp + j;
              load = smax(load, s.c_comp[c] + s.c_tp[c] + s.c_pp[c] + s.c_hbm[c]);
            }
          } else {
            load = -kInf;
          }
          double m = warp_max(load);
          if (m > worst) {
            const unsigned bal = __ballot_sync(kFull, j < pp && load == m);
            worst = m;
            bn = j0 + __ffs(bal) - 1;
          }
        }
        if (s.split_best[bn] <= 1) break;
        double step_best = best;
        bool found = false;
        for (int side = 0; side < 2; ++side) {
          const int nb = side == 0 ? bn - 1 : bn + 1;
          if (nb < 0 || nb >= pp) continue;
          copy_i32(s.split_trial, s.split_best, pp);
          if (lane == 0) {
            --s.split_trial[bn];
            ++s.split_trial[nb];
          }
          __syncwarp();
          const double c = total_with_split(P, cfg, s, t, s.split_trial);
          if (c < step_best) {
            step_best = c;
            copy_i32(s.split_step, s.split_trial, pp);
            found = true;
          }
        }
        if (!found) break;
        best = step_best;
        copy_i32(s.split_best, s.split_step, pp);
        copy_i32(sl_t, s.split_best, pp);
      }
    }
  }
  if (!touched) {
    copy_i32(s.sl, s.sl_save, nsl);
    return;
  }
  if (!check_memory(P, cfg, s)) {
    copy_i32(s.sl, s.sl_save, nsl);
    return;
  }
  const E2E after = end_to_end(P, cfg, s);
  E2E before;
  if (have_cur) {
    before = cur;
  } else {
    copy_i32(s.sl_save2, s.sl, nsl);
    copy_i32(s.sl, s.sl_save, nsl);
    before = end_to_end(P, cfg, s);
    copy_i32(s.sl, s.sl_save2, nsl);
  }
  have_cur = true;
  if (after.e2e < before.e2e) {
    cur = after;
    changed = true;
  } else {
    copy_i32(s.sl, s.sl_save, nsl);
    cur = before;
  }
}

__global__ void __launch_bounds__(32)
eval_kernel(DevProblem P, DevCostConfig cfg, Carve cv, int32_t kb_flags,
            const uint8_t* __restrict__ recs, const int64_t* __restrict__ off,
            const int32_t* __restrict__ modes, int32_t uniform_mode, int n, int64_t stride,
            uint8_t* __restrict__ out_recs, EvalResult* __restrict__ res,
            double* __restrict__ per_task, double* __restrict__ required) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ws2 s;
  const int lane = threadIdx.x & 31;
  if (lane == 0) carve2(s, smem, cv);
  __syncwarp();
  for (int p = blockIdx.x; p < n; p += gridDim.x) {
    const int64_t rec_at = off ? off[p] : static_cast<int64_t>(p) * stride;
    const uint8_t* rec = recs + rec_at;
    const int mode = modes ? modes[p] : uniform_mode;
    // ---- stage the plan ----
    if (lane < 20) reinterpret_cast<int32_t*>(&s.h)[lane] = reinterpret_cast<const int32_t*>(rec)[lane];
    __syncwarp();
    if (lane == 0) {
      rec_offsets(s.h, s.o);
      s.memo_tp_ok = 0;
      s.memo_pp_ok = 0;
      s.bridge_ok = 0;
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
    for (int t = 0; t < P.n_tasks; ++t) apportion(P, s, t);
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
          have_cur = balance_data_dev(P, cfg, s, cur, ch);
          if (ch) r.flags |= kResWeights;
        }
        if ((chain && (kb_flags & 2)) || mode == kModeBalanceLayers) {
          balance_layers_dev(P, cfg, s, have_cur, cur, ch);
          if (ch) r.flags |= kResLayers;
        }
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
    if (lane == 0) res[p] = r;
    __syncwarp();
  }
}

}  // namespace dev

int eval_smem_bytes(const Carve& c) { return carve2_bytes(c); }

cudaError_t launch_eval(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                        int32_t kb_flags, const uint8_t* d_recs, const int64_t* d_off,
                        const int32_t* d_modes, int32_t uniform_mode, int n, int64_t stride,
                        uint8_t* d_out,
                        EvalResult* d_res, double* d_per_task, double* d_required,
                        int n_sm, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cv.bytes = carve2_bytes(cv);
  static int configured_bytes = 0;
  if (cv.bytes > 48 * 1024 && cv.bytes > configured_bytes) {
    cudaError_t e = cudaFuncSetAttribute(dev::eval_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, cv.bytes);
    if (e != cudaSuccess) return e;
    configured_bytes = cv.bytes;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::eval_kernel, 32,
                                                                cv.bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = n < n_sm * per_sm ? n : n_sm * per_sm;
  dev::eval_kernel<<<grid, 32, cv.bytes, st>>>(P, cfg, cv, kb_flags, d_recs, d_off, d_modes,
                                               uniform_mode, n, stride, d_out, d_res, d_per_task,
                                               d_required);
  return cudaGetLastError();
}

}  // namespace hpg
