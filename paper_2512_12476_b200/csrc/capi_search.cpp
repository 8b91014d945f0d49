// C ABI: search, single-arm GA, result accessors and the config-5 sweep.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>

#include "engine.hpp"
#include "eval_launch.hpp"
#include "search.hpp"
#include "sweep.hpp"

using namespace hpg;

struct hpg_ctx {
  Ctx* impl;
};

struct hpg_search_result {
  SearchOut out;
  // chosen plan as a one-plan table
  int32_t n_groups = 0;
  std::vector<int32_t> task_group, gpu_counts, dp, pp, tp, stage_layers, devices, groups_flat;
  std::vector<int64_t> sl_off, w_off, dev_off;
  std::vector<double> weights;
};

namespace {

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (err && errlen > 0) std::snprintf(err, errlen, "%s", msg.c_str());
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    set_err(err, errlen, "");
    return HPG_OK;
  } catch (const UsageError& e) {
    set_err(err, errlen, e.what());
    return HPG_USAGE;
  } catch (const InputError& e) {
    set_err(err, errlen, e.what());
    return HPG_INPUT;
  } catch (const InfeasibleError& e) {
    set_err(err, errlen, e.what());
    return HPG_INFEASIBLE;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return HPG_INTERNAL;
  } catch (...) {
    set_err(err, errlen, "unknown engine failure");
    return HPG_INTERNAL;
  }
}

hpg_search_result* wrap(SearchOut&& s, const Problem& P) {
  auto* r = new hpg_search_result();
  r->out = std::move(s);
  if (r->out.has_plan) {
    const SearchOut& o = r->out;
    const int T = P.T;
    r->n_groups = static_cast<int32_t>(o.plan_groups.size());
    r->task_group.assign(T, 0);
    for (size_t g = 0; g < o.plan_groups.size(); ++g)
      for (int sl : o.plan_groups[g]) {
        r->task_group[sl] = static_cast<int32_t>(g);
        r->groups_flat.push_back(sl);
      }
    r->gpu_counts.assign(T, 0);
    for (size_t g = 0; g < o.plan_counts.size(); ++g) r->gpu_counts[g] = o.plan_counts[g];
    const Cand& c = o.plan;
    for (int t = 0; t < T; ++t) {
      r->dp.push_back(c.hdr().dp[t]);
      r->pp.push_back(c.hdr().pp[t]);
      r->tp.push_back(c.hdr().tp[t]);
      r->sl_off.push_back(c.o.sl[t]);
      r->w_off.push_back(c.o.w[t]);
      r->dev_off.push_back(c.o.dev[t]);
    }
    r->stage_layers.assign(c.sl(), c.sl() + c.o.sl[T]);
    r->weights.assign(c.w(), c.w() + c.o.w[T]);
    for (int i = 0; i < c.o.dev[T]; ++i) r->devices.push_back(c.dev()[i]);
  }
  return r;
}

// ---- sweep tables ----

struct SweepHost {
  SweepTablesDev tb{};
  void* blob = nullptr;
};

SweepTablesDev& sweep_tables(Ctx& C) {
  if (C.d_sweep_tables) return C.sweep_tb;
  const Problem& P = C.prob;
  if (P.N < P.T) throw InputError("sweep needs at least as many devices as workflow tasks");
  const auto tgs = enumerate_task_groupings(P, false);
  std::vector<int8_t> grp(tgs.size() * kMaxTasks, -1), ng(tgs.size());
  for (size_t i = 0; i < tgs.size(); ++i) {
    ng[i] = static_cast<int8_t>(tgs[i].size());
    for (size_t g = 0; g < tgs[i].size(); ++g)
      for (int s : tgs[i][g]) grp[i * kMaxTasks + s] = static_cast<int8_t>(g);
  }
  const int N = P.N, T = P.T;
  std::vector<int32_t> off(T * (N + 1) + 1, 0);
  std::vector<int16_t> opt;
  int idx = 0;
  for (int s = 0; s < T; ++s) {
    for (int c = 0; c <= N; ++c) {
      off[s * (N + 1) + c] = idx;
      if (c == 0) continue;
      for (int dp = 1; dp <= c; ++dp) {
        if (c % dp) continue;
        const int rest = c / dp;
        for (int pp = 1; pp <= rest; ++pp) {
          if (rest % pp) continue;
          const int tp = rest / pp;
          if (pp > P.tasks[s].nl || tp > P.max_node_size) continue;
          opt.push_back(static_cast<int16_t>(dp));
          opt.push_back(static_cast<int16_t>(pp));
          opt.push_back(static_cast<int16_t>(tp));
          ++idx;
        }
      }
    }
  }
  off[T * (N + 1)] = idx;
  const size_t b_grp = grp.size(), b_ng = ng.size(), b_off = 4 * off.size(), b_opt = 2 * opt.size();
  const size_t o_ng = (b_grp + 15) & ~size_t(15);
  const size_t o_off = (o_ng + b_ng + 15) & ~size_t(15);
  const size_t o_opt = (o_off + b_off + 15) & ~size_t(15);
  const size_t total = o_opt + b_opt + 16;
  std::vector<uint8_t> blob(total, 0);
  std::memcpy(blob.data(), grp.data(), b_grp);
  std::memcpy(blob.data() + o_ng, ng.data(), b_ng);
  std::memcpy(blob.data() + o_off, off.data(), b_off);
  std::memcpy(blob.data() + o_opt, opt.data(), b_opt);
  SweepHost h;
  cuda_check(cudaMalloc(&h.blob, total), "cudaMalloc sweep tables");
  cuda_check(cudaMemcpy(h.blob, blob.data(), total, cudaMemcpyHostToDevice), "H2D sweep tables");
  uint8_t* b = static_cast<uint8_t*>(h.blob);
  h.tb.n_dev = N;
  h.tb.n_tasks = T;
  h.tb.n_tgs = static_cast<int32_t>(tgs.size());
  h.tb.tg_group = reinterpret_cast<const int8_t*>(b);
  h.tb.tg_ng = reinterpret_cast<const int8_t*>(b + o_ng);
  h.tb.opt_off = reinterpret_cast<const int32_t*>(b + o_off);
  h.tb.opt = reinterpret_cast<const int16_t*>(b + o_opt);
  h.tb.gen_slot = C.dprob.gen_slot;
  h.tb.train6_slot = C.dprob.train6_slot;
  h.tb.train_mask = 0;
  for (int s = 0; s < T; ++s)
    if (C.dprob.task[s].kind == kTraining) h.tb.train_mask |= 1 << s;
  C.d_sweep_tables = h.blob;
  C.sweep_tb = h.tb;
  return C.sweep_tb;
}

struct SweepAcc {
  double best = kInf;
  uint64_t best_k = ~0ull, nf = 0, x = 0, bytes = 0;
  float gen_ms = 0, eval_ms = 0, total_ms = 0;
  int64_t launches = 0;
  uint64_t global_slab_plans = 0;
};

// Plans [k0, k0 + count) in chunks: gen_kernel writes a chunk's compact plan
// records into HBM, sweep_kernel scores them (end_to_end_cost, per-plan
// carve) and folds them into per-warp (argmin, feasible count, checksum)
// partials that persist across chunks. Chunks follow each other on the
// context's stream with no host round trip; the partials come back once.
// With costs/feasible requested, each chunk's per-plan results are copied out.
void run_sweep(Ctx& C, uint64_t seed, uint64_t k0, uint64_t count, double* costs,
               uint8_t* feasible, SweepAcc& acc) {
  const Problem& P = C.prob;
  SweepTablesDev& tb = sweep_tables(C);
  const int64_t stride = (80 + P.T * P.N + 7) & ~int64_t(7);
  const int64_t chunk = static_cast<int64_t>(std::min<uint64_t>(std::max<uint64_t>(count, 1), 1ull << 21));
  const bool want = costs || feasible;
  C.d_recs.reserve(static_cast<size_t>(chunk) * stride);
  if (want) C.d_res.reserve(chunk);
  C.d_best.reserve(2);
  static const int warps_env = [] {
    const char* v = std::getenv("HPG_SWEEP_WARPS");  // diagnostics: 2, 4 or 8 plan-warps per CTA
    return v ? std::atoi(v) : 8;
  }();
  static const int slab_env = [] {
    const char* v = std::getenv("HPG_SWEEP_SLAB");  // diagnostics: cap the per-warp slab (bytes)
    return v ? std::atoi(v) : 0;
  }();
  static const int sync_env = [] {
    // CTA-wide phase barriers (plan + per-task; 2 = plan only, 0 = none):
    // measured 1.88 -> 2.51 M plans/s on c4 (r02c), with ordering 2.91 (r02f)
    const char* v = std::getenv("HPG_SWEEP_SYNC");
    return v ? std::atoi(v) : 1;
  }();
  static const int sort_env = [] {
    const char* v = std::getenv("HPG_SWEEP_SORT");  // work-class ordering (0 = off)
    return v ? std::atoi(v) : 1;
  }();
  SweepLaunch L;
  L.sync = sync_env;
  cuda_check(sweep_plan(P.N, P.T, C.n_sm, warps_env, slab_env, L), "sweep_kernel configuration");
  const int64_t nwarps = static_cast<int64_t>(L.grid) * L.warps;
  C.d_sweep_gslab.reserve(static_cast<size_t>(nwarps * L.gslab_bytes));
  C.d_sweep_part.reserve(static_cast<size_t>(nwarps) * sizeof(SweepPartial) + 16);
  L.gslab = C.d_sweep_gslab.p;
  L.part = reinterpret_cast<SweepPartial*>(C.d_sweep_part.p);
  L.n_global = reinterpret_cast<unsigned long long*>(C.d_sweep_part.p +
                                                      nwarps * sizeof(SweepPartial));
  std::vector<SweepPartial> hp(static_cast<size_t>(nwarps), SweepPartial{kInf, ~0ull, 0, 0});
  SweepOrder ord;
  if (sort_env) {
    const size_t kb = (4 * static_cast<size_t>(chunk) + 255) & ~size_t(255);
    C.d_sweep_order.reserve(2 * kb + (sizeof(uint32_t) << kSweepKeyBits));
    ord.keys = reinterpret_cast<uint32_t*>(C.d_sweep_order.p);
    ord.order = reinterpret_cast<uint32_t*>(C.d_sweep_order.p + kb);
    ord.hist = reinterpret_cast<uint32_t*>(C.d_sweep_order.p + 2 * kb);
  }
  const DevCostConfig cfg = to_dev_cfg(default_cost_config());
  cudaStream_t st = C.stream;
  cuda_check(cudaMemcpyAsync(L.part, hp.data(), sizeof(SweepPartial) * nwarps,
                             cudaMemcpyHostToDevice, st), "H2D sweep partials");
  cuda_check(cudaMemsetAsync(L.n_global, 0, 8, st), "memset");
  cuda_check(cudaMemsetAsync(C.d_best.p, 0, 16, st), "memset");
  // independent random plans share no rings: the ring memo would only fill
  DevProblem sweep_prob = C.dprob;
  sweep_prob.ring_cache = nullptr;
  const int64_t n_chunks = (static_cast<int64_t>(count) + chunk - 1) / chunk;
  std::vector<cudaEvent_t> ev(static_cast<size_t>(3 * std::max<int64_t>(n_chunks, 1)));
  for (auto& e : ev) cuda_check(cudaEventCreate(&e), "event");
  std::vector<EvalResult> r;
  int64_t ci = 0;
  for (uint64_t done = 0; done < count; ++ci) {
    const int64_t n = static_cast<int64_t>(std::min<uint64_t>(chunk, count - done));
    const uint64_t kk = k0 + done;
    cudaEventRecord(ev[3 * ci], st);
    cuda_check(launch_gen(tb, seed, kk, n, C.d_recs.p, stride, C.d_best.p,
                          sort_env ? &ord : nullptr, st), "gen_kernel");
    if (sort_env) {
      cuda_check(launch_order(ord, n, st), "order kernels");
      acc.launches += 2;
      C.launches += 2;
    }
    cudaEventRecord(ev[3 * ci + 1], st);
    cuda_check(launch_sweep(sweep_prob, cfg, C.d_recs.p, stride, n, kk, L,
                            sort_env ? ord.order : nullptr, want ? C.d_res.p : nullptr, st),
               "sweep_kernel");
    cudaEventRecord(ev[3 * ci + 2], st);
    acc.launches += 2;
    C.launches += 2;
    C.plans_evaluated += n;
    if (want) {
      r.resize(static_cast<size_t>(n));
      cuda_check(cudaMemcpyAsync(r.data(), C.d_res.p, sizeof(EvalResult) * n,
                                 cudaMemcpyDeviceToHost, st), "D2H results");
      cuda_check(cudaStreamSynchronize(st), "sweep");
      for (int64_t i = 0; i < n; ++i) {
        if (costs) costs[done + i] = r[i].cost;
        if (feasible) feasible[done + i] = (r[i].flags & kResFeasOut) ? 1 : 0;
      }
    }
    done += n;
  }
  unsigned long long tail[2] = {0, 0};
  cuda_check(cudaMemcpyAsync(hp.data(), L.part, sizeof(SweepPartial) * nwarps,
                             cudaMemcpyDeviceToHost, st), "D2H sweep partials");
  cuda_check(cudaMemcpyAsync(&tail[0], C.d_best.p, 8, cudaMemcpyDeviceToHost, st), "D2H bytes");
  cuda_check(cudaMemcpyAsync(&tail[1], L.n_global, 8, cudaMemcpyDeviceToHost, st), "D2H spills");
  cuda_check(cudaStreamSynchronize(st), "sweep");
  for (int64_t c = 0; c < ci; ++c) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[3 * c], ev[3 * c + 1]);
    cudaEventElapsedTime(&b, ev[3 * c + 1], ev[3 * c + 2]);
    acc.gen_ms += a;
    acc.eval_ms += b;
  }
  if (ci > 0) cudaEventElapsedTime(&acc.total_ms, ev[0], ev[3 * (ci - 1) + 2]);
  for (auto& e : ev) cudaEventDestroy(e);
  for (const SweepPartial& p : hp) {
    acc.nf += p.n_feasible;
    acc.x ^= p.xor_bits;
    if (p.best < acc.best || (p.best == acc.best && p.best_k < acc.best_k)) {
      acc.best = p.best;
      acc.best_k = p.best_k;
    }
  }
  acc.bytes = tail[0];
  acc.global_slab_plans = tail[1];
}

}  // namespace

extern "C" {

int hpg_search(hpg_ctx* ctx, const hpg_knobs* knobs, hpg_search_result** out, char* err,
               size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !knobs || !out) throw UsageError("hpg_search: null argument");
    *out = nullptr;
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const Knobs K = knobs_from_c(C.prob, *knobs);
    if (K.budget < 1) throw UsageError("search budget must be >= 1");
    *out = wrap(nested_sha_search(C, K, nullptr), C.prob);
  });
}

int hpg_nccl_unique_id(uint8_t id_out[128], char* err, size_t errlen) {
  return guarded(err, errlen, [&] { dist_unique_id(id_out); });
}

int hpg_search_dist(hpg_ctx* ctx, const hpg_knobs* knobs, int rank, int world,
                    const uint8_t nccl_id[128], hpg_search_result** out, char* err,
                    size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !knobs || !out) throw UsageError("hpg_search_dist: null argument");
    *out = nullptr;
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const Knobs K = knobs_from_c(C.prob, *knobs);
    if (K.budget < 1) throw UsageError("search budget must be >= 1");
    if (world <= 1) {
      *out = wrap(nested_sha_search(C, K, nullptr), C.prob);
      return;
    }
    // the communicator is created on the first sharded search of a context
    // (nccl_id consumed then) and reused afterwards
    if (!C.dist.comm || C.dist.rank != rank || C.dist.world != world) {
      if (C.dist.comm) dist_destroy(C.dist);
      dist_init(C.dist, rank, world, nccl_id, C.device);
    }
    *out = wrap(nested_sha_search(C, K, &C.dist), C.prob);
  });
}

int hpg_ga_search(hpg_ctx* ctx, const int32_t* task_group, int32_t n_groups,
                  const int32_t* gpu_counts, int64_t budget_slice, uint64_t rng_seed,
                  const hpg_knobs* knobs, hpg_search_result** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !knobs || !out || !task_group || !gpu_counts)
      throw UsageError("hpg_ga_search: null argument");
    *out = nullptr;
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const Knobs K = knobs_from_c(C.prob, *knobs);
    Grouping tg(n_groups);
    for (int s = 0; s < C.prob.T; ++s) {
      if (task_group[s] < 0 || task_group[s] >= n_groups)
        throw InputError("task grouping must cover every workflow task");
      tg[task_group[s]].push_back(s);
    }
    std::vector<int> counts(gpu_counts, gpu_counts + n_groups);
    *out = wrap(ga_search(C, tg, counts, budget_slice, rng_seed, K), C.prob);
  });
}

int hpg_exhaustive(hpg_ctx* ctx, const hpg_knobs* knobs, hpg_search_result** out, char* err,
                   size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !knobs || !out) throw UsageError("hpg_exhaustive: null argument");
    *out = nullptr;
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    *out = wrap(exhaustive_search(C, knobs_from_c(C.prob, *knobs)), C.prob);
  });
}

int hpg_exhaustive_estimate(hpg_ctx* ctx, const hpg_knobs* knobs, double* estimate, char* err,
                            size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !knobs || !estimate)
      throw UsageError("hpg_exhaustive_estimate: null argument");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    *estimate = exhaustive_space_estimate(C.prob, knobs_from_c(C.prob, *knobs));
  });
}

int hpg_result_info(const hpg_search_result* r, hpg_search_info* info) {
  if (!r || !info) return HPG_USAGE;
  const SearchOut& o = r->out;
  info->budget = o.budget;
  info->consumed = o.consumed;
  info->seed = o.seed;
  info->has_plan = o.has_plan ? 1 : 0;
  info->n_b_m = static_cast<int32_t>(o.b_m.size());
  info->n_trace = static_cast<int32_t>(o.trace.size());
  info->n_arms = static_cast<int32_t>(o.arms.size());
  info->n_halvings = static_cast<int32_t>(o.halvings.size());
  info->n_survivor_sets = static_cast<int32_t>(o.survivors.size());
  info->task_groupings = o.task_groupings;
  info->wall_s = o.wall_s;
  info->time_to_best_s = o.time_to_best_s;
  info->gpu_launches = o.launches;
  info->waves = o.waves;
  info->plans_evaluated_gpu = o.plans_gpu;
  info->h2d_bytes = o.h2d_bytes;
  info->d2h_bytes = o.d2h_bytes;
  info->eval_kernel_ms = o.eval_ms;
  info->eval_launches = o.eval_launches;
  info->canonical_bytes = o.canonical_bytes;
  info->host_ms = o.host_ms;
  info->batch_ms = o.batch_ms;
  return HPG_OK;
}

int hpg_result_b_m(const hpg_search_result* r, int64_t* b_m) {
  if (!r || !b_m) return HPG_USAGE;
  std::copy(r->out.b_m.begin(), r->out.b_m.end(), b_m);
  return HPG_OK;
}

int hpg_result_trace(const hpg_search_result* r, int64_t* consumed, double* cost) {
  if (!r) return HPG_USAGE;
  for (size_t i = 0; i < r->out.trace.size(); ++i) {
    if (consumed) consumed[i] = r->out.trace[i].first;
    if (cost) cost[i] = r->out.trace[i].second;
  }
  return HPG_OK;
}

int hpg_result_arms(const hpg_search_result* r, int64_t* tg_index, int64_t* gg_index,
                    double* best_cost, int64_t* evals) {
  if (!r) return HPG_USAGE;
  for (size_t i = 0; i < r->out.arms.size(); ++i) {
    const ArmRec& a = r->out.arms[i];
    if (tg_index) tg_index[i] = a.tg;
    if (gg_index) gg_index[i] = a.gg;
    if (best_cost) best_cost[i] = a.best;
    if (evals) evals[i] = a.evals;
  }
  return HPG_OK;
}

int hpg_result_halvings(const hpg_search_result* r, int32_t* level, int64_t* before,
                        int64_t* after, double* survivor_worst, double* eliminated_best) {
  if (!r) return HPG_USAGE;
  for (size_t i = 0; i < r->out.halvings.size(); ++i) {
    const Halving& h = r->out.halvings[i];
    if (level) level[i] = h.level;
    if (before) before[i] = h.before;
    if (after) after[i] = h.after;
    if (survivor_worst) survivor_worst[i] = h.survivor_worst;
    if (eliminated_best) eliminated_best[i] = h.eliminated_best;
  }
  return HPG_OK;
}

int hpg_result_survivor_sizes(const hpg_search_result* r, int32_t* sizes) {
  if (!r || !sizes) return HPG_USAGE;
  for (size_t i = 0; i < r->out.survivors.size(); ++i)
    sizes[i] = static_cast<int32_t>(r->out.survivors[i].size());
  return HPG_OK;
}

int hpg_result_survivors(const hpg_search_result* r, int64_t* idx) {
  if (!r || !idx) return HPG_USAGE;
  size_t k = 0;
  for (const auto& s : r->out.survivors)
    for (int64_t v : s) idx[k++] = v;
  return HPG_OK;
}

int hpg_result_plan(const hpg_search_result* r, hpg_plan_table* plan, int32_t* groups_flat,
                    double* estimated_cost_s, uint64_t* prov_seed, int64_t* prov_budget) {
  if (!r) return HPG_USAGE;
  if (!r->out.has_plan) return HPG_INFEASIBLE;
  if (plan) {
    plan->n_plans = 1;
    plan->n_groups = &r->n_groups;
    plan->task_group = r->task_group.data();
    plan->gpu_counts = r->gpu_counts.data();
    plan->dp = r->dp.data();
    plan->pp = r->pp.data();
    plan->tp = r->tp.data();
    plan->sl_off = r->sl_off.data();
    plan->stage_layers = r->stage_layers.data();
    plan->w_off = r->w_off.data();
    plan->weights = r->weights.data();
    plan->dev_off = r->dev_off.data();
    plan->devices = r->devices.data();
  }
  if (groups_flat) std::copy(r->groups_flat.begin(), r->groups_flat.end(), groups_flat);
  if (estimated_cost_s) *estimated_cost_s = r->out.est_cost;
  if (prov_seed) *prov_seed = r->out.seed;
  if (prov_budget) *prov_budget = r->out.prov_budget >= 0 ? r->out.prov_budget : r->out.consumed;
  return HPG_OK;
}

int hpg_result_breakdown(const hpg_search_result* r, double* per_task, double* reshard_s,
                         double* sync_s, double* end_to_end_s, uint8_t* memory_feasible) {
  if (!r) return HPG_USAGE;
  if (!r->out.has_plan) return HPG_INFEASIBLE;
  if (per_task) std::copy(r->out.per_task.begin(), r->out.per_task.end(), per_task);
  if (reshard_s) *reshard_s = r->out.reshard_s;
  if (sync_s) *sync_s = r->out.sync_s;
  if (end_to_end_s) *end_to_end_s = r->out.e2e;
  if (memory_feasible) *memory_feasible = r->out.feasible ? 1 : 0;
  return HPG_OK;
}

void hpg_result_free(hpg_search_result* r) { delete r; }

int hpg_sweep(hpg_ctx* ctx, uint64_t seed, uint64_t k0, uint64_t count, double* costs,
              uint8_t* feasible, double* best_cost, uint64_t* best_k, uint64_t* n_feasible,
              char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl) throw UsageError("hpg_sweep: null context");
    SweepAcc acc;
    const DeviceScope on_device(ctx->impl->device);
    run_sweep(*ctx->impl, seed, k0, count, costs, feasible, acc);
    if (best_cost) *best_cost = acc.best;
    if (best_k) *best_k = acc.best_k;
    if (n_feasible) *n_feasible = acc.nf;
  });
}

int hpg_sweep_resident(hpg_ctx* ctx, uint64_t seed, uint64_t k0, uint64_t count,
                       hpg_sweep_stats* stats, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !stats) throw UsageError("hpg_sweep_resident: null argument");
    SweepAcc acc;
    const DeviceScope on_device(ctx->impl->device);
    run_sweep(*ctx->impl, seed, k0, count, nullptr, nullptr, acc);
    stats->best_cost = acc.best;
    stats->best_k = acc.best_k;
    stats->n_feasible = acc.nf;
    stats->xor_bits = acc.x;
    stats->canonical_bytes = acc.bytes;
    stats->total_ms = acc.total_ms;
    stats->eval_ms = acc.eval_ms;
    stats->gen_ms = acc.gen_ms;
    stats->launches = acc.launches;
    stats->global_slab_plans = acc.global_slab_plans;
  });
}

int hpg_sweep_dist(hpg_ctx* ctx, uint64_t seed, uint64_t total, int rank, int world,
                   const uint8_t nccl_id[128], hpg_sweep_stats* stats, char* err,
                   size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !stats) throw UsageError("hpg_sweep_dist: null argument");
    if (world < 1 || rank < 0 || rank >= world) throw UsageError("hpg_sweep_dist: bad rank/world");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    // contiguous plan-index shard of this rank
    const uint64_t k0 = static_cast<uint64_t>((static_cast<unsigned __int128>(total) * rank) / world);
    const uint64_t k1 =
        static_cast<uint64_t>((static_cast<unsigned __int128>(total) * (rank + 1)) / world);
    SweepAcc acc;
    run_sweep(C, seed, k0, k1 - k0, nullptr, nullptr, acc);
    SweepPartial mine{acc.best, acc.best_k, acc.nf, acc.x};
    if (world > 1) {
      if (!C.dist.comm || C.dist.rank != rank || C.dist.world != world) {
        if (C.dist.comm) dist_destroy(C.dist);
        dist_init(C.dist, rank, world, nccl_id, C.device);
      }
      // one all-gather of the 32-byte (cost, k, feasible count, checksum) partials
      std::vector<SweepPartial> all(static_cast<size_t>(world));
      C.d_xch_send.reserve(sizeof(SweepPartial));
      C.d_xch_recv.reserve(sizeof(SweepPartial) * world);
      cuda_check(cudaMemcpyAsync(C.d_xch_send.p, &mine, sizeof(mine), cudaMemcpyHostToDevice,
                                 C.stream), "H2D sweep partial");
      dist_allgather(C.dist, C.d_xch_send.p, C.d_xch_recv.p, sizeof(SweepPartial), C.stream);
      cuda_check(cudaMemcpyAsync(all.data(), C.d_xch_recv.p, sizeof(SweepPartial) * world,
                                 cudaMemcpyDeviceToHost, C.stream), "D2H sweep partials");
      cuda_check(cudaStreamSynchronize(C.stream), "sweep all-gather");
      mine = SweepPartial{kInf, ~0ull, 0, 0};
      for (const SweepPartial& p : all) {
        mine.n_feasible += p.n_feasible;
        mine.xor_bits ^= p.xor_bits;
        if (p.best < mine.best || (p.best == mine.best && p.best_k < mine.best_k)) {
          mine.best = p.best;
          mine.best_k = p.best_k;
        }
      }
    }
    stats->best_cost = mine.best;
    stats->best_k = mine.best_k;
    stats->n_feasible = mine.n_feasible;
    stats->xor_bits = mine.xor_bits;
    stats->canonical_bytes = acc.bytes;
    stats->total_ms = acc.total_ms;
    stats->eval_ms = acc.eval_ms;
    stats->gen_ms = acc.gen_ms;
    stats->launches = acc.launches;
    stats->global_slab_plans = acc.global_slab_plans;
  });
}

}  // extern "C"
