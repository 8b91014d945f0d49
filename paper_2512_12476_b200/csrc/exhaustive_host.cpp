// Host side of exhaustive_search / exhaustive_space_estimate
// (search.cpp:837-1031): block enumeration, symmetry classes, the per-block
// device pipeline of exhaustive.cu + eval_kernel, and the first-minimum merge.
#include "exhaustive.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <map>
#include <string>

#include "eval_launch.hpp"
#include "search.hpp"

namespace hpg {

namespace {

double factorial_d(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

struct Opt {
  int dp, pp, tp;
};

// enumerate_layouts (search.cpp:127-150)
std::vector<Opt> layout_options(int group_size, int64_t nl, int max_tp) {
  std::vector<Opt> out;
  for (int dp = 1; dp <= group_size; ++dp) {
    if (group_size % dp != 0) continue;
    const int rest = group_size / dp;
    for (int pp = 1; pp <= rest; ++pp) {
      if (rest % pp != 0) continue;
      const int tp = rest / pp;
      if (pp > nl || tp > max_tp) continue;
      out.push_back({dp, pp, tp});
    }
  }
  return out;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// std::ostream << double with the default flags (precision 6, %g)
std::string g6(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%g", v);
  return buf;
}

}  // namespace

// exhaustive_space_estimate (search.cpp:851-882), same double arithmetic
double exhaustive_space_estimate(const Problem& P, const Knobs& K) {
  const int n = P.N;
  double total = 0.0;
  for (const Grouping& tg : enumerate_task_groupings(P, false)) {
    const int k = static_cast<int>(tg.size());
    if (k > n) continue;
    for (const auto& comp : compositions(n, k, 1)) {
      double medium_ways = factorial_d(n);
      for (int c : comp) medium_ways /= factorial_d(c);
      double per_plan = 1.0;
      for (int g = 0; g < k; ++g) {
        for (int s : tg[g]) {
          const auto opts = layout_options(comp[g], P.tasks[s].nl, P.max_node_size);
          per_plan *= static_cast<double>(std::max<size_t>(1, opts.size())) * factorial_d(comp[g]);
        }
      }
      total += medium_ways * per_plan;
      if (total > K.exhaustive_cap * 1e3) return total;  // far over budget already
    }
  }
  return total;
}

SearchOut exhaustive_search(Ctx& ctx, const Knobs& K) {
  reset_ring_memo(ctx);
  const Problem& P = ctx.prob;
  const double t0 = now_s();
  const int64_t launches0 = ctx.launches, plans0 = ctx.plans_evaluated;
  const double estimate = exhaustive_space_estimate(P, K);
  if (estimate > K.exhaustive_cap) {
    throw InputError("exhaustive search space estimate " + std::to_string(estimate) +
                     " exceeds cap " + std::to_string(K.exhaustive_cap));
  }
  const int n = P.N, T = P.T;
  if (n > kExhMaxDevices)
    throw InputError("engine limit: exhaustive_search supports at most 20 devices");
  // symmetry classes: identical and co-resident devices (search.cpp:897-907)
  uint8_t cls[kExhMaxDevices] = {};
  {
    std::map<std::string, int> ids;
    for (int i = 0; i < n; ++i) {
      const std::string key = P.dev_model[i] + '|' + g6(P.comp_tflops[i]) + '|' +
                              g6(P.mem_gb[i]) + '|' + g6(P.hbm_gbps[i]) + '|' +
                              g6(P.intra_gbps[i]) + '|' + P.dev_node[i] + '|' +
                              P.dev_region[i];
      cls[i] = static_cast<uint8_t>(
          ids.emplace(key, static_cast<int>(ids.size())).first->second);
    }
  }
  const DevCostConfig cfg = K.cost_config();
  Carve cv{};
  cv.n_dev = n;
  cv.n_tasks = T;
  cv.max_w = cv.max_sl = cv.max_slots = cv.max_cells = cv.max_dpk = T * n;
  const int64_t stride = (80 + T * n + 7) & ~int64_t(7);
  // ---- pass 1: the blocks, in enumeration order ----
  struct BlockRef {
    ExhBlock B;
    const Grouping* tg;
    std::vector<int> comp;
    int part_off, part_n;
  };
  std::vector<BlockRef> blocks;
  SearchOut S;
  const auto tgs = enumerate_task_groupings(P, false);
  S.task_groupings = static_cast<int64_t>(tgs.size());
  int64_t raw_total = 0;
  uint64_t max_raw = 0;
  int key_max = 8, parts = 0;
  for (const Grouping& tg : tgs) {
    const int k = static_cast<int>(tg.size());
    if (k > n) continue;
    for (const auto& comp : compositions(n, k, 1)) {
      ExhBlock B{};
      B.n = n;
      B.T = T;
      B.k = k;
      B.fact[0] = 1;
      for (int i = 1; i <= kExhMaxDevices; ++i) B.fact[i] = B.fact[i - 1] * i;
      for (int i = 0; i < n; ++i) B.cls[i] = cls[i];
      bool any_empty = false;
      int t = 0;
      long double raw = 1.0L;
      for (int g = 0; g < k; ++g) {
        B.comp[g] = comp[g];
        for (int s : tg[g]) {
          const auto opts = layout_options(comp[g], P.tasks[s].nl, P.max_node_size);
          if (opts.empty()) any_empty = true;
          if (opts.size() > static_cast<size_t>(kExhMaxOpts))
            throw InputError("engine limit: more than 64 layout options for one task");
          B.order[t] = s;
          B.grp[t] = g;
          B.nopt[t] = static_cast<int32_t>(opts.size());
          for (size_t o = 0; o < opts.size(); ++o) {
            B.opt[t][o][0] = static_cast<int16_t>(opts[o].dp);
            B.opt[t][o][1] = static_cast<int16_t>(opts[o].pp);
            B.opt[t][o][2] = static_cast<int16_t>(opts[o].tp);
          }
          B.perms[t] = B.fact[comp[g]];
          raw *= static_cast<long double>(opts.size()) * static_cast<long double>(B.perms[t]);
          ++t;
        }
      }
      if (any_empty) continue;
      uint64_t mult = B.fact[n];
      for (int g = 0; g < k; ++g) mult /= B.fact[comp[g]];
      B.multinom = mult;
      raw *= static_cast<long double>(mult);
      if (raw > static_cast<long double>(1ull << 25))
        throw InputError("engine limit: exhaustive block exceeds 2^25 raw candidates");
      B.raw = static_cast<uint64_t>(raw);
      int kb = T;
      for (int p = 0; p < T; ++p) kb += 2 * B.comp[B.grp[p]];
      B.key_bytes = (kb + 7) & ~7;
      B.rec_stride = static_cast<int32_t>(stride);
      raw_total += static_cast<int64_t>(B.raw);
      max_raw = std::max(max_raw, B.raw);
      key_max = std::max(key_max, B.key_bytes);
      const int pn = static_cast<int>(
          std::min<uint64_t>(static_cast<uint64_t>(2 * ctx.n_sm), (B.raw + 1023) / 1024));
      blocks.push_back({B, &tg, comp, parts, std::max(1, pn)});
      parts += std::max(1, pn);
    }
  }
  // ---- pass 2: every block queued back to back on the context stream ----
  // (buffers live in the context; stream order makes their reuse safe)
  uint64_t H = 1;
  while (H < 2 * std::max<uint64_t>(max_raw, 1)) H <<= 1;
  DevBuf<uint8_t>& keys = ctx.d_exh_keys;
  DevBuf<uint8_t>& recs = ctx.d_exh_recs;
  DevBuf<unsigned long long>& table = ctx.d_exh_table;
  DevBuf<unsigned long long>& slot = ctx.d_exh_slot;
  DevBuf<unsigned long long>& counts = ctx.d_exh_count;
  DevBuf<EvalResult>& res = ctx.d_exh_res;
  keys.reserve(max_raw * key_max);
  table.reserve(H);
  slot.reserve(max_raw);
  recs.reserve(max_raw * stride);
  res.reserve(max_raw);
  ctx.d_modes.reserve(max_raw);
  counts.reserve(blocks.size() + 1);
  ctx.d_exh_part.reserve(sizeof(ExhPartial) * (parts + 1));
  ExhPartial* part_p = reinterpret_cast<ExhPartial*>(ctx.d_exh_part.p);
  const int64_t scratch = eval_scratch_doubles(n, ctx.max_nl);
  ctx.d_scratch.reserve(static_cast<size_t>(32 * ctx.n_sm) * scratch);
  cudaStream_t st = ctx.stream;
  cuda_check(cudaMemsetAsync(counts.p, 0, 8 * (blocks.size() + 1), st), "memset counts");
  for (size_t bi = 0; bi < blocks.size(); ++bi) {
    const ExhBlock& B = blocks[bi].B;
    const uint64_t R = B.raw;
    uint64_t h = 1;
    while (h < 2 * R) h <<= 1;
    cuda_check(cudaMemsetAsync(table.p, 0xff, h * 8, st), "memset table");
    cuda_check(launch_exh_keys(B, R, keys.p, st), "exh_key_kernel");
    cuda_check(launch_exh_insert(B, R, keys.p, table.p, h - 1, slot.p, st), "exh_insert_kernel");
    cuda_check(launch_exh_reps(B, R, table.p, slot.p, recs.p, ctx.d_modes.p, counts.p + bi, st),
               "exh_rep_kernel");
    int grid = 0;
    cuda_check(eval_grid(cv, static_cast<int>(R), ctx.n_sm, grid), "eval occupancy");
    cuda_check(launch_eval(ctx.dprob, cfg, cv, 0, recs.p, nullptr, ctx.d_modes.p, 0,
                           static_cast<int>(R), stride, nullptr, nullptr, res.p, nullptr, nullptr,
                           ctx.d_scratch.p, scratch, grid, st),
               "eval_kernel");
    cuda_check(launch_exh_reduce(res.p, static_cast<int64_t>(R), part_p + blocks[bi].part_off,
                                 blocks[bi].part_n, st),
               "exh_reduce_kernel");
    ctx.launches += 5;
    ++ctx.eval_launches;
    ctx.plans_evaluated += static_cast<int64_t>(R);
  }
  std::vector<unsigned long long> hc(blocks.size() + 1);
  std::vector<ExhPartial> hp(parts + 1);
  cuda_check(cudaMemcpyAsync(hc.data(), counts.p, 8 * hc.size(), cudaMemcpyDeviceToHost, st),
             "D2H counts");
  if (parts)
    cuda_check(cudaMemcpyAsync(hp.data(), part_p, sizeof(ExhPartial) * parts,
                               cudaMemcpyDeviceToHost, st),
               "D2H partials");
  cuda_check(cudaStreamSynchronize(st), "exhaustive");
  // ---- merge: blocks in enumeration order, strict < keeps the first minimum ----
  int64_t explored = 0;
  double best = kInf;
  int best_block = -1;
  uint64_t best_idx = 0;
  for (size_t bi = 0; bi < blocks.size(); ++bi) {
    explored += static_cast<int64_t>(hc[bi]);
    ExhPartial bb{kInf, ~0ull};
    for (int q = 0; q < blocks[bi].part_n; ++q) {
      const ExhPartial& p = hp[blocks[bi].part_off + q];
      if (p.best < bb.best || (p.best == bb.best && p.best_idx < bb.best_idx)) bb = p;
    }
    if (bb.best_idx != ~0ull && bb.best < best) {
      best = bb.best;
      best_block = static_cast<int>(bi);
      best_idx = bb.best_idx;
    }
  }
  S.consumed = explored;
  S.budget = raw_total;
  if (best_block >= 0) {
    const ExhBlock& BB = blocks[best_block].B;
    int oi[kMaxTasks];
    uint8_t devs[kMaxTasks * kExhMaxDevices];
    exh_decode(BB, best_idx, oi, devs);
    int dp[kMaxTasks], pp[kMaxTasks], tp[kMaxTasks];
    for (int p = 0; p < T; ++p) {
      const int s = BB.order[p];
      dp[s] = BB.opt[p][oi[p]][0];
      pp[s] = BB.opt[p][oi[p]][1];
      tp[s] = BB.opt[p][oi[p]][2];
    }
    Cand c;
    init_cand(c, T, dp, pp, tp, P);
    c.ng = static_cast<int>(blocks[best_block].tg->size());
    for (int p = 0; p < T; ++p) {
      const int s = BB.order[p];
      const int m = BB.comp[BB.grp[p]];
      for (int i = 0; i < m; ++i) c.dev()[c.o.dev[s] + i] = devs[p * n + i];
    }
    S.has_plan = true;
    S.plan = std::move(c);
    S.plan_groups = *blocks[best_block].tg;
    S.plan_counts = blocks[best_block].comp;
    Batch b;
    b.cands.push_back(&S.plan);
    b.modes.push_back(kModeE2E);
    BatchOut bo;
    run_batch(ctx, b, cfg, 0, false, true, false, bo);
    S.per_task = bo.per_task;
    S.reshard_s = bo.res[0].reshard_s;
    S.sync_s = bo.res[0].sync_s;
    S.e2e = bo.res[0].cost;
    S.feasible = (bo.res[0].flags & kResFeasOut) != 0;
    S.est_cost = S.e2e;
    S.prov_budget = 0;  // exhaustive plans keep the default provenance
  }
  S.wall_s = now_s() - t0;
  S.launches = ctx.launches - launches0;
  S.plans_gpu = ctx.plans_evaluated - plans0;
  return S;
}

}  // namespace hpg
