// Host side of the search: enumerations, candidate generation, the per-arm GA
// (coroutines) and the nested successive-halving schedule, executed in
// lockstep waves against eval_kernel. Reference: proj/src/search.cpp,
// proj/src/combinatorics.cpp, proj/include/hetplan/rng.hpp.
#include "search.hpp"
#include "dist_exchange.hpp"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstddef>
#include <chrono>
#include <coroutine>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <set>

#include "eval_launch.hpp"
#include "host_pool.hpp"
#include "rng_jump.hpp"

namespace hpg {

namespace {

int ceil_log2(size_t n) {
  int r = 0;
  size_t v = 1;
  while (v < n) {
    v <<= 1;
    ++r;
  }
  return r;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

DevCostConfig Knobs::cost_config() const {
  hpg_cost_config c = default_cost_config();
  c.recompute = recompute ? 1 : 0;
  c.reshard_override = reshard_override;
  c.sync_override = sync_override;
  return to_dev_cfg(c);
}

Knobs knobs_from_c(const Problem& P, const hpg_knobs& k) {
  Knobs o;
  o.budget = k.budget;
  o.seed = k.seed;
  o.population = k.population;
  o.locality_bias = k.locality_bias;
  o.quantize = k.quantize_gpu_counts;
  o.adjacent = k.level1_filter_adjacent != 0;
  o.level1_cap = k.level1_cap;
  o.gg_arm_cap = k.gg_arm_cap;
  o.swap_pair_sample = k.swap_pair_sample;
  o.balance_data = k.balance_data != 0;
  o.balance_layers = k.balance_layers != 0;
  o.recompute = k.recompute != 0;
  o.reshard_override = k.reshard_override;
  o.sync_override = k.sync_override;
  o.exhaustive_cap = k.exhaustive_cap;
  // parse_knobs_json validation (search.cpp:75-83)
  if (o.population < 1 || o.swap_pair_sample < 0 || o.gg_arm_cap < 1)
    throw InputError("knobs: population and gg_arm_cap must be >= 1");
  if (o.locality_bias < 0 || o.locality_bias > 1)
    throw InputError("knobs: locality_bias must be within [0, 1]");
  if (k.n_tg_override > 0) {
    o.has_tg_override = true;
    for (int i = 0; i < k.n_tg_override; ++i) {
      int ng = 0;
      for (int s = 0; s < P.T; ++s) ng = std::max(ng, k.tg_override[i * P.T + s] + 1);
      Grouping g(ng);
      for (int s = 0; s < P.T; ++s) {
        const int gi = k.tg_override[i * P.T + s];
        if (gi < 0) throw InputError("task grouping must cover every workflow task");
        g[gi].push_back(s);
      }
      for (const auto& grp : g)
        if (grp.empty()) throw InputError("task groups must be non-empty");
      o.tg_override.push_back(std::move(g));
    }
  }
  return o;
}

// ---- enumerations ----

std::vector<Grouping> enumerate_task_groupings(const Problem& P, bool adjacent) {
  // set_partitions in restricted-growth-string order (combinatorics.cpp:10-46)
  const int n = P.T;
  std::vector<Grouping> out;
  std::vector<int> a(n, 0);
  while (true) {
    const int blocks = *std::max_element(a.begin(), a.end()) + 1;
    Grouping g(blocks);
    for (int i = 0; i < n; ++i) g[a[i]].push_back(i);
    bool keep = true;
    if (adjacent) {  // level1_filter "adjacent" (search.cpp:636-656)
      for (const auto& group : g) {
        if (group.size() < 2) continue;
        bool adj = false;
        for (int x : group)
          for (int y : group)
            if (P.dep_edges.count({P.tasks[x].id, P.tasks[y].id})) adj = true;
        if (!adj) keep = false;
      }
    }
    if (keep) out.push_back(std::move(g));
    int i = n - 1;
    for (; i > 0; --i) {
      int prefix_max = 0;
      for (int j = 0; j < i; ++j) prefix_max = std::max(prefix_max, a[j]);
      if (a[i] <= prefix_max) {
        ++a[i];
        std::fill(a.begin() + i + 1, a.end(), 0);
        break;
      }
    }
    if (i == 0) break;
  }
  return out;
}

std::vector<std::vector<int>> compositions(int total, int parts, int quantum) {
  std::vector<std::vector<int>> out;
  if (parts <= 0 || total < parts) return out;
  if (quantum > 1) {
    if (total % quantum != 0) return out;
    out = compositions(total / quantum, parts, 1);
    for (auto& c : out)
      for (auto& v : c) v *= quantum;
    return out;
  }
  std::vector<int> cur;
  std::function<void(int, int)> rec = [&](int remaining, int slots) {
    if (slots == 1) {
      cur.push_back(remaining);
      out.push_back(cur);
      cur.pop_back();
      return;
    }
    for (int v = 1; v <= remaining - (slots - 1); ++v) {
      cur.push_back(v);
      rec(remaining - v, slots - 1);
      cur.pop_back();
    }
  };
  rec(total, parts);
  return out;
}

double composition_count(int total, int parts, int quantum) {
  if (parts <= 0 || total < parts) return 0.0;
  if (quantum > 1) {
    if (total % quantum != 0) return 0.0;
    return composition_count(total / quantum, parts, 1);
  }
  double r = 1.0;
  for (int i = 1; i <= parts - 1; ++i) {
    r = r * static_cast<double>(total - parts + i) / static_cast<double>(i);
  }
  return r;
}

std::vector<int> sample_composition(int total, int parts, int quantum, Rng& rng) {
  if (quantum > 1 && total % quantum == 0 && total / quantum >= parts) {
    auto scaled = sample_composition(total / quantum, parts, 1, rng);
    for (auto& v : scaled) v *= quantum;
    return scaled;
  }
  std::vector<int> cuts;
  while (static_cast<int>(cuts.size()) < parts - 1) {
    const int c = 1 + static_cast<int>(rng.bounded(static_cast<uint64_t>(total - 1)));
    if (std::find(cuts.begin(), cuts.end(), c) == cuts.end()) cuts.push_back(c);
  }
  std::sort(cuts.begin(), cuts.end());
  std::vector<int> comp;
  int prev = 0;
  for (int c : cuts) {
    comp.push_back(c - prev);
    prev = c;
  }
  comp.push_back(total - prev);
  return comp;
}

namespace {

struct Layout {
  int dp, pp, tp;
};

// enumerate_layouts (search.cpp:127-150)
std::vector<Layout> enumerate_layouts(int group_size, int64_t nl, int max_tp) {
  std::vector<Layout> out;
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

// ---- candidate generation (search.cpp:152-234, 318-421) ----

struct ArmLayouts {
  std::vector<int> task_order;                // slots, group order
  std::vector<std::vector<Layout>> options;   // per slot
  bool feasible = true;
};

ArmLayouts build_arm_layouts(const Problem& P, const Grouping& tg, const std::vector<int>& counts) {
  ArmLayouts al;
  al.options.resize(P.T);
  for (size_t g = 0; g < tg.size(); ++g) {
    for (int s : tg[g]) {
      auto opts = enumerate_layouts(counts[g], P.tasks[s].nl, P.max_node_size);
      if (opts.empty()) al.feasible = false;
      al.task_order.push_back(s);
      al.options[s] = std::move(opts);
    }
  }
  return al;
}

void medium_assignment(const Problem& P, double bias, Rng& rng, std::vector<int>& flat) {
  flat.clear();
  const int R = static_cast<int>(P.region_nodes.size());
  int regions[kMaxDevices];
  for (int r = 0; r < R; ++r) regions[r] = r;
  rng.shuffle(regions, R);
  int nodes[kMaxDevices];
  for (int ri = 0; ri < R; ++ri) {
    const auto& rn = P.region_nodes[regions[ri]];
    const int nn = static_cast<int>(rn.size());
    for (int k = 0; k < nn; ++k) nodes[k] = k;
    rng.shuffle(nodes, nn);
    for (int k = 0; k < nn; ++k)
      for (int d : rn[nodes[k]]) flat.push_back(d);
  }
  for (size_t i = flat.size(); i > 1; --i) {
    const bool scramble = rng.uniform() < (1.0 - bias);
    const uint64_t pick = rng.bounded(i);
    if (scramble) std::swap(flat[i - 1], flat[pick]);
  }
}

// random_fine_assignment: node blocks (lexicographic node names) shuffled,
// devices shuffled within a block.
void fine_assignment(const Problem& P, const int* group_devs, int n, Rng& rng, uint8_t* out) {
  // bucket the group's devices by node (insertion order kept), nodes listed
  // in lexicographic name order = ascending node rank
  int cnt[kMaxDevices];
  const int R = P.n_nodes;
  for (int r = 0; r < R; ++r) cnt[r] = 0;
  for (int i = 0; i < n; ++i) ++cnt[P.node_rank[group_devs[i]]];
  int ranks[kMaxDevices], start[kMaxDevices];
  int nr = 0, acc = 0;
  for (int r = 0; r < R; ++r) {
    if (!cnt[r]) continue;
    ranks[nr++] = r;
    start[r] = acc;
    acc += cnt[r];
  }
  int bucket[kMaxDevices], fill[kMaxDevices];
  for (int k = 0; k < nr; ++k) fill[ranks[k]] = start[ranks[k]];
  for (int i = 0; i < n; ++i) bucket[fill[P.node_rank[group_devs[i]]]++] = group_devs[i];
  rng.shuffle(ranks, nr);
  int pos = 0;
  for (int k = 0; k < nr; ++k) {
    int* b = bucket + start[ranks[k]];
    const int nb = cnt[ranks[k]];
    rng.shuffle(b, nb);
    for (int i = 0; i < nb; ++i) out[pos++] = static_cast<uint8_t>(b[i]);
  }
}

struct ArmEnv {
  const Problem& P;
  const Knobs& K;
  const Grouping& tg;
  const std::vector<int>& counts;
  ArmLayouts al;
};

// make_candidate's layout part (decode_layout_combo, search.cpp:283-316): the
// record with its layouts, unit weights and uniform splits, devices unset
void candidate_layouts(const ArmEnv& e, int64_t combo, Cand& c) {
  const Problem& P = e.P;
  int dp[kMaxTasks], pp[kMaxTasks], tp[kMaxTasks];
  for (int s : e.al.task_order) {
    const auto& opts = e.al.options[s];
    const Layout& l = opts[static_cast<size_t>(combo) % opts.size()];
    combo /= static_cast<int64_t>(opts.size());
    dp[s] = l.dp;
    pp[s] = l.pp;
    tp[s] = l.tp;
  }
  init_cand(c, P.T, dp, pp, tp, P);
  c.ng = static_cast<int>(e.tg.size());
}

void make_candidate(const ArmEnv& e, int64_t combo, Rng& rng, Cand& c) {
  const Problem& P = e.P;
  candidate_layouts(e, combo, c);
  std::vector<int> flat;
  flat.reserve(P.N);
  medium_assignment(P, e.K.locality_bias, rng, flat);
  int cursor = 0;
  for (size_t g = 0; g < e.tg.size(); ++g) {
    const int cnt = e.counts[g];
    for (int s : e.tg[g]) fine_assignment(P, flat.data() + cursor, cnt, rng, c.dev() + c.o.dev[s]);
    cursor += cnt;
  }
}

// group_device_set (search.cpp:336-341) is the group's device set sorted by
// device-id string; kept as a bitmask in id-rank space so the idx-th entry is
// a select over four words instead of a sort.
struct RankSet {
  uint64_t w[kMaxDevices / 64];
};

void group_rank_set(const ArmEnv& e, const Cand& c, size_t g, RankSet& rs, int& n) {
  const int s = e.tg[g].front();
  n = c.size(s);
  for (auto& x : rs.w) x = 0;
  const uint8_t* d = c.dev() + c.o.dev[s];
  for (int i = 0; i < n; ++i) {
    const int r = e.P.id_rank[d[i]];
    rs.w[r >> 6] |= 1ull << (r & 63);
  }
}

int select_rank(const ArmEnv& e, const RankSet& rs, uint64_t idx) {
  for (int k = 0; k < kMaxDevices / 64; ++k) {
    const uint64_t pc = static_cast<uint64_t>(__builtin_popcountll(rs.w[k]));
    if (idx >= pc) {
      idx -= pc;
      continue;
    }
    uint64_t x = rs.w[k];
    for (uint64_t i = 0; i < idx; ++i) x &= x - 1;
    return e.P.by_id_rank[64 * k + __builtin_ctzll(x)];
  }
  return -1;
}

bool random_move(const ArmEnv& e, Cand& c, int level, Rng& rng) {
  if (level == 3) {
    const size_t ng = e.tg.size();
    if (ng < 2) return false;
    const size_t g1 = rng.bounded(ng);
    size_t g2 = rng.bounded(ng - 1);
    if (g2 >= g1) ++g2;
    RankSet d1, d2;
    int n1, n2;
    group_rank_set(e, c, g1, d1, n1);
    group_rank_set(e, c, g2, d2, n2);
    // GCC evaluates the two bounded() arguments right to left
    // (search.cpp:378-379): the d2 index is drawn first.
    const int b = select_rank(e, d2, rng.bounded(static_cast<uint64_t>(n2)));
    const int a = select_rank(e, d1, rng.bounded(static_cast<uint64_t>(n1)));
    for (int s : e.tg[g1]) {
      uint8_t* d = c.dev() + c.o.dev[s];
      for (int i = 0; i < c.size(s); ++i)
        if (d[i] == a) {
          d[i] = static_cast<uint8_t>(b);
          break;
        }
    }
    for (int s : e.tg[g2]) {
      uint8_t* d = c.dev() + c.o.dev[s];
      for (int i = 0; i < c.size(s); ++i)
        if (d[i] == b) {
          d[i] = static_cast<uint8_t>(a);
          break;
        }
    }
    return true;
  }
  int eligible[kMaxTasks];
  int ne = 0;
  for (int s = 0; s < e.P.T; ++s)
    if (c.size(s) >= 2) eligible[ne++] = s;
  if (ne == 0) return false;
  const int s = eligible[rng.bounded(static_cast<uint64_t>(ne))];
  const size_t n = static_cast<size_t>(c.size(s));
  const size_t p1 = rng.bounded(n);
  size_t p2 = rng.bounded(n - 1);
  if (p2 >= p1) ++p2;
  uint8_t* d = c.dev() + c.o.dev[s];
  std::swap(d[p1], d[p2]);
  return true;
}

bool mutate(const ArmEnv& e, Cand& c, Rng& rng) {
  const bool has_l3 = e.tg.size() >= 2;
  bool has_l5 = false;
  for (int s = 0; s < e.P.T; ++s)
    if (c.size(s) >= 2) has_l5 = true;
  if (!has_l3 && !has_l5) return false;
  int level;
  if (has_l3 && has_l5) {
    level = rng.bounded(2) == 0 ? 3 : 5;
  } else {
    level = has_l3 ? 3 : 5;
  }
  return random_move(e, c, level, rng);
}

// ---- coroutine plumbing ----

struct EvalReq {
  std::vector<Cand> cands;
  std::vector<EvalResult> res;
  // init chunk: `gen_count` new candidates (combinations gen_combo0...) drawn
  // from gen_rng, generated by the scheduler (host or device); gen_snaps[c] =
  // the stream state after candidate c
  bool gen = false;
  const ArmEnv* env = nullptr;
  Rng gen_rng;
  int64_t gen_combo0 = 0;
  int gen_count = 0;
  std::vector<Rng> gen_snaps;
  std::vector<Rng> gen_starts;  // device generation: each candidate's start state
};

// the generator's view of an arm: groups, counts and the fine-assignment
// order of make_candidate (task slots group by group)
GenItem gen_item_of(const ArmEnv& e) {
  GenItem it{};
  it.bias = e.K.locality_bias;
  it.n_groups = static_cast<int32_t>(e.tg.size());
  int no = 0;
  for (size_t g = 0; g < e.tg.size(); ++g) {
    it.counts[g] = e.counts[g];
    for (int s : e.tg[g]) {
      it.order_slot[no] = static_cast<int8_t>(s);
      it.order_group[no] = static_cast<int8_t>(g);
      ++no;
    }
  }
  it.n_order = no;
  return it;
}

struct ArmCoro {
  struct promise_type {
    EvalReq* pending = nullptr;
    std::exception_ptr exc;
    ArmCoro get_return_object() {
      return ArmCoro{std::coroutine_handle<promise_type>::from_promise(*this)};
    }
    std::suspend_always initial_suspend() noexcept { return {}; }
    std::suspend_always final_suspend() noexcept { return {}; }
    void return_void() {}
    void unhandled_exception() { exc = std::current_exception(); }
  };
  std::coroutine_handle<promise_type> h;
  ArmCoro() = default;
  explicit ArmCoro(std::coroutine_handle<promise_type> hh) : h(hh) {}
  ArmCoro(ArmCoro&& o) noexcept : h(o.h) { o.h = nullptr; }
  ArmCoro& operator=(ArmCoro&& o) noexcept {
    if (h) h.destroy();
    h = o.h;
    o.h = nullptr;
    return *this;
  }
  ~ArmCoro() {
    if (h) h.destroy();
  }
};

struct EvalAwait {
  EvalReq* req;
  bool await_ready() const noexcept { return false; }
  void await_suspend(std::coroutine_handle<ArmCoro::promise_type> h) noexcept {
    h.promise().pending = req;
  }
  void await_resume() const noexcept {}
};

struct Improvement {
  int64_t local_idx;  // 1-based evaluation index inside the run
  double cost;
  Cand plan;
  double t_wall;
};

struct Member {
  Cand plan;
  double cost;
  uint64_t seq;
};

struct ArmRun {
  int64_t ti = 0, gi = 0;
  int64_t slice = 0;
  Rng rng;
  int64_t used = 0;
  double best = kInf;
  std::vector<Improvement> impr;
  // ga_search result (best inserted member, search.cpp:464-469)
  bool has_best_member = false;
  Cand best_member;
  double best_member_cost = kInf;
  std::unique_ptr<ArmEnv> env;
  ArmCoro coro;
  double* clock = nullptr;
  int owner = 0;  // rank that runs it (multi-GPU)
  int64_t n_offspring = 0, n_spec_hit = 0;  // diagnostics
  double t_make = 0, t_mut = 0, t_swap = 0, t_spec = 0;  // diagnostics (s)
  int64_t w_init = 0, w_mut = 0, w_swap = 0, w_redraw = 0;  // diagnostics: waves by kind
  int64_t n_make = 0;
  // population (ga_run's locals, kept here so the device can take over)
  std::vector<Member> pop;
  uint64_t seq = 0;
  bool device_ga = false;  // hand the offspring loop to ga_kernel after init
  bool handoff = false;
};

// ga_run (search.cpp:437-565) as a coroutine.
ArmCoro ga_run(ArmRun& run) {
  ArmEnv& e = *run.env;
  const Knobs& K = e.K;
  Rng& rng = run.rng;
  const int64_t slice = run.slice;
  if (slice <= 0) co_return;
  if (!e.al.feasible) co_return;
  if (run.device_ga) {  // the whole run goes to the device (ga_kernel.cuh)
    run.handoff = true;
    co_return;
  }
  std::vector<Member>& pop = run.pop;
  uint64_t& seq = run.seq;
  auto score = [&](const Cand& c, double cost) {
    ++run.used;
    if (cost < run.best) {
      run.best = cost;
      run.impr.push_back({run.used, cost, c, *run.clock});
    }
  };
  auto insert_member = [&](const Cand& plan, double cost) {
    if (cost < run.best_member_cost) {
      run.best_member_cost = cost;
      run.best_member = plan;
      run.has_best_member = true;
    }
    Member m{plan, cost, seq++};
    auto pos = std::upper_bound(pop.begin(), pop.end(), m, [](const Member& a, const Member& b) {
      return a.cost != b.cost ? a.cost < b.cost : a.seq < b.seq;
    });
    pop.insert(pos, std::move(m));
    if (static_cast<int>(pop.size()) > K.population) pop.pop_back();
  };
  EvalReq req;
  std::vector<Rng> snaps, snaps5;

  // init: cycle layout combinations (speculative chunks, one wave each)
  const int64_t init_target =
      std::max<int64_t>(1, std::min({slice, static_cast<int64_t>(K.population), slice / 2}));
  const int64_t attempt_cap = 64 + 16 * init_target;
  int64_t attempts = 0, combo = 0, chunk = 0;
  while (static_cast<int64_t>(pop.size()) < init_target && run.used < slice &&
         attempts < attempt_cap) {
    const int64_t need = init_target - static_cast<int64_t>(pop.size());
    chunk = std::min(attempt_cap - attempts, std::max(chunk * 2, 2 * need + 2));
    // the scheduler makes the chunk (make_candidate x chunk from this stream
    // position, on the device when the wave is wide) and returns the stream
    // state after each candidate
    req.cands.clear();
    req.gen = true;
    req.env = &e;
    req.gen_rng = rng;
    req.gen_combo0 = combo;
    req.gen_count = static_cast<int>(chunk);
    run.n_make += chunk;
    ++run.w_init;  // diagnostics
    co_await EvalAwait{&req};
    req.gen = false;
    const int64_t combo0 = combo;
    combo += chunk;
    rng = req.gen_snaps.back();
    for (int64_t c = 0; c < chunk; ++c) {
      ++attempts;
      if (!(req.res[c].flags & kResFeasIn)) continue;
      score(req.cands[c], req.res[c].cost);
      insert_member(req.cands[c], req.res[c].cost);
      if (static_cast<int64_t>(pop.size()) >= init_target) {
        rng = req.gen_snaps[c];
        combo = combo0 + c + 1;
        break;
      }
    }
  }
  if (pop.empty()) co_return;

  // offspring generations. Each offspring is a mutation wave (up to 8 trials
  // and the unmutated parent, first feasible trial wins) followed by a swap
  // wave. The next offspring's mutation stage depends on this offspring only
  // through the RNG position and the population after insertion; both are
  // known in advance when the swap walk accepts nothing, so its trials ride
  // along in the swap wave and are used only if that turns out to hold
  // (exact: the RNG state is compared, everything else follows from it).
  struct MutStage {
    std::vector<Cand> cands;  // ntr trials + the unmutated parent
    std::vector<EvalResult> res;
    std::vector<Rng> snaps;
    Rng start, after_all;
    int ntr = 0;
  };
  // draws the trials (+ the parent) straight into `out`; m keeps the snapshots
  auto draw_mut = [&](Rng r, const Cand& parent, MutStage& m, std::vector<Cand>& out) {
    m.snaps.clear();
    m.ntr = 0;
    for (int tries = 0; tries < 8; ++tries) {
      out.push_back(parent);
      if (!mutate(e, out.back(), r)) {
        out.pop_back();
        break;
      }
      m.snaps.push_back(r);
      ++m.ntr;
    }
    m.after_all = r;
    out.push_back(parent);
  };
  // speculative next mutation stage from RNG state r, assuming (child, cost)
  // is inserted as it stands; appended to req after index base
  MutStage spec;
  auto speculate = [&](const Rng& r, const Cand& ch, double ch_cost) {
    const bool ins =
        static_cast<int>(pop.size()) < K.population || ch_cost < pop.back().cost;
    size_t pos = pop.size(), n_spec = pop.size();
    if (ins) {
      pos = 0;
      while (pos < pop.size() && !(pop[pos].cost > ch_cost)) ++pos;
      n_spec = std::min(pop.size() + 1, static_cast<size_t>(K.population));
    }
    Rng rr = r;
    const size_t i = static_cast<size_t>(rr.bounded(n_spec));
    const Cand& parent = !ins || i < pos ? pop[i].plan : (i == pos ? ch : pop[i - 1].plan);
    draw_mut(rr, parent, spec, req.cands);
    spec.start = r;
  };
  auto same_rng = [](const Rng& a, const Rng& b) {
    return a.seed == b.seed && a.s[0] == b.s[0] && a.s[1] == b.s[1] && a.s[2] == b.s[2] &&
           a.s[3] == b.s[3];
  };
  MutStage cur;
  bool have_spec = false;
  int64_t streak = 0;
  while (run.used < slice && streak < 64) {
    ++run.n_offspring;
    if (have_spec && same_rng(spec.start, rng)) {
      ++run.n_spec_hit;
      std::swap(cur, spec);
    } else {
      Rng r = rng;
      const size_t i = static_cast<size_t>(r.bounded(pop.size()));
      req.cands.clear();
      const double tu0 = now_s();
      draw_mut(r, pop[i].plan, cur, req.cands);
      run.t_mut += now_s() - tu0;
      ++run.w_mut;  // diagnostics
      co_await EvalAwait{&req};
      cur.res = req.res;
      cur.cands = std::move(req.cands);
    }
    have_spec = false;
    const int ntr = cur.ntr;
    int chosen = -1;
    for (int i = 0; i < ntr; ++i) {
      if (cur.res[i].flags & kResFeasIn) {
        chosen = i;
        break;
      }
    }
    Cand child;
    double cost;
    if (chosen >= 0) {
      rng = cur.snaps[chosen];
      child = std::move(cur.cands[chosen]);
      cost = cur.res[chosen].cost;
    } else {
      rng = cur.after_all;
      if (!(cur.res[ntr].flags & kResFeasIn)) {
        ++streak;
        continue;
      }
      child = std::move(cur.cands[ntr]);
      cost = cur.res[ntr].cost;
    }
    streak = 0;
    score(child, cost);
    // improving swaps, first improvement per level (search.cpp:534-558).
    // Both levels' trials are drawn from the current child and scored in one
    // wave; the level-5 set stays valid unless a level-3 trial is accepted
    // (then level 5 is redrawn from the new child, as the reference does).
    // walk(): the sequential trial loop over already-scored trials
    // [b, b+n); returns 1 accepted, 2 budget stop, 0 ran out.
    auto walk = [&](int b, int n, const Rng& before, const std::vector<Rng>& sn) {
      for (int t = 0; t < n; ++t) {
        if (run.used >= slice) {
          rng = t == 0 ? before : sn[t - 1];
          return 2;
        }
        if (!(req.res[b + t].flags & kResFeasIn)) continue;
        const double c2 = req.res[b + t].cost;
        score(req.cands[b + t], c2);
        if (c2 < cost) {
          child = std::move(req.cands[b + t]);
          cost = c2;
          rng = sn[t];
          return 1;
        }
      }
      if (n > 0) rng = sn.back();
      return 0;
    };
    auto draw = [&](int level, std::vector<Rng>& sn) {
      int ng = 0;
      for (int t = 0; t < K.swap_pair_sample; ++t) {
        Cand cand = child;
        if (!random_move(e, cand, level, rng)) break;
        req.cands.push_back(std::move(cand));
        sn.push_back(rng);
        ++ng;
      }
      return ng;
    };
    // keeps the speculative stage at req[base...] if the walk accepted nothing
    auto take_spec = [&](int base, int w) {
      if (w != 0) return;
      const int ns = spec.ntr + 1;
      spec.res.assign(req.res.begin() + base, req.res.begin() + base + ns);
      spec.cands.resize(ns);
      for (int k = 0; k < ns; ++k) spec.cands[k] = std::move(req.cands[base + k]);
      have_spec = true;
    };
    if (run.used < slice) {
      req.cands.clear();
      snaps.clear();
      snaps5.clear();
      const Rng before3 = rng;
      const double ts0 = now_s();
      const int n3 = draw(3, snaps);
      const Rng before5 = rng;
      const int n5 = draw(5, snaps5);
      run.t_swap += now_s() - ts0;
      if (n3 + n5 > 0) {
        const int base = static_cast<int>(req.cands.size());
        const double tp0 = now_s();
        speculate(n5 > 0 ? snaps5.back() : before5, child, cost);
        run.t_spec += now_s() - tp0;
        ++run.w_swap;  // diagnostics
        co_await EvalAwait{&req};
        rng = before5;  // stream position after the level-3 draws (walk may rewind it)
        const int w3 = walk(0, n3, before3, snaps);
        if (w3 == 0 && run.used < slice) {
          rng = before5;
          take_spec(base, walk(n3, n5, before5, snaps5));
        } else if (w3 == 1 && run.used < slice) {
          req.cands.clear();
          snaps5.clear();
          const Rng b5 = rng;
          const int m5 = draw(5, snaps5);
          if (m5 > 0) {
            const int base5 = static_cast<int>(req.cands.size());
            speculate(snaps5.back(), child, cost);
            ++run.w_redraw;  // diagnostics
            co_await EvalAwait{&req};
            take_spec(base5, walk(0, m5, b5, snaps5));
          }
        }
      } else {
        rng = before5;
      }
    }
    if (static_cast<int>(pop.size()) < K.population || cost < pop.back().cost) {
      insert_member(child, cost);
    }
  }
}

// ga_run of every run of a lockstep round on the device, in one persistent
// launch (ga_kernel.cuh): init chunks, offspring, speculation. The host
// hands over the arm (layout options, groups, RNG stream, slice) and gets
// back the run's budget use, best, improvements and best member, exactly as
// the coroutine would have left them.
bool device_ga_enabled(const Knobs& K) {
  static const int env = [] {
    const char* v = std::getenv("HPG_DEVICE_GA");  // 0 = host GA (lockstep waves)
    return v ? std::atoi(v) : 1;
  }();
  return env != 0 && K.population >= 1 && K.population <= kGaMaxPop &&
         K.swap_pair_sample >= 0 && K.swap_pair_sample <= kGaMaxSps;
}

void device_ga(Ctx& ctx, const Knobs& K, const std::vector<ArmRun*>& runs, double& clock,
               int64_t& waves) {
  const int n = static_cast<int>(runs.size());
  if (n == 0) return;
  const double t_prep0 = now_s();
  const Problem& P = ctx.prob;
  const DevCostConfig cfg = K.cost_config();
  const GenTablesDev& gt = gen_tables(ctx);
  const int kb = (K.balance_data ? 1 : 0) | (K.balance_layers ? 2 : 0);
  const int pop_cap = K.population, sps = K.swap_pair_sample;
  const int max_wave = 2 * sps + kGaTrials + 1;
  std::vector<int> nodes_per_region;
  for (const auto& rn : P.region_nodes) nodes_per_region.push_back(static_cast<int>(rn.size()));
  // per run: layout options, record bound, init sizes; shared slot stride
  Carve cv{};
  cv.n_dev = P.N;
  cv.n_tasks = P.T;
  int stride = 16;
  int init_cap = 1;
  int64_t remaining = 0;
  std::vector<short4> opts;
  std::vector<Poly256> jumps;
  std::map<int32_t, int32_t> jump_at;  // gen_draws -> first polynomial
  // the host writes (and ships) only a run's head: its set-up fields, the GA
  // scalars and the population slot map; the population costs, mutation /
  // speculation stages and swap snapshots behind it are written by the
  // device before they are read
  constexpr size_t kRunHead = offsetof(GaRun, pop_cost);
  std::unique_ptr<GaRun[]> gr(new GaRun[static_cast<size_t>(std::max(n, 1))]);
  // pass 1 (host pool): per run, its layout-option count, draw count per
  // candidate and record bounds
  struct RunPrep {
    int64_t n_opts = 0, gen_draws = 0;
    int mw = 0, msl = 0, mslots = 0, mcells = 0, mdpk = 0, mrec = 0;
  };
  std::vector<RunPrep> rp(n);
  host_parallel_for(n, n >= 64, [&](int i) {
    const ArmEnv& e = *runs[i]->env;
    RunPrep& q = rp[i];
    for (size_t gi = 0; gi < e.tg.size(); ++gi) {
      for (int s : e.tg[gi]) {
        int xdp = 0, xpp = 0, xcell = 0, xdpk = 0, xrec = 0;
        for (const Layout& l : e.al.options[s]) {
          xdp = std::max(xdp, l.dp);
          xpp = std::max(xpp, l.pp);
          xcell = std::max(xcell, l.dp * l.pp);
          xdpk = std::max(xdpk, l.pp * l.tp);
          xrec = std::max(xrec, 8 * l.dp + 4 * l.pp);
        }
        q.n_opts += static_cast<int64_t>(e.al.options[s].size());
        q.mw += xdp;
        q.msl += xpp;
        q.mcells += xcell;
        q.mdpk += xdpk;
        q.mrec += xrec;
        q.mslots += e.counts[gi];
      }
    }
    q.gen_draws = gen_draws_per_candidate(P.N, nodes_per_region.data(),
                                          static_cast<int>(nodes_per_region.size()), gen_item_of(e));
  });
  // round-wide bounds, option offsets, jump tables per distinct draw count
  // (first-appearance order; the tables themselves built in parallel)
  std::vector<int64_t> opt_base(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    const RunPrep& q = rp[i];
    opt_base[i + 1] = opt_base[i] + q.n_opts;
    stride = std::max(stride, (static_cast<int>(sizeof(RecHeader)) + q.mrec + q.mslots + 15) & ~15);
    cv.max_w = std::max(cv.max_w, q.mw);
    cv.max_sl = std::max(cv.max_sl, q.msl);
    cv.max_slots = std::max(cv.max_slots, q.mslots);
    cv.max_cells = std::max(cv.max_cells, q.mcells);
    cv.max_dpk = std::max(cv.max_dpk, q.mdpk);
    remaining += runs[i]->slice;
  }
  std::vector<int64_t> ds;
  for (int i = 0; i < n; ++i)
    if (jump_at.emplace(static_cast<int32_t>(rp[i].gen_draws), 0).second) ds.push_back(rp[i].gen_draws);
  std::vector<JumpTable> tables(ds.size());
  host_parallel_for(static_cast<int>(ds.size()), ds.size() >= 2, [&](int i) {
    tables[i] = jump_table(static_cast<uint64_t>(ds[i]), kGaJumps);
  });
  for (size_t i = 0; i < ds.size(); ++i) {
    // x^(L*D) for L = 1..127: lane offsets and strides of a team of four
    jump_at[static_cast<int32_t>(ds[i])] = static_cast<int32_t>(jumps.size());
    jumps.insert(jumps.end(), tables[i]->begin(), tables[i]->begin() + kGaJumps);
  }
  opts.resize(static_cast<size_t>(opt_base[n]));
  // pass 2 (host pool): the GaRun of every run and its layout options
  host_parallel_for(n, n >= 64, [&](int i) {
    const ArmRun& r = *runs[i];
    const ArmEnv& e = *r.env;
    GaRun& g = gr[i];
    std::memset(static_cast<void*>(&g), 0, kRunHead);
    g.slice = r.slice;
    g.ng = static_cast<int32_t>(e.tg.size());
    g.opt_base = opt_base[i];
    int k = 0;
    int64_t at = opt_base[i];
    for (size_t gi = 0; gi < e.tg.size(); ++gi) {
      g.gstart[gi] = k;
      g.counts[gi] = e.counts[gi];
      for (int s : e.tg[gi]) {
        g.gslot[k] = s;
        g.opt_off[k] = static_cast<int32_t>(at - g.opt_base);
        for (const Layout& l : e.al.options[s])
          opts[at++] = make_short4(static_cast<short>(l.dp), static_cast<short>(l.pp),
                                   static_cast<short>(l.tp), 0);
        ++k;
      }
    }
    g.gstart[e.tg.size()] = k;
    g.opt_off[k] = static_cast<int32_t>(at - g.opt_base);
    g.gen_draws = static_cast<int32_t>(rp[i].gen_draws);
    g.jump_off = jump_at.at(g.gen_draws);
    const int64_t it = std::max<int64_t>(
        1, std::min({r.slice, static_cast<int64_t>(K.population), r.slice / 2}));
    g.init_target = static_cast<int32_t>(it);
    g.attempt_cap = 64 + 16 * it;
    g.rng = r.rng;
    g.best = kInf;
    g.best_member_cost = kInf;
    g.state = kGaInit;
    for (int m = 0; m < pop_cap; ++m) g.pop_slot[m] = 2 + m;
  });
  for (int i = 0; i < n; ++i) init_cap = std::max<int>(init_cap, static_cast<int>(gr[i].attempt_cap));
  const int res_per_run = std::max(2 * max_wave, init_cap);
  const int64_t gen_bytes =
      (2 * (gt.n_regions + gt.max_nodes_per_region + 4 * gt.n_nodes) + 2 * gt.n_dev + 15) & ~15;
  const int n_slots = 2 + pop_cap + res_per_run;
  const int64_t run_bytes = static_cast<int64_t>(n_slots) * stride;
  for (int i = 0; i < n; ++i) {
    gr[i].pool_off = run_bytes * i;
    gr[i].rec_stride = stride;
  }
  // work ring: at most one wave per run in flight plus the idle workers' tickets
  const int max_workers = 16 * ctx.n_sm;
  const int64_t want_q = 2 * (static_cast<int64_t>(n) * (res_per_run + 1) + 4 * max_workers);
  uint64_t q_cap = 1024;
  while (static_cast<int64_t>(q_cap) < want_q) q_cap <<= 1;
  // improvements: every evaluation can improve its run's best, so the device
  // list is sized by the round's budget (32 B per unit in HBM); the pinned
  // host staging holds only a bounded prefix (a round usually records a few
  // per run) and a longer list is read into pageable memory
  const int64_t impr_cap = std::max<int64_t>(1, remaining);
  const int64_t impr_pre = std::min<int64_t>(impr_cap, 8 * static_cast<int64_t>(n) + 64);
  auto al = [](int64_t x) { return (x + 255) & ~int64_t(255); };
  const int64_t o_runs = 0, o_pool = al(o_runs + static_cast<int64_t>(sizeof(GaRun)) * n),
                o_res = al(o_pool + run_bytes * n),
                o_qpay = al(o_res + static_cast<int64_t>(sizeof(EvalResult)) * n * res_per_run),
                o_qseq = al(o_qpay + 8 * static_cast<int64_t>(q_cap)),
                o_ctl = al(o_qseq + 8 * static_cast<int64_t>(q_cap)),
                o_impr = al(o_ctl + 8 * kGaCtlWords),
                o_rank = al(o_impr + static_cast<int64_t>(sizeof(GaImpr)) * impr_cap),
                o_opts = al(o_rank + 8 * 256),
                o_snaps = al(o_opts + 8 * static_cast<int64_t>(opts.size())),
                o_gscr = al(o_snaps + static_cast<int64_t>(sizeof(Rng)) * n * init_cap),
                o_jump = al(o_gscr + static_cast<int64_t>(max_workers) * 32 * gen_bytes),
                d_total = al(o_jump + 32 * static_cast<int64_t>(jumps.size()));
  // one generous allocation per context (reallocating inside a search is slow)
  ctx.d_ga.reserve(std::max<int64_t>(d_total, int64_t{512} << 20));
  uint8_t* D = ctx.d_ga.p;
  // host staging: [runs | ctl | ranks | queue seeds | options], results reuse it
  const int64_t h_runs = 0, h_ctl = al(sizeof(GaRun) * static_cast<int64_t>(n)),
                h_rank = al(h_ctl + 8 * kGaCtlWords), h_qpay = al(h_rank + 8 * 256),
                h_qseq = al(h_qpay + 8 * static_cast<int64_t>(n)),
                h_opts = al(h_qseq + 8 * static_cast<int64_t>(n)),
                h_jump = al(h_opts + 8 * static_cast<int64_t>(opts.size())),
                h_best = al(h_jump + 32 * static_cast<int64_t>(jumps.size())),
                h_imp = al(h_best + 2 * static_cast<int64_t>(stride) * n),
                h_total = al(h_imp + static_cast<int64_t>(sizeof(GaImpr)) * impr_pre);
  // staging sized generously once per context: pinned allocations are slow
  ctx.h_ga.reserve(std::max<int64_t>(h_total, int64_t{32} << 20));
  uint8_t* H = ctx.h_ga.p;
  for (int i = 0; i < n; ++i)
    std::memcpy(H + h_runs + static_cast<int64_t>(sizeof(GaRun)) * i, &gr[i], kRunHead);
  GaRun* hr = reinterpret_cast<GaRun*>(H + h_runs);
  unsigned long long* hctl = reinterpret_cast<unsigned long long*>(H + h_ctl);
  std::memset(hctl, 0, 8 * kGaCtlWords);
  hctl[kGaCtlTail] = static_cast<unsigned long long>(n);
  int32_t* hrank = reinterpret_cast<int32_t*>(H + h_rank);
  for (int d = 0; d < 256; ++d) {
    hrank[d] = d < P.N ? P.id_rank[d] : 0;
    hrank[256 + d] = d < P.N ? P.by_id_rank[d] : 0;
  }
  uint2* hq = reinterpret_cast<uint2*>(H + h_qpay);
  unsigned long long* hs = reinterpret_cast<unsigned long long*>(H + h_qseq);
  for (int i = 0; i < n; ++i) {
    hq[i] = make_uint2(static_cast<unsigned>(i), 0xffffffffu);
    hs[i] = static_cast<unsigned long long>(i) + 1;
  }
  std::memcpy(H + h_opts, opts.data(), 8 * opts.size());
  std::memcpy(H + h_jump, jumps.data(), 32 * jumps.size());
  cudaStream_t st = ctx.stream;
  cuda_check(cudaMemcpy2DAsync(D + o_runs, sizeof(GaRun), H + h_runs, sizeof(GaRun), kRunHead, n,
                               cudaMemcpyHostToDevice, st), "H2D ga runs");
  cuda_check(cudaMemcpyAsync(D + o_ctl, H + h_ctl, 8 * kGaCtlWords, cudaMemcpyHostToDevice, st), "H2D ga ctl");
  cuda_check(cudaMemcpyAsync(D + o_rank, H + h_rank, 8 * 256, cudaMemcpyHostToDevice, st), "H2D ga ranks");
  cuda_check(cudaMemsetAsync(D + o_qseq, 0, 8 * q_cap, st), "ga queue clear");
  cuda_check(cudaMemcpyAsync(D + o_qpay, H + h_qpay, 8 * n, cudaMemcpyHostToDevice, st), "H2D ga queue");
  cuda_check(cudaMemcpyAsync(D + o_qseq, H + h_qseq, 8 * n, cudaMemcpyHostToDevice, st), "H2D ga queue");
  if (!opts.empty())
    cuda_check(cudaMemcpyAsync(D + o_opts, H + h_opts, 8 * opts.size(), cudaMemcpyHostToDevice, st),
               "H2D ga layout options");
  cuda_check(cudaMemcpyAsync(D + o_jump, H + h_jump, 32 * jumps.size(), cudaMemcpyHostToDevice, st),
             "H2D ga jump polynomials");
  GaParams G{};
  G.runs = reinterpret_cast<GaRun*>(D + o_runs);
  G.n_runs = n;
  G.pop_cap = pop_cap;
  G.sps = sps;
  G.max_wave = max_wave;
  G.pool = D + o_pool;
  G.res = reinterpret_cast<EvalResult*>(D + o_res);
  G.id_rank = reinterpret_cast<const int32_t*>(D + o_rank);
  G.by_id_rank = reinterpret_cast<const int32_t*>(D + o_rank) + 256;
  G.q_pay = reinterpret_cast<uint2*>(D + o_qpay);
  G.q_seq = reinterpret_cast<unsigned long long*>(D + o_qseq);
  G.q_mask = q_cap - 1;
  G.ctl = reinterpret_cast<unsigned long long*>(D + o_ctl);
  G.impr = reinterpret_cast<GaImpr*>(D + o_impr);
  G.impr_cap = impr_cap;
  G.kb_flags = kb;
  G.n_tasks = P.T;
  G.max_stride = stride;
  static const int split_env = [] {
    const char* e = std::getenv("HPG_GA_SPLIT_RUNS");  // diagnostics: live-run threshold
    return e ? std::atoi(e) : -1;
  }();
  G.split_runs = split_env;  // -1: grid / 16 (launch_ga_offspring)
  G.opts = reinterpret_cast<const short4*>(D + o_opts);
  G.init_snaps = reinterpret_cast<Rng*>(D + o_snaps);
  G.jumps = reinterpret_cast<const uint64_t*>(D + o_jump);
  G.gen_scratch = D + o_gscr;
  G.init_cap = init_cap;
  G.res_per_run = res_per_run;
  // interleaved per-lane generation scratch: int16 regions | nodes | 4 x nodes,
  // uint8 flat | bucket; in shared memory when the evaluation carve holds it
  G.gen_smem = 2 * (gt.n_regions + gt.max_nodes_per_region + 4 * gt.n_nodes) + 2 * gt.n_dev;
  {
    Carve c1 = cv;
    c1.cls_smem = 0;
    c1.n_warps = 1;
    G.gen_in_smem = 32 * G.gen_smem <= carve2_bytes(c1) ? 1 : 0;
  }
  G.n_regions = gt.n_regions;
  G.n_nodes = gt.n_nodes;
  G.max_nodes_per_region = gt.max_nodes_per_region;
  G.n_dev = gt.n_dev;
  G.bias = K.locality_bias;
  G.region_off = gt.region_off;
  G.node_off = gt.node_off;
  G.node_devs = gt.node_devs;
  G.node_rank = gt.node_rank;
  for (int t = 0; t < P.T; ++t) G.task_nl[t] = P.tasks[t].nl;
  static const char* ga_log = std::getenv("HPG_GA_LOG");  // diagnostics only
  G.prof = ga_log ? 1 : 0;
  const int64_t scratch = eval_scratch_doubles(P.N, ctx.max_nl);
  ctx.d_scratch.reserve(static_cast<size_t>(32 * ctx.n_sm) * scratch);
  const int64_t h2d = static_cast<int64_t>(kRunHead) * n + 8 * kGaCtlWords + 8 * 256 +
                      16 * static_cast<int64_t>(n) + 8 * static_cast<int64_t>(opts.size()) +
                      32 * static_cast<int64_t>(jumps.size());
  const double t_launch = now_s();
  cuda_check(cudaEventRecord(ctx.ev0, st), "event");
  int grid = 0;
  // diagnostics (HPG_GA_LOG): the evaluation phase accumulators run inside
  // the GA kernel too (one shared dummy per-plan slot block)
  static long long* d_prof_dummy = nullptr;
  if (ga_log) {
    if (!d_prof_dummy) cuda_check(cudaMalloc(&d_prof_dummy, sizeof(long long) * 64), "profile alloc");
    cuda_check(eval_set_plan_profile(d_prof_dummy), "profile symbol");
  }
  cuda_check(launch_ga_offspring(ctx.dprob, cfg, cv, G, ctx.d_scratch.p, scratch, ctx.n_sm, grid, st),
             "ga_kernel launch");
  if (grid > max_workers) throw InternalError("ga_kernel grid exceeds its scratch");
  cuda_check(cudaEventRecord(ctx.ev1, st), "event");
  ++ctx.launches;
  ++ctx.eval_launches;
  // results: run states and control words, the two kept plans per run, then
  // the improvements
  // only the run summary the host reads (used, best, counters, flags): the
  // GaRun prefix before the population and stage state
  constexpr size_t kRunSummary = offsetof(GaRun, pop_slot);
  cuda_check(cudaMemcpy2DAsync(H + h_runs, sizeof(GaRun), D + o_runs, sizeof(GaRun), kRunSummary, n,
                               cudaMemcpyDeviceToHost, st), "D2H ga runs");
  cuda_check(cudaMemcpyAsync(H + h_ctl, D + o_ctl, 8 * kGaCtlWords, cudaMemcpyDeviceToHost, st), "D2H ga ctl");
  cuda_check(cudaMemcpy2DAsync(H + h_best, 2 * stride, D + o_pool, run_bytes, 2 * stride, n,
                               cudaMemcpyDeviceToHost, st), "D2H ga best plans");
  // improvements: the bounded prefix rides in the same batch; only a longer
  // list costs a second round trip
  cuda_check(cudaMemcpyAsync(H + h_imp, D + o_impr, sizeof(GaImpr) * impr_pre,
                             cudaMemcpyDeviceToHost, st), "D2H ga improvements");
  cuda_check(cudaStreamSynchronize(st), "ga_kernel");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx.ev0, ctx.ev1);
  ctx.eval_ms += ms;
  const int64_t n_impr = static_cast<int64_t>(hctl[kGaCtlImpr]);
  if (n_impr > impr_cap) throw InternalError("device GA improvement list overflow");
  std::vector<GaImpr> imp(reinterpret_cast<GaImpr*>(H + h_imp),
                          reinterpret_cast<GaImpr*>(H + h_imp) + std::min(n_impr, impr_pre));
  if (n_impr > impr_pre) {
    imp.resize(static_cast<size_t>(n_impr));
    cuda_check(cudaMemcpy(imp.data() + impr_pre, D + o_impr + sizeof(GaImpr) * impr_pre,
                          sizeof(GaImpr) * (n_impr - impr_pre), cudaMemcpyDeviceToHost),
               "D2H ga improvements");
  }
  ctx.plans_evaluated += static_cast<int64_t>(hctl[kGaCtlEvals]);
  ctx.canonical_bytes += static_cast<int64_t>(hctl[kGaCtlBytes]);
  ctx.h2d_bytes += h2d;
  ctx.d2h_bytes += static_cast<int64_t>(offsetof(GaRun, pop_slot)) * n + 8 * kGaCtlWords +
                   2 * static_cast<int64_t>(stride) * n +
                   static_cast<int64_t>(sizeof(GaImpr)) * std::max(n_impr, impr_pre);
  const unsigned long long t0_dev = hctl[kGaCtlT0];
  auto cand_at = [&](const uint8_t* rec, int ng) {
    Cand c;
    const int32_t bytes = *reinterpret_cast<const int32_t*>(rec);
    c.rec.assign(rec, rec + bytes);
    rec_offsets(c.hdr(), c.o);
    c.ng = ng;
    return c;
  };
  std::stable_sort(imp.begin(), imp.end(), [](const GaImpr& a, const GaImpr& b) {
    return a.run != b.run ? a.run < b.run : a.local_idx < b.local_idx;
  });
  for (int i = 0; i < n; ++i) {
    const GaRun& g = hr[i];
    ArmRun& r = *runs[i];
    const int ng = static_cast<int>(r.env->tg.size());
    r.used = g.used;
    r.best = g.best;
    r.n_offspring += g.n_offspring;
    r.w_mut += g.n_waves;
    if (g.best_member_flags & 2) {
      r.best_member = cand_at(H + h_best + 2 * static_cast<int64_t>(stride) * i, ng);
      r.best_member_cost = g.best_member_cost;
      r.has_best_member = true;
    }
  }
  for (size_t k = 0; k < imp.size(); ++k) {
    const GaImpr& x = imp[k];
    ArmRun& r = *runs[x.run];
    const double t = t_launch + 1e-9 * static_cast<double>(x.t - t0_dev);
    r.impr.push_back(Improvement{x.local_idx, x.cost, Cand{}, t});
    const bool last = k + 1 == imp.size() || imp[k + 1].run != x.run;
    if (last && (hr[x.run].impr_flags & 1))
      r.impr.back().plan = cand_at(H + h_best + 2 * static_cast<int64_t>(stride) * x.run + stride,
                                   static_cast<int>(r.env->tg.size()));
  }
  int64_t mx = 0;
  for (int i = 0; i < n; ++i) mx = std::max<int64_t>(mx, hr[i].n_waves);
  waves += mx;
  clock = now_s();
  if (ga_log) {
    cuda_check(eval_set_plan_profile(nullptr), "profile symbol");
    unsigned long long acc[32];
    cuda_check(eval_phase_acc(acc), "phase acc");
    if (FILE* f = std::fopen(ga_log, "a")) {
      // cumulative evaluation phases (kcycles): geometry, TP rings, PP pairs,
      // exact searches of open TP cells (kcycles, count), TP cells with 3-8
      // vertices
      std::fprintf(f, "  phases: geometry %.1f tp %.1f pp %.1f open %.1f n_open %llu cells %llu\n",
                   1e-3 * acc[12], 1e-3 * acc[13], 1e-3 * acc[14], 1e-3 * acc[28], acc[29], acc[30]);
      std::fclose(f);
    }
    if (FILE* f = std::fopen(ga_log, "a")) {
      // runs grid stride evals impr max_waves prep_ms kernel_ms total_ms |
      // step_kcycles_avg steps eval_kcycles_avg evals
      const unsigned long long* pf = hctl + kGaCtlProf;
      std::fprintf(f, "%d %d %d %llu %lld %lld %.3f %.3f %.3f | %.1f %llu %.1f %llu\n", n, grid,
                   stride, hctl[kGaCtlEvals], static_cast<long long>(n_impr),
                   static_cast<long long>(mx), 1e3 * (t_launch - t_prep0), ms,
                   1e3 * (clock - t_prep0), pf[1] ? 1e-3 * pf[0] / pf[1] : 0.0, pf[1],
                   pf[3] ? 1e-3 * pf[2] / pf[3] : 0.0, pf[3]);
      // sub-phases (kcycles per step): load store draw spec walk3 insert mut/init score
      std::fprintf(f, "   ");
      for (int q = 0; q < 8; ++q)
        std::fprintf(f, " %.1f", pf[1] ? 1e-3 * hctl[100 + q] / pf[1] : 0.0);
      // init chunks: kcycles per chunk, chunks, candidates
      std::fprintf(f, " | init %.1f %llu %llu | lane1 jump0 %.1f jumps %.1f total %.1f\n",
                   hctl[109] ? 1e-3 * hctl[108] / hctl[109] : 0.0, hctl[109], hctl[110],
                   hctl[109] ? 1e-3 * hctl[111] / hctl[109] : 0.0,
                   hctl[109] ? 1e-3 * hctl[97] / hctl[109] : 0.0,
                   hctl[109] ? 1e-3 * hctl[98] / hctl[109] : 0.0);
      std::fprintf(f, "    make: layouts %.1f medium %.1f fine %.1f kcycles (n %llu) gen_in_smem %d\n",
                   hctl[127] ? 1e-3 * hctl[99] / hctl[127] : 0.0,
                   hctl[127] ? 1e-3 * hctl[125] / hctl[127] : 0.0,
                   hctl[127] ? 1e-3 * hctl[126] / hctl[127] : 0.0, hctl[127], G.gen_in_smem);
      std::fclose(f);
    }
  }
}

// Runs all arm coroutines to completion, batching their requests per wave.
void run_lockstep(Ctx& ctx, const Knobs& K, std::vector<ArmRun*>& runs, double& clock,
                  int64_t& waves) {
  const DevCostConfig cfg = K.cost_config();
  const int kb = (K.balance_data ? 1 : 0) | (K.balance_layers ? 2 : 0);
  double th = now_s();
  const bool dev_ga = device_ga_enabled(K);
  // arms are independent: their GA steps (candidate generation, population
  // bookkeeping) run on a host thread pool; only the GPU wave is shared
  const int nr = static_cast<int>(runs.size());
host_parallel_for(nr, nr >= 16, [&](int i) {
    ArmRun* r = runs[i];
    r->clock = &clock;
    r->device_ga = dev_ga;
    r->coro = ga_run(*r);
    r->coro.h.resume();
  });
  for (ArmRun* r : runs)
    if (r->coro.h.promise().exc) std::rethrow_exception(r->coro.h.promise().exc);
  ctx.host_ms += 1e3 * (now_s() - th);
  Batch b;
  BatchOut bo;
  std::vector<std::pair<ArmRun*, int>> owners;
  std::vector<size_t> first;
  // init chunks can be made on the device (one thread per candidate, the
  // stream stepped to each start on the host). Measured on c3/c4 at B = 1e4
  // it costs more wave latency (the generator runs ahead of the evaluation,
  // ~0.5 ms per wave) than it saves host time, so the host pool makes them
  // unless HPG_DEVICE_GEN_MIN sets a threshold (runs per wave; 0 = always).
  static const int dev_gen_min = [] {
    const char* v = std::getenv("HPG_DEVICE_GEN_MIN");
    return v ? std::atoi(v) : (1 << 30);
  }();
  std::vector<EvalReq*> gens;
  std::vector<int> gen_first_out;
  std::vector<int> nodes_per_region;
  for (const auto& rn : ctx.prob.region_nodes) nodes_per_region.push_back(static_cast<int>(rn.size()));
  while (true) {
    b.cands.clear();
    b.modes.clear();
    b.gen.clear();
    b.gen_item.clear();
    b.gen_starts.clear();
    b.n_gen = 0;
    owners.clear();
    gens.clear();
    int64_t wave = 0;
    for (ArmRun* r : runs) {
      if (r->coro.h.done()) continue;
      EvalReq* q = r->coro.h.promise().pending;
      if (!q) continue;
      if (q->gen) gens.push_back(q);
      wave += q->gen ? q->gen_count : static_cast<int64_t>(q->cands.size());
    }
    const bool device_gen = !gens.empty() && static_cast<int>(gens.size()) >= dev_gen_min &&
                            wave <= 32768;
    if (!gens.empty()) {
      const double tg = now_s();
      // host: make_candidate x count (stream states recorded); device: the
      // layouts only, the device assignment follows on the GPU
      host_parallel_for(static_cast<int>(gens.size()), gens.size() >= 16, [&](int i) {
        EvalReq* q = gens[i];
        q->cands.resize(q->gen_count);
        q->gen_snaps.resize(q->gen_count);
        if (device_gen) {
          // layouts here; the stream stepped to every candidate's start (each
          // draws the same count), the assignments on the device
          GenItem it = gen_item_of(*q->env);
          const int64_t draws = gen_draws_per_candidate(ctx.prob.N, nodes_per_region.data(),
                                                        static_cast<int>(nodes_per_region.size()), it);
          q->gen_starts.resize(q->gen_count);
          Rng rng = q->gen_rng;
          for (int c = 0; c < q->gen_count; ++c) {
            candidate_layouts(*q->env, q->gen_combo0 + c, q->cands[c]);
            q->gen_starts[c] = rng;
            for (int64_t d = 0; d < draws; ++d) rng.next();
            q->gen_snaps[c] = rng;
          }
        } else {
          Rng rng = q->gen_rng;
          for (int c = 0; c < q->gen_count; ++c) {
            make_candidate(*q->env, q->gen_combo0 + c, rng, q->cands[c]);
            q->gen_snaps[c] = rng;
          }
        }
      });
      ctx.host_ms += 1e3 * (now_s() - tg);
    }
    gen_first_out.clear();
    for (ArmRun* r : runs) {
      if (r->coro.h.done()) continue;
      EvalReq* q = r->coro.h.promise().pending;
      if (!q) continue;
      if (q->gen && device_gen) {
        GenItem it = gen_item_of(*q->env);
        it.first = static_cast<int32_t>(b.cands.size());
        it.first_out = b.n_gen;
        it.count = q->gen_count;
        gen_first_out.push_back(b.n_gen);
        for (int c = 0; c < q->gen_count; ++c) {
          b.gen_item.push_back(static_cast<int32_t>(b.gen.size()));
          b.gen_starts.push_back(q->gen_starts[c]);
        }
        b.gen.push_back(it);
        b.n_gen += q->gen_count;
      } else {
        gen_first_out.push_back(-1);
      }
      for (size_t i = 0; i < q->cands.size(); ++i) {
        b.cands.push_back(&q->cands[i]);
        b.modes.push_back(kModeEvaluate);
      }
      owners.emplace_back(r, static_cast<int>(q->cands.size()));
    }
    if (owners.empty()) break;
    const double tb = now_s();
    run_batch(ctx, b, cfg, kb, true, false, false, bo);
    ++waves;
    clock = now_s();
    ctx.batch_ms += 1e3 * (clock - tb);
    first.resize(owners.size());
    size_t k = 0;
    for (size_t o = 0; o < owners.size(); ++o) {
      first[o] = k;
      k += owners[o].second;
    }
    const int no = static_cast<int>(owners.size());
    host_parallel_for(no, no >= 16, [&](int o) {
      ArmRun* r = owners[o].first;
      const int cnt = owners[o].second;
      EvalReq* q = r->coro.h.promise().pending;
      q->res.resize(cnt);
      const int gj = gen_first_out[o];
      for (int i = 0; i < cnt; ++i) {
        const size_t kk = first[o] + i;
        q->res[i] = bo.res[kk];
        Cand& c = q->cands[i];
        if (gj >= 0)  // device-generated: its device slots
          std::memcpy(c.dev(), bo.gen_devs + bo.gen_dev_off[gj + i], c.o.dev[ctx.prob.T]);
        apply_ws(ctx.prob, c, bo.out_ws + bo.ws_off[kk]);
      }
      r->coro.h.promise().pending = nullptr;
      r->coro.h.resume();
    });
    for (auto& [r, cnt] : owners)
      if (r->coro.h.promise().exc) std::rethrow_exception(r->coro.h.promise().exc);
    ctx.host_ms += 1e3 * (now_s() - clock);
  }
  std::vector<ArmRun*> handed;
  for (ArmRun* r : runs)
    if (r->handoff) handed.push_back(r);
  if (!handed.empty()) {
    const double tb = now_s();
    device_ga(ctx, K, handed, clock, waves);
    ctx.batch_ms += 1e3 * (now_s() - tb);
  }
  static const char* spec_log = std::getenv("HPG_SPEC_LOG");  // diagnostics only
  if (spec_log) {
    if (FILE* f = std::fopen(spec_log, "a")) {
      int64_t off = 0, hit = 0, used = 0, nm = 0, mx = 0, wi = 0, wm = 0, ws = 0, wr = 0;
      double tm = 0, tu = 0, ts = 0, tp = 0;
      for (ArmRun* r : runs) {
        off += r->n_offspring;
        hit += r->n_spec_hit;
        used += r->used;
        nm += r->n_make;
        tm += r->t_make;
        tu += r->t_mut;
        ts += r->t_swap;
        tp += r->t_spec;
        const int64_t w = r->w_init + r->w_mut + r->w_swap + r->w_redraw;
        if (w > mx) {
          mx = w;
          wi = r->w_init;
          wm = r->w_mut;
          ws = r->w_swap;
          wr = r->w_redraw;
        }
      }
      std::fprintf(f,
                   "runs %zu used %lld offspring %lld spec_hits %lld waves_total %lld "
                   "make %lld %.2fms mut %.2fms swap %.2fms spec %.2fms | longest run waves %lld "
                   "(init %lld mut %lld swap %lld redraw %lld)\n",
                   runs.size(), static_cast<long long>(used), static_cast<long long>(off),
                   static_cast<long long>(hit), static_cast<long long>(waves),
                   static_cast<long long>(nm), 1e3 * tm, 1e3 * tu, 1e3 * ts, 1e3 * tp,
                   static_cast<long long>(mx), static_cast<long long>(wi), static_cast<long long>(wm),
                   static_cast<long long>(ws), static_cast<long long>(wr));
      std::fclose(f);
    }
  }
}

// best_half (search.cpp:590-620) for many segments at once, on the device.
struct Segment {
  std::vector<int64_t> arms;   // ascending
  std::vector<double> scores;  // per arm
};

void best_half_batch(Ctx& ctx, std::vector<Segment>& segs, int level,
                     std::vector<std::vector<int64_t>>& keep_out, std::vector<Halving>& ev_out,
                     std::vector<bool>& has_event) {
  const int ns = static_cast<int>(segs.size());
  keep_out.assign(ns, {});
  ev_out.assign(ns, Halving{});
  has_event.assign(ns, false);
  std::vector<int32_t> off(1, 0);
  std::vector<double> sc;
  std::vector<int32_t> idx;
  std::vector<int> seg_of;
  for (int s = 0; s < ns; ++s) {
    if (segs[s].arms.size() <= 1) {
      keep_out[s] = segs[s].arms;
      continue;
    }
    for (size_t i = 0; i < segs[s].arms.size(); ++i) {
      sc.push_back(segs[s].scores[i]);
      idx.push_back(static_cast<int32_t>(segs[s].arms[i]));
    }
    off.push_back(static_cast<int32_t>(sc.size()));
    seg_of.push_back(s);
  }
  const int nk = static_cast<int>(seg_of.size());
  if (nk == 0) return;
  const double t_bh = now_s();
  const size_t n = sc.size();
  ctx.d_scores.reserve(n);
  ctx.d_arm_idx.reserve(n);
  ctx.d_keep.reserve(n);
  ctx.d_seg_off.reserve(nk + 1);
  ctx.d_events.reserve(2 * nk);
  cudaStream_t st = ctx.stream;
  cuda_check(cudaMemcpyAsync(ctx.d_scores.p, sc.data(), 8 * n, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(ctx.d_arm_idx.p, idx.data(), 4 * n, cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(cudaMemcpyAsync(ctx.d_seg_off.p, off.data(), 4 * (nk + 1), cudaMemcpyHostToDevice, st), "H2D");
  cuda_check(launch_best_half(ctx.d_scores.p, ctx.d_seg_off.p, ctx.d_arm_idx.p, nk, ctx.d_keep.p,
                              ctx.d_events.p, st),
             "best_half launch");
  ++ctx.launches;
  std::vector<int32_t> keep(n);
  std::vector<double> ev(2 * nk);
  cuda_check(cudaMemcpyAsync(keep.data(), ctx.d_keep.p, 4 * n, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(ev.data(), ctx.d_events.p, 16 * nk, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "best_half");
  ctx.best_half_ms += 1e3 * (now_s() - t_bh);
  ++ctx.best_half_calls;
  for (int k = 0; k < nk; ++k) {
    const int s = seg_of[k];
    for (int i = off[k]; i < off[k + 1]; ++i)
      if (keep[i]) keep_out[s].push_back(idx[i]);
    std::sort(keep_out[s].begin(), keep_out[s].end());
    Halving h;
    h.level = level;
    h.before = off[k + 1] - off[k];
    h.after = (h.before + 1) / 2;
    h.survivor_worst = ev[2 * k];
    h.eliminated_best = ev[2 * k + 1];
    ev_out[s] = h;
    has_event[s] = true;
  }
}

struct TgArm {
  Grouping tg;
  std::vector<std::vector<int>> ggs;
  std::vector<double> best;
  std::vector<int64_t> alive;
  std::vector<int64_t> rec;
};

// ---- multi-GPU: per-run records all-gathered after every lockstep round ----

// NCCL all-gather over the context's communicator, staged through HBM
class NcclTransport : public Transport {
 public:
  NcclTransport(Ctx& ctx, Dist& d) : ctx_(ctx), d_(d) {}
  int rank() const override { return d_.rank; }
  int world() const override { return d_.world; }
  void allgather(const void* send, void* recv, size_t bytes) override {
    DevBuf<uint8_t>& snd = ctx_.d_xch_send;
    DevBuf<uint8_t>& rcv = ctx_.d_xch_recv;
    snd.reserve(bytes + 8);
    rcv.reserve(bytes * d_.world + 8);
    if (bytes == 0) return;
    cuda_check(cudaMemcpyAsync(snd.p, send, bytes, cudaMemcpyHostToDevice, ctx_.stream), "H2D");
    dist_allgather(d_, snd.p, rcv.p, bytes, ctx_.stream);
    cuda_check(cudaMemcpyAsync(recv, rcv.p, bytes * d_.world, cudaMemcpyDeviceToHost, ctx_.stream),
               "D2H");
    cuda_check(cudaStreamSynchronize(ctx_.stream), "allgather");
    ctx_.h2d_bytes += static_cast<int64_t>(bytes);
    ctx_.d2h_bytes += static_cast<int64_t>(bytes * d_.world);
  }

 private:
  Ctx& ctx_;
  Dist& d_;
};

// Every rank ends with identical (used, best, improvement list) for every run
// of the round; improvement plans stay with the owning rank.
void exchange_runs(Ctx& ctx, Dist& d, std::vector<ArmRun*>& all, double now) {
  const size_t R = all.size();
  std::vector<int> owner(R);
  std::vector<RunRecord> rec(R);
  std::vector<std::vector<ImprRecord>> imp(R);
  for (size_t r = 0; r < R; ++r) {
    owner[r] = all[r]->owner;
    rec[r] = RunRecord{all[r]->used, all[r]->best};
    if (owner[r] == d.rank)
      for (const auto& im : all[r]->impr)
        imp[r].push_back(ImprRecord{static_cast<int64_t>(r), im.local_idx, im.cost});
  }
  NcclTransport tr(ctx, d);
  exchange_round(tr, owner, rec, imp);
  for (size_t r = 0; r < R; ++r) {
    if (owner[r] == d.rank) continue;
    all[r]->used = rec[r].used;
    all[r]->best = rec[r].best;
    all[r]->impr.clear();
    for (const ImprRecord& x : imp[r]) all[r]->impr.push_back(Improvement{x.local_idx, x.cost, Cand{}, now});
  }
}

}  // namespace

SearchOut nested_sha_search(Ctx& ctx, const Knobs& K, Dist* dist) {
  (void)dist;
  if (K.budget < 1) throw UsageError("search budget must be >= 1");
  reset_ring_memo(ctx);
  const Problem& P = ctx.prob;
  const double t0 = now_s();
  const int64_t launches0 = ctx.launches, plans0 = ctx.plans_evaluated;
  const int64_t h2d0 = ctx.h2d_bytes, d2h0 = ctx.d2h_bytes, el0 = ctx.eval_launches,
                cb0 = ctx.canonical_bytes;
  const double ems0 = ctx.eval_ms, hms0 = ctx.host_ms, bms0 = ctx.batch_ms;
  const Rng base_rng(K.seed);
  SearchOut S;
  S.budget = K.budget;
  S.seed = K.seed;

  std::vector<Grouping> tgs = K.has_tg_override ? K.tg_override : enumerate_task_groupings(P, K.adjacent);
  if (K.level1_cap > 0 && tgs.size() > static_cast<size_t>(K.level1_cap)) tgs.resize(K.level1_cap);
  S.task_groupings = static_cast<int64_t>(tgs.size());

  const int n_devices = P.N;
  // level-2 arms of every task grouping: independent per grouping (each
  // sampled from its own fork of the base stream), built on the host pool
  std::vector<TgArm> arms(tgs.size());
  host_parallel_for(static_cast<int>(tgs.size()), tgs.size() >= 16, [&](int ti) {
    TgArm& arm = arms[ti];
    arm.tg = tgs[ti];
    const int k = static_cast<int>(arm.tg.size());
    if (k <= n_devices) {
      int q = K.quantize;
      double count = composition_count(n_devices, k, q);
      if (count == 0) {
        q = 1;
        count = composition_count(n_devices, k, q);
      }
      if (count <= K.gg_arm_cap) {
        arm.ggs = compositions(n_devices, k, q);
      } else {
        std::set<std::vector<int>> seen;
        std::vector<int> balanced(k, n_devices / k);
        for (int i = 0; i < n_devices % k; ++i) ++balanced[i];
        seen.insert(balanced);
        arm.ggs.push_back(balanced);
        Rng rng = base_rng.fork(0xA001 + ti);
        for (int64_t tries = 0; static_cast<int>(arm.ggs.size()) < K.gg_arm_cap &&
                                tries < 50LL * K.gg_arm_cap;
             ++tries) {
          auto comp = sample_composition(n_devices, k, q, rng);
          if (seen.insert(comp).second) arm.ggs.push_back(std::move(comp));
        }
      }
    }
    arm.best.assign(arm.ggs.size(), kInf);
  });
  // arm records in (task grouping, GPU grouping) order
  for (size_t ti = 0; ti < arms.size(); ++ti) {
    TgArm& arm = arms[ti];
    for (size_t gi = 0; gi < arm.ggs.size(); ++gi) {
      arm.alive.push_back(static_cast<int64_t>(gi));
      arm.rec.push_back(static_cast<int64_t>(S.arms.size()));
      ArmRec r;
      r.tg = static_cast<int64_t>(ti);
      r.gg = static_cast<int64_t>(gi);
      S.arms.push_back(r);
    }
  }

  const double t_setup = now_s();
  double t_env = 0, t_run = 0, t_inc = 0;  // diagnostics: round phases (s)
  const double bh0 = ctx.best_half_ms;
  const int64_t bhc0 = ctx.best_half_calls;
  double incumbent = kInf;
  Cand inc_plan;
  int inc_owner = 0;
  int64_t inc_ti = -1, inc_gi = -1;
  double inc_time = t0;
  int64_t consumed = 0;
  double clock = t0;
  int64_t waves = 0;

  std::vector<int64_t> surv(tgs.size());
  std::iota(surv.begin(), surv.end(), 0);
  const int denom_out = std::max(1, ceil_log2(tgs.size()));
  for (int m = 0; m < denom_out; ++m) {
    const int64_t b_m = K.budget / (static_cast<int64_t>(surv.size()) * denom_out);
    S.b_m.push_back(b_m);
    // participating task groupings and their round budget b
    std::vector<std::pair<int64_t, int64_t>> parts;
    if (b_m >= 1) {
      for (int64_t ti : surv) parts.emplace_back(ti, b_m);
    } else {
      int64_t ob = K.budget / denom_out;
      if (ob == 0 && m == 0) ob = K.budget;
      for (int64_t ti : surv) {
        if (static_cast<int64_t>(parts.size()) >= ob) break;
        parts.emplace_back(ti, 1);
      }
    }
    struct Part {
      int64_t ti, b;
      std::vector<int64_t> entry, cur;
      int rounds, denom_in;
      std::vector<Halving> events;
      std::vector<std::vector<int64_t>> surv_sets;
      std::vector<std::vector<std::unique_ptr<ArmRun>>> runs;  // per n, in gi order
    };
    std::vector<Part> ps;
    for (auto& [ti, b] : parts) {
      if (arms[ti].alive.empty()) continue;
      Part p;
      p.ti = ti;
      p.b = b;
      p.entry = arms[ti].alive;
      p.cur = p.entry;
      p.denom_in = std::max(1, ceil_log2(p.entry.size()));
      p.rounds = p.denom_in;
      ps.push_back(std::move(p));
    }
    int max_rounds = 0;
    for (auto& p : ps) max_rounds = std::max(max_rounds, p.rounds);
    for (int n = 0; n < max_rounds; ++n) {
      // one NVTX range per SHA round (outer m, inner n): nsys / ncu --nvtx
      char range_name[48];
      std::snprintf(range_name, sizeof(range_name), "hpg SHA round m=%d n=%d", m, n);
      nvtxRangePushA(range_name);
      const double t_round0 = now_s();
      std::vector<ArmRun*> batch;
      // the round's runs in sequential order: (part, gi, slice); their state
      // (RNG fork, layout options) is built on the host pool below
      struct RunSpec {
        Part* p;
        int64_t gi, slice;
      };
      std::vector<RunSpec> specs;
      for (auto& p : ps) {
        p.runs.emplace_back();
        if (n >= p.rounds) continue;
        const int64_t b_mn = p.b / (static_cast<int64_t>(p.cur.size()) * p.denom_in);
        if (b_mn >= 1) {
          for (int64_t gi : p.cur) specs.push_back({&p, gi, b_mn});
        } else {
          int64_t rb = p.b / p.denom_in;
          if (rb == 0 && n == 0) rb = p.b;
          int64_t spent = 0;
          for (int64_t gi : p.cur) {
            if (spent >= rb) break;
            specs.push_back({&p, gi, 1});
            ++spent;
          }
        }
      }
      std::vector<std::unique_ptr<ArmRun>> made(specs.size());
      host_parallel_for(static_cast<int>(specs.size()), specs.size() >= 32, [&](int i) {
        const RunSpec& sp = specs[i];
        auto r = std::make_unique<ArmRun>();
        r->ti = sp.p->ti;
        r->gi = sp.gi;
        r->slice = sp.slice;
        const uint64_t salt = (static_cast<uint64_t>(sp.p->ti) << 40) |
                              (static_cast<uint64_t>(sp.gi) << 16) |
                              (static_cast<uint64_t>(m) << 8) | static_cast<uint64_t>(n);
        r->rng = base_rng.fork(salt);
        const TgArm& arm = arms[sp.p->ti];
        r->env.reset(new ArmEnv{P, K, arm.tg, arm.ggs[sp.gi],
                                build_arm_layouts(P, arm.tg, arm.ggs[sp.gi])});
        made[i] = std::move(r);
      });
      for (size_t i = 0; i < specs.size(); ++i) {
        batch.push_back(made[i].get());
        specs[i].p->runs.back().push_back(std::move(made[i]));
      }
      const double t_env_done = now_s();
      t_env += t_env_done - t_round0;
      if (dist && dist->world > 1) {
        // runs dealt over the ranks by budget (longest slice first to the
        // least-loaded rank, dist_exchange.cpp deal_runs), then all-gathered
        std::vector<int64_t> slices(batch.size());
        for (size_t r = 0; r < batch.size(); ++r) slices[r] = batch[r]->slice;
        const std::vector<int> owner = deal_runs(slices, dist->world);
        std::vector<ArmRun*> mine;
        for (size_t r = 0; r < batch.size(); ++r) {
          batch[r]->owner = owner[r];
          if (batch[r]->owner == dist->rank) mine.push_back(batch[r]);
        }
        run_lockstep(ctx, K, mine, clock, waves);
        exchange_runs(ctx, *dist, batch, clock);
      } else {
        run_lockstep(ctx, K, batch, clock, waves);
      }
      const double t_run_done = now_s();
      t_run += t_run_done - t_env_done;
      // fold run results into the arm records
      for (auto& p : ps) {
        if (n >= p.rounds) continue;
        TgArm& arm = arms[p.ti];
        for (auto& r : p.runs.back()) {
          ArmRec& rec = S.arms[arm.rec[r->gi]];
          rec.evals += r->used;
          rec.best = std::min(rec.best, r->best);
          arm.best[r->gi] = rec.best;
        }
      }
      std::vector<Segment> segs;
      std::vector<Part*> owners;
      for (auto& p : ps) {
        if (n >= p.rounds) continue;
        Segment sg;
        sg.arms = p.cur;
        for (int64_t gi : p.cur) sg.scores.push_back(arms[p.ti].best[gi]);
        segs.push_back(std::move(sg));
        owners.push_back(&p);
      }
      std::vector<std::vector<int64_t>> keep;
      std::vector<Halving> ev;
      std::vector<bool> has_ev;
      best_half_batch(ctx, segs, 2, keep, ev, has_ev);
      for (size_t s = 0; s < owners.size(); ++s) {
        owners[s]->cur = keep[s];
        if (has_ev[s]) {
          owners[s]->events.push_back(ev[s]);
          owners[s]->surv_sets.push_back(keep[s]);
        }
      }
      nvtxRangePop();
    }
    {
      std::vector<Segment> segs;
      for (auto& p : ps) {
        Segment sg;
        sg.arms = p.entry;
        for (int64_t gi : p.entry) sg.scores.push_back(arms[p.ti].best[gi]);
        segs.push_back(std::move(sg));
      }
      std::vector<std::vector<int64_t>> keep;
      std::vector<Halving> ev;
      std::vector<bool> has_ev;
      best_half_batch(ctx, segs, 2, keep, ev, has_ev);
      for (size_t s = 0; s < ps.size(); ++s) {
        arms[ps[s].ti].alive = keep[s];
        if (has_ev[s]) {
          ps[s].events.push_back(ev[s]);
          ps[s].surv_sets.push_back(keep[s]);
        }
      }
    }
    const double t_inc0 = now_s();
    // sequential order: task groupings in survivor order, rounds, arms
    for (auto& p : ps) {
      for (size_t i = 0; i < p.events.size(); ++i) {
        S.halvings.push_back(p.events[i]);
        S.survivors.push_back(p.surv_sets[i]);
      }
      for (auto& list : p.runs) {
        for (auto& r : list) {
          for (auto& im : r->impr) {
            if (im.cost < incumbent) {
              incumbent = im.cost;
              inc_plan = im.plan;
              inc_owner = r->owner;
              inc_ti = r->ti;
              inc_gi = r->gi;
              inc_time = im.t_wall;
              S.trace.emplace_back(consumed + im.local_idx, im.cost);
            }
          }
          consumed += r->used;
        }
      }
    }
    t_inc += now_s() - t_inc0;
    // level-1 halving over task groupings (tg score = min over all gg arms)
    std::vector<Segment> segs(1);
    segs[0].arms = surv;
    for (int64_t ti : surv) {
      double best = kInf;
      for (double c : arms[ti].best) best = std::min(best, c);
      segs[0].scores.push_back(best);
    }
    std::vector<std::vector<int64_t>> keep;
    std::vector<Halving> ev;
    std::vector<bool> has_ev;
    best_half_batch(ctx, segs, 1, keep, ev, has_ev);
    surv = keep[0];
    if (has_ev[0]) {
      S.halvings.push_back(ev[0]);
      S.survivors.push_back(keep[0]);
    }
  }
  S.consumed = consumed;
  const double t_rounds = now_s();
  if (consumed > K.budget) throw InternalError("search overspent its budget");
  if (inc_ti >= 0 && dist && dist->world > 1) {
    // the incumbent's plan lives on the rank that evaluated it
    NcclTransport tr(ctx, *dist);
    const int64_t sz = dist->rank == inc_owner ? static_cast<int64_t>(inc_plan.rec.size()) : 0;
    std::vector<int64_t> gsz(dist->world);
    tr.allgather(&sz, gsz.data(), 8);
    const int64_t bytes = gsz[inc_owner];
    std::vector<uint8_t> mine(bytes, 0);
    if (dist->rank == inc_owner) std::memcpy(mine.data(), inc_plan.rec.data(), bytes);
    std::vector<uint8_t> all(static_cast<size_t>(bytes) * dist->world);
    tr.allgather(mine.data(), all.data(), static_cast<size_t>(bytes));
    inc_plan.rec.assign(all.begin() + static_cast<int64_t>(inc_owner) * bytes,
                        all.begin() + static_cast<int64_t>(inc_owner + 1) * bytes);
    rec_offsets(inc_plan.hdr(), inc_plan.o);
    inc_plan.ng = static_cast<int>(arms[inc_ti].tg.size());
  }
  if (inc_ti >= 0) {
    S.has_plan = true;
    S.plan = inc_plan;
    S.plan_groups = arms[inc_ti].tg;
    S.plan_counts = arms[inc_ti].ggs[inc_gi];
    // breakdown of the incumbent (end_to_end_cost with the search's config)
    Batch b;
    b.cands.push_back(&S.plan);
    b.modes.push_back(kModeE2E);
    BatchOut bo;
    run_batch(ctx, b, K.cost_config(), 0, false, true, false, bo);
    S.per_task = bo.per_task;
    S.reshard_s = bo.res[0].reshard_s;
    S.sync_s = bo.res[0].sync_s;
    S.e2e = bo.res[0].cost;
    S.feasible = (bo.res[0].flags & kResFeasOut) != 0;
    S.est_cost = S.e2e;
  }
  S.wall_s = now_s() - t0;
  S.time_to_best_s = S.has_plan ? inc_time - t0 : 0.0;
  S.launches = ctx.launches - launches0;
  S.plans_gpu = ctx.plans_evaluated - plans0;
  S.waves = waves;
  S.h2d_bytes = ctx.h2d_bytes - h2d0;
  S.d2h_bytes = ctx.d2h_bytes - d2h0;
  S.eval_launches = ctx.eval_launches - el0;
  S.canonical_bytes = ctx.canonical_bytes - cb0;
  S.eval_ms = ctx.eval_ms - ems0;
  S.host_ms = ctx.host_ms - hms0;
  S.batch_ms = ctx.batch_ms - bms0;
  static const char* phase_log = std::getenv("HPG_GA_LOG");  // diagnostics only
  if (phase_log) {
    if (FILE* f = std::fopen(phase_log, "a")) {
      std::fprintf(f,
                   "search: setup %.3f ms, rounds %.3f ms (run set-up %.3f, GA rounds %.3f, "
                   "incumbent merge %.3f, best_half %.3f ms in %lld calls, device GA %.3f ms), "
                   "final %.3f ms, total %.3f ms\n",
                   1e3 * (t_setup - t0), 1e3 * (t_rounds - t_setup), 1e3 * t_env, 1e3 * t_run,
                   1e3 * t_inc, ctx.best_half_ms - bh0,
                   static_cast<long long>(ctx.best_half_calls - bhc0), S.eval_ms,
                   1e3 * (now_s() - t_rounds), 1e3 * S.wall_s);
      std::fclose(f);
    }
  }
  return S;
}

SearchOut ga_search(Ctx& ctx, const Grouping& tg, const std::vector<int>& counts, int64_t slice,
                    uint64_t seed, const Knobs& K) {
  if (slice < 1) throw UsageError("ga_search needs a budget of at least 1 evaluation");
  reset_ring_memo(ctx);
  const Problem& P = ctx.prob;
  if (counts.size() != tg.size()) throw InputError("gpu grouping must list one count per task group");
  const double t0 = now_s();
  const int64_t launches0 = ctx.launches, plans0 = ctx.plans_evaluated;
  ArmRun r;
  r.slice = slice;
  r.rng = Rng(seed);
  r.env.reset(new ArmEnv{P, K, tg, counts, build_arm_layouts(P, tg, counts)});
  std::vector<ArmRun*> runs{&r};
  double clock = t0;
  int64_t waves = 0;
  run_lockstep(ctx, K, runs, clock, waves);
  SearchOut S;
  S.budget = slice;
  S.seed = seed;
  S.consumed = r.used;
  ArmRec rec;
  rec.best = r.best_member_cost;
  rec.evals = r.used;
  S.arms.push_back(rec);
  for (auto& im : r.impr) S.trace.emplace_back(im.local_idx, im.cost);
  if (r.has_best_member) {
    S.has_plan = true;
    S.plan = r.best_member;
    S.plan_groups = tg;
    S.plan_counts = counts;
    Batch b;
    b.cands.push_back(&S.plan);
    b.modes.push_back(kModeE2E);
    BatchOut bo;
    run_batch(ctx, b, K.cost_config(), 0, false, true, false, bo);
    S.per_task = bo.per_task;
    S.reshard_s = bo.res[0].reshard_s;
    S.sync_s = bo.res[0].sync_s;
    S.e2e = bo.res[0].cost;
    S.feasible = (bo.res[0].flags & kResFeasOut) != 0;
    S.est_cost = r.best_member_cost;
  }
  S.wall_s = now_s() - t0;
  S.launches = ctx.launches - launches0;
  S.plans_gpu = ctx.plans_evaluated - plans0;
  S.waves = waves;
  return S;
}

}  // namespace hpg
