// hetplan_b200.cpp — see hetplan_b200.hpp. Pure type conversion: hetplan's
// std::map/std::string plan model <-> the engine's struct-of-arrays tables.
#include "hetplan_b200.hpp"

#include <cstring>
#include <stdexcept>
#include <string>

#include "hetplan/errors.hpp"
#include "hpg.h"

namespace hetplan::b200 {
namespace {

void check(int rc, const char* err) {
  if (rc == HPG_OK) return;
  if (rc == HPG_USAGE) throw UsageError(err);
  if (rc == HPG_INPUT) throw InputError(err);
  throw std::runtime_error(std::string("B200 engine: ") + err);
}

int kind_of(TaskKind k) {
  return k == TaskKind::kGeneration ? 0 : (k == TaskKind::kInference ? 1 : 2);
}

struct ProblemC {
  std::vector<hpg_task> tasks;
  std::vector<int32_t> edges;
  std::vector<hpg_device> devs;
  std::vector<hpg_region_link> links;
  hpg_problem p{};
};

void make_problem(const WorkflowGraph& wf, const DeviceTopology& topo, ProblemC& c) {
  for (const RlTask& t : wf.tasks) {
    c.tasks.push_back(hpg_task{t.id, kind_of(t.kind), t.model.hidden_size,
                               t.model.intermediate_size, t.model.num_layers,
                               t.model.include_embedding ? 1 : 0, t.model.vocab_size,
                               t.precision_bytes});
  }
  for (const auto& [a, b] : wf.dep_edges) {
    c.edges.push_back(a);
    c.edges.push_back(b);
  }
  for (const Device& d : topo.devices()) {
    c.devs.push_back(hpg_device{d.id.c_str(), d.gpu_model.c_str(), d.comp_tflops, d.mem_gb,
                                d.hbm_gbps, d.intra_node_gbps, d.node.c_str(), d.region.c_str()});
  }
  for (const RegionLink& l : topo.region_links()) {
    c.links.push_back(hpg_region_link{l.src.c_str(), l.dst.c_str(), l.latency_ms, l.bandwidth_gbps});
  }
  hpg_problem& p = c.p;
  p.algorithm = wf.algorithm == RlAlgorithm::kPpo ? 0 : 1;
  p.mode = wf.mode == RunMode::kSync ? 0 : 1;
  p.eta = wf.eta;
  p.global_batch = wf.batch.global_batch;
  p.responses_per_prompt = wf.batch.responses_per_prompt;
  p.seq_in = wf.batch.seq_in;
  p.seq_out = wf.batch.seq_out;
  p.micro_batch_size = wf.batch.micro_batch_size;
  p.n_tasks = static_cast<int32_t>(c.tasks.size());
  p.tasks = c.tasks.data();
  p.n_dep_edges = static_cast<int32_t>(c.edges.size() / 2);
  p.dep_edges = c.edges.data();
  p.n_devices = static_cast<int32_t>(c.devs.size());
  p.devices = c.devs.data();
  p.n_region_links = static_cast<int32_t>(c.links.size());
  p.region_links = c.links.data();
  p.intra_region_latency_ms = topo.defaults().intra_region_latency_ms;
  p.intra_region_bandwidth_gbps = topo.defaults().intra_region_bandwidth_gbps;
}

struct TableC {
  std::vector<int32_t> n_groups, task_group, counts, dp, pp, tp, sl, dev;
  std::vector<int64_t> sl_off, w_off, dev_off;
  std::vector<double> w;
  hpg_plan_table t{};
};

// resolve_plan's lookups (plan.cpp:257-349): missing layouts/assignments and
// unknown device ids raise InputError here; the engine validates the rest.
void make_table(const std::vector<const Plan*>& plans, const WorkflowGraph& wf,
                const DeviceTopology& topo, TableC& c) {
  const int T = static_cast<int>(wf.tasks.size());
  for (const Plan* pl : plans) {
    c.n_groups.push_back(static_cast<int32_t>(pl->task_grouping.groups.size()));
    for (const RlTask& t : wf.tasks) c.task_group.push_back(pl->task_grouping.group_of(t.id));
    for (int g = 0; g < T; ++g)
      c.counts.push_back(g < static_cast<int>(pl->gpu_grouping.counts.size())
                             ? pl->gpu_grouping.counts[g]
                             : 0);
    for (const RlTask& t : wf.tasks) {
      auto lit = pl->layouts.find(t.id);
      if (lit == pl->layouts.end())
        throw InputError("plan missing layout for task " + std::to_string(t.id));
      auto ait = pl->assignment.find(t.id);
      if (ait == pl->assignment.end())
        throw InputError("plan missing assignment for task " + std::to_string(t.id));
      const ParallelLayout& l = lit->second;
      c.dp.push_back(l.dp);
      c.pp.push_back(l.pp);
      c.tp.push_back(l.tp);
      c.sl_off.push_back(static_cast<int64_t>(c.sl.size()));
      c.sl.insert(c.sl.end(), l.stage_layers.begin(), l.stage_layers.end());
      c.w_off.push_back(static_cast<int64_t>(c.w.size()));
      c.w.insert(c.w.end(), l.replica_batch_weights.begin(), l.replica_batch_weights.end());
      c.dev_off.push_back(static_cast<int64_t>(c.dev.size()));
      for (const std::string& id : ait->second) c.dev.push_back(topo.device_index(id));
    }
  }
  hpg_plan_table& t = c.t;
  t.n_plans = static_cast<int32_t>(plans.size());
  t.n_groups = c.n_groups.data();
  t.task_group = c.task_group.data();
  t.gpu_counts = c.counts.data();
  t.dp = c.dp.data();
  t.pp = c.pp.data();
  t.tp = c.tp.data();
  t.sl_off = c.sl_off.data();
  t.stage_layers = c.sl.data();
  t.w_off = c.w_off.data();
  t.weights = c.w.data();
  t.dev_off = c.dev_off.data();
  t.devices = c.dev.data();
}

hpg_cost_config cfg_c(const CostModelConfig& c) {
  hpg_cost_config o;
  o.recompute = c.recompute ? 1 : 0;
  o.reshard_override = c.reshard_override;
  o.sync_override = c.sync_override;
  o.dbs_override = c.dbs_override;
  o.train_bytes_per_param = c.memory.train_bytes_per_param;
  o.infer_bytes_per_param = c.memory.infer_bytes_per_param;
  o.kv_bytes_per_elem = c.memory.kv_bytes_per_elem;
  o.dbs_cap = c.memory.dbs_cap;
  o.act_factor = c.memory.act_factor;
  return o;
}

CostBreakdown breakdown_of(const WorkflowGraph& wf, const double* per_task, double reshard,
                           double sync, double e2e, bool feasible) {
  CostBreakdown bd;
  for (size_t t = 0; t < wf.tasks.size(); ++t) {
    const double* v = per_task + 7 * t;
    bd.per_task[wf.tasks[t].id] = TaskCost{v[0], v[1], v[2], v[3], v[4], v[5], v[6]};
  }
  bd.reshard_s = reshard;
  bd.sync_s = sync;
  bd.end_to_end_s = e2e;
  bd.memory_feasible = feasible;
  return bd;
}

}  // namespace

Engine::Engine(const WorkflowGraph& wf, const DeviceTopology& topo, int cuda_device)
    : wf_(wf), topo_(topo) {
  ProblemC pc;
  make_problem(wf, topo, pc);
  char err[1024];
  check(hpg_create(&pc.p, cuda_device, &ctx_, err, sizeof(err)), err);
}

Engine::~Engine() { hpg_destroy(ctx_); }

std::vector<CostBreakdown> Engine::end_to_end_cost(const std::vector<Plan>& plans,
                                                   const CostModelConfig& cfg) {
  std::vector<const Plan*> ps;
  for (const Plan& p : plans) ps.push_back(&p);
  TableC tc;
  make_table(ps, wf_, topo_, tc);
  const size_t n = plans.size(), T = wf_.tasks.size();
  std::vector<double> e2e(n), rs(n), sy(n), pt(n * T * 7);
  std::vector<uint8_t> feas(n);
  hpg_eval_out out{e2e.data(), feas.data(), pt.data(), rs.data(), sy.data()};
  const hpg_cost_config c = cfg_c(cfg);
  char err[1024];
  check(hpg_eval(ctx_, &tc.t, &c, &out, err, sizeof(err)), err);
  std::vector<CostBreakdown> r;
  for (size_t i = 0; i < n; ++i)
    r.push_back(breakdown_of(wf_, pt.data() + i * T * 7, rs[i], sy[i], e2e[i], feas[i] != 0));
  return r;
}

TaskCostDetail Engine::task_cost_detail(const ResolvedTask& rt, const CostModelConfig& cfg,
                                        std::span<const double> resident_weight_bytes) {
  int slot = -1;
  for (size_t i = 0; i < wf_.tasks.size(); ++i)
    if (wf_.tasks[i].id == rt.task_id) slot = static_cast<int>(i);
  if (slot < 0 || !rt.layout) throw InputError("resolved task is not part of the workflow");
  const ParallelLayout& l = *rt.layout;
  hpg_resolved_task t{};
  t.task_slot = slot;
  t.dp = l.dp;
  t.pp = l.pp;
  t.tp = l.tp;
  std::vector<int32_t> sl(l.stage_layers.begin(), l.stage_layers.end());
  std::vector<int32_t> dv(rt.devices.begin(), rt.devices.end());
  t.stage_layers = sl.data();
  t.nm_replica = rt.nm_replica.data();
  t.devices = dv.data();
  if (!resident_weight_bytes.empty() &&
      resident_weight_bytes.size() != static_cast<size_t>(topo_.size()))
    throw InputError("resident weight bytes must have one entry per device");
  const hpg_cost_config c = cfg_c(cfg);
  double agg[7];
  std::vector<double> stage(4 * static_cast<size_t>(l.dp) * l.pp), bubble(l.dp);
  char err[1024];
  check(hpg_task_cost(ctx_, &t, &c, resident_weight_bytes.empty() ? nullptr : resident_weight_bytes.data(),
                      agg, stage.data(), bubble.data(), err, sizeof(err)),
        err);
  TaskCostDetail d;
  d.agg = TaskCost{agg[0], agg[1], agg[2], agg[3], agg[4], agg[5], agg[6]};
  d.stage.assign(l.dp, std::vector<StagePiece>(l.pp));
  for (int i = 0; i < l.dp; ++i)
    for (int j = 0; j < l.pp; ++j) {
      const double* q = stage.data() + 4 * (static_cast<size_t>(i) * l.pp + j);
      d.stage[i][j] = StagePiece{q[0], q[1], q[2], q[3]};
    }
  d.bubble_replica = bubble;
  d.nm_replica = rt.nm_replica;
  return d;
}

double Engine::min_ring_bottleneck(std::span<const int> devices, double volume_bytes) {
  std::vector<int32_t> dv(devices.begin(), devices.end());
  double out = 0;
  char err[1024];
  check(hpg_ring_bottleneck(ctx_, dv.data(), static_cast<int32_t>(dv.size()), volume_bytes, &out,
                            err, sizeof(err)),
        err);
  return out;
}

double Engine::min_pair_cost(std::span<const int> src, std::span<const int> dst,
                             double volume_bytes) {
  std::vector<int32_t> a(src.begin(), src.end()), b(dst.begin(), dst.end());
  double out = 0;
  char err[1024];
  check(hpg_pair_cost(ctx_, a.data(), static_cast<int32_t>(a.size()), b.data(),
                      static_cast<int32_t>(b.size()), volume_bytes, &out, err, sizeof(err)),
        err);
  return out;
}

std::vector<MemoryViolation> Engine::check_memory(const Plan& plan, const MemoryModel& mm) {
  TableC tc;
  make_table({&plan}, wf_, topo_, tc);
  CostModelConfig cfg;
  cfg.memory = mm;
  const hpg_cost_config c = cfg_c(cfg);
  uint8_t feas = 0;
  std::vector<double> req(topo_.size());
  char err[1024];
  check(hpg_check_memory(ctx_, &tc.t, &c, &feas, req.data(), err, sizeof(err)), err);
  std::vector<MemoryViolation> v;
  for (int d = 0; d < topo_.size(); ++d)
    if (req[d] > topo_.device(d).mem()) v.push_back({topo_.device(d).id, req[d], topo_.device(d).mem()});
  return v;
}

static Plan balanced(hpg_ctx* ctx, const Plan& plan, const WorkflowGraph& wf,
                     const DeviceTopology& topo, const CostModelConfig& cfg, int which) {
  TableC tc;
  make_table({&plan}, wf, topo, tc);
  const hpg_cost_config c = cfg_c(cfg);
  std::vector<int32_t> sl(tc.sl.size());
  std::vector<double> w(tc.w.size());
  char err[1024];
  check(hpg_balance(ctx, &tc.t, &c, which, sl.data(), w.data(), nullptr, err, sizeof(err)), err);
  Plan out = plan;
  for (size_t s = 0; s < wf.tasks.size(); ++s) {
    ParallelLayout& l = out.layouts.at(wf.tasks[s].id);
    for (int j = 0; j < l.pp; ++j) l.stage_layers[j] = sl[tc.sl_off[s] + j];
    for (int i = 0; i < l.dp; ++i) l.replica_batch_weights[i] = w[tc.w_off[s] + i];
  }
  return out;
}

Plan Engine::balance_data(const Plan& plan, const CostModelConfig& cfg) {
  return balanced(ctx_, plan, wf_, topo_, cfg, 1);
}

Plan Engine::balance_layers(const Plan& plan, const CostModelConfig& cfg) {
  return balanced(ctx_, plan, wf_, topo_, cfg, 2);
}

namespace {

hpg_knobs knobs_to_c(const SearchKnobs& k) {
  hpg_knobs kn;
  hpg_knobs_default(&kn);
  kn.budget = k.budget;
  kn.seed = k.seed;
  kn.population = k.population;
  kn.locality_bias = k.locality_bias;
  kn.quantize_gpu_counts = k.quantize_gpu_counts;
  kn.level1_filter_adjacent = k.level1_filter == "adjacent" ? 1 : 0;
  kn.level1_cap = k.level1_cap;
  kn.gg_arm_cap = k.gg_arm_cap;
  kn.swap_pair_sample = k.swap_pair_sample;
  kn.balance_data = k.balance_data;
  kn.balance_layers = k.balance_layers;
  kn.balance_seqlen = k.balance_seqlen;
  kn.recompute = k.recompute;
  kn.reshard_override = k.reshard_override;
  kn.sync_override = k.sync_override;
  kn.exhaustive_cap = k.exhaustive_cap;
  return kn;
}

// the chosen plan + breakdown of a result handle (has_plan checked by caller)
void read_plan(hpg_search_result* r, const WorkflowGraph& wf, const DeviceTopology& topo,
               Plan& plan, CostBreakdown& bd) {
  hpg_plan_table pt;
  const int T = static_cast<int>(wf.tasks.size());
  std::vector<int32_t> gflat(T);
  double est = 0;
  uint64_t pseed = 0;
  int64_t pbudget = 0;
  hpg_result_plan(r, &pt, gflat.data(), &est, &pseed, &pbudget);
  plan.task_grouping.groups.assign(pt.n_groups[0], {});
  for (int s_ : gflat) plan.task_grouping.groups[pt.task_group[s_]].push_back(wf.tasks[s_].id);
  for (int g = 0; g < pt.n_groups[0]; ++g) plan.gpu_grouping.counts.push_back(pt.gpu_counts[g]);
  for (int t = 0; t < T; ++t) {
    ParallelLayout l;
    l.dp = pt.dp[t];
    l.pp = pt.pp[t];
    l.tp = pt.tp[t];
    l.stage_layers.assign(pt.stage_layers + pt.sl_off[t], pt.stage_layers + pt.sl_off[t] + l.pp);
    l.replica_batch_weights.assign(pt.weights + pt.w_off[t], pt.weights + pt.w_off[t] + l.dp);
    std::vector<std::string> ids;
    for (int e = 0; e < l.dp * l.pp * l.tp; ++e)
      ids.push_back(topo.device(pt.devices[pt.dev_off[t] + e]).id);
    plan.layouts[wf.tasks[t].id] = std::move(l);
    plan.assignment[wf.tasks[t].id] = std::move(ids);
  }
  plan.provenance.seed = pseed;
  plan.provenance.budget = pbudget;
  plan.estimated_cost_s = est;
  std::vector<double> ptk(T * 7);
  double rs = 0, sy = 0, e2e = 0;
  uint8_t mf = 0;
  hpg_result_breakdown(r, ptk.data(), &rs, &sy, &e2e, &mf);
  bd = breakdown_of(wf, ptk.data(), rs, sy, e2e, mf != 0);
}

}  // namespace

SearchResult Engine::nested_sha_search(const SearchKnobs& k,
                                       const std::vector<TaskGrouping>* tg_override) {
  hpg_knobs kn = knobs_to_c(k);
  std::vector<int32_t> tgo;
  if (tg_override) {
    for (const TaskGrouping& tg : *tg_override)
      for (const RlTask& t : wf_.tasks) tgo.push_back(tg.group_of(t.id));
    kn.n_tg_override = static_cast<int32_t>(tg_override->size());
    kn.tg_override = tgo.data();
  }
  hpg_search_result* r = nullptr;
  char err[1024];
  check(hpg_search(ctx_, &kn, &r, err, sizeof(err)), err);
  hpg_search_info info;
  hpg_result_info(r, &info);
  SearchResult out;
  SearchState& s = out.state;
  s.budget = k.budget;
  s.consumed = info.consumed;
  s.seed = k.seed;
  s.task_groupings = static_cast<size_t>(info.task_groupings);
  s.b_m.resize(info.n_b_m);
  hpg_result_b_m(r, s.b_m.data());
  std::vector<int64_t> tc(info.n_trace);
  std::vector<double> tv(info.n_trace);
  hpg_result_trace(r, tc.data(), tv.data());
  for (int i = 0; i < info.n_trace; ++i) s.trace.emplace_back(tc[i], tv[i]);
  std::vector<int64_t> a0(info.n_arms), a1(info.n_arms), a3(info.n_arms);
  std::vector<double> a2(info.n_arms);
  hpg_result_arms(r, a0.data(), a1.data(), a2.data(), a3.data());
  for (int i = 0; i < info.n_arms; ++i)
    s.arms.push_back(ArmRecord{static_cast<size_t>(a0[i]), static_cast<size_t>(a1[i]), a2[i], a3[i]});
  std::vector<int32_t> hl(info.n_halvings);
  std::vector<int64_t> hb(info.n_halvings), ha(info.n_halvings);
  std::vector<double> hw(info.n_halvings), he(info.n_halvings);
  hpg_result_halvings(r, hl.data(), hb.data(), ha.data(), hw.data(), he.data());
  for (int i = 0; i < info.n_halvings; ++i)
    s.halvings.push_back(HalvingEvent{hl[i], static_cast<size_t>(hb[i]),
                                      static_cast<size_t>(ha[i]), hw[i], he[i]});
  if (info.has_plan) {
    Plan plan;
    read_plan(r, wf_, topo_, plan, out.breakdown);
    out.plan = std::move(plan);
  }
  hpg_result_free(r);
  return out;
}

ExhaustiveResult Engine::exhaustive_search(const SearchKnobs& k) {
  const hpg_knobs kn = knobs_to_c(k);
  hpg_search_result* r = nullptr;
  char err[1024];
  check(hpg_exhaustive(ctx_, &kn, &r, err, sizeof(err)), err);
  hpg_search_info info;
  hpg_result_info(r, &info);
  ExhaustiveResult out;
  out.explored = info.consumed;
  if (info.has_plan) {
    Plan plan;
    read_plan(r, wf_, topo_, plan, out.breakdown);
    out.cost = out.breakdown.end_to_end_s;
    out.plan = std::move(plan);
  }
  hpg_result_free(r);
  return out;
}

double Engine::exhaustive_space_estimate(const SearchKnobs& k) {
  const hpg_knobs kn = knobs_to_c(k);
  double est = 0;
  char err[1024];
  check(hpg_exhaustive_estimate(ctx_, &kn, &est, err, sizeof(err)), err);
  return est;
}

CostBreakdown end_to_end_cost(const Plan& plan, const WorkflowGraph& wf,
                              const DeviceTopology& topo, const CostModelConfig& cfg) {
  Engine e(wf, topo);
  return e.end_to_end_cost({plan}, cfg).at(0);
}

SearchResult nested_sha_search(const WorkflowGraph& wf, const DeviceTopology& topo,
                               const SearchKnobs& knobs,
                               const std::vector<TaskGrouping>* tg_override) {
  Engine e(wf, topo);
  return e.nested_sha_search(knobs, tg_override);
}

ExhaustiveResult exhaustive_search(const WorkflowGraph& wf, const DeviceTopology& topo,
                                   const SearchKnobs& knobs) {
  Engine e(wf, topo);
  return e.exhaustive_search(knobs);
}

TaskCostDetail task_cost_detail(const WorkflowGraph& wf, const ResolvedTask& rt,
                                const DeviceTopology& topo, const CostModelConfig& cfg,
                                std::span<const double> resident_weight_bytes) {
  Engine e(wf, topo);
  return e.task_cost_detail(rt, cfg, resident_weight_bytes);
}

TaskCost task_cost(const WorkflowGraph& wf, const ResolvedTask& rt, const DeviceTopology& topo,
                   const CostModelConfig& cfg) {
  return b200::task_cost_detail(wf, rt, topo, cfg, {}).agg;
}

namespace {
// a one-task workflow: the engine context needs one, link costs never read it
const WorkflowGraph& placeholder_workflow() {
  static const WorkflowGraph wf = [] {
    WorkflowGraph w;
    RlTask t;
    t.id = 6;
    t.kind = TaskKind::kTraining;
    t.model.hidden_size = 8;
    t.model.intermediate_size = 16;
    t.model.num_layers = 1;
    w.tasks.push_back(t);
    return w;
  }();
  return wf;
}
}  // namespace

double min_ring_bottleneck(std::span<const int> devices, double volume_bytes,
                           const DeviceTopology& topo) {
  Engine e(placeholder_workflow(), topo);
  return e.min_ring_bottleneck(devices, volume_bytes);
}

double min_pair_cost(std::span<const int> src, std::span<const int> dst, double volume_bytes,
                     const DeviceTopology& topo) {
  Engine e(placeholder_workflow(), topo);
  return e.min_pair_cost(src, dst, volume_bytes);
}

}  // namespace hetplan::b200
