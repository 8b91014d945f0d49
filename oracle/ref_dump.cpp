// ref_dump — TEST INFRASTRUCTURE ONLY (oracle side, never the product).
//
// Drives the UNMODIFIED reference planner (compiled in place from
// /root/reference/proj/src by oracle/Makefile) through its public API and
// emits golden vectors for the B200 engine's parity tests, plus the timed CPU
// baseline legs of bench.py. Doubles are written as C99 hex floats ("%a") so
// the fixtures are bit-exact.
//
// Commands:
//   fixtures OUTDIR                      c1..c4 (+acc7/acc10) workflow/topology JSON
//   evalplans WF TOPO SEED N OUT         random plans: e2e, memory, balance, evaluate
//   fuzz SEED N OUT                      acceptance-#1-style random instances
//   search WF TOPO BUDGET SEED OUT [knobs.json]   nested_sha_search + survivor replay
//   searchfuzz SEED N OUT                tiny random searches (acceptance #3/#4 style)
//   exhaustive SEED N OUT                exhaustive_search goldens (acceptance #2 + fuzz)
//   cli OUT                              reference CLI (cmd_plan/estimate/compare/scenario)
//   sweep WF TOPO SEED K0 COUNT OUT      config-5 generator
//   time_search WF TOPO BUDGET SEED [knobs.json]  one timed search, JSON line
//   time_sweep WF TOPO SEED K0 COUNT THREADS      timed sweep sample, JSON line
#include <atomic>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <numeric>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"

#include "hetplan/balance.hpp"
#include "hetplan/cli.hpp"
#include "hetplan/combinatorics.hpp"
#include "hetplan/cost_model.hpp"
#include "hetplan/errors.hpp"
#include "hetplan/plan.hpp"
#include "hetplan/rng.hpp"
#include "hetplan/search.hpp"
#include "hetplan/topology.hpp"
#include "hetplan/workflow.hpp"
#include "test_util.hpp"

using namespace hetplan;
using json = nlohmann::json;

namespace {

std::string hx(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%a", v);
  return buf;
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream out(path);
  if (!out) {
    throw std::runtime_error("cannot write " + path);
  }
  out << text;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) {
    throw std::runtime_error("cannot read " + path);
  }
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// ---- engine-neutral JSON encodings (hex doubles) ----

json workflow_json(const WorkflowGraph& wf) {
  json j;
  j["algorithm"] = to_string(wf.algorithm);
  j["mode"] = to_string(wf.mode);
  j["eta"] = hx(wf.eta);
  j["batch"] = {{"global_batch", wf.batch.global_batch},
                {"responses_per_prompt", wf.batch.responses_per_prompt},
                {"seq_in", wf.batch.seq_in},
                {"seq_out", wf.batch.seq_out},
                {"micro_batch_size", wf.batch.micro_batch_size}};
  json tasks = json::array();
  for (const RlTask& t : wf.tasks) {
    tasks.push_back({{"id", t.id},
                     {"kind", static_cast<int>(t.kind)},
                     {"model_name", t.model_name},
                     {"hidden_size", t.model.hidden_size},
                     {"intermediate_size", t.model.intermediate_size},
                     {"num_layers", t.model.num_layers},
                     {"include_embedding", t.model.include_embedding},
                     {"vocab_size", t.model.vocab_size},
                     {"precision_bytes", t.precision_bytes}});
  }
  j["tasks"] = tasks;
  json edges = json::array();
  for (const auto& [a, b] : wf.dep_edges) {
    edges.push_back({a, b});
  }
  j["dep_edges"] = edges;
  return j;
}

json topology_json(const DeviceTopology& topo) {
  json devs = json::array();
  for (const Device& d : topo.devices()) {
    devs.push_back({{"id", d.id},
                    {"gpu_model", d.gpu_model},
                    {"comp_tflops", hx(d.comp_tflops)},
                    {"mem_gb", hx(d.mem_gb)},
                    {"hbm_gbps", hx(d.hbm_gbps)},
                    {"intra_node_gbps", hx(d.intra_node_gbps)},
                    {"node", d.node},
                    {"region", d.region}});
  }
  json links = json::array();
  for (const RegionLink& rl : topo.region_links()) {
    links.push_back({{"src", rl.src},
                     {"dst", rl.dst},
                     {"latency_ms", hx(rl.latency_ms)},
                     {"bandwidth_gbps", hx(rl.bandwidth_gbps)}});
  }
  return {{"devices", devs},
          {"region_links", links},
          {"defaults",
           {{"intra_region_latency_ms", hx(topo.defaults().intra_region_latency_ms)},
            {"intra_region_bandwidth_gbps",
             hx(topo.defaults().intra_region_bandwidth_gbps)}}}};
}

json cfg_json(const CostModelConfig& c) {
  return {{"recompute", c.recompute},
          {"reshard_override", hx(c.reshard_override)},
          {"sync_override", hx(c.sync_override)},
          {"dbs_override", hx(c.dbs_override)},
          {"memory",
           {{"train_bytes_per_param", hx(c.memory.train_bytes_per_param)},
            {"infer_bytes_per_param", hx(c.memory.infer_bytes_per_param)},
            {"kv_bytes_per_elem", hx(c.memory.kv_bytes_per_elem)},
            {"dbs_cap", c.memory.dbs_cap},
            {"act_factor", hx(c.memory.act_factor)}}}};
}

json plan_json(const Plan& p, const DeviceTopology& topo) {
  json j;
  j["groups"] = p.task_grouping.groups;
  j["counts"] = p.gpu_grouping.counts;
  json layouts = json::object();
  for (const auto& [id, l] : p.layouts) {
    json w = json::array();
    for (double x : l.replica_batch_weights) {
      w.push_back(hx(x));
    }
    layouts[std::to_string(id)] = {{"dp", l.dp},
                                   {"pp", l.pp},
                                   {"tp", l.tp},
                                   {"stage_layers", l.stage_layers},
                                   {"weights", w}};
  }
  j["layouts"] = layouts;
  json asg = json::object();
  for (const auto& [id, devs] : p.assignment) {
    std::vector<int> idx;
    for (const auto& d : devs) {
      idx.push_back(topo.device_index(d));
    }
    asg[std::to_string(id)] = idx;
  }
  j["assignment"] = asg;
  j["estimated_cost_s"] = hx(p.estimated_cost_s);
  j["provenance"] = {{"seed", p.provenance.seed}, {"budget", p.provenance.budget}};
  return j;
}

json breakdown_json(const CostBreakdown& bd) {
  json pt = json::object();
  for (const auto& [id, c] : bd.per_task) {
    pt[std::to_string(id)] = {hx(c.comp), hx(c.tp), hx(c.pp), hx(c.dp),
                              hx(c.bubble), hx(c.hbm), hx(c.total)};
  }
  return {{"per_task", pt},
          {"reshard_s", hx(bd.reshard_s)},
          {"sync_s", hx(bd.sync_s)},
          {"end_to_end_s", hx(bd.end_to_end_s)},
          {"memory_feasible", bd.memory_feasible}};
}

SearchKnobs knobs_from(const std::string& path) {
  return path.empty() ? SearchKnobs{} : load_knobs(path);
}

json knobs_json(const SearchKnobs& k) {
  return {{"budget", k.budget},
          {"seed", k.seed},
          {"population", k.population},
          {"locality_bias", hx(k.locality_bias)},
          {"quantize_gpu_counts", k.quantize_gpu_counts},
          {"level1_filter", k.level1_filter},
          {"level1_cap", k.level1_cap},
          {"gg_arm_cap", k.gg_arm_cap},
          {"swap_pair_sample", k.swap_pair_sample},
          {"balance_data", k.balance_data},
          {"balance_layers", k.balance_layers},
          {"recompute", k.recompute},
          {"reshard_override", hx(k.reshard_override)},
          {"sync_override", hx(k.sync_override)}};
}

// ---- config-5 generator, written here against the
// reference's own primitives so the CPU leg and the GPU generator agree ----

Plan gen_a5(const WorkflowGraph& wf, const DeviceTopology& topo,
            const std::vector<TaskGrouping>& tgs, std::uint64_t seed,
            std::uint64_t k) {
  Rng rng = Rng(seed).fork(k);
  const int n = topo.size();
  Plan p;
  p.task_grouping = tgs[rng.bounded(tgs.size())];
  const int ng = static_cast<int>(p.task_grouping.groups.size());
  p.gpu_grouping.counts = sample_composition(n, ng, 1, rng);
  for (int g = 0; g < ng; ++g) {
    for (int id : p.task_grouping.groups[g]) {
      auto opts = enumerate_layouts(p.gpu_grouping.counts[g], wf.task(id).model,
                                    wf.batch, topo.max_devices_per_node());
      p.layouts[id] = opts[rng.bounded(opts.size())];
    }
  }
  std::vector<int> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  rng.shuffle(perm);
  int cursor = 0;
  for (int g = 0; g < ng; ++g) {
    std::vector<int> gd(perm.begin() + cursor,
                        perm.begin() + cursor + p.gpu_grouping.counts[g]);
    cursor += p.gpu_grouping.counts[g];
    for (int id : p.task_grouping.groups[g]) {
      std::vector<int> a = gd;
      rng.shuffle(a);
      std::vector<std::string> ids;
      for (int d : a) {
        ids.push_back(topo.device(d).id);
      }
      p.assignment[id] = std::move(ids);
    }
  }
  return p;
}

// ---- fixtures ----

WorkflowGraph make_wf(RlAlgorithm algo, std::int64_t h1, std::int64_t h2,
                      std::int64_t nl, std::int64_t mbs) {
  ModelSpec m;
  m.hidden_size = h1;
  m.intermediate_size = h2;
  m.num_layers = nl;
  BatchConfig b;
  b.global_batch = 1024;
  b.responses_per_prompt = 8;
  b.seq_in = 1024;
  b.seq_out = 1024;
  b.micro_batch_size = mbs;
  std::map<std::string, ModelSpec> models{{"actor", m}, {"reward", m}, {"reference", m}};
  if (algo == RlAlgorithm::kPpo) {
    models["critic"] = m;
  }
  return build_workflow(algo, RunMode::kSync, models, b, 0.5);
}

std::string workflow_file_json(const WorkflowGraph& wf) {
  // reference sample format (proj/samples/workflow-*.json)
  json j;
  j["algorithm"] = to_string(wf.algorithm);
  j["mode"] = to_string(wf.mode);
  j["eta"] = wf.eta;
  j["batch"] = {{"global_batch", wf.batch.global_batch},
                {"responses_per_prompt", wf.batch.responses_per_prompt},
                {"seq_in", wf.batch.seq_in},
                {"seq_out", wf.batch.seq_out},
                {"micro_batch_size", wf.batch.micro_batch_size}};
  json models = json::object();
  for (const RlTask& t : wf.tasks) {
    models[t.model_name] = {{"hidden_size", t.model.hidden_size},
                            {"intermediate_size", t.model.intermediate_size},
                            {"num_layers", t.model.num_layers}};
  }
  j["models"] = models;
  return j.dump(2) + "\n";
}

DeviceTopology c4_topology() {
  const char* types[4] = {"A100", "L40S", "L4", "H100"};
  const double spec[4][4] = {{312.0, 40.0, 2039.0, 600.0},
                             {366.0, 48.0, 864.0, 64.0},
                             {121.0, 24.0, 300.0, 64.0},
                             {989.0, 80.0, 3350.0, 900.0}};
  const char* regions[4] = {"virginia", "ohio", "paris", "frankfurt"};
  std::vector<Device> devs;
  for (int i = 0; i < 128; ++i) {
    const int t = (i / 8) % 4;
    Device d;
    d.id = std::string(types[t]) + "-" + std::to_string(i);
    d.gpu_model = types[t];
    d.comp_tflops = spec[t][0];
    d.mem_gb = spec[t][1];
    d.hbm_gbps = spec[t][2];
    d.intra_node_gbps = spec[t][3];
    d.region = regions[(i / 32) % 4];
    d.node = d.region + "-n" + std::to_string(i / 8);
    devs.push_back(d);
  }
  Rng rng(7);
  std::vector<RegionLink> links;
  for (int a = 0; a < 4; ++a) {
    for (int b = a + 1; b < 4; ++b) {
      const double lat = rng.uniform(5.0, 60.0);
      const double bw = rng.uniform(0.9, 5.0);
      links.push_back({regions[a], regions[b], lat, bw});
    }
  }
  TopologyDefaults def;
  def.intra_region_latency_ms = 0.1;
  def.intra_region_bandwidth_gbps = 100.0;
  return DeviceTopology::make(devs, links, def);
}

int cmd_fixtures(const std::string& dir) {
  struct Cfg {
    std::string name;
    WorkflowGraph wf;
    DeviceTopology topo;
  };
  std::vector<Cfg> cfgs;
  {
    ScenarioOptions o;
    o.inventory = {{4, "A100"}, {4, "L40S"}};
    o.seed = 7;
    cfgs.push_back({"c1", parse_workflow_json(read_file(
                              "/root/reference/proj/samples/workflow-ppo-4b.json")),
                    generate_scenario(1, o)});
  }
  {
    ScenarioOptions o;
    o.inventory = {{16, "A100"}, {16, "L40S"}};
    o.seed = 7;
    cfgs.push_back({"c2", make_wf(RlAlgorithm::kGrpo, 3584, 18944, 28, 2),
                    generate_scenario(1, o)});
  }
  {
    ScenarioOptions o;
    o.seed = 7;
    cfgs.push_back({"c3", make_wf(RlAlgorithm::kPpo, 5120, 13824, 48, 1),
                    generate_scenario(2, o)});
  }
  cfgs.push_back({"c4", make_wf(RlAlgorithm::kPpo, 5120, 27648, 64, 1), c4_topology()});
  {
    ScenarioOptions o;
    o.seed = 7;
    cfgs.push_back({"acc10", make_wf(RlAlgorithm::kPpo, 2560, 9728, 36, 1),
                    generate_scenario(3, o)});
  }
  {
    ScenarioOptions o;
    o.seed = 7;
    cfgs.push_back({"acc7mixed", make_wf(RlAlgorithm::kGrpo, 4096, 12288, 36, 2),
                    generate_scenario(1, o)});
    ScenarioOptions a;
    a.inventory = {{24, "A100"}};
    a.seed = 7;
    cfgs.push_back({"acc7a100", make_wf(RlAlgorithm::kGrpo, 4096, 12288, 36, 2),
                    generate_scenario(1, a)});
  }
  for (const Cfg& c : cfgs) {
    write_file(dir + "/" + c.name + ".workflow.json", workflow_file_json(c.wf));
    write_file(dir + "/" + c.name + ".topology.json", serialize_topology(c.topo));
  }
  std::printf("wrote %zu configs to %s\n", cfgs.size(), dir.c_str());
  return 0;
}

// evaluate() of search.cpp:259-279 restated through public calls
CostBreakdown evaluate_like_search(Plan& plan, const WorkflowGraph& wf,
                                   const DeviceTopology& topo,
                                   const SearchKnobs& k) {
  const CostModelConfig cfg = k.cost_config();
  if (k.balance_data) {
    plan = balance_data(plan, wf, topo, cfg);
  }
  if (k.balance_layers) {
    plan = balance_layers(plan, wf, topo, cfg);
  }
  return end_to_end_cost(plan, wf, topo, cfg);
}

json one_plan_record(const Plan& plan, const WorkflowGraph& wf,
                     const DeviceTopology& topo, const CostModelConfig& cfg,
                     bool with_search_eval) {
  json r;
  r["plan"] = plan_json(plan, topo);
  r["e2e"] = breakdown_json(end_to_end_cost(plan, wf, topo, cfg));
  const auto viol = check_memory(plan, topo, wf, cfg.memory);
  json v = json::array();
  for (const auto& m : viol) {
    v.push_back({topo.device_index(m.device_id), hx(m.required_bytes),
                 hx(m.capacity_bytes)});
  }
  r["violations"] = v;
  const Plan bdp = balance_data(plan, wf, topo, cfg);
  r["balance_data"] = plan_json(bdp, topo);
  const Plan blp = balance_layers(plan, wf, topo, cfg);
  r["balance_layers"] = plan_json(blp, topo);
  if (with_search_eval) {
    SearchKnobs k;
    Plan p = plan;
    const CostBreakdown bd = evaluate_like_search(p, wf, topo, k);
    r["evaluate"] = {{"plan", plan_json(p, topo)}, {"bd", breakdown_json(bd)}};
  }
  return r;
}

int cmd_evalplans(const std::string& wfp, const std::string& tpp,
                  std::uint64_t seed, int n, const std::string& out) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  const auto tgs = enumerate_task_groupings(wf);
  SearchKnobs k;
  const CostModelConfig cfg = k.cost_config();
  Rng rng(seed);
  json recs = json::array();
  for (int i = 0; i < n; ++i) {
    std::optional<Plan> plan;
    if (i % 2 == 0) {
      plan = gen_a5(wf, topo, tgs, seed, static_cast<std::uint64_t>(i));
    } else {
      plan = testutil::random_plan(wf, topo, rng);
    }
    if (!plan) {
      continue;
    }
    recs.push_back(one_plan_record(*plan, wf, topo, cfg, true));
  }
  json j;
  j["workflow"] = workflow_json(wf);
  j["topology"] = topology_json(topo);
  j["cfg"] = cfg_json(cfg);
  j["records"] = recs;
  write_file(out, j.dump() + "\n");
  std::printf("wrote %zu records to %s\n", recs.size(), out.c_str());
  return 0;
}

WorkflowGraph random_workflow(Rng& rng) {
  const auto algo = rng.bounded(2) == 0 ? RlAlgorithm::kPpo : RlAlgorithm::kGrpo;
  const auto mode = rng.bounded(2) == 0 ? RunMode::kSync : RunMode::kAsync;
  auto rnd_model = [&]() {
    ModelSpec m = testutil::tiny_model(
        4 + 4 * static_cast<std::int64_t>(rng.bounded(8)),
        8 + 8 * static_cast<std::int64_t>(rng.bounded(8)),
        1 + static_cast<std::int64_t>(rng.bounded(8)));
    if (rng.bounded(4) == 0) {
      m.include_embedding = true;
      m.vocab_size = 16 + static_cast<std::int64_t>(rng.bounded(200));
    }
    return m;
  };
  const auto batch = testutil::tiny_batch(
      1 + static_cast<std::int64_t>(rng.bounded(32)),
      1 + static_cast<std::int64_t>(rng.bounded(4)),
      1 + static_cast<std::int64_t>(rng.bounded(128)),
      static_cast<std::int64_t>(rng.bounded(128)),
      1 + static_cast<std::int64_t>(rng.bounded(4)));
  const double eta = rng.uniform();
  const int shape = static_cast<int>(rng.bounded(3));
  if (shape == 0) {
    // full workflow, one shared model
    return testutil::full_workflow(algo, mode, rnd_model(), batch, eta);
  }
  if (shape == 1) {
    std::map<std::string, ModelSpec> models{{"actor", rnd_model()},
                                            {"critic", rnd_model()},
                                            {"reward", rnd_model()},
                                            {"reference", rnd_model()}};
    WorkflowGraph wf = build_workflow(algo, mode, models, batch, eta);
    for (RlTask& t : wf.tasks) {
      if (rng.bounded(6) == 0) {
        t.precision_bytes = 4;
      }
    }
    return wf;
  }
  // task subset (tiny search instances)
  std::vector<int> ids;
  for (int id = 1; id <= 6; ++id) {
    if (rng.bounded(2) == 0) {
      ids.push_back(id);
    }
  }
  if (ids.empty()) {
    ids.push_back(1 + static_cast<int>(rng.bounded(6)));
  }
  std::map<int, ModelSpec> tm;
  for (int id : ids) {
    tm[id] = rnd_model();
  }
  return testutil::subset_workflow_models(tm, batch, mode, eta);
}

CostModelConfig random_cfg(Rng& rng) {
  CostModelConfig cfg;
  cfg.recompute = rng.bounded(2) == 0;
  const int d = static_cast<int>(rng.bounded(3));
  cfg.dbs_override = d == 0 ? -1.0 : (d == 1 ? 1.0 + static_cast<double>(rng.bounded(4))
                                             : rng.uniform(0.5, 6.0));
  if (rng.bounded(2) == 0) {
    cfg.reshard_override = rng.bounded(3) == 0 ? 0.0 : rng.uniform(0.0, 3.0);
  }
  if (rng.bounded(2) == 0) {
    cfg.sync_override = rng.uniform(0.0, 3.0);
  }
  if (rng.bounded(3) == 0) {
    cfg.memory.train_bytes_per_param = rng.uniform(8.0, 24.0);
    cfg.memory.infer_bytes_per_param = rng.uniform(1.0, 4.0);
    cfg.memory.kv_bytes_per_elem = rng.uniform(1.0, 4.0);
    cfg.memory.dbs_cap = 1 + static_cast<int>(rng.bounded(4));
    cfg.memory.act_factor = rng.uniform(1.0, 8.0);
  }
  return cfg;
}

int cmd_fuzz(std::uint64_t seed, int n, const std::string& out) {
  Rng rng(seed);
  json recs = json::array();
  int made = 0;
  while (made < n) {
    const WorkflowGraph wf = random_workflow(rng);
    const DeviceTopology topo = testutil::random_topology(rng, 8);
    const auto plan = testutil::random_plan(wf, topo, rng);
    if (!plan) {
      continue;
    }
    const CostModelConfig cfg = random_cfg(rng);
    json r = one_plan_record(*plan, wf, topo, cfg, false);
    r["workflow"] = workflow_json(wf);
    r["topology"] = topology_json(topo);
    r["cfg"] = cfg_json(cfg);
    recs.push_back(r);
    ++made;
  }
  write_file(out, json{{"records", recs}}.dump() + "\n");
  std::printf("wrote %d fuzz records to %s\n", made, out.c_str());
  return 0;
}

// ---- search with per-halving survivor replay ----

int ceil_log2(std::size_t n) {
  int r = 0;
  std::size_t v = 1;
  while (v < n) {
    v <<= 1;
    ++r;
  }
  return r;
}

// Replays nested_sha_search's schedule (search.cpp:624-835) through the public
// ga_search entry point so the survivor set of every halving round can be
// logged; the reference's SearchState does not expose it (search.hpp:79-103).
// Cross-checked against the real search's arms/halvings by the caller.
json replay_survivors(const WorkflowGraph& wf, const DeviceTopology& topo,
                      const SearchKnobs& knobs, std::vector<ArmRecord>& arms_out,
                      std::vector<HalvingEvent>& halvings_out) {
  const Rng base_rng(knobs.seed);
  std::function<bool(const TaskGrouping&)> filter;
  if (knobs.level1_filter == "adjacent") {
    filter = [&wf](const TaskGrouping& tg) {
      for (const auto& group : tg.groups) {
        if (group.size() < 2) continue;
        bool adjacent = false;
        for (int a : group)
          for (int b : group)
            if (wf.dep_edges.count({a, b}) != 0) adjacent = true;
        if (!adjacent) return false;
      }
      return true;
    };
  }
  std::vector<TaskGrouping> tgs = enumerate_task_groupings(wf, filter);
  if (knobs.level1_cap > 0 && tgs.size() > static_cast<std::size_t>(knobs.level1_cap)) {
    tgs.resize(knobs.level1_cap);
  }
  const int n_devices = topo.size();
  struct TgArm {
    std::vector<GpuGrouping> ggs;
    std::vector<double> best;
    std::vector<std::size_t> alive;
    std::vector<std::size_t> rec;
  };
  std::vector<TgArm> tga;
  arms_out.clear();
  for (std::size_t ti = 0; ti < tgs.size(); ++ti) {
    TgArm arm;
    const int k = static_cast<int>(tgs[ti].groups.size());
    if (k <= n_devices) {
      int q = knobs.quantize_gpu_counts;
      double count = composition_count(n_devices, k, q);
      if (count == 0) {
        q = 1;
        count = composition_count(n_devices, k, q);
      }
      if (count <= knobs.gg_arm_cap) {
        arm.ggs = enumerate_gpu_groupings(n_devices, k, q);
      } else {
        std::set<std::vector<int>> seen;
        std::vector<int> balanced(k, n_devices / k);
        for (int i = 0; i < n_devices % k; ++i) ++balanced[i];
        seen.insert(balanced);
        arm.ggs.push_back(GpuGrouping{balanced});
        Rng rng = base_rng.fork(0xA001 + ti);
        for (std::int64_t tries = 0; static_cast<int>(arm.ggs.size()) < knobs.gg_arm_cap &&
                                     tries < 50LL * knobs.gg_arm_cap;
             ++tries) {
          auto comp = sample_composition(n_devices, k, q, rng);
          if (seen.insert(comp).second) arm.ggs.push_back(GpuGrouping{std::move(comp)});
        }
      }
    }
    arm.best.assign(arm.ggs.size(), std::numeric_limits<double>::infinity());
    for (std::size_t gi = 0; gi < arm.ggs.size(); ++gi) {
      arm.alive.push_back(gi);
      arm.rec.push_back(arms_out.size());
      ArmRecord r;
      r.tg_index = ti;
      r.gg_index = gi;
      arms_out.push_back(r);
    }
    tga.push_back(std::move(arm));
  }
  json survivors = json::array();
  auto best_half = [&](const std::vector<std::size_t>& arms, auto score, int level) {
    if (arms.size() <= 1) return arms;
    std::vector<std::size_t> order = arms;
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
      const double sa = score(a), sb = score(b);
      if (sa != sb) return sa < sb;
      return a < b;
    });
    const std::size_t keep = (order.size() + 1) / 2;
    std::vector<std::size_t> surv(order.begin(), order.begin() + keep);
    HalvingEvent ev;
    ev.level = level;
    ev.before = order.size();
    ev.after = keep;
    ev.survivor_worst = score(surv.back());
    ev.eliminated_best = score(order[keep]);
    halvings_out.push_back(ev);
    std::sort(surv.begin(), surv.end());
    survivors.push_back(surv);
    return surv;
  };
  std::int64_t consumed = 0;
  auto run_arm = [&](std::size_t ti, std::size_t gi, std::int64_t slice, int m, int n) {
    if (consumed >= knobs.budget || slice < 1) return;
    TgArm& arm = tga[ti];
    const std::uint64_t salt = (static_cast<std::uint64_t>(ti) << 40) |
                               (static_cast<std::uint64_t>(gi) << 16) |
                               (static_cast<std::uint64_t>(m) << 8) |
                               static_cast<std::uint64_t>(n);
    const GaResult r = ga_search(tgs[ti], arm.ggs[gi], wf, topo, slice,
                                 base_rng.fork(salt), knobs);
    ArmRecord& rec = arms_out[arm.rec[gi]];
    rec.evals += r.evals;
    rec.best_cost = std::min(rec.best_cost, r.cost);
    consumed += r.evals;
    arm.best[gi] = rec.best_cost;
  };
  auto run_tg_round = [&](std::size_t ti, std::int64_t b, int m) {
    TgArm& arm = tga[ti];
    if (arm.alive.empty()) return;
    const std::vector<std::size_t> entry = arm.alive;
    const int denom_in = std::max(1, ceil_log2(entry.size()));
    std::vector<std::size_t> cur = entry;
    for (int n = 0; n < std::max(1, ceil_log2(entry.size())); ++n) {
      const std::int64_t b_mn = b / (static_cast<std::int64_t>(cur.size()) * denom_in);
      if (b_mn >= 1) {
        for (std::size_t gi : cur) run_arm(ti, gi, b_mn, m, n);
      } else {
        std::int64_t rb = b / denom_in;
        if (rb == 0 && n == 0) rb = b;
        std::int64_t spent = 0;
        for (std::size_t gi : cur) {
          if (spent >= rb || consumed >= knobs.budget) break;
          run_arm(ti, gi, 1, m, n);
          ++spent;
        }
      }
      cur = best_half(cur, [&](std::size_t gi) { return arm.best[gi]; }, 2);
    }
    arm.alive = best_half(entry, [&](std::size_t gi) { return arm.best[gi]; }, 2);
  };
  auto tg_score = [&](std::size_t ti) {
    double best = std::numeric_limits<double>::infinity();
    for (double c : tga[ti].best) best = std::min(best, c);
    return best;
  };
  std::vector<std::size_t> surv;
  for (std::size_t ti = 0; ti < tgs.size(); ++ti) surv.push_back(ti);
  const int denom_out = std::max(1, ceil_log2(tgs.size()));
  for (int m = 0; m < denom_out; ++m) {
    const std::int64_t b_m = knobs.budget / (static_cast<std::int64_t>(surv.size()) * denom_out);
    if (b_m >= 1) {
      for (std::size_t ti : surv) run_tg_round(ti, b_m, m);
    } else {
      std::int64_t ob = knobs.budget / denom_out;
      if (ob == 0 && m == 0) ob = knobs.budget;
      std::int64_t spent = 0;
      for (std::size_t ti : surv) {
        if (spent >= ob || consumed >= knobs.budget) break;
        run_tg_round(ti, 1, m);
        ++spent;
      }
    }
    surv = best_half(surv, tg_score, 1);
  }
  return survivors;
}

json search_record(const WorkflowGraph& wf, const DeviceTopology& topo,
                   const SearchKnobs& knobs, bool replay, double* wall_out) {
  const auto t0 = std::chrono::steady_clock::now();
  const SearchResult res = nested_sha_search(wf, topo, knobs);
  const double wall =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (wall_out) *wall_out = wall;
  json j;
  j["knobs"] = knobs_json(knobs);
  const SearchState& s = res.state;
  j["consumed"] = s.consumed;
  j["budget"] = s.budget;
  j["b_m"] = s.b_m;
  j["task_groupings"] = s.task_groupings;
  json tr = json::array();
  for (const auto& [c, v] : s.trace) tr.push_back({c, hx(v)});
  j["trace"] = tr;
  json arms = json::array();
  for (const auto& a : s.arms) {
    arms.push_back({a.tg_index, a.gg_index, hx(a.best_cost), a.evals});
  }
  j["arms"] = arms;
  json hv = json::array();
  for (const auto& h : s.halvings) {
    hv.push_back({h.level, h.before, h.after, hx(h.survivor_worst), hx(h.eliminated_best)});
  }
  j["halvings"] = hv;
  j["has_plan"] = res.plan.has_value();
  if (res.plan) {
    j["plan"] = plan_json(*res.plan, topo);
    j["breakdown"] = breakdown_json(res.breakdown);
  }
  j["wall_s"] = wall;
  if (replay) {
    std::vector<ArmRecord> arms2;
    std::vector<HalvingEvent> halv2;
    json surv = replay_survivors(wf, topo, knobs, arms2, halv2);
    bool ok = arms2.size() == s.arms.size() && halv2.size() == s.halvings.size();
    for (std::size_t i = 0; ok && i < arms2.size(); ++i) {
      ok = arms2[i].best_cost == s.arms[i].best_cost && arms2[i].evals == s.arms[i].evals;
    }
    for (std::size_t i = 0; ok && i < halv2.size(); ++i) {
      ok = halv2[i].before == s.halvings[i].before && halv2[i].after == s.halvings[i].after &&
           halv2[i].survivor_worst == s.halvings[i].survivor_worst &&
           halv2[i].eliminated_best == s.halvings[i].eliminated_best &&
           halv2[i].level == s.halvings[i].level;
    }
    j["survivors"] = surv;
    j["replay_consistent"] = ok;
    if (!ok) {
      std::fprintf(stderr, "WARNING: survivor replay diverged from nested_sha_search\n");
    }
  }
  return j;
}

int cmd_search(const std::string& wfp, const std::string& tpp, std::int64_t budget,
               std::uint64_t seed, const std::string& out, const std::string& knobs_path) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  SearchKnobs k = knobs_from(knobs_path);
  k.budget = budget;
  k.seed = seed;
  double wall = 0;
  json j = search_record(wf, topo, k, true, &wall);
  j["workflow"] = workflow_json(wf);
  j["topology"] = topology_json(topo);
  write_file(out, j.dump() + "\n");
  std::printf("search consumed %" PRId64 " in %.3f s, replay %s -> %s\n",
              j["consumed"].get<std::int64_t>(), wall,
              j["replay_consistent"].get<bool>() ? "consistent" : "DIVERGED", out.c_str());
  return j["replay_consistent"].get<bool>() ? 0 : 1;
}


// ga_search (search.hpp:127-135) on its own: for a few arms of a fixture
// (task grouping from enumerate_task_groupings, GPU grouping from
// enumerate_gpu_groupings) and slices/seeds, the best member's plan and
// cost, the evaluations used and its breakdown.
int cmd_ga(const std::string& wfp, const std::string& tpp, const std::string& out,
           const std::string& knobs_path) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  SearchKnobs k = knobs_from(knobs_path);
  const auto tgs = enumerate_task_groupings(wf);
  json recs = json::array();
  Rng pick(2024);
  for (int c = 0; c < 12; ++c) {
    const TaskGrouping& tg = tgs[pick.bounded(tgs.size())];
    const auto ggs = enumerate_gpu_groupings(topo.size(), static_cast<int>(tg.groups.size()), 1);
    if (ggs.empty()) continue;
    const GpuGrouping& gg = ggs[pick.bounded(ggs.size())];
    const std::int64_t slice = 1 + static_cast<std::int64_t>(pick.bounded(c < 6 ? 40 : 400));
    const std::uint64_t seed = pick.next();
    const GaResult r = ga_search(tg, gg, wf, topo, slice, Rng(seed), k);
    json j;
    j["groups"] = tg.groups;
    j["counts"] = gg.counts;
    j["slice"] = slice;
    j["seed"] = std::to_string(seed);
    j["evals"] = r.evals;
    j["cost"] = hx(r.cost);
    j["has_plan"] = r.plan.has_value();
    if (r.plan) {
      j["plan"] = plan_json(*r.plan, topo);
      j["breakdown"] = breakdown_json(r.breakdown);
    }
    recs.push_back(j);
  }
  json o;
  o["knobs"] = knobs_json(k);
  o["workflow"] = workflow_json(wf);
  o["topology"] = topology_json(topo);
  o["records"] = recs;
  write_file(out, o.dump() + "\n");
  std::printf("ga %zu records -> %s\n", recs.size(), out.c_str());
  return 0;
}

int cmd_searchfuzz(std::uint64_t seed, int n, const std::string& out) {
  Rng rng(seed);
  json recs = json::array();
  bool all_ok = true;
  for (int i = 0; i < n; ++i) {
    const auto algo = rng.bounded(2) == 0 ? RlAlgorithm::kPpo : RlAlgorithm::kGrpo;
    WorkflowGraph wf;
    if (rng.bounded(3) == 0) {
      wf = random_workflow(rng);
    } else {
      wf = testutil::full_workflow(
          algo, rng.bounded(2) == 0 ? RunMode::kSync : RunMode::kAsync,
          testutil::tiny_model(8LL << rng.bounded(3), 16LL << rng.bounded(3),
                               1 + static_cast<std::int64_t>(rng.bounded(6))),
          testutil::tiny_batch(1 + rng.bounded(8), 1 + rng.bounded(2), 1 + rng.bounded(32),
                               rng.bounded(32), 1 + rng.bounded(2)),
          rng.uniform());
    }
    const DeviceTopology topo = testutil::random_topology(rng, 8);
    SearchKnobs k;
    k.budget = 1 + static_cast<std::int64_t>(rng.bounded(400));
    k.seed = rng.next();
    k.balance_data = rng.bounded(4) != 0;
    k.balance_layers = rng.bounded(4) != 0;
    k.recompute = rng.bounded(2) == 0;
    k.population = 1 + static_cast<int>(rng.bounded(20));
    k.locality_bias = rng.uniform();
    k.swap_pair_sample = static_cast<int>(rng.bounded(10));
    k.gg_arm_cap = 1 + static_cast<int>(rng.bounded(12));
    k.quantize_gpu_counts = 1 + static_cast<int>(rng.bounded(2));
    k.level1_filter = rng.bounded(3) == 0 ? "adjacent" : "off";
    k.level1_cap = rng.bounded(3) == 0 ? 1 + static_cast<int>(rng.bounded(8)) : 0;
    if (rng.bounded(4) == 0) k.reshard_override = rng.uniform(0.0, 2.0);
    if (rng.bounded(4) == 0) k.sync_override = rng.uniform(0.0, 2.0);
    json r = search_record(wf, topo, k, true, nullptr);
    all_ok = all_ok && r["replay_consistent"].get<bool>();
    r["workflow"] = workflow_json(wf);
    r["topology"] = topology_json(topo);
    recs.push_back(r);
  }
  write_file(out, json{{"records", recs}}.dump() + "\n");
  std::printf("wrote %d search records to %s (replay %s)\n", n, out.c_str(),
              all_ok ? "consistent" : "DIVERGED");
  return all_ok ? 0 : 1;
}

// ---- exhaustive_search goldens (search.cpp:837-1031; acceptance #2) ----

json exh_record(const std::string& name, const WorkflowGraph& wf, const DeviceTopology& topo,
                const SearchKnobs& k) {
  json r;
  r["name"] = name;
  r["workflow"] = workflow_json(wf);
  r["topology"] = topology_json(topo);
  r["knobs"] = knobs_json(k);
  r["exhaustive_cap"] = hx(k.exhaustive_cap);
  r["estimate"] = hx(exhaustive_space_estimate(wf, topo, k));
  try {
    const auto t0 = std::chrono::steady_clock::now();
    const ExhaustiveResult ex = exhaustive_search(wf, topo, k);
    if (std::getenv("HPG_REF_TIMING"))  // timing probes only, not in the goldens
      r["ref_wall_s"] =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r["explored"] = ex.explored;
    r["cost"] = hx(ex.cost);
    r["has_plan"] = ex.plan.has_value();
    if (ex.plan) {
      r["plan"] = plan_json(*ex.plan, topo);
      r["breakdown"] = breakdown_json(ex.breakdown);
    }
  } catch (const InputError& e) {
    r["error"] = e.what();
  }
  return r;
}

// two regions x two single-GPU nodes (the level-5 swap / SHA test fixture shape)
DeviceTopology two_region_pairs() {
  std::vector<Device> devs(4);
  for (int i = 0; i < 4; ++i) {
    Device& d = devs[i];
    d.id = "dev-" + std::to_string(i);
    d.gpu_model = "synthetic";
    d.comp_tflops = 10;
    d.mem_gb = 640;
    d.hbm_gbps = 1000;
    d.intra_node_gbps = 600;
    d.region = i < 2 ? "east" : "west";
    d.node = d.region + "-n" + std::to_string(i % 2);
  }
  return DeviceTopology::make(devs, {{"east", "west", 50.0, 1.0}}, TopologyDefaults{0.05, 100.0});
}

int cmd_exhaustive(std::uint64_t seed, int n_fuzz, const std::string& out) {
  json recs = json::array();
  auto quiet = [](std::int64_t budget, std::uint64_t s) {
    SearchKnobs k;
    k.budget = budget;
    k.seed = s;
    k.balance_data = false;
    k.balance_layers = false;
    return k;
  };
  // acceptance #2's twenty instances (acceptance.cpp:116-141)
  for (int i = 0; i < 20; ++i) {
    Rng rng(5000 + i);
    std::map<int, ModelSpec> models;
    if (i % 4 == 0) {
      models[6] = testutil::tiny_model(8, 16, 2 + i % 3);
    } else if (i % 4 == 1) {
      models[2] = testutil::tiny_model(8, 16, 2);
      models[6] = testutil::tiny_model(8, 16, 4);
    } else if (i % 4 == 2) {
      models[1] = testutil::tiny_model(8, 16, 2);
      models[6] = testutil::tiny_model(8, 16, 2);
    } else {
      models[2] = testutil::tiny_model(8, 16, 2);
      models[3] = testutil::tiny_model(16, 32, 2);
    }
    const auto wf = testutil::subset_workflow_models(
        models, testutil::tiny_batch(4, 1, 8, 4, 1),
        i % 2 == 0 ? RunMode::kSync : RunMode::kAsync, 0.25);
    const int n_devices = 2 + static_cast<int>(rng.bounded(3));
    const DeviceTopology topo = i % 3 == 0
                                    ? testutil::uniform_topology(n_devices, 1e13, 1e12, 64.0, 2)
                                    : testutil::random_topology(rng, 4);
    recs.push_back(exh_record("acc2_" + std::to_string(i), wf, topo, quiet(0, 0)));
  }
  // test_search.cpp:284-320 shapes, the two-region fixture, the cap guard
  recs.push_back(exh_record(
      "one_task_one_device",
      testutil::subset_workflow({2}, testutil::tiny_model(4, 8, 2), testutil::tiny_batch()),
      testutil::uniform_topology(1, 1e13, 1e12, 64.0, 1), quiet(0, 0)));
  recs.push_back(exh_record(
      "train_two_same_node",
      testutil::subset_workflow({6}, testutil::tiny_model(4, 8, 2), testutil::tiny_batch()),
      testutil::uniform_topology(2, 1e13, 1e12, 64.0, 2), quiet(0, 0)));
  recs.push_back(exh_record("cap_guard",
                            testutil::subset_workflow({1, 2, 6}, testutil::tiny_model(4, 8, 2),
                                                      testutil::tiny_batch()),
                            testutil::uniform_topology(16, 1e13, 1e12, 64.0, 8), quiet(0, 0)));
  recs.push_back(exh_record(
      "two_region_train",
      testutil::subset_workflow({6}, testutil::tiny_model(8, 16, 2),
                                testutil::tiny_batch(8, 1, 16, 0, 1)),
      two_region_pairs(), quiet(0, 0)));
  {
    std::map<int, ModelSpec> models{{2, testutil::tiny_model(8, 16, 2)},
                                    {6, testutil::tiny_model(8, 16, 4)}};
    recs.push_back(exh_record("two_region_pair",
                              testutil::subset_workflow_models(
                                  models, testutil::tiny_batch(4, 1, 8, 0, 1), RunMode::kSync, 0.0),
                              two_region_pairs(), quiet(0, 0)));
  }
  // fuzz: random workflows on small random / uniform / duplicated-type pools
  Rng rng(seed);
  for (int i = 0; i < n_fuzz; ++i) {
    WorkflowGraph wf = random_workflow(rng);
    DeviceTopology topo;
    const int shape = static_cast<int>(rng.bounded(3));
    if (shape == 0) {
      topo = testutil::random_topology(rng, 5);
    } else if (shape == 1) {
      topo = testutil::uniform_topology(1 + static_cast<int>(rng.bounded(6)),
                                        rng.uniform(1e12, 4e14), rng.uniform(1e11, 3e12),
                                        rng.uniform(8.0, 96.0), 1 + static_cast<int>(rng.bounded(4)));
    } else {
      // two device types over two nodes (symmetry classes with repeats)
      const int n = 2 + static_cast<int>(rng.bounded(5));
      std::vector<Device> devs(n);
      for (int d = 0; d < n; ++d) {
        Device& x = devs[d];
        x.id = "g" + std::to_string(d);
        const bool big = rng.bounded(2) == 0;
        x.gpu_model = big ? "big" : "small";
        x.comp_tflops = big ? 312.0 : 181.0;
        x.mem_gb = big ? 80.0 : 48.0;
        x.hbm_gbps = big ? 2039.0 : 864.0;
        x.intra_node_gbps = big ? 600.0 : 64.0;
        x.region = "r0";
        x.node = "n" + std::to_string(rng.bounded(2));
      }
      topo = DeviceTopology::make(devs, {}, TopologyDefaults{0.1, 100.0});
    }
    SearchKnobs k = quiet(0, 0);
    k.recompute = rng.bounded(2) == 0;
    if (rng.bounded(4) == 0) k.reshard_override = rng.uniform(0.0, 2.0);
    if (rng.bounded(4) == 0) k.sync_override = rng.uniform(0.0, 2.0);
    if (rng.bounded(3) == 0) k.exhaustive_cap = 1e4 * (1 + static_cast<double>(rng.bounded(100)));
    recs.push_back(exh_record("fuzz_" + std::to_string(i), wf, topo, k));
  }
  write_file(out, json{{"records", recs}}.dump() + "\n");
  std::printf("wrote %zu exhaustive records to %s\n", recs.size(), out.c_str());
  return 0;
}

// ---- CLI goldens: the reference's own cmd_* (cli.cpp:76-283) on fixed
// command lines; paths relative to the repo root, {tmp} = a scratch dir ----

std::string subst_tmp(std::string s, const std::string& tmp) {
  for (size_t p = s.find(tmp); p != std::string::npos; p = s.find(tmp, p)) {
    s.replace(p, tmp.size(), "{tmp}");
    p += 5;
  }
  return s;
}

int cmd_cli(const std::string& out_path) {
  char tmpl[] = "/tmp/hpg_cli_XXXXXX";
  const std::string tmp = mkdtemp(tmpl);
  json cases = json::array();
  auto file_text = [&](const std::string& path) {
    std::ifstream in(path);
    std::stringstream ss;
    ss << in.rdbuf();
    return subst_tmp(ss.str(), tmp);
  };
  auto record = [&](const std::string& name, const std::vector<std::string>& argv, int rc,
                    const std::string& out, const std::string& err,
                    const std::vector<std::string>& files) {
    json c;
    c["name"] = name;
    c["args"] = argv;
    c["rc"] = rc;
    c["stdout"] = subst_tmp(out, tmp);
    c["stderr"] = subst_tmp(err, tmp);
    json f = json::object();
    for (const auto& fn : files) f[fn] = file_text(tmp + "/" + fn);
    c["files"] = f;
    cases.push_back(c);
  };
  const std::string K = "tests/golden/cli/knobs.json";
  auto fx = [](const std::string& c, const char* kind) {
    return "fixtures/" + c + "." + kind + ".json";
  };
  auto plan = [&](const std::string& name, const std::string& cfg, const std::string& knobs,
                  std::optional<std::int64_t> budget, std::optional<std::uint64_t> seed,
                  const std::string& out_file, const std::string& format) {
    PlanArgs a;
    a.workflow_path = fx(cfg, "workflow");
    a.topology_path = fx(cfg, "topology");
    a.knobs_path = knobs;
    a.out_path = tmp + "/" + out_file;
    a.budget = budget;
    a.seed = seed;
    a.format = format;
    std::ostringstream o, e;
    const int rc = cmd_plan(a, o, e);
    std::vector<std::string> argv = {"plan", "--workflow", a.workflow_path, "--topology",
                                     a.topology_path};
    if (!knobs.empty()) argv.insert(argv.end(), {"--knobs", knobs});
    if (budget) argv.insert(argv.end(), {"--budget", std::to_string(*budget)});
    if (seed) argv.insert(argv.end(), {"--seed", std::to_string(*seed)});
    argv.insert(argv.end(), {"--out", "{tmp}/" + out_file, "--format", format});
    record(name, argv, rc, o.str(), e.str(), rc == 0 ? std::vector<std::string>{out_file}
                                                     : std::vector<std::string>{});
  };
  plan("plan_c1_json", "c1", "", 1000, 42, "p1.json", "json");
  plan("plan_c1_text", "c1", K, std::nullopt, 7, "p2.json", "text");
  plan("plan_c2_knobs", "c2", K, 300, 11, "p3.json", "json");
  auto estimate = [&](const std::string& name, const std::string& cfg, const std::string& pfile,
                      const std::string& knobs, const std::string& format) {
    EstimateArgs a;
    a.plan_path = tmp + "/" + pfile;
    a.workflow_path = fx(cfg, "workflow");
    a.topology_path = fx(cfg, "topology");
    a.knobs_path = knobs;
    a.format = format;
    std::ostringstream o, e;
    const int rc = cmd_estimate(a, o, e);
    std::vector<std::string> argv = {"estimate", "--plan", "{tmp}/" + pfile, "--workflow",
                                     a.workflow_path, "--topology", a.topology_path};
    if (!knobs.empty()) argv.insert(argv.end(), {"--knobs", knobs});
    argv.insert(argv.end(), {"--format", format});
    record(name, argv, rc, o.str(), e.str(), {});
  };
  estimate("estimate_json", "c1", "p1.json", "", "json");
  estimate("estimate_text_knobs", "c1", "p2.json", K, "text");
  estimate("estimate_missing_plan", "c1", "nope.json", "", "json");
  {
    // a plan file naming an unknown device
    std::string t = file_text(tmp + "/p1.json");
    const auto pos = t.find("\"a100-00\"");
    if (pos != std::string::npos) t.replace(pos, 9, "\"zz-99\"");
    std::ofstream(tmp + "/bad.json") << subst_tmp(t, "{tmp}");
    estimate("estimate_unknown_device", "c1", "bad.json", "", "json");
  }
  auto compare = [&](const std::string& name, const std::vector<std::string>& pfiles,
                     const std::string& knobs, const std::string& format) {
    CompareArgs a;
    for (const auto& p : pfiles) a.plan_paths.push_back(tmp + "/" + p);
    a.workflow_path = fx("c1", "workflow");
    a.topology_path = fx("c1", "topology");
    a.knobs_path = knobs;
    a.format = format;
    std::ostringstream o, e;
    const int rc = cmd_compare(a, o, e);
    std::vector<std::string> argv = {"compare"};
    for (const auto& p : pfiles) argv.push_back("{tmp}/" + p);
    argv.insert(argv.end(), {"--workflow", a.workflow_path, "--topology", a.topology_path});
    if (!knobs.empty()) argv.insert(argv.end(), {"--knobs", knobs});
    argv.insert(argv.end(), {"--format", format});
    record(name, argv, rc, o.str(), e.str(), {});
  };
  compare("compare_json", {"p2.json", "p1.json"}, "", "json");
  compare("compare_text", {"p1.json", "p2.json", "p1.json"}, K, "text");
  compare("compare_one_plan", {"p1.json"}, "", "json");
  auto scenario = [&](const std::string& name, int id, const std::string& gpus,
                      std::optional<std::uint64_t> seed, int node_size,
                      const std::string& edge, const std::string& out_file) {
    ScenarioArgs a;
    a.scenario_id = id;
    a.gpus = gpus;
    a.seed = seed;
    a.out_path = tmp + "/" + out_file;
    a.node_size = node_size;
    a.edge_gpus = edge;
    std::ostringstream o, e;
    const int rc = cmd_scenario(a, o, e);
    std::vector<std::string> argv = {"scenario", "--id", std::to_string(id)};
    if (!gpus.empty()) argv.insert(argv.end(), {"--gpus", gpus});
    if (seed) argv.insert(argv.end(), {"--seed", std::to_string(*seed)});
    argv.insert(argv.end(), {"--out", "{tmp}/" + out_file, "--node-size",
                             std::to_string(node_size), "--edge-gpus", edge});
    record(name, argv, rc, o.str(), e.str(), rc == 0 ? std::vector<std::string>{out_file}
                                                     : std::vector<std::string>{});
  };
  scenario("scenario1_default", 1, "", 3, 8, "L4", "s1.json");
  scenario("scenario1_mixed", 1, "6xA100,3xL4,5xL40S", 3, 4, "L4", "s1b.json");
  scenario("scenario2_edges", 2, "8xA100,8xL40S,4xL4", 9, 8, "L4,L40S", "s2.json");
  scenario("scenario3", 3, "", 11, 8, "L4", "s3.json");
  scenario("scenario4", 4, "10xL40S,6xA100", 5, 8, "L4", "s4.json");
  scenario("scenario_bad_inventory", 1, "24A100", 1, 8, "L4", "sx.json");
  scenario("scenario_unknown_model", 1, "4xH200", 1, 8, "L4", "sx.json");
  scenario("scenario_bad_id", 9, "", 1, 8, "L4", "sx.json");
  {
    PlanArgs a;  // usage error: no topology
    a.workflow_path = fx("c1", "workflow");
    std::ostringstream o, e;
    const int rc = cmd_plan(a, o, e);
    record("plan_missing_topology", {"plan", "--workflow", a.workflow_path, "--seed", "1"}, rc,
           o.str(), e.str(), {});
  }
  // ---- error paths: defective plan / topology / workflow files through
  // cmd_estimate (resolve_plan, DeviceTopology::make, build_workflow
  // validation; JSON schema errors) ----
  const json good_plan = json::parse(file_text(tmp + "/p1.json"));
  const json good_topo = json::parse(read_file(fx("c1", "topology")));
  const json good_wf = json::parse(read_file(fx("c1", "workflow")));
  auto err_case = [&](const std::string& name, const json& plan, const json& topo,
                      const json& wf) {
    const std::string pf = name + ".plan.json", tf = name + ".topo.json",
                      wff = name + ".wf.json";
    write_file(tmp + "/" + pf, plan.dump(2) + "\n");
    write_file(tmp + "/" + tf, topo.dump(2) + "\n");
    write_file(tmp + "/" + wff, wf.dump(2) + "\n");
    EstimateArgs a;
    a.plan_path = tmp + "/" + pf;
    a.workflow_path = tmp + "/" + wff;
    a.topology_path = tmp + "/" + tf;
    std::ostringstream o, e;
    const int rc = cmd_estimate(a, o, e);
    const std::vector<std::string> argv = {"estimate",   "--plan",     "{tmp}/" + pf,
                                           "--workflow", "{tmp}/" + wff, "--topology",
                                           "{tmp}/" + tf};
    record(name, argv, rc, o.str(), e.str(), {});
    json& c = cases.back();
    c["inputs"] = {{pf, plan.dump(2) + "\n"}, {tf, topo.dump(2) + "\n"}, {wff, wf.dump(2) + "\n"}};
  };
  auto P = [&](auto f) {
    json p = good_plan;
    f(p);
    return p;
  };
  auto T = [&](auto f) {
    json t = good_topo;
    f(t);
    return t;
  };
  auto W = [&](auto f) {
    json w = good_wf;
    f(w);
    return w;
  };
  const std::string l6 = "6";  // a task id of the c1 PPO workflow
  err_case("err_plan_empty_groups", P([](json& p) { p["task_groups"] = json::array(); }),
           good_topo, good_wf);
  err_case("err_plan_task_twice", P([](json& p) { p["task_groups"][0].push_back(p["task_groups"][0][0]); }),
           good_topo, good_wf);
  err_case("err_plan_unknown_task", P([](json& p) { p["task_groups"][0].push_back(9); }),
           good_topo, good_wf);
  err_case("err_plan_counts_len", P([](json& p) { p["gpu_counts"].push_back(1); }), good_topo,
           good_wf);
  err_case("err_plan_counts_sum", P([](json& p) { p["gpu_counts"][0] = p["gpu_counts"][0].get<int>() + 1; }),
           good_topo, good_wf);
  err_case("err_plan_missing_layout", P([&](json& p) { p["layouts"].erase(l6); }), good_topo,
           good_wf);
  err_case("err_plan_stage_sum", P([&](json& p) { p["layouts"][l6]["stage_layers"][0] = 1000; }),
           good_topo, good_wf);
  err_case("err_plan_weights", P([&](json& p) { p["layouts"][l6]["replica_batch_weights"][0] = 7.0; }),
           good_topo, good_wf);
  err_case("err_plan_dp_zero", P([&](json& p) { p["layouts"][l6]["dp"] = 0; }), good_topo,
           good_wf);
  err_case("err_plan_unknown_device", P([](json& p) {
             for (auto& [k, v] : p["assignment"].items()) {
               v = "nope";
               break;
             }
           }),
           good_topo, good_wf);
  err_case("err_plan_schema", P([](json& p) { p.erase("gpu_counts"); }), good_topo, good_wf);
  err_case("err_topo_no_devices", good_plan, T([](json& t) { t["devices"] = json::array(); }),
           good_wf);
  err_case("err_topo_dup_id", good_plan, T([](json& t) { t["devices"][1]["id"] = t["devices"][0]["id"]; }),
           good_wf);
  err_case("err_topo_bad_attr", good_plan, T([](json& t) { t["devices"][2]["mem_gb"] = -1.0; }),
           good_wf);
  err_case("err_topo_no_region_link", good_plan, T([](json& t) { t["devices"][3]["region"] = "mars"; }),
           good_wf);
  err_case("err_topo_bad_defaults", good_plan,
           T([](json& t) { t["defaults"]["intra_region_bandwidth_gbps"] = 0.0; }), good_wf);
  err_case("err_topo_schema", good_plan, T([](json& t) { t["devices"][0].erase("node"); }),
           good_wf);
  err_case("err_wf_eta", good_plan, good_topo, W([](json& w) { w["eta"] = 1.5; }));
  err_case("err_wf_batch", good_plan, good_topo, W([](json& w) { w["batch"]["global_batch"] = 0; }));
  err_case("err_wf_missing_model", good_plan, good_topo, W([](json& w) { w["models"].erase("critic"); }));
  err_case("err_wf_layers", good_plan, good_topo,
           W([](json& w) { w["models"]["actor"]["num_layers"] = 0; }));
  err_case("err_wf_algorithm", good_plan, good_topo, W([](json& w) { w["algorithm"] = "dpo"; }));
  err_case("err_wf_parse", good_plan, good_topo, json("not an object"));
  write_file(out_path, json{{"cases", cases}}.dump(1) + "\n");
  std::printf("wrote %zu CLI cases to %s\n", cases.size(), out_path.c_str());
  return 0;
}

struct SweepStats {
  std::uint64_t feasible = 0;
  double best = std::numeric_limits<double>::infinity();
  std::uint64_t best_k = 0;
  std::uint64_t xor_bits = 0;  // XOR of e2e bit patterns, order independent
};

void sweep_range(const WorkflowGraph& wf, const DeviceTopology& topo,
                 const std::vector<TaskGrouping>& tgs, std::uint64_t seed,
                 std::uint64_t k0, std::uint64_t k1, SweepStats& st,
                 std::vector<double>* costs, std::vector<int>* feas) {
  for (std::uint64_t k = k0; k < k1; ++k) {
    const Plan p = gen_a5(wf, topo, tgs, seed, k);
    const CostBreakdown bd = end_to_end_cost(p, wf, topo, CostModelConfig{});
    std::uint64_t bits;
    std::memcpy(&bits, &bd.end_to_end_s, 8);
    st.xor_bits ^= bits;
    if (costs) costs->push_back(bd.end_to_end_s);
    if (feas) feas->push_back(bd.memory_feasible ? 1 : 0);
    if (bd.memory_feasible) {
      ++st.feasible;
      if (bd.end_to_end_s < st.best) {
        st.best = bd.end_to_end_s;
        st.best_k = k;
      }
    }
  }
}

int cmd_sweep(const std::string& wfp, const std::string& tpp, std::uint64_t seed,
              std::uint64_t k0, std::uint64_t count, const std::string& out) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  const auto tgs = enumerate_task_groupings(wf);
  SweepStats st;
  std::vector<double> costs;
  std::vector<int> feas;
  sweep_range(wf, topo, tgs, seed, k0, k0 + count, st, &costs, &feas);
  json c = json::array();
  for (double v : costs) c.push_back(hx(v));
  json j = {{"seed", seed}, {"k0", k0}, {"count", count}, {"costs", c}, {"feasible", feas},
            {"n_feasible", st.feasible}, {"best", hx(st.best)}, {"best_k", st.best_k}};
  write_file(out, j.dump() + "\n");
  std::printf("sweep %" PRIu64 " plans: %" PRIu64 " feasible, best %.9g at k=%" PRIu64 "\n",
              count, st.feasible, st.best, st.best_k);
  return 0;
}

int cmd_time_search(const std::string& wfp, const std::string& tpp, std::int64_t budget,
                    std::uint64_t seed, const std::string& knobs_path) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  SearchKnobs k = knobs_from(knobs_path);
  k.budget = budget;
  k.seed = seed;
  const auto t0 = std::chrono::steady_clock::now();
  const SearchResult res = nested_sha_search(wf, topo, k);
  const double wall =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const auto& s = res.state;
  const std::int64_t last = s.trace.empty() ? 0 : s.trace.back().first;
  std::printf(
      "{\"consumed\": %" PRId64 ", \"wall_s\": %.6f, \"plans_per_s\": %.3f, "
      "\"best\": \"%s\", \"best_dec\": %.17g, \"last_improvement\": %" PRId64
      ", \"time_to_best_est_s\": %.6f}\n",
      s.consumed, wall, s.consumed / wall,
      hx(res.plan ? res.breakdown.end_to_end_s : -1.0).c_str(),
      res.plan ? res.breakdown.end_to_end_s : -1.0, last,
      s.consumed ? wall * static_cast<double>(last) / static_cast<double>(s.consumed) : 0.0);
  return 0;
}

int cmd_time_sweep(const std::string& wfp, const std::string& tpp, std::uint64_t seed,
                   std::uint64_t k0, std::uint64_t count, int threads) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  const auto tgs = enumerate_task_groupings(wf);
  std::vector<SweepStats> st(threads);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const std::uint64_t a = k0 + count * t / threads, b = k0 + count * (t + 1) / threads;
    pool.emplace_back([&, t, a, b] { sweep_range(wf, topo, tgs, seed, a, b, st[t], nullptr, nullptr); });
  }
  for (auto& th : pool) th.join();
  const double wall =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  SweepStats all;
  for (const auto& s : st) {
    all.feasible += s.feasible;
    all.xor_bits ^= s.xor_bits;
    if (s.best < all.best || (s.best == all.best && s.best_k < all.best_k)) {
      all.best = s.best;
      all.best_k = s.best_k;
    }
  }
  std::printf(
      "{\"count\": %" PRIu64 ", \"threads\": %d, \"wall_s\": %.6f, \"plans_per_s\": %.3f, "
      "\"n_feasible\": %" PRIu64 ", \"best\": \"%s\", \"best_k\": %" PRIu64
      ", \"xor_bits\": \"%016" PRIx64 "\"}\n",
      count, threads, wall, count / wall, all.feasible, hx(all.best).c_str(), all.best_k,
      all.xor_bits);
  return 0;
}

// Stratified config-5 sample (SURVEY.md §8 D1 CPU baseline + parity set):
// `blocks` contiguous runs of `block_len` plans, block b starting at
// k = b * (total / blocks), so the sample spans the whole [0, total) range.
// All `threads` host threads share the blocks (static interleave). Prints a
// timing line; with `out`, writes per-plan records in sample order:
// k (u64), e2e bits (u64), memory_feasible (u64).
int cmd_sample_sweep(const std::string& wfp, const std::string& tpp, std::uint64_t seed,
                     std::uint64_t total, std::uint64_t blocks, std::uint64_t block_len,
                     int threads, const std::string& out) {
  const WorkflowGraph wf = parse_workflow_json(read_file(wfp));
  const DeviceTopology topo = parse_topology_json(read_file(tpp));
  const auto tgs = enumerate_task_groupings(wf);
  const std::uint64_t stride = total / blocks;
  std::vector<SweepStats> st(blocks);
  std::vector<std::vector<double>> costs(blocks);
  std::vector<std::vector<int>> feas(blocks);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (std::uint64_t b = t; b < blocks; b += threads) {
        const std::uint64_t a = b * stride;
        sweep_range(wf, topo, tgs, seed, a, a + block_len, st[b], &costs[b], &feas[b]);
      }
    });
  }
  for (auto& th : pool) th.join();
  const double wall =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  SweepStats all;
  for (const auto& s : st) {
    all.feasible += s.feasible;
    all.xor_bits ^= s.xor_bits;
    if (s.best < all.best || (s.best == all.best && s.best_k < all.best_k)) {
      all.best = s.best;
      all.best_k = s.best_k;
    }
  }
  if (!out.empty()) {
    std::FILE* f = std::fopen(out.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + out);
    for (std::uint64_t b = 0; b < blocks; ++b) {
      for (std::uint64_t i = 0; i < block_len; ++i) {
        std::uint64_t rec[3];
        rec[0] = b * stride + i;
        std::memcpy(&rec[1], &costs[b][i], 8);
        rec[2] = static_cast<std::uint64_t>(feas[b][i]);
        std::fwrite(rec, sizeof(rec), 1, f);
      }
    }
    std::fclose(f);
  }
  const std::uint64_t count = blocks * block_len;
  std::printf(
      "{\"count\": %" PRIu64 ", \"blocks\": %" PRIu64 ", \"block_len\": %" PRIu64
      ", \"stride\": %" PRIu64 ", \"threads\": %d, \"wall_s\": %.6f, \"plans_per_s\": %.3f, "
      "\"n_feasible\": %" PRIu64 ", \"best\": \"%s\", \"best_dec\": %.17g, \"best_k\": %" PRIu64
      ", \"xor_bits\": \"%016" PRIx64 "\"}\n",
      count, blocks, block_len, stride, threads, wall, count / wall, all.feasible,
      hx(all.best).c_str(), all.best, all.best_k, all.xor_bits);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_dump <command> ...\n");
    return 2;
  }
  const std::string cmd = argv[1];
  auto arg = [&](int i) -> std::string {
    if (i >= argc) {
      std::fprintf(stderr, "missing argument %d for %s\n", i, cmd.c_str());
      std::exit(2);
    }
    return argv[i];
  };
  try {
    if (cmd == "fixtures") return cmd_fixtures(arg(2));
    if (cmd == "rngpin") {  // same lines as tests/host_units.cpp prints
      const uint64_t seed = std::stoull(arg(2));
      Rng s(seed);
      const uint64_t a = s.next(), b = s.next(), c = s.next();
      std::printf("draws %" PRIu64 " %" PRIu64 " %" PRIu64 "\n", a, b, c);
      Rng f = Rng(seed).fork(7);
      const uint64_t x = f.next();
      const uint64_t y = f.bounded(100);
      const double z = f.uniform();
      std::printf("fork7 %" PRIu64 " bounded100 %" PRIu64 " uniform %.17g\n", x, y, z);
      return 0;
    }
    if (cmd == "evalplans")
      return cmd_evalplans(arg(2), arg(3), std::stoull(arg(4)), std::stoi(arg(5)), arg(6));
    if (cmd == "fuzz") return cmd_fuzz(std::stoull(arg(2)), std::stoi(arg(3)), arg(4));
    if (cmd == "search")
      return cmd_search(arg(2), arg(3), std::stoll(arg(4)), std::stoull(arg(5)), arg(6),
                        argc > 7 ? argv[7] : "");
    if (cmd == "ga") return cmd_ga(arg(2), arg(3), arg(4), argc > 5 ? arg(5) : "");
    if (cmd == "searchfuzz") return cmd_searchfuzz(std::stoull(arg(2)), std::stoi(arg(3)), arg(4));
    if (cmd == "exhaustive") return cmd_exhaustive(std::stoull(arg(2)), std::stoi(arg(3)), arg(4));
    if (cmd == "cli") return cmd_cli(arg(2));
    if (cmd == "sweep")
      return cmd_sweep(arg(2), arg(3), std::stoull(arg(4)), std::stoull(arg(5)),
                       std::stoull(arg(6)), arg(7));
    if (cmd == "time_search")
      return cmd_time_search(arg(2), arg(3), std::stoll(arg(4)), std::stoull(arg(5)),
                             argc > 6 ? argv[6] : "");
    if (cmd == "sample_sweep")
      return cmd_sample_sweep(arg(2), arg(3), std::stoull(arg(4)), std::stoull(arg(5)),
                              std::stoull(arg(6)), std::stoull(arg(7)), std::stoi(arg(8)),
                              argc > 9 ? argv[9] : "");
    if (cmd == "time_sweep")
      return cmd_time_sweep(arg(2), arg(3), std::stoull(arg(4)), std::stoull(arg(5)),
                            std::stoull(arg(6)), std::stoi(arg(7)));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_dump: %s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
