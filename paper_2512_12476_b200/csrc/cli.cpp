// hetplan_b200 — the reference command line (proj/src/cli.cpp:76-283,
// proj/tools/hetplan_main.cpp) on the B200 engine: plan / estimate / compare /
// scenario, plus exhaustive (search.cpp:884-1031) and the fleet scenario
// generator.
//
// The search and the cost model run on the GPU through the C ABI
// (include/hpg.h). JSON is read and written with nlohmann::json, the
// reference's I/O library (the 3.11.3 copy shipped in this image), with the
// reference's schema, key order and dump(2) layout, so plan files, topology
// files and JSON reports are byte-identical to the reference CLI's for the
// same inputs (wall-clock fields aside). Exit codes follow cli.hpp:12-16.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"

#include "hpg.h"

using json = nlohmann::json;

namespace {

constexpr int kExitOk = 0, kExitUsage = 2, kExitInput = 3, kExitInfeasible = 4,
              kExitInternal = 5;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(int rc, const char* err) {
  if (rc == HPG_OK) return;
  if (rc == HPG_USAGE) throw UsageError(err);
  if (rc == HPG_INPUT) throw InputError(err);
  throw std::runtime_error(err);
}

std::string read_file(const std::string& path, const std::string& what) {
  std::ifstream in(path);
  if (!in) throw InputError("cannot open " + what + " file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void write_file(const std::string& path, const std::string& what, const std::string& text) {
  std::ofstream out(path);
  if (!out) throw InputError("cannot write " + what + " file: " + path);
  out << text;
}

// ---- workflow (workflow.cpp:16-33, 97-146, 161-232) ----

struct Workflow {
  int algorithm = 0;  // 0 ppo, 1 grpo
  int mode = 0;       // 0 sync, 1 async
  double eta = 0.5;
  int64_t global_batch = 0, rpp = 0, seq_in = 0, seq_out = 0, mbs = 0;
  std::vector<hpg_task> tasks;  // id order
  std::vector<std::string> model_names;
  std::set<std::pair<int, int>> edges;
  bool has_task(int id) const {
    for (const hpg_task& t : tasks)
      if (t.id == id) return true;
    return false;
  }
  int slot_of(int id) const {
    for (size_t s = 0; s < tasks.size(); ++s)
      if (tasks[s].id == id) return static_cast<int>(s);
    return -1;
  }
};

struct Model {
  int64_t h1 = 0, h2 = 0, nl = 0;
  bool emb = false;
  int64_t vocab = 0;
};

Workflow parse_workflow(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw InputError(std::string("workflow JSON parse error: ") + e.what());
  }
  try {
    Workflow wf;
    const std::string algo = j.at("algorithm").get<std::string>();
    if (algo == "ppo") {
      wf.algorithm = 0;
    } else if (algo == "grpo") {
      wf.algorithm = 1;
    } else {
      throw InputError("unknown algorithm '" + algo + "'");
    }
    const std::string mode = j.at("mode").get<std::string>();
    if (mode == "sync") {
      wf.mode = 0;
    } else if (mode == "async") {
      wf.mode = 1;
    } else {
      throw InputError("unknown mode '" + mode + "'");
    }
    wf.eta = j.value("eta", 0.5);
    const json& jb = j.at("batch");
    wf.global_batch = jb.at("global_batch").get<int64_t>();
    wf.rpp = jb.at("responses_per_prompt").get<int64_t>();
    wf.seq_in = jb.at("seq_in").get<int64_t>();
    wf.seq_out = jb.at("seq_out").get<int64_t>();
    wf.mbs = jb.at("micro_batch_size").get<int64_t>();
    std::map<std::string, Model> models;
    for (const auto& [name, jm] : j.at("models").items()) {
      Model m;
      m.h1 = jm.at("hidden_size").get<int64_t>();
      m.h2 = jm.at("intermediate_size").get<int64_t>();
      m.nl = jm.at("num_layers").get<int64_t>();
      if (jm.contains("include_embedding")) m.emb = jm.at("include_embedding").get<bool>();
      if (jm.contains("vocab_size")) m.vocab = jm.at("vocab_size").get<int64_t>();
      models[name] = m;
    }
    // build_workflow
    if (wf.eta < 0.0 || wf.eta > 1.0) throw InputError("eta must be within [0, 1]");
    if (wf.global_batch < 1 || wf.rpp < 1 || wf.mbs < 1)
      throw InputError("batch sizes must be >= 1");
    if (wf.seq_in < 1 || wf.seq_out < 0)
      throw InputError("seq_in must be >= 1 and seq_out >= 0");
    const std::vector<int> ids =
        wf.algorithm == 0 ? std::vector<int>{1, 2, 3, 4, 5, 6} : std::vector<int>{1, 2, 3, 6};
    static const char* names[7] = {"", "actor", "reward", "reference", "critic", "critic", "actor"};
    for (int id : ids) {
      const std::string name = names[id];
      auto it = models.find(name);
      if (it == models.end())
        throw InputError("missing model spec '" + name + "' required by task " +
                         std::to_string(id));
      const Model& m = it->second;
      if (m.h1 < 1 || m.h2 < 1 || m.nl < 1)
        throw InputError(
            "model spec requires hidden_size, intermediate_size and num_layers >= 1");
      if (m.emb && m.vocab < 1) throw InputError("include_embedding requires vocab_size >= 1");
      hpg_task t{};
      t.id = id;
      t.kind = id == 1 ? 0 : (id <= 4 ? 1 : 2);
      t.hidden_size = m.h1;
      t.intermediate_size = m.h2;
      t.num_layers = m.nl;
      t.include_embedding = m.emb ? 1 : 0;
      t.vocab_size = m.vocab;
      t.precision_bytes = 2;
      wf.tasks.push_back(t);
      wf.model_names.push_back(name);
    }
    std::vector<int> inf, trn;
    for (const hpg_task& t : wf.tasks) {
      if (t.kind == 1) inf.push_back(t.id);
      if (t.kind == 2) trn.push_back(t.id);
    }
    for (int i : inf) wf.edges.emplace(1, i);
    for (int i : inf)
      for (int tr : trn) wf.edges.emplace(i, tr);
    if (j.contains("precision_bytes")) {
      for (const auto& [name, jp] : j.at("precision_bytes").items())
        for (size_t s = 0; s < wf.tasks.size(); ++s)
          if (wf.model_names[s] == name) wf.tasks[s].precision_bytes = jp.get<int>();
    }
    return wf;
  } catch (const json::exception& e) {
    throw InputError(std::string("workflow JSON schema error: ") + e.what());
  }
}

// ---- topology (topology.cpp:132-211) ----

struct Device {
  std::string id, gpu_model;
  double comp_tflops = 0, mem_gb = 0, hbm_gbps = 0, intra_node_gbps = 0;
  std::string node, region;
};
struct RegionLink {
  std::string src, dst;
  double latency_ms = 0, bandwidth_gbps = 0;
};
struct Topology {
  std::vector<Device> devices;
  std::vector<RegionLink> links;
  double intra_region_latency_ms = 0.1, intra_region_bandwidth_gbps = 100.0;
  int index_of(const std::string& id) const {
    for (size_t i = 0; i < devices.size(); ++i)
      if (devices[i].id == id) return static_cast<int>(i);
    throw InputError("unknown device id '" + id + "'");
  }
};

Topology parse_topology(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw InputError(std::string("topology JSON parse error: ") + e.what());
  }
  try {
    Topology t;
    for (const json& jd : j.at("devices")) {
      Device d;
      d.id = jd.at("id").get<std::string>();
      d.gpu_model = jd.at("gpu_model").get<std::string>();
      d.comp_tflops = jd.at("comp_tflops").get<double>();
      d.mem_gb = jd.at("mem_gb").get<double>();
      d.hbm_gbps = jd.at("hbm_gbps").get<double>();
      d.intra_node_gbps = jd.at("intra_node_gbps").get<double>();
      d.node = jd.at("node").get<std::string>();
      d.region = jd.at("region").get<std::string>();
      t.devices.push_back(std::move(d));
    }
    if (j.contains("region_links")) {
      for (const json& jl : j.at("region_links")) {
        RegionLink rl;
        rl.src = jl.at("src").get<std::string>();
        rl.dst = jl.at("dst").get<std::string>();
        rl.latency_ms = jl.at("latency_ms").get<double>();
        rl.bandwidth_gbps = jl.at("bandwidth_gbps").get<double>();
        t.links.push_back(std::move(rl));
      }
    }
    if (j.contains("defaults")) {
      const json& jd = j.at("defaults");
      t.intra_region_latency_ms = jd.value("intra_region_latency_ms", t.intra_region_latency_ms);
      t.intra_region_bandwidth_gbps =
          jd.value("intra_region_bandwidth_gbps", t.intra_region_bandwidth_gbps);
    }
    return t;
  } catch (const json::exception& e) {
    throw InputError(std::string("topology JSON schema error: ") + e.what());
  }
}

std::string serialize_topology(const Topology& topo) {
  json jdevs = json::array();
  for (const Device& d : topo.devices) {
    jdevs.push_back({{"id", d.id},
                     {"gpu_model", d.gpu_model},
                     {"comp_tflops", d.comp_tflops},
                     {"mem_gb", d.mem_gb},
                     {"hbm_gbps", d.hbm_gbps},
                     {"intra_node_gbps", d.intra_node_gbps},
                     {"node", d.node},
                     {"region", d.region}});
  }
  json jlinks = json::array();
  for (const RegionLink& rl : topo.links) {
    jlinks.push_back({{"src", rl.src},
                      {"dst", rl.dst},
                      {"latency_ms", rl.latency_ms},
                      {"bandwidth_gbps", rl.bandwidth_gbps}});
  }
  json j = {{"devices", jdevs},
            {"region_links", jlinks},
            {"defaults",
             {{"intra_region_latency_ms", topo.intra_region_latency_ms},
              {"intra_region_bandwidth_gbps", topo.intra_region_bandwidth_gbps}}}};
  return j.dump(2) + "\n";
}

// ---- knobs (search.cpp:46-94) ----

struct Knobs {
  int64_t budget = 1000;
  uint64_t seed = 0;
  bool seed_set = false;
  int population = 16;
  double locality_bias = 0.8;
  int quantize_gpu_counts = 1;
  std::string level1_filter = "off";
  int level1_cap = 0;
  int gg_arm_cap = 64;
  int swap_pair_sample = 8;
  bool balance_data = true, balance_layers = true, balance_seqlen = true, recompute = true;
  double reshard_override = -1.0, sync_override = -1.0, exhaustive_cap = 1e6;

  hpg_knobs to_c() const {
    hpg_knobs k;
    hpg_knobs_default(&k);
    k.budget = budget;
    k.seed = seed;
    k.population = population;
    k.locality_bias = locality_bias;
    k.quantize_gpu_counts = quantize_gpu_counts;
    k.level1_filter_adjacent = level1_filter == "adjacent" ? 1 : 0;
    k.level1_cap = level1_cap;
    k.gg_arm_cap = gg_arm_cap;
    k.swap_pair_sample = swap_pair_sample;
    k.balance_data = balance_data;
    k.balance_layers = balance_layers;
    k.balance_seqlen = balance_seqlen;
    k.recompute = recompute;
    k.reshard_override = reshard_override;
    k.sync_override = sync_override;
    k.exhaustive_cap = exhaustive_cap;
    return k;
  }
  hpg_cost_config cost_config() const {  // SearchKnobs::cost_config (search.cpp:38-44)
    hpg_cost_config c;
    hpg_cost_config_default(&c);
    c.recompute = recompute;
    c.reshard_override = reshard_override;
    c.sync_override = sync_override;
    return c;
  }
};

Knobs parse_knobs(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw InputError(std::string("knobs JSON parse error: ") + e.what());
  }
  Knobs k;
  try {
    k.budget = j.value("budget", k.budget);
    k.seed = j.value("seed", k.seed);
    k.seed_set = j.contains("seed");
    k.population = j.value("population", k.population);
    k.locality_bias = j.value("locality_bias", k.locality_bias);
    k.quantize_gpu_counts = j.value("quantize_gpu_counts", k.quantize_gpu_counts);
    k.level1_filter = j.value("level1_filter", k.level1_filter);
    k.level1_cap = j.value("level1_cap", k.level1_cap);
    k.gg_arm_cap = j.value("gg_arm_cap", k.gg_arm_cap);
    k.swap_pair_sample = j.value("swap_pair_sample", k.swap_pair_sample);
    k.balance_data = j.value("balance_data", k.balance_data);
    k.balance_layers = j.value("balance_layers", k.balance_layers);
    k.balance_seqlen = j.value("balance_seqlen", k.balance_seqlen);
    k.recompute = j.value("recompute", k.recompute);
    k.reshard_override = j.value("reshard_override", k.reshard_override);
    k.sync_override = j.value("sync_override", k.sync_override);
    k.exhaustive_cap = j.value("exhaustive_cap", k.exhaustive_cap);
  } catch (const json::exception& e) {
    throw InputError(std::string("knobs JSON schema error: ") + e.what());
  }
  if (k.population < 1 || k.swap_pair_sample < 0 || k.gg_arm_cap < 1)
    throw InputError("knobs: population and gg_arm_cap must be >= 1");
  if (k.locality_bias < 0 || k.locality_bias > 1)
    throw InputError("knobs: locality_bias must be within [0, 1]");
  if (k.level1_filter != "off" && k.level1_filter != "adjacent")
    throw InputError("knobs: level1_filter must be \"off\" or \"adjacent\"");
  return k;
}

Knobs knobs_for(const std::string& path) {
  return path.empty() ? Knobs{} : parse_knobs(read_file(path, "knobs"));
}

// ---- plans (plan.cpp:19-87, 257-349, 384-556) ----

struct Layout {
  int dp = 1, pp = 1, tp = 1;
  std::vector<int> stage_layers;
  std::vector<double> weights;
  int flat(int i, int j, int k) const { return (i * pp + j) * tp + k; }
  int size() const { return dp * pp * tp; }
};
struct TaskCost {
  double comp = 0, tp = 0, pp = 0, dp = 0, bubble = 0, hbm = 0, total = 0;
};
struct Breakdown {
  std::map<int, TaskCost> per_task;
  double reshard_s = 0, sync_s = 0, end_to_end_s = 0;
  bool memory_feasible = true;
};
struct Plan {
  std::vector<std::vector<int>> groups;
  std::vector<int> counts;
  std::map<int, Layout> layouts;
  std::map<int, std::vector<std::string>> assignment;
  uint64_t prov_seed = 0;
  int64_t prov_budget = 0;
  double estimated_cost_s = -1.0;
};

Plan parse_plan(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw InputError(std::string("plan JSON parse error: ") + e.what());
  }
  try {
    Plan p;
    p.groups = j.at("task_groups").get<std::vector<std::vector<int>>>();
    p.counts = j.at("gpu_counts").get<std::vector<int>>();
    for (const auto& [key, jl] : j.at("layouts").items()) {
      Layout l;
      l.dp = jl.at("dp").get<int>();
      l.pp = jl.at("pp").get<int>();
      l.tp = jl.at("tp").get<int>();
      l.stage_layers = jl.at("stage_layers").get<std::vector<int>>();
      if (jl.contains("replica_batch_weights")) {
        l.weights = jl.at("replica_batch_weights").get<std::vector<double>>();
      } else {
        l.weights.assign(l.dp, 1.0);
      }
      p.layouts[std::stoi(key)] = l;
    }
    const json& ja = j.at("assignment");
    for (const auto& [id, l] : p.layouts) {
      std::vector<std::string> devs(l.size());
      for (int i = 0; i < l.dp; ++i)
        for (int j2 = 0; j2 < l.pp; ++j2)
          for (int k = 0; k < l.tp; ++k) {
            std::ostringstream key;
            key << id << ',' << i << ',' << j2 << ',' << k;
            if (!ja.contains(key.str()))
              throw InputError("plan assignment missing tasklet " + key.str());
            devs[l.flat(i, j2, k)] = ja.at(key.str()).get<std::string>();
          }
      p.assignment[id] = std::move(devs);
    }
    if (j.contains("provenance")) {
      p.prov_seed = j.at("provenance").at("seed").get<uint64_t>();
      p.prov_budget = j.at("provenance").at("budget").get<int64_t>();
    }
    p.estimated_cost_s = j.value("estimated_cost_s", -1.0);
    return p;
  } catch (const json::exception& e) {
    throw InputError(std::string("plan JSON schema error: ") + e.what());
  }
}

json layout_json(const Layout& l) {
  return {{"dp", l.dp},
          {"pp", l.pp},
          {"tp", l.tp},
          {"stage_layers", l.stage_layers},
          {"replica_batch_weights", l.weights}};
}

json breakdown_json(const Breakdown& bd) {
  json per_task = json::object();
  for (const auto& [id, tc] : bd.per_task) {
    per_task[std::to_string(id)] = {{"comp", tc.comp}, {"tp", tc.tp},         {"pp", tc.pp},
                                    {"dp", tc.dp},     {"bubble", tc.bubble}, {"hbm", tc.hbm},
                                    {"total", tc.total}};
  }
  return {{"per_task", per_task},
          {"reshard_s", bd.reshard_s},
          {"sync_s", bd.sync_s},
          {"end_to_end_s", bd.end_to_end_s},
          {"memory_feasible", bd.memory_feasible}};
}

std::string serialize_plan(const Plan& plan, const Breakdown* bd) {
  json jlayouts = json::object();
  for (const auto& [id, l] : plan.layouts) jlayouts[std::to_string(id)] = layout_json(l);
  json jassign = json::object();
  for (const auto& [id, devs] : plan.assignment) {
    auto lit = plan.layouts.find(id);
    if (lit == plan.layouts.end())
      throw InputError("plan has assignment for task without layout");
    const Layout& l = lit->second;
    for (int i = 0; i < l.dp; ++i)
      for (int j = 0; j < l.pp; ++j)
        for (int k = 0; k < l.tp; ++k) {
          std::ostringstream key;
          key << id << ',' << i << ',' << j << ',' << k;
          jassign[key.str()] = devs.at(l.flat(i, j, k));
        }
  }
  json j = {{"task_groups", plan.groups},
            {"gpu_counts", plan.counts},
            {"layouts", jlayouts},
            {"assignment", jassign},
            {"provenance", {{"seed", plan.prov_seed}, {"budget", plan.prov_budget}}},
            {"estimated_cost_s", plan.estimated_cost_s}};
  if (bd) j["cost_breakdown"] = breakdown_json(*bd);
  return j.dump(2) + "\n";
}

// resolve_plan's structural checks, in the reference's order (plan.cpp:257-349);
// the engine repeats them on the device-index table it receives
void validate_plan(const Plan& p, const Workflow& wf, const Topology& topo) {
  if (p.groups.empty()) throw InputError("task grouping must contain at least one group");
  std::set<int> seen;
  for (const auto& g : p.groups) {
    if (g.empty()) throw InputError("task groups must be non-empty");
    for (int id : g) {
      if (!wf.has_task(id))
        throw InputError("task grouping references unknown task " + std::to_string(id));
      if (!seen.insert(id).second)
        throw InputError("task " + std::to_string(id) + " appears in more than one group");
    }
  }
  if (seen.size() != wf.tasks.size())
    throw InputError("task grouping must cover every workflow task");
  if (p.counts.size() != p.groups.size())
    throw InputError("gpu_counts must list one entry per task group");
  int64_t sum = 0;
  for (int c : p.counts) {
    if (c < 1) throw InputError("gpu_counts entries must be >= 1");
    sum += c;
  }
  if (sum != static_cast<int64_t>(topo.devices.size()))
    throw InputError("gpu_counts must sum to the device count (" +
                     std::to_string(topo.devices.size()) + ")");
  std::vector<std::set<int>> group_sets(p.groups.size());
  for (size_t g = 0; g < p.groups.size(); ++g) {
    for (int id : p.groups[g]) {
      const hpg_task& task = wf.tasks[wf.slot_of(id)];
      auto lit = p.layouts.find(id);
      if (lit == p.layouts.end())
        throw InputError("plan missing layout for task " + std::to_string(id));
      const Layout& l = lit->second;
      if (l.dp < 1 || l.pp < 1 || l.tp < 1) throw InputError("dp, pp and tp must be >= 1");
      if (l.pp > task.num_layers) throw InputError("pp exceeds layer count");
      if (static_cast<int>(l.stage_layers.size()) != l.pp)
        throw InputError("stage_layers must have one entry per pipeline stage");
      int64_t total = 0;
      for (int x : l.stage_layers) {
        if (x < 1) throw InputError("every pipeline stage needs at least one layer");
        total += x;
      }
      if (total != task.num_layers)
        throw InputError("stage_layers must sum to the model layer count");
      if (static_cast<int>(l.weights.size()) != l.dp)
        throw InputError("replica_batch_weights must have one entry per replica");
      double wsum = 0;
      for (double w : l.weights) {
        if (!(w > 0)) throw InputError("replica batch weights must be positive");
        wsum += w;
      }
      if (std::abs(wsum - l.dp) > 1e-6 * l.dp)
        throw InputError("replica batch weights must sum to dp");
      if (l.size() != p.counts[g])
        throw InputError("task " + std::to_string(id) +
                         ": dp*pp*tp must equal its group's GPU count");
      auto ait = p.assignment.find(id);
      if (ait == p.assignment.end())
        throw InputError("plan missing assignment for task " + std::to_string(id));
      if (static_cast<int>(ait->second.size()) != l.size())
        throw InputError("task " + std::to_string(id) + ": assignment must cover every tasklet");
      std::set<int> used;
      for (const std::string& dev : ait->second) {
        if (!used.insert(topo.index_of(dev)).second)
          throw InputError("task " + std::to_string(id) + ": device '" + dev +
                           "' hosts more than one tasklet");
      }
      if (group_sets[g].empty()) {
        group_sets[g] = used;
      } else if (group_sets[g] != used) {
        throw InputError("co-located tasks in group " + std::to_string(g) +
                         " must share the same device set");
      }
    }
  }
  std::set<int> all;
  for (const auto& gs : group_sets)
    for (int d : gs)
      if (!all.insert(d).second)
        throw InputError("device '" + topo.devices[d].id + "' appears in more than one GPU group");
}

// ---- the engine behind the C ABI ----

class Engine {
 public:
  Engine(const Workflow& wf, const Topology& topo) : wf_(wf), topo_(topo) {
    for (const Device& d : topo.devices)
      devs_.push_back({d.id.c_str(), d.gpu_model.c_str(), d.comp_tflops, d.mem_gb, d.hbm_gbps,
                       d.intra_node_gbps, d.node.c_str(), d.region.c_str()});
    for (const RegionLink& l : topo.links)
      links_.push_back({l.src.c_str(), l.dst.c_str(), l.latency_ms, l.bandwidth_gbps});
    for (const auto& [a, b] : wf.edges) {
      edges_.push_back(a);
      edges_.push_back(b);
    }
    hpg_problem p{};
    p.algorithm = wf.algorithm;
    p.mode = wf.mode;
    p.eta = wf.eta;
    p.global_batch = wf.global_batch;
    p.responses_per_prompt = wf.rpp;
    p.seq_in = wf.seq_in;
    p.seq_out = wf.seq_out;
    p.micro_batch_size = wf.mbs;
    p.n_tasks = static_cast<int32_t>(wf.tasks.size());
    p.tasks = wf.tasks.data();
    p.n_dep_edges = static_cast<int32_t>(wf.edges.size());
    p.dep_edges = edges_.data();
    p.n_devices = static_cast<int32_t>(devs_.size());
    p.devices = devs_.data();
    p.n_region_links = static_cast<int32_t>(links_.size());
    p.region_links = links_.data();
    p.intra_region_latency_ms = topo.intra_region_latency_ms;
    p.intra_region_bandwidth_gbps = topo.intra_region_bandwidth_gbps;
    char err[1024];
    check(hpg_create(&p, 0, &ctx_, err, sizeof(err)), err);
  }
  ~Engine() {
    if (ctx_) hpg_destroy(ctx_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  Breakdown estimate(const Plan& plan, const hpg_cost_config& cfg) {
    validate_plan(plan, wf_, topo_);
    const int T = static_cast<int>(wf_.tasks.size());
    const int32_t ng = static_cast<int32_t>(plan.groups.size());
    std::vector<int32_t> task_group(T), counts(T, 0), dp(T), pp(T), tp(T), sls, devices;
    std::vector<int64_t> sl_off(T), w_off(T), dev_off(T);
    std::vector<double> ws;
    for (size_t g = 0; g < plan.groups.size(); ++g) {
      counts[g] = plan.counts[g];
      for (int id : plan.groups[g]) task_group[wf_.slot_of(id)] = static_cast<int32_t>(g);
    }
    for (int s = 0; s < T; ++s) {
      const int id = wf_.tasks[s].id;
      const Layout& l = plan.layouts.at(id);
      dp[s] = l.dp;
      pp[s] = l.pp;
      tp[s] = l.tp;
      sl_off[s] = static_cast<int64_t>(sls.size());
      sls.insert(sls.end(), l.stage_layers.begin(), l.stage_layers.end());
      w_off[s] = static_cast<int64_t>(ws.size());
      ws.insert(ws.end(), l.weights.begin(), l.weights.end());
      dev_off[s] = static_cast<int64_t>(devices.size());
      for (const std::string& d : plan.assignment.at(id)) devices.push_back(topo_.index_of(d));
    }
    hpg_plan_table t{1,          &ng,       task_group.data(), counts.data(), dp.data(),
                     pp.data(),  tp.data(), sl_off.data(),     sls.data(),    w_off.data(),
                     ws.data(),  dev_off.data(), devices.data()};
    double e2e = 0, rs = 0, sy = 0;
    uint8_t feas = 0;
    std::vector<double> per_task(static_cast<size_t>(T) * 7);
    hpg_eval_out out{&e2e, &feas, per_task.data(), &rs, &sy};
    char err[1024];
    check(hpg_eval(ctx_, &t, &cfg, &out, err, sizeof(err)), err);
    return breakdown_of(per_task.data(), rs, sy, e2e, feas != 0);
  }

  // nested_sha_search / exhaustive_search: plan + breakdown of the result
  struct Found {
    bool has_plan = false;
    Plan plan;
    Breakdown bd;
    hpg_search_info info{};
    std::vector<std::pair<int64_t, double>> trace;
  };
  Found search(const Knobs& k, bool exhaustive) {
    const hpg_knobs kc = k.to_c();
    hpg_search_result* r = nullptr;
    char err[1024];
    check(exhaustive ? hpg_exhaustive(ctx_, &kc, &r, err, sizeof(err))
                     : hpg_search(ctx_, &kc, &r, err, sizeof(err)),
          err);
    Found f;
    hpg_result_info(r, &f.info);
    std::vector<int64_t> tc(f.info.n_trace);
    std::vector<double> tv(f.info.n_trace);
    hpg_result_trace(r, tc.data(), tv.data());
    for (int i = 0; i < f.info.n_trace; ++i) f.trace.emplace_back(tc[i], tv[i]);
    if (f.info.has_plan) {
      const int T = static_cast<int>(wf_.tasks.size());
      hpg_plan_table t{};
      std::vector<int32_t> gflat(T);
      double est = 0;
      uint64_t pseed = 0;
      int64_t pbud = 0;
      hpg_result_plan(r, &t, gflat.data(), &est, &pseed, &pbud);
      f.has_plan = true;
      Plan& p = f.plan;
      p.groups.assign(t.n_groups[0], {});
      for (int s : gflat) p.groups[t.task_group[s]].push_back(wf_.tasks[s].id);
      for (int g = 0; g < t.n_groups[0]; ++g) p.counts.push_back(t.gpu_counts[g]);
      for (int s = 0; s < T; ++s) {
        Layout l;
        l.dp = t.dp[s];
        l.pp = t.pp[s];
        l.tp = t.tp[s];
        l.stage_layers.assign(t.stage_layers + t.sl_off[s], t.stage_layers + t.sl_off[s] + l.pp);
        l.weights.assign(t.weights + t.w_off[s], t.weights + t.w_off[s] + l.dp);
        std::vector<std::string> ids;
        for (int e = 0; e < l.size(); ++e) ids.push_back(topo_.devices[t.devices[t.dev_off[s] + e]].id);
        p.layouts[wf_.tasks[s].id] = l;
        p.assignment[wf_.tasks[s].id] = std::move(ids);
      }
      p.estimated_cost_s = est;
      p.prov_seed = pseed;
      p.prov_budget = pbud;
      std::vector<double> per_task(static_cast<size_t>(T) * 7);
      double rs = 0, sy = 0, e2e = 0;
      uint8_t mf = 0;
      hpg_result_breakdown(r, per_task.data(), &rs, &sy, &e2e, &mf);
      f.bd = breakdown_of(per_task.data(), rs, sy, e2e, mf != 0);
    }
    hpg_result_free(r);
    return f;
  }

 private:
  Breakdown breakdown_of(const double* per_task, double rs, double sy, double e2e, bool feas) {
    Breakdown bd;
    for (size_t s = 0; s < wf_.tasks.size(); ++s) {
      const double* v = per_task + 7 * s;
      bd.per_task[wf_.tasks[s].id] = TaskCost{v[0], v[1], v[2], v[3], v[4], v[5], v[6]};
    }
    bd.reshard_s = rs;
    bd.sync_s = sy;
    bd.end_to_end_s = e2e;
    bd.memory_feasible = feas;
    return bd;
  }

  const Workflow& wf_;
  const Topology& topo_;
  std::vector<hpg_device> devs_;
  std::vector<hpg_region_link> links_;
  std::vector<int32_t> edges_;
  hpg_ctx* ctx_ = nullptr;
};

// ---- scenario synthesis (topology.cpp:222-391) + the fleet generator ----

struct GpuSpec {
  double comp_tflops, mem_gb, hbm_gbps, intra_node_gbps;
};
const std::map<std::string, GpuSpec>& gpu_catalog() {
  // topology.cpp:228-236, plus H100 as SURVEY.md App. A.4 defines it (fleet only)
  static const std::map<std::string, GpuSpec> c = {{"A100", {312.0, 40.0, 2039.0, 600.0}},
                                                    {"L40S", {366.0, 48.0, 864.0, 64.0}},
                                                    {"L4", {121.0, 24.0, 300.0, 64.0}}};
  return c;
}
const std::map<std::string, GpuSpec>& fleet_catalog() {
  static const std::map<std::string, GpuSpec> c = {{"A100", {312.0, 40.0, 2039.0, 600.0}},
                                                    {"L40S", {366.0, 48.0, 864.0, 64.0}},
                                                    {"L4", {121.0, 24.0, 300.0, 64.0}},
                                                    {"H100", {989.0, 80.0, 3350.0, 900.0}}};
  return c;
}

std::string lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return std::tolower(c); });
  return s;
}

struct InventoryItem {
  int count;
  std::string gpu_model;
};

std::vector<InventoryItem> parse_inventory(const std::string& text) {
  std::vector<InventoryItem> items;
  std::stringstream ss(text);
  std::string part;
  while (std::getline(ss, part, ',')) {
    auto x = part.find('x');
    if (x == std::string::npos) x = part.find('*');
    if (x == std::string::npos || x == 0 || x + 1 >= part.size())
      throw UsageError("bad inventory entry '" + part + "' (expected COUNTxMODEL, e.g. 24xA100)");
    InventoryItem item;
    try {
      item.count = std::stoi(part.substr(0, x));
    } catch (const std::exception&) {
      throw UsageError("bad inventory count in '" + part + "'");
    }
    item.gpu_model = part.substr(x + 1);
    items.push_back(std::move(item));
  }
  if (items.empty()) throw UsageError("empty inventory");
  return items;
}

// Rng (rng.hpp:10-65): splitmix64 seeding, xoshiro256**, uniform()
struct Rng {
  uint64_t s[4];
  static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  }
  explicit Rng(uint64_t seed) {
    uint64_t v = seed;
    for (int i = 0; i < 4; ++i) v = s[i] = mix64(v);
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform(double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(next() >> 11) * 0x1.0p-53);
  }
};

std::vector<Device> inventory_devices(const std::vector<InventoryItem>& inv) {
  std::vector<Device> devs;
  std::map<std::string, int> per_model;
  for (const InventoryItem& item : inv) {
    auto it = gpu_catalog().find(item.gpu_model);
    if (it == gpu_catalog().end())
      throw InputError("unknown GPU model '" + item.gpu_model + "' (known: A100, L40S, L4)");
    if (item.count < 1) throw InputError("inventory counts must be >= 1");
    for (int k = 0; k < item.count; ++k) {
      Device d;
      char buf[16];
      std::snprintf(buf, sizeof(buf), "%02d", per_model[item.gpu_model]++);
      d.id = lower(item.gpu_model) + "-" + buf;
      d.gpu_model = item.gpu_model;
      d.comp_tflops = it->second.comp_tflops;
      d.mem_gb = it->second.mem_gb;
      d.hbm_gbps = it->second.hbm_gbps;
      d.intra_node_gbps = it->second.intra_node_gbps;
      devs.push_back(std::move(d));
    }
  }
  return devs;
}

struct ScenarioOptions {
  std::vector<InventoryItem> inventory{{24, "A100"}, {24, "L40S"}, {16, "L4"}};
  uint64_t seed = 0;
  int node_size = 8;
  std::vector<std::string> edge_models{"L4"};
};

// generate_scenario (topology.cpp:310-391)
Topology generate_scenario(int id, const ScenarioOptions& o) {
  if (id < 1 || id > 4) throw UsageError("scenario id must be 1..4");
  Topology t;
  t.devices = inventory_devices(o.inventory);
  if (id == 1) {
    std::map<std::string, int> per_model;
    for (Device& d : t.devices) {
      const int k = per_model[d.gpu_model]++;
      d.region = "local";
      d.node = lower(d.gpu_model) + "-node-" + std::to_string(k / std::max(1, o.node_size));
    }
    return t;
  }
  for (Device& d : t.devices) d.node = "host-" + d.id;
  if (id == 2) {
    auto is_edge = [&](const Device& d) {
      return std::find(o.edge_models.begin(), o.edge_models.end(), d.gpu_model) !=
             o.edge_models.end();
    };
    std::set<std::string> used;
    std::string ohio;
    for (Device& d : t.devices) {
      if (is_edge(d)) {
        d.region = "virginia-edge";
      } else {
        if (ohio.empty()) ohio = d.gpu_model;
        d.region = d.gpu_model == ohio ? "ohio" : "virginia";
      }
      used.insert(d.region);
    }
    auto add = [&](const std::string& a, const std::string& b, double ms, double gbps) {
      if (used.count(a) && used.count(b)) t.links.push_back({a, b, ms, gbps});
    };
    add("ohio", "virginia", 10.0, 5.0);
    add("ohio", "virginia-edge", 10.0, 1.0);
    add("virginia", "virginia-edge", t.intra_region_latency_ms, 1.0);
    return t;
  }
  const std::vector<std::string> regions =
      id == 3 ? std::vector<std::string>{"paris", "stockholm", "london", "ireland", "spain",
                                         "zurich", "frankfurt", "milan"}
              : std::vector<std::string>{"virginia", "ohio", "paris", "stockholm", "london",
                                         "ireland", "spain", "zurich"};
  for (size_t i = 0; i < t.devices.size(); ++i) t.devices[i].region = regions[i % regions.size()];
  const double d_lo = 5.0, d_hi = id == 3 ? 30.0 : 60.0;
  const double b_lo = id == 3 ? 1.9 : 0.9, b_hi = 5.0;
  Rng rng(o.seed);
  for (size_t a = 0; a < regions.size(); ++a)
    for (size_t b = a + 1; b < regions.size(); ++b) {
      const double lat = rng.uniform(d_lo, d_hi);
      const double bw = rng.uniform(b_lo, b_hi);
      t.links.push_back({regions[a], regions[b], lat, bw});
    }
  return t;
}

// Fleet generator: N GPU types x R regions, config-4 style.
// Device i takes the next type in round-robin blocks of node_size (types
// whose inventory is used up drop out), its id is <TYPE>-<i>, its region is
// regions[(i / ceil(n / R)) % R] and its node <region>-n<i / node_size>. One
// link per region pair a < b: latency uniform(lat_lo, lat_hi) ms then
// bandwidth uniform(bw_lo, bw_hi) Gbps from Rng(seed); defaults 0.1 ms /
// 100 Gbps. With 32xA100,32xL40S,32xL4,32xH100 over
// virginia,ohio,paris,frankfurt, node size 8, seed 7, 5-60 ms and 0.9-5 Gbps
// this is fixtures/c4.topology.json (App. A.4) byte for byte.
struct FleetOptions {
  std::vector<InventoryItem> inventory;
  std::vector<std::string> regions;
  int node_size = 8;
  uint64_t seed = 7;
  double lat_lo = 5.0, lat_hi = 60.0, bw_lo = 0.9, bw_hi = 5.0;
};

Topology generate_fleet(const FleetOptions& o) {
  if (o.inventory.empty()) throw UsageError("fleet needs --gpus");
  if (o.regions.empty()) throw UsageError("fleet needs at least one region");
  if (o.node_size < 1) throw UsageError("node size must be >= 1");
  std::vector<int> left;
  int n = 0;
  for (const InventoryItem& it : o.inventory) {
    if (!fleet_catalog().count(it.gpu_model))
      throw InputError("unknown GPU model '" + it.gpu_model + "' (known: A100, H100, L40S, L4)");
    if (it.count < 1) throw InputError("inventory counts must be >= 1");
    left.push_back(it.count);
    n += it.count;
  }
  Topology t;
  const int R = static_cast<int>(o.regions.size());
  const int per_region = (n + R - 1) / R;
  size_t type = 0;
  int in_block = 0;
  for (int i = 0; i < n; ++i) {
    while (left[type] == 0 || in_block == o.node_size) {
      type = (type + 1) % left.size();
      in_block = 0;
    }
    const InventoryItem& it = o.inventory[type];
    const GpuSpec& g = fleet_catalog().at(it.gpu_model);
    Device d;
    d.id = it.gpu_model + "-" + std::to_string(i);
    d.gpu_model = it.gpu_model;
    d.comp_tflops = g.comp_tflops;
    d.mem_gb = g.mem_gb;
    d.hbm_gbps = g.hbm_gbps;
    d.intra_node_gbps = g.intra_node_gbps;
    d.region = o.regions[(i / per_region) % R];
    d.node = d.region + "-n" + std::to_string(i / o.node_size);
    t.devices.push_back(std::move(d));
    --left[type];
    ++in_block;
  }
  Rng rng(o.seed);
  for (int a = 0; a < R; ++a)
    for (int b = a + 1; b < R; ++b) {
      const double lat = rng.uniform(o.lat_lo, o.lat_hi);
      const double bw = rng.uniform(o.bw_lo, o.bw_hi);
      t.links.push_back({o.regions[a], o.regions[b], lat, bw});
    }
  t.intra_region_latency_ms = 0.1;
  t.intra_region_bandwidth_gbps = 100.0;
  return t;
}

// ---- reports (cli.cpp:21-53) ----

void print_breakdown_text(const Breakdown& bd, std::ostream& out) {
  out << std::left << std::setw(6) << "task" << std::right << std::setw(12) << "comp"
      << std::setw(12) << "tp" << std::setw(12) << "pp" << std::setw(12) << "dp" << std::setw(12)
      << "bubble" << std::setw(12) << "hbm" << std::setw(12) << "total" << "\n";
  for (const auto& [id, tc] : bd.per_task) {
    out << std::left << std::setw(6) << id << std::right << std::fixed << std::setprecision(4)
        << std::setw(12) << tc.comp << std::setw(12) << tc.tp << std::setw(12) << tc.pp
        << std::setw(12) << tc.dp << std::setw(12) << tc.bubble << std::setw(12) << tc.hbm
        << std::setw(12) << tc.total << "\n";
  }
  out << "reshard_s    " << bd.reshard_s << "\n";
  out << "sync_s       " << bd.sync_s << "\n";
  out << "end_to_end_s " << bd.end_to_end_s << "\n";
  out << "memory_ok    " << (bd.memory_feasible ? "yes" : "no") << "\n";
  out.unsetf(std::ios::fixed);
}

int run_guarded(std::ostream& err, const std::function<int()>& body) {
  try {
    return body();
  } catch (const UsageError& e) {
    err << "usage error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const InputError& e) {
    err << "input error: " << e.what() << "\n";
    return kExitInput;
  } catch (const std::exception& e) {
    err << "internal error: " << e.what() << "\n";
    return kExitInternal;
  }
}

// ---- commands ----

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;
  std::vector<std::string> positional;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
};

int cmd_plan(const Args& a, std::ostream& out, std::ostream& err, bool exhaustive) {
  return run_guarded(err, [&]() -> int {
    const std::string wf_path = a.get("--workflow"), topo_path = a.get("--topology");
    const std::string out_path = a.get("--out", "plan.json"), format = a.get("--format", "json");
    if (wf_path.empty() || topo_path.empty())
      throw UsageError(std::string(exhaustive ? "exhaustive" : "plan") +
                       " requires --workflow and --topology");
    const Workflow wf = parse_workflow(read_file(wf_path, "workflow"));
    const Topology topo = parse_topology(read_file(topo_path, "topology"));
    Engine eng(wf, topo);
    Knobs knobs = knobs_for(a.get("--knobs"));
    if (a.has("--budget") && std::stoll(a.get("--budget")) >= 0)
      knobs.budget = std::stoll(a.get("--budget"));
    bool drew_seed = false;
    if (a.has("--seed") && std::stoll(a.get("--seed")) >= 0) {
      knobs.seed = std::stoull(a.get("--seed"));
    } else if (!knobs.seed_set) {
      knobs.seed = std::random_device{}();
      drew_seed = true;
    }
    if (!exhaustive && knobs.budget < 1) throw UsageError("budget must be >= 1");
    const auto start = std::chrono::steady_clock::now();
    const Engine::Found res = eng.search(knobs, exhaustive);
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    if (!res.has_plan) {
      err << "no memory-feasible plan found for this workflow on this topology\n";
      return kExitInfeasible;
    }
    write_file(out_path, "plan", serialize_plan(res.plan, &res.bd));
    json trace = json::array();
    for (const auto& [evals, cost] : res.trace) trace.push_back({evals, cost});
    json layouts = json::object();
    for (const auto& [id, l] : res.plan.layouts)
      layouts[std::to_string(id)] = {
          {"dp", l.dp}, {"pp", l.pp}, {"tp", l.tp}, {"stage_layers", l.stage_layers}};
    json report = {{"seed", knobs.seed},
                   {"budget", knobs.budget},
                   {"consumed", res.info.consumed},
                   {"task_groupings", res.info.task_groupings},
                   {"arms", static_cast<size_t>(res.info.n_arms)},
                   {"final_cost_s", res.bd.end_to_end_s},
                   {"plan_file", out_path},
                   {"wall_clock_s", wall},
                   {"plan_summary",
                    {{"task_groups", res.plan.groups},
                     {"gpu_counts", res.plan.counts},
                     {"layouts", layouts}}},
                   {"trace", trace},
                   {"cost_breakdown", breakdown_json(res.bd)}};
    if (exhaustive) {
      report.erase("trace");
      report.erase("arms");
      report["explored"] = res.info.consumed;
      report["raw_candidates"] = res.info.budget;
    }
    if (format == "text") {
      out << "seed           " << knobs.seed << (drew_seed ? "  (drawn)" : "") << "\n";
      out << "budget         " << knobs.budget << " (consumed " << res.info.consumed << ")\n";
      out << "task groupings " << res.info.task_groupings << ", arms " << res.info.n_arms << "\n";
      out << "final cost     " << res.bd.end_to_end_s << " s\n";
      out << "wall clock     " << wall << " s\n";
      out << "plan file      " << out_path << "\n";
      out << "task groups    ";
      for (const auto& g : res.plan.groups) {
        out << "[";
        for (size_t i = 0; i < g.size(); ++i) out << (i ? "," : "") << g[i];
        out << "]";
      }
      out << "  gpu counts ";
      for (size_t i = 0; i < res.plan.counts.size(); ++i)
        out << (i ? "," : "") << res.plan.counts[i];
      out << "\n";
      for (const auto& [id, l] : res.plan.layouts)
        out << "  task " << id << ": dp=" << l.dp << " pp=" << l.pp << " tp=" << l.tp << "\n";
      out << "incumbent trace (evals -> cost):\n";
      for (const auto& [evals, cost] : res.trace)
        out << "  " << std::setw(8) << evals << "  " << cost << "\n";
      print_breakdown_text(res.bd, out);
    } else {
      out << report.dump(2) << "\n";
    }
    return kExitOk;
  });
}

int cmd_estimate(const Args& a, std::ostream& out, std::ostream& err) {
  return run_guarded(err, [&]() -> int {
    const std::string plan_path = a.get("--plan"), wf_path = a.get("--workflow"),
                      topo_path = a.get("--topology"), format = a.get("--format", "json");
    if (plan_path.empty() || wf_path.empty() || topo_path.empty())
      throw UsageError("estimate requires --plan, --workflow and --topology");
    const Workflow wf = parse_workflow(read_file(wf_path, "workflow"));
    const Topology topo = parse_topology(read_file(topo_path, "topology"));
    Engine eng(wf, topo);
    const Knobs knobs = knobs_for(a.get("--knobs"));
    const Plan plan = parse_plan(read_file(plan_path, "plan"));
    const Breakdown bd = eng.estimate(plan, knobs.cost_config());
    if (format == "text") {
      print_breakdown_text(bd, out);
    } else {
      out << breakdown_json(bd).dump(2) << "\n";
    }
    return kExitOk;
  });
}

int cmd_compare(const Args& a, std::ostream& out, std::ostream& err) {
  return run_guarded(err, [&]() -> int {
    if (a.positional.size() < 2) throw UsageError("compare requires at least two plan files");
    const std::string wf_path = a.get("--workflow"), topo_path = a.get("--topology"),
                      format = a.get("--format", "json");
    if (wf_path.empty() || topo_path.empty())
      throw UsageError("compare requires --workflow and --topology");
    const Workflow wf = parse_workflow(read_file(wf_path, "workflow"));
    const Topology topo = parse_topology(read_file(topo_path, "topology"));
    Engine eng(wf, topo);
    const Knobs knobs = knobs_for(a.get("--knobs"));
    struct Entry {
      std::string path;
      Breakdown bd;
    };
    std::vector<Entry> entries;
    for (const std::string& path : a.positional)
      entries.push_back({path, eng.estimate(parse_plan(read_file(path, "plan")),
                                            knobs.cost_config())});
    std::stable_sort(entries.begin(), entries.end(), [](const Entry& x, const Entry& y) {
      return x.bd.end_to_end_s < y.bd.end_to_end_s;
    });
    const double best = entries.front().bd.end_to_end_s;
    if (format == "text") {
      out << std::left << std::setw(4) << "#" << std::setw(32) << "plan" << std::right
          << std::setw(14) << "cost_s" << std::setw(14) << "delta_s" << "\n";
      for (size_t i = 0; i < entries.size(); ++i)
        out << std::left << std::setw(4) << i + 1 << std::setw(32) << entries[i].path
            << std::right << std::setw(14) << entries[i].bd.end_to_end_s << std::setw(14)
            << entries[i].bd.end_to_end_s - best << "\n";
    } else {
      json ranked = json::array();
      for (const Entry& e : entries)
        ranked.push_back({{"plan", e.path},
                          {"end_to_end_s", e.bd.end_to_end_s},
                          {"delta_s", e.bd.end_to_end_s - best},
                          {"cost_breakdown", breakdown_json(e.bd)}});
      out << ranked.dump(2) << "\n";
    }
    return kExitOk;
  });
}

std::vector<std::string> split_csv(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, ','))
    if (!x.empty()) out.push_back(x);
  return out;
}

int cmd_scenario(const Args& a, std::ostream& out, std::ostream& err) {
  return run_guarded(err, [&]() -> int {
    const std::string id = a.get("--id");
    const std::string out_path = a.get("--out", "topology.json");
    bool drew_seed = false;
    uint64_t seed = 0;
    if (a.has("--seed") && std::stoll(a.get("--seed")) >= 0) {
      seed = std::stoull(a.get("--seed"));
    } else {
      seed = std::random_device{}();
      drew_seed = true;
    }
    Topology topo;
    std::string label = id;
    if (id == "fleet") {
      FleetOptions o;
      o.inventory = parse_inventory(a.get("--gpus", "32xA100,32xL40S,32xL4,32xH100"));
      o.regions = split_csv(a.get("--regions", "virginia,ohio,paris,frankfurt"));
      o.node_size = std::stoi(a.get("--node-size", "8"));
      o.seed = seed;
      if (a.has("--latency-ms")) {
        const auto v = split_csv(a.get("--latency-ms"));
        if (v.size() != 2) throw UsageError("--latency-ms takes LO,HI");
        o.lat_lo = std::stod(v[0]);
        o.lat_hi = std::stod(v[1]);
      }
      if (a.has("--bandwidth-gbps")) {
        const auto v = split_csv(a.get("--bandwidth-gbps"));
        if (v.size() != 2) throw UsageError("--bandwidth-gbps takes LO,HI");
        o.bw_lo = std::stod(v[0]);
        o.bw_hi = std::stod(v[1]);
      }
      topo = generate_fleet(o);
    } else {
      if (id.empty()) throw UsageError("scenario requires --id");
      ScenarioOptions o;
      if (a.has("--gpus") && !a.get("--gpus").empty()) o.inventory = parse_inventory(a.get("--gpus"));
      o.seed = seed;
      o.node_size = std::stoi(a.get("--node-size", "8"));
      o.edge_models = split_csv(a.get("--edge-gpus", "L4"));
      int sid = 0;
      try {
        sid = std::stoi(id);
      } catch (const std::exception&) {
        throw UsageError("scenario id must be 1..4 or fleet");
      }
      topo = generate_scenario(sid, o);
    }
    write_file(out_path, "topology", serialize_topology(topo));
    out << "scenario " << label << ": " << topo.devices.size() << " devices -> " << out_path
        << " (seed " << seed << (drew_seed ? ", drawn" : "") << ")\n";
    return kExitOk;
  });
}

void usage(std::ostream& o) {
  o << "hetplan_b200: plan search for RL fine-tuning workflows on heterogeneous GPU pools "
       "(B200 engine)\n"
       "  plan       --workflow W --topology T [--knobs K] [--budget B] [--seed S] "
       "[--out plan.json] [--format json|text]\n"
       "  estimate   --plan P --workflow W --topology T [--knobs K] [--format json|text]\n"
       "  compare    PLAN PLAN... --workflow W --topology T [--knobs K] [--format json|text]\n"
       "  scenario   --id 1..4|fleet [--gpus 24xA100,...] [--seed S] [--out topology.json]\n"
       "             [--node-size 8] [--edge-gpus L4] [--regions a,b,...]\n"
       "             [--latency-ms LO,HI] [--bandwidth-gbps LO,HI]\n"
       "  exhaustive --workflow W --topology T [--knobs K] [--out plan.json] "
       "[--format json|text]\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return kExitUsage;
  }
  Args a;
  a.cmd = argv[1];
  static const std::set<std::string> with_value = {
      "--workflow", "--topology", "--knobs",      "--budget",     "--seed",
      "--out",      "--format",   "--plan",       "--id",         "--gpus",
      "--node-size", "--edge-gpus", "--regions", "--latency-ms", "--bandwidth-gbps"};
  for (int i = 2; i < argc; ++i) {
    const std::string s = argv[i];
    if (s == "--help" || s == "-h") {
      usage(std::cout);
      return kExitOk;
    }
    if (with_value.count(s)) {
      if (i + 1 >= argc) {
        std::cerr << s << ": missing value\n";
        return kExitUsage;
      }
      a.opt[s] = argv[++i];
    } else if (s.rfind("--", 0) == 0) {
      std::cerr << "unknown option " << s << "\n";
      return kExitUsage;
    } else {
      a.positional.push_back(s);
    }
  }
  const std::string fmt = a.get("--format", "json");
  if (fmt != "json" && fmt != "text") {
    std::cerr << "--format: " << fmt << " not in {json,text}\n";
    return kExitUsage;
  }
  if (a.cmd == "plan") return cmd_plan(a, std::cout, std::cerr, false);
  if (a.cmd == "exhaustive") return cmd_plan(a, std::cout, std::cerr, true);
  if (a.cmd == "estimate") return cmd_estimate(a, std::cout, std::cerr);
  if (a.cmd == "compare") return cmd_compare(a, std::cout, std::cerr);
  if (a.cmd == "scenario") return cmd_scenario(a, std::cout, std::cerr);
  usage(std::cerr);
  return kExitUsage;
}
