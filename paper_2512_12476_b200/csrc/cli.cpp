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
#include "rng.hpp"

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

// ---- JSON schema codec ----
//
// Every record type of the CLI's files (workflow models, devices, region
// links, knobs, layouts, cost rows) is described once as a list of fields.
// A field is required (read with json::at, whose out_of_range error names the
// first missing key in list order, so lists follow the order the reference's
// parser reads keys) or optional (json::value with the record's current value
// as default). Writing needs no ordering: nlohmann::json objects keep their
// keys sorted, so the dump(2) bytes depend only on the key/value set.

template <class R>
struct Field {
  const char* key;
  std::function<void(R&, const json&)> read;
  std::function<void(const R&, json&)> write;
};

template <class R, class M>
Field<R> required(const char* key, M R::*m) {
  return {key, [key, m](R& r, const json& j) { r.*m = j.at(key).template get<M>(); },
          [key, m](const R& r, json& j) { j[key] = r.*m; }};
}

template <class R, class M>
Field<R> optional_field(const char* key, M R::*m) {
  return {key, [key, m](R& r, const json& j) { r.*m = j.value(key, r.*m); },
          [key, m](const R& r, json& j) { j[key] = r.*m; }};
}

template <class R>
void read_record(R& r, const json& j, const std::vector<Field<R>>& fields) {
  for (const Field<R>& f : fields) f.read(r, j);
}

template <class R>
json write_record(const R& r, const std::vector<Field<R>>& fields) {
  json j = json::object();
  for (const Field<R>& f : fields) f.write(r, j);
  return j;
}

// parse `text` as `what` JSON and run `body` on it, mapping nlohmann's
// parse / schema exceptions onto the reference's InputError messages
template <class T, class Body>
T decode(const std::string& text, const char* what, Body&& body) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw InputError(std::string(what) + " JSON parse error: " + e.what());
  }
  try {
    return body(j);
  } catch (const json::exception& e) {
    throw InputError(std::string(what) + " JSON schema error: " + e.what());
  }
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
  bool has_task(int id) const { return slot_of(id) >= 0; }
  int slot_of(int id) const {
    const auto it = std::find_if(tasks.begin(), tasks.end(),
                                 [id](const hpg_task& t) { return t.id == id; });
    return it == tasks.end() ? -1 : static_cast<int>(it - tasks.begin());
  }
};

struct Model {
  int64_t hidden_size = 0, intermediate_size = 0, num_layers = 0;
  bool include_embedding = false;
  int64_t vocab_size = 0;
};

const std::vector<Field<Workflow>>& batch_fields() {
  static const std::vector<Field<Workflow>> f = {
      required("global_batch", &Workflow::global_batch),
      required("responses_per_prompt", &Workflow::rpp), required("seq_in", &Workflow::seq_in),
      required("seq_out", &Workflow::seq_out), required("micro_batch_size", &Workflow::mbs)};
  return f;
}

const std::vector<Field<Model>>& model_fields() {
  static const std::vector<Field<Model>> f = {
      required("hidden_size", &Model::hidden_size),
      required("intermediate_size", &Model::intermediate_size),
      required("num_layers", &Model::num_layers),
      optional_field("include_embedding", &Model::include_embedding),
      optional_field("vocab_size", &Model::vocab_size)};
  return f;
}

// the value of `name` among `choices` (its index), or InputError
int choose(const std::string& name, std::initializer_list<const char*> choices, const char* what) {
  int i = 0;
  for (const char* c : choices) {
    if (name == c) return i;
    ++i;
  }
  throw InputError(std::string("unknown ") + what + " '" + name + "'");
}

// PPO runs tasks 1..6, GRPO drops the critic (tasks 4, 5); each task's
// model role and kind (generation 0, inference 1, training 2)
struct TaskRole {
  int id;
  const char* model;
  int kind;
};
constexpr TaskRole kRoles[] = {{1, "actor", 0},  {2, "reward", 1}, {3, "reference", 1},
                               {4, "critic", 1}, {5, "critic", 2}, {6, "actor", 2}};

Workflow parse_workflow(const std::string& text) {
  return decode<Workflow>(text, "workflow", [](const json& j) {
    Workflow wf;
    wf.algorithm = choose(j.at("algorithm").get<std::string>(), {"ppo", "grpo"}, "algorithm");
    wf.mode = choose(j.at("mode").get<std::string>(), {"sync", "async"}, "mode");
    wf.eta = j.value("eta", 0.5);
    read_record(wf, j.at("batch"), batch_fields());
    std::map<std::string, Model> models;
    for (const auto& [name, jm] : j.at("models").items()) read_record(models[name], jm, model_fields());
    // build_workflow's checks
    if (!(wf.eta >= 0.0 && wf.eta <= 1.0)) throw InputError("eta must be within [0, 1]");
    if (std::min({wf.global_batch, wf.rpp, wf.mbs}) < 1) throw InputError("batch sizes must be >= 1");
    if (wf.seq_in < 1 || wf.seq_out < 0) throw InputError("seq_in must be >= 1 and seq_out >= 0");
    for (const TaskRole& role : kRoles) {
      if (wf.algorithm == 1 && (role.id == 4 || role.id == 5)) continue;
      const auto it = models.find(role.model);
      if (it == models.end())
        throw InputError(std::string("missing model spec '") + role.model +
                         "' required by task " + std::to_string(role.id));
      const Model& m = it->second;
      if (std::min({m.hidden_size, m.intermediate_size, m.num_layers}) < 1)
        throw InputError("model spec requires hidden_size, intermediate_size and num_layers >= 1");
      if (m.include_embedding && m.vocab_size < 1)
        throw InputError("include_embedding requires vocab_size >= 1");
      wf.tasks.push_back(hpg_task{role.id, role.kind, m.hidden_size, m.intermediate_size,
                                  m.num_layers, m.include_embedding ? 1 : 0, m.vocab_size, 2});
      wf.model_names.emplace_back(role.model);
    }
    // dependencies: generation feeds every inference task, which feeds every
    // training task
    for (const hpg_task& a : wf.tasks) {
      if (a.kind != 1) continue;
      wf.edges.emplace(1, a.id);
      for (const hpg_task& b : wf.tasks)
        if (b.kind == 2) wf.edges.emplace(a.id, b.id);
    }
    if (j.contains("precision_bytes")) {
      for (const auto& [name, jp] : j.at("precision_bytes").items())
        for (size_t s = 0; s < wf.tasks.size(); ++s)
          if (wf.model_names[s] == name) wf.tasks[s].precision_bytes = jp.get<int>();
    }
    return wf;
  });
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

const std::vector<Field<Device>>& device_fields() {
  static const std::vector<Field<Device>> f = {
      required("id", &Device::id),
      required("gpu_model", &Device::gpu_model),
      required("comp_tflops", &Device::comp_tflops),
      required("mem_gb", &Device::mem_gb),
      required("hbm_gbps", &Device::hbm_gbps),
      required("intra_node_gbps", &Device::intra_node_gbps),
      required("node", &Device::node),
      required("region", &Device::region)};
  return f;
}

const std::vector<Field<RegionLink>>& link_fields() {
  static const std::vector<Field<RegionLink>> f = {
      required("src", &RegionLink::src), required("dst", &RegionLink::dst),
      required("latency_ms", &RegionLink::latency_ms),
      required("bandwidth_gbps", &RegionLink::bandwidth_gbps)};
  return f;
}

const std::vector<Field<Topology>>& topology_default_fields() {
  static const std::vector<Field<Topology>> f = {
      optional_field("intra_region_latency_ms", &Topology::intra_region_latency_ms),
      optional_field("intra_region_bandwidth_gbps", &Topology::intra_region_bandwidth_gbps)};
  return f;
}

template <class R>
std::vector<R> read_list(const json& arr, const std::vector<Field<R>>& fields) {
  std::vector<R> out;
  for (const json& item : arr) read_record(out.emplace_back(), item, fields);
  return out;
}

template <class R>
json write_list(const std::vector<R>& items, const std::vector<Field<R>>& fields) {
  json arr = json::array();
  for (const R& r : items) arr.push_back(write_record(r, fields));
  return arr;
}

Topology parse_topology(const std::string& text) {
  return decode<Topology>(text, "topology", [](const json& j) {
    Topology t;
    t.devices = read_list(j.at("devices"), device_fields());
    if (j.contains("region_links")) t.links = read_list(j.at("region_links"), link_fields());
    if (j.contains("defaults")) read_record(t, j.at("defaults"), topology_default_fields());
    return t;
  });
}

std::string serialize_topology(const Topology& topo) {
  json j = json::object();
  j["devices"] = write_list(topo.devices, device_fields());
  j["region_links"] = write_list(topo.links, link_fields());
  j["defaults"] = write_record(topo, topology_default_fields());
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

const std::vector<Field<Knobs>>& knob_fields() {
  static const std::vector<Field<Knobs>> f = {
      optional_field("budget", &Knobs::budget),
      optional_field("seed", &Knobs::seed),
      optional_field("population", &Knobs::population),
      optional_field("locality_bias", &Knobs::locality_bias),
      optional_field("quantize_gpu_counts", &Knobs::quantize_gpu_counts),
      optional_field("level1_filter", &Knobs::level1_filter),
      optional_field("level1_cap", &Knobs::level1_cap),
      optional_field("gg_arm_cap", &Knobs::gg_arm_cap),
      optional_field("swap_pair_sample", &Knobs::swap_pair_sample),
      optional_field("balance_data", &Knobs::balance_data),
      optional_field("balance_layers", &Knobs::balance_layers),
      optional_field("balance_seqlen", &Knobs::balance_seqlen),
      optional_field("recompute", &Knobs::recompute),
      optional_field("reshard_override", &Knobs::reshard_override),
      optional_field("sync_override", &Knobs::sync_override),
      optional_field("exhaustive_cap", &Knobs::exhaustive_cap)};
  return f;
}

Knobs parse_knobs(const std::string& text) {
  Knobs k = decode<Knobs>(text, "knobs", [](const json& j) {
    Knobs r;
    read_record(r, j, knob_fields());
    r.seed_set = j.contains("seed");
    return r;
  });
  if (k.population < 1 || k.swap_pair_sample < 0 || k.gg_arm_cap < 1)
    throw InputError("knobs: population and gg_arm_cap must be >= 1");
  if (!(k.locality_bias >= 0 && k.locality_bias <= 1))
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

const std::vector<Field<Layout>>& layout_fields() {
  static const std::vector<Field<Layout>> f = {
      required("dp", &Layout::dp), required("pp", &Layout::pp), required("tp", &Layout::tp),
      required("stage_layers", &Layout::stage_layers),
      // unit weights when absent (make_layout, plan.cpp:89-100)
      {"replica_batch_weights",
       [](Layout& l, const json& j) {
         if (j.contains("replica_batch_weights"))
           l.weights = j.at("replica_batch_weights").get<std::vector<double>>();
         else
           l.weights.assign(l.dp, 1.0);
       },
       [](const Layout& l, json& j) { j["replica_batch_weights"] = l.weights; }}};
  return f;
}

const std::vector<Field<TaskCost>>& task_cost_fields() {
  static const std::vector<Field<TaskCost>> f = {
      required("comp", &TaskCost::comp), required("tp", &TaskCost::tp),
      required("pp", &TaskCost::pp), required("dp", &TaskCost::dp),
      required("bubble", &TaskCost::bubble), required("hbm", &TaskCost::hbm),
      required("total", &TaskCost::total)};
  return f;
}

const std::vector<Field<Breakdown>>& breakdown_fields() {
  static const std::vector<Field<Breakdown>> f = {
      required("reshard_s", &Breakdown::reshard_s), required("sync_s", &Breakdown::sync_s),
      required("end_to_end_s", &Breakdown::end_to_end_s),
      required("memory_feasible", &Breakdown::memory_feasible)};
  return f;
}

// "task,replica,stage,shard" keys of the plan file's assignment map
std::string tasklet_key(int task, int i, int j, int k) {
  return std::to_string(task) + "," + std::to_string(i) + "," + std::to_string(j) + "," +
         std::to_string(k);
}

// visits a layout's tasklets in flat (replica, stage, shard) order
template <class F>
void for_tasklets(int task, const Layout& l, F&& f) {
  for (int i = 0; i < l.dp; ++i)
    for (int j = 0; j < l.pp; ++j)
      for (int k = 0; k < l.tp; ++k) f(tasklet_key(task, i, j, k), l.flat(i, j, k));
}

Plan parse_plan(const std::string& text) {
  return decode<Plan>(text, "plan", [](const json& j) {
    Plan p;
    p.groups = j.at("task_groups").get<std::vector<std::vector<int>>>();
    p.counts = j.at("gpu_counts").get<std::vector<int>>();
    for (const auto& [key, jl] : j.at("layouts").items())
      read_record(p.layouts[std::stoi(key)], jl, layout_fields());
    const json& ja = j.at("assignment");
    for (const auto& [task, l] : p.layouts) {
      std::vector<std::string> devs(l.size());
      for_tasklets(task, l, [&](const std::string& key, int at) {
        if (!ja.contains(key)) throw InputError("plan assignment missing tasklet " + key);
        devs[at] = ja.at(key).get<std::string>();
      });
      p.assignment[task] = std::move(devs);
    }
    if (j.contains("provenance")) {
      const json& jp = j.at("provenance");
      p.prov_seed = jp.at("seed").get<uint64_t>();
      p.prov_budget = jp.at("budget").get<int64_t>();
    }
    p.estimated_cost_s = j.value("estimated_cost_s", -1.0);
    return p;
  });
}

json breakdown_json(const Breakdown& bd) {
  json j = write_record(bd, breakdown_fields());
  json rows = json::object();
  for (const auto& [task, tc] : bd.per_task) rows[std::to_string(task)] = write_record(tc, task_cost_fields());
  j["per_task"] = rows;
  return j;
}

std::string serialize_plan(const Plan& plan, const Breakdown* bd) {
  json layouts = json::object(), assign = json::object();
  for (const auto& [task, l] : plan.layouts) layouts[std::to_string(task)] = write_record(l, layout_fields());
  for (const auto& [task, devs] : plan.assignment) {
    const auto lit = plan.layouts.find(task);
    if (lit == plan.layouts.end()) throw InputError("plan has assignment for task without layout");
    for_tasklets(task, lit->second,
                 [&](const std::string& key, int at) { assign[key] = devs.at(at); });
  }
  json j = json::object();
  j["task_groups"] = plan.groups;
  j["gpu_counts"] = plan.counts;
  j["layouts"] = layouts;
  j["assignment"] = assign;
  j["provenance"] = json{{"seed", plan.prov_seed}, {"budget", plan.prov_budget}};
  j["estimated_cost_s"] = plan.estimated_cost_s;
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
// GPU model catalogue: the reference scenarios know A100 / L40S / L4
// (topology.cpp:228-236); the fleet generator adds H100
struct CatalogEntry {
  const char* model;
  GpuSpec spec;
  bool in_scenarios;
};
constexpr CatalogEntry kCatalog[] = {{"A100", {312.0, 40.0, 2039.0, 600.0}, true},
                                     {"L40S", {366.0, 48.0, 864.0, 64.0}, true},
                                     {"L4", {121.0, 24.0, 300.0, 64.0}, true},
                                     {"H100", {989.0, 80.0, 3350.0, 900.0}, false}};

const GpuSpec* lookup_gpu(const std::string& model, bool fleet) {
  for (const CatalogEntry& e : kCatalog)
    if (model == e.model && (fleet || e.in_scenarios)) return &e.spec;
  return nullptr;
}

Device make_device(std::string id, const std::string& model, const GpuSpec& g) {
  Device d;
  d.id = std::move(id);
  d.gpu_model = model;
  d.comp_tflops = g.comp_tflops;
  d.mem_gb = g.mem_gb;
  d.hbm_gbps = g.hbm_gbps;
  d.intra_node_gbps = g.intra_node_gbps;
  return d;
}

std::string lowercase(const std::string& s) {
  std::string r;
  r.reserve(s.size());
  for (unsigned char c : s) r.push_back(static_cast<char>(std::tolower(c)));
  return r;
}

struct InventoryItem {
  int count;
  std::string gpu_model;
};

// "24xA100,16*L4": comma-separated COUNTxMODEL entries ('x' or '*'); an empty
// entry between commas is an error, a trailing comma is not
std::vector<InventoryItem> parse_inventory(const std::string& text) {
  std::vector<std::string> parts;
  size_t from = 0;
  while (from < text.size()) {
    const size_t comma = text.find(',', from);
    const size_t to = comma == std::string::npos ? text.size() : comma;
    parts.push_back(text.substr(from, to - from));
    from = to + 1;
  }
  std::vector<InventoryItem> items;
  for (const std::string& part : parts) {
    size_t sep = part.find('x');
    if (sep == std::string::npos) sep = part.find('*');
    if (sep == std::string::npos || sep == 0 || sep + 1 >= part.size())
      throw UsageError("bad inventory entry '" + part + "' (expected COUNTxMODEL, e.g. 24xA100)");
    int count = 0;
    try {
      count = std::stoi(part.substr(0, sep));
    } catch (const std::exception&) {
      throw UsageError("bad inventory count in '" + part + "'");
    }
    items.push_back(InventoryItem{count, part.substr(sep + 1)});
  }
  if (items.empty()) throw UsageError("empty inventory");
  return items;
}

// inventory_devices (topology.cpp:240-265): "<model lowercase>-NN", numbered
// per model in inventory order
std::vector<Device> inventory_devices(const std::vector<InventoryItem>& inv) {
  std::vector<Device> devs;
  std::map<std::string, int> next_index;
  for (const InventoryItem& item : inv) {
    const GpuSpec* g = lookup_gpu(item.gpu_model, false);
    if (!g) throw InputError("unknown GPU model '" + item.gpu_model + "' (known: A100, L40S, L4)");
    if (item.count < 1) throw InputError("inventory counts must be >= 1");
    int& k = next_index[item.gpu_model];
    for (int c = 0; c < item.count; ++c, ++k) {
      std::string num = std::to_string(k);
      if (num.size() < 2) num.insert(0, 2 - num.size(), '0');
      devs.push_back(make_device(lowercase(item.gpu_model) + "-" + num, item.gpu_model, *g));
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

// one link per region pair a < b, latency then bandwidth drawn uniformly from
// Rng(seed), in pair order
void random_region_links(Topology& t, const std::vector<std::string>& regions, uint64_t seed,
                         double lat_lo, double lat_hi, double bw_lo, double bw_hi) {
  hpg::Rng rng(seed);
  for (size_t a = 0; a < regions.size(); ++a)
    for (size_t b = a + 1; b < regions.size(); ++b) {
      RegionLink l;
      l.src = regions[a];
      l.dst = regions[b];
      l.latency_ms = rng.uniform(lat_lo, lat_hi);
      l.bandwidth_gbps = rng.uniform(bw_lo, bw_hi);
      t.links.push_back(std::move(l));
    }
}

// Scenario 1: one region, nodes of node_size GPUs of one model.
void scenario_single_region(Topology& t, int node_size) {
  std::map<std::string, int> seen;
  for (Device& d : t.devices) {
    const int k = seen[d.gpu_model]++;
    d.region = "local";
    d.node = lowercase(d.gpu_model) + "-node-" + std::to_string(k / std::max(1, node_size));
  }
}

// Scenario 2: the first non-edge model in ohio, other non-edge models in
// virginia, edge models in virginia-edge; fixed cross-region rules.
void scenario_edge(Topology& t, const std::vector<std::string>& edge_models) {
  std::string ohio_model;
  std::set<std::string> regions;
  for (Device& d : t.devices) {
    const bool edge =
        std::find(edge_models.begin(), edge_models.end(), d.gpu_model) != edge_models.end();
    if (edge) {
      d.region = "virginia-edge";
    } else {
      if (ohio_model.empty()) ohio_model = d.gpu_model;
      d.region = d.gpu_model == ohio_model ? "ohio" : "virginia";
    }
    regions.insert(d.region);
  }
  struct Rule {
    const char* a;
    const char* b;
    double ms, gbps;
  };
  const Rule rules[] = {{"ohio", "virginia", 10.0, 5.0},
                        {"ohio", "virginia-edge", 10.0, 1.0},
                        {"virginia", "virginia-edge", t.intra_region_latency_ms, 1.0}};
  for (const Rule& r : rules)
    if (regions.count(r.a) && regions.count(r.b)) t.links.push_back({r.a, r.b, r.ms, r.gbps});
}

// generate_scenario (topology.cpp:310-391)
Topology generate_scenario(int id, const ScenarioOptions& o) {
  if (id < 1 || id > 4) throw UsageError("scenario id must be 1..4");
  Topology t;
  t.devices = inventory_devices(o.inventory);
  if (id == 1) {
    scenario_single_region(t, o.node_size);
    return t;
  }
  for (Device& d : t.devices) d.node = "host-" + d.id;
  if (id == 2) {
    scenario_edge(t, o.edge_models);
    return t;
  }
  // scenarios 3 (Europe, 5-30 ms, 1.9-5 Gbps) and 4 (US + Europe, 5-60 ms,
  // 0.9-5 Gbps): devices dealt round-robin over eight regions
  static const std::vector<std::string> europe = {"paris",   "stockholm", "london", "ireland",
                                                  "spain",   "zurich",    "frankfurt", "milan"};
  static const std::vector<std::string> transatlantic = {"virginia", "ohio",  "paris",  "stockholm",
                                                         "london",   "ireland", "spain", "zurich"};
  const std::vector<std::string>& regions = id == 3 ? europe : transatlantic;
  for (size_t i = 0; i < t.devices.size(); ++i) t.devices[i].region = regions[i % regions.size()];
  if (id == 3)
    random_region_links(t, regions, o.seed, 5.0, 30.0, 1.9, 5.0);
  else
    random_region_links(t, regions, o.seed, 5.0, 60.0, 0.9, 5.0);
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
    if (!lookup_gpu(it.gpu_model, true))
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
    const std::string& model = o.inventory[type].gpu_model;
    Device d = make_device(model + "-" + std::to_string(i), model, *lookup_gpu(model, true));
    d.region = o.regions[(i / per_region) % R];
    d.node = d.region + "-n" + std::to_string(i / o.node_size);
    t.devices.push_back(std::move(d));
    --left[type];
    ++in_block;
  }
  random_region_links(t, o.regions, o.seed, o.lat_lo, o.lat_hi, o.bw_lo, o.bw_hi);
  t.intra_region_latency_ms = 0.1;
  t.intra_region_bandwidth_gbps = 100.0;
  return t;
}

// ---- reports (cli.cpp:21-53) ----

// the text breakdown: a task-id column of width 6 (left), seven 12-wide
// right-aligned cost columns in fixed 4-decimal notation, then the totals.
// The stream stays in 4-digit precision afterwards, as the reference's does.
void print_breakdown_text(const Breakdown& bd, std::ostream& out) {
  static const char* const kCols[] = {"comp", "tp", "pp", "dp", "bubble", "hbm", "total"};
  out << std::left << std::setw(6) << "task" << std::right;
  for (const char* c : kCols) out << std::setw(12) << c;
  out << "\n";
  for (const auto& [task, tc] : bd.per_task) {
    const double row[] = {tc.comp, tc.tp, tc.pp, tc.dp, tc.bubble, tc.hbm, tc.total};
    out << std::left << std::setw(6) << task << std::right << std::fixed << std::setprecision(4);
    for (double v : row) out << std::setw(12) << v;
    out << "\n";
  }
  const std::pair<const char*, double> totals[] = {
      {"reshard_s    ", bd.reshard_s}, {"sync_s       ", bd.sync_s}, {"end_to_end_s ", bd.end_to_end_s}};
  for (const auto& [label, v] : totals) out << label << v << "\n";
  out << "memory_ok    " << (bd.memory_feasible ? "yes" : "no") << "\n";
  out.unsetf(std::ios::fixed);
}

// run_guarded (cli.cpp:55-68): errors become a one-line report and an exit code
int run_guarded(std::ostream& err, const std::function<int()>& body) {
  const char* kind = nullptr;
  int code = kExitOk;
  std::string what;
  try {
    return body();
  } catch (const UsageError& e) {
    kind = "usage error: ";
    code = kExitUsage;
    what = e.what();
  } catch (const InputError& e) {
    kind = "input error: ";
    code = kExitInput;
    what = e.what();
  } catch (const std::exception& e) {
    kind = "internal error: ";
    code = kExitInternal;
    what = e.what();
  }
  err << kind << what << "\n";
  return code;
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
