// shim_check — the reference's own entry points vs the B200 engine behind the
// reference-side adapter (hetplan_b200.hpp), on the same inputs, through the
// reference's own types. Prints one JSON line per case; exit status = number
// of mismatching cases. Built by oracle/Makefile (target `shim`), run on a GPU.
//
// Cases: the reference acceptance criteria #7 (mixed pool vs 24xA100, B=5000)
// and #10 (desk-scale, B=1000) (proj/tests/acceptance.cpp:379-420, 552-588),
// the survey configs c1..c4 at B=1000, and 200 random plans per config for
// end_to_end_cost, and exhaustive_search on acceptance #2's twenty instances.
// Equality = byte-identical serialize_plan(plan, &breakdown)
// plus identical SearchState (b_m, trace, arms, halvings).
#include <chrono>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <string>

#include "hetplan/cost_model.hpp"
#include "hetplan/plan.hpp"
#include "hetplan/search.hpp"
#include "hetplan/topology.hpp"
#include "hetplan/workflow.hpp"
#include "hetplan_b200.hpp"
#include "test_util.hpp"

using namespace hetplan;

namespace {

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

std::string read(const std::string& p) {
  std::ifstream in(p);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

bool same_state(const SearchState& a, const SearchState& b) {
  if (a.consumed != b.consumed || a.b_m != b.b_m || a.trace != b.trace ||
      a.arms.size() != b.arms.size() || a.halvings.size() != b.halvings.size())
    return false;
  for (size_t i = 0; i < a.arms.size(); ++i) {
    if (a.arms[i].tg_index != b.arms[i].tg_index || a.arms[i].gg_index != b.arms[i].gg_index ||
        a.arms[i].best_cost != b.arms[i].best_cost || a.arms[i].evals != b.arms[i].evals)
      return false;
  }
  for (size_t i = 0; i < a.halvings.size(); ++i) {
    const auto &x = a.halvings[i], &y = b.halvings[i];
    if (x.level != y.level || x.before != y.before || x.after != y.after ||
        x.survivor_worst != y.survivor_worst || x.eliminated_best != y.eliminated_best)
      return false;
  }
  return true;
}

int run_search(const char* name, const WorkflowGraph& wf, const DeviceTopology& topo,
               const SearchKnobs& k) {
  const double t0 = now();
  const SearchResult ref = nested_sha_search(wf, topo, k);
  const double t1 = now();
  b200::Engine eng(wf, topo);
  eng.nested_sha_search(k);  // warm-up (context buffers)
  const double t2 = now();
  const SearchResult gpu = eng.nested_sha_search(k);
  const double t3 = now();
  const bool plan_eq = ref.plan.has_value() == gpu.plan.has_value() &&
                       (!ref.plan || serialize_plan(*ref.plan, &ref.breakdown) ==
                                         serialize_plan(*gpu.plan, &gpu.breakdown));
  const bool ok = plan_eq && same_state(ref.state, gpu.state);
  std::printf(
      "{\"case\": \"%s\", \"budget\": %lld, \"ok\": %s, \"plan_bytes_identical\": %s, "
      "\"consumed\": %lld, \"best\": %.17g, \"ref_s\": %.4f, \"b200_s\": %.4f, \"speedup\": %.1f}\n",
      name, static_cast<long long>(k.budget), ok ? "true" : "false", plan_eq ? "true" : "false",
      static_cast<long long>(gpu.state.consumed),
      gpu.plan ? gpu.breakdown.end_to_end_s : -1.0, t1 - t0, t3 - t2, (t1 - t0) / (t3 - t2));
  std::fflush(stdout);
  return ok ? 0 : 1;
}

int run_costs(const char* name, const WorkflowGraph& wf, const DeviceTopology& topo) {
  Rng rng(2026);
  std::vector<Plan> plans;
  while (plans.size() < 200) {
    auto p = testutil::random_plan(wf, topo, rng);
    if (p) plans.push_back(*p);
  }
  b200::Engine eng(wf, topo);
  const auto got = eng.end_to_end_cost(plans);
  int bad = 0;
  for (size_t i = 0; i < plans.size(); ++i) {
    const CostBreakdown want = end_to_end_cost(plans[i], wf, topo);
    if (!(want == got[i])) ++bad;
  }
  std::printf("{\"case\": \"%s end_to_end_cost x200\", \"ok\": %s, \"mismatches\": %d}\n", name,
              bad ? "false" : "true", bad);
  std::fflush(stdout);
  return bad ? 1 : 0;
}

// exhaustive_search on acceptance #2's twenty instances (acceptance.cpp:116-141)
int run_exhaustive() {
  int bad = 0, n = 0;
  double ref_s = 0, gpu_s = 0;
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
        models, testutil::tiny_batch(4, 1, 8, 4, 1), i % 2 == 0 ? RunMode::kSync : RunMode::kAsync,
        0.25);
    const int n_devices = 2 + static_cast<int>(rng.bounded(3));
    const DeviceTopology topo = i % 3 == 0
                                    ? testutil::uniform_topology(n_devices, 1e13, 1e12, 64.0, 2)
                                    : testutil::random_topology(rng, 4);
    SearchKnobs k;
    k.balance_data = false;
    k.balance_layers = false;
    const double t0 = now();
    const ExhaustiveResult ref = exhaustive_search(wf, topo, k);
    const double t1 = now();
    b200::Engine eng(wf, topo);
    const ExhaustiveResult gpu = eng.exhaustive_search(k);
    const double t2 = now();
    ref_s += t1 - t0;
    gpu_s += t2 - t1;
    ++n;
    const bool ok = ref.explored == gpu.explored && ref.cost == gpu.cost &&
                    ref.plan.has_value() == gpu.plan.has_value() &&
                    (!ref.plan || serialize_plan(*ref.plan, &ref.breakdown) ==
                                      serialize_plan(*gpu.plan, &gpu.breakdown));
    if (!ok) ++bad;
  }
  std::printf("{\"case\": \"exhaustive_search acceptance#2 x%d\", \"ok\": %s, \"mismatches\": %d, "
              "\"ref_s\": %.4f, \"b200_s_incl_staging\": %.4f}\n",
              n, bad ? "false" : "true", bad, ref_s, gpu_s);
  std::fflush(stdout);
  return bad ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string fx = argc > 1 ? argv[1] : "fixtures";
  int failures = 0;
  SearchKnobs k;
  k.seed = 42;
  // acceptance #10 and #7 (proj/tests/acceptance.cpp:552-588, 379-420)
  {
    const auto wf = parse_workflow_json(read(fx + "/acc10.workflow.json"));
    const auto topo = parse_topology_json(read(fx + "/acc10.topology.json"));
    k.budget = 1000;
    failures += run_search("acceptance#10 PPO-4B scenario 3", wf, topo, k);
  }
  for (const char* c : {"acc7mixed", "acc7a100"}) {
    const auto wf = parse_workflow_json(read(fx + "/" + c + ".workflow.json"));
    const auto topo = parse_topology_json(read(fx + "/" + c + ".topology.json"));
    k.budget = 5000;
    failures += run_search(c, wf, topo, k);
  }
  for (const char* c : {"c1", "c2", "c3", "c4"}) {
    const auto wf = parse_workflow_json(read(fx + "/" + c + ".workflow.json"));
    const auto topo = parse_topology_json(read(fx + "/" + c + ".topology.json"));
    k.budget = 1000;
    failures += run_search(c, wf, topo, k);
    failures += run_costs(c, wf, topo);
  }
  failures += run_exhaustive();
  return failures;
}
