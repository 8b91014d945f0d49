// hetplan_b200 — reference-side adapter: the hetplan API (same names, same
// argument meaning, same exceptions) implemented over the B200 engine's C ABI
// (include/hpg.h). A hetplan maintainer adds this header + hetplan_b200.cpp to
// proj/src and links libhpg.so; call sites switch from hetplan::X to
// hetplan::b200::X (or keep an Engine per problem to amortise staging).
//
// Compiled against the reference headers (proj/include/hetplan/*.hpp); it is
// not part of the engine library itself.
#pragma once

#include <memory>
#include <optional>
#include <span>
#include <vector>

#include "hetplan/balance.hpp"
#include "hetplan/cost_model.hpp"
#include "hetplan/plan.hpp"
#include "hetplan/search.hpp"
#include "hetplan/topology.hpp"
#include "hetplan/workflow.hpp"

struct hpg_ctx;

namespace hetplan::b200 {

// One (workflow, topology) staged on one GPU. Throws InputError / UsageError
// like the reference; engine faults surface as std::runtime_error.
class Engine {
 public:
  Engine(const WorkflowGraph& wf, const DeviceTopology& topo, int cuda_device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // end_to_end_cost (cost_model.hpp:115-117), batched
  std::vector<CostBreakdown> end_to_end_cost(const std::vector<Plan>& plans,
                                             const CostModelConfig& cfg = {});
  // task_cost_detail / task_cost (cost_model.hpp:103-111) of one resolved task
  TaskCostDetail task_cost_detail(const ResolvedTask& rt, const CostModelConfig& cfg = {},
                                  std::span<const double> resident_weight_bytes = {});
  // min_ring_bottleneck / min_pair_cost (cost_model.hpp:49-56)
  double min_ring_bottleneck(std::span<const int> devices, double volume_bytes);
  double min_pair_cost(std::span<const int> src, std::span<const int> dst, double volume_bytes);
  // check_memory (plan.hpp:116-119)
  std::vector<MemoryViolation> check_memory(const Plan& plan, const MemoryModel& mm = {});
  // balance_data / balance_layers (balance.hpp:23-31)
  Plan balance_data(const Plan& plan, const CostModelConfig& cfg = {});
  Plan balance_layers(const Plan& plan, const CostModelConfig& cfg = {});
  // nested_sha_search (search.hpp:115-118)
  SearchResult nested_sha_search(const SearchKnobs& knobs,
                                 const std::vector<TaskGrouping>* tg_override = nullptr);
  // exhaustive_search / exhaustive_space_estimate (search.hpp:137-155)
  ExhaustiveResult exhaustive_search(const SearchKnobs& knobs);
  double exhaustive_space_estimate(const SearchKnobs& knobs);

 private:
  const WorkflowGraph& wf_;
  const DeviceTopology& topo_;
  hpg_ctx* ctx_ = nullptr;
};

// Free-function forms with the reference signatures (stage the problem per
// call; prefer Engine for repeated calls).
CostBreakdown end_to_end_cost(const Plan& plan, const WorkflowGraph& wf,
                              const DeviceTopology& topo, const CostModelConfig& cfg = {});
SearchResult nested_sha_search(const WorkflowGraph& wf, const DeviceTopology& topo,
                               const SearchKnobs& knobs,
                               const std::vector<TaskGrouping>* tg_override = nullptr);
ExhaustiveResult exhaustive_search(const WorkflowGraph& wf, const DeviceTopology& topo,
                                   const SearchKnobs& knobs);
TaskCostDetail task_cost_detail(const WorkflowGraph& wf, const ResolvedTask& rt,
                                const DeviceTopology& topo, const CostModelConfig& cfg = {},
                                std::span<const double> resident_weight_bytes = {});
TaskCost task_cost(const WorkflowGraph& wf, const ResolvedTask& rt, const DeviceTopology& topo,
                   const CostModelConfig& cfg = {});
// link costs depend on the topology only: staged with a placeholder workflow
double min_ring_bottleneck(std::span<const int> devices, double volume_bytes,
                           const DeviceTopology& topo);
double min_pair_cost(std::span<const int> src, std::span<const int> dst, double volume_bytes,
                     const DeviceTopology& topo);

}  // namespace hetplan::b200
