/* hpg.h — C ABI of the B200-native HetRL plan-search engine.
 *
 * Drop-in boundary for the scheduler hot path of the reference planner
 * ("hetplan", /root/reference/proj). Every entry point below replaces one
 * reference C++ call; the reference interface it stands in for is cited on
 * each declaration (file:line under proj/). Plain C types only: no torch, no
 * STL, no exceptions. Every call returns an int status that mirrors the
 * reference CLI's exit codes (proj/include/hetplan/cli.hpp:12-16):
 *
 *   HPG_OK 0, HPG_USAGE 2 (UsageError), HPG_INPUT 3 (InputError),
 *   HPG_INFEASIBLE 4 (no feasible plan), HPG_INTERNAL 5 (CUDA/engine fault)
 *
 * and copies a human-readable message into the caller's `err` buffer.
 * Inputs are copied at the call; outputs go to caller-owned arrays or to an
 * opaque result handle. A context is bound to one CUDA device and is not
 * thread-safe; separate contexts are. There is no CPU fallback: without a
 * usable sm_100 device hpg_create fails with HPG_INTERNAL.
 */
#ifndef HPG_H_
#define HPG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPG_OK 0
#define HPG_USAGE 2
#define HPG_INPUT 3
#define HPG_INFEASIBLE 4
#define HPG_INTERNAL 5

#define HPG_ABI_VERSION 3

/* ---- problem: workflow + topology (workflow.hpp:67-77, topology.hpp:24-104) ---- */

typedef struct {
  const char* id;          /* Device::id */
  const char* gpu_model;   /* Device::gpu_model */
  double comp_tflops;      /* FP16 TFLOPS */
  double mem_gb;           /* GB (x1e9) */
  double hbm_gbps;         /* GB/s (x1e9) */
  double intra_node_gbps;  /* GB/s (x1e9) */
  const char* node;
  const char* region;
} hpg_device;

typedef struct {
  const char* src;
  const char* dst;
  double latency_ms;
  double bandwidth_gbps;   /* Gbps (x1.25e8 B/s) */
} hpg_region_link;

typedef struct {
  int32_t id;              /* 1..6 (workflow.cpp:64-81) */
  int32_t kind;            /* 0 generation, 1 inference, 2 training */
  int64_t hidden_size;     /* h1 */
  int64_t intermediate_size; /* h2 */
  int64_t num_layers;      /* nl */
  int32_t include_embedding;
  int64_t vocab_size;
  int32_t precision_bytes;
} hpg_task;

typedef struct {
  int32_t algorithm;       /* 0 ppo, 1 grpo */
  int32_t mode;            /* 0 sync, 1 async */
  double eta;
  int64_t global_batch, responses_per_prompt, seq_in, seq_out, micro_batch_size;
  int32_t n_tasks;         /* tasks in id order */
  const hpg_task* tasks;
  int32_t n_dep_edges;     /* WorkflowGraph::dep_edges as (producer, consumer) pairs */
  const int32_t* dep_edges;
  int32_t n_devices;       /* DeviceTopology::make inputs (topology.cpp:44-113) */
  const hpg_device* devices;
  int32_t n_region_links;
  const hpg_region_link* region_links;
  double intra_region_latency_ms;     /* TopologyDefaults */
  double intra_region_bandwidth_gbps;
} hpg_problem;

/* CostModelConfig + MemoryModel (cost_model.hpp:13-28, plan.hpp:83-89) */
typedef struct {
  int32_t recompute;
  double reshard_override;
  double sync_override;
  double dbs_override;
  double train_bytes_per_param;
  double infer_bytes_per_param;
  double kv_bytes_per_elem;
  int32_t dbs_cap;
  double act_factor;
} hpg_cost_config;

/* ---- plans (plan.hpp:15-70) ----
 * Struct-of-arrays table of n plans. Per plan p and task slot t (workflow
 * order): task_group[p*T+t] = index of the task's group (groups ordered as in
 * TaskGrouping::groups; order of tasks inside a group = slot order),
 * gpu_counts[p*T+g] for g < n_groups[p], layout dp/pp/tp, stage_layers
 * (pp entries at sl_off), replica_batch_weights (dp entries at w_off) and the
 * flat (replica, stage, shard) device assignment as topology indices
 * (dp*pp*tp entries at dev_off). */
typedef struct {
  int32_t n_plans;
  const int32_t* n_groups;
  const int32_t* task_group;
  const int32_t* gpu_counts;
  const int32_t* dp;
  const int32_t* pp;
  const int32_t* tp;
  const int64_t* sl_off;
  const int32_t* stage_layers;
  const int64_t* w_off;
  const double* weights;
  const int64_t* dev_off;
  const int32_t* devices;
} hpg_plan_table;

/* CostBreakdown (plan.hpp:149-161); per_task rows are TaskCost
 * (comp, tp, pp, dp, bubble, hbm, total) in workflow task order. */
typedef struct {
  double* end_to_end_s;      /* [n] */
  uint8_t* memory_feasible;  /* [n] */
  double* per_task;          /* optional [n * T * 7] */
  double* reshard_s;         /* optional [n] */
  double* sync_s;            /* optional [n] */
} hpg_eval_out;

/* SearchKnobs (search.hpp:17-39) */
typedef struct {
  int64_t budget;
  uint64_t seed;
  int32_t population;
  double locality_bias;
  int32_t quantize_gpu_counts;
  int32_t level1_filter_adjacent; /* "adjacent" = 1, "off" = 0 */
  int32_t level1_cap;
  int32_t gg_arm_cap;
  int32_t swap_pair_sample;
  int32_t balance_data;
  int32_t balance_layers;
  int32_t balance_seqlen;  /* parsed, unused by the search */
  int32_t recompute;
  double reshard_override;
  double sync_override;
  /* optional tg_override (search.hpp:115-118): n_tg_override task groupings,
   * each as a per-task group index (n_tg_override * T entries) */
  int32_t n_tg_override;
  const int32_t* tg_override;
  double exhaustive_cap;   /* exhaustive_search raw-space cap (search.hpp:35) */
} hpg_knobs;

typedef struct hpg_ctx hpg_ctx;
typedef struct hpg_search_result hpg_search_result;

int hpg_abi_version(void);

void hpg_cost_config_default(hpg_cost_config* cfg);   /* CostModelConfig{} */
void hpg_knobs_default(hpg_knobs* knobs);             /* SearchKnobs{} */

/* Stages the problem on `cuda_device` (DeviceTopology::make validation and
 * link matrix, topology.cpp:44-113; workflow constants). */
int hpg_create(const hpg_problem* problem, int cuda_device, hpg_ctx** out, char* err,
               size_t errlen);
void hpg_destroy(hpg_ctx* ctx);
/* Re-validates and re-uploads a (possibly different) problem into an existing
 * context, keeping its device buffers, streams and NCCL communicator. */
int hpg_restage(hpg_ctx* ctx, const hpg_problem* problem, char* err, size_t errlen);

/* DeviceTopology::max_devices_per_node (topology.hpp:79) */
int hpg_max_devices_per_node(const hpg_ctx* ctx);
/* DeviceTopology::link (topology.hpp:75): latency_s, bandwidth_bps */
int hpg_link(const hpg_ctx* ctx, int a, int b, double* latency_s, double* bandwidth_bps);

/* end_to_end_cost (cost_model.hpp:115-117) over a batch of plans; plans are
 * validated like resolve_plan (plan.cpp:257-349). */
int hpg_eval(hpg_ctx* ctx, const hpg_plan_table* plans, const hpg_cost_config* cfg,
             hpg_eval_out* out, char* err, size_t errlen);

/* check_memory (plan.hpp:116-119): feasible[n]; optional required[n * N]
 * bytes per device (violations are the devices with required > mem). */
int hpg_check_memory(hpg_ctx* ctx, const hpg_plan_table* plans, const hpg_cost_config* cfg,
                     uint8_t* feasible, double* required, char* err, size_t errlen);

/* balance_data / balance_layers (balance.hpp:23-31) and the search's
 * evaluate() chain (search.cpp:259-279: balance_data -> balance_layers ->
 * end_to_end_cost). which: 1 data, 2 layers, 3 both (evaluate).
 * out_stage_layers / out_weights use the input's sl_off / w_off layout;
 * out_e2e[n] = end-to-end cost of the returned plan (optional). */
int hpg_balance(hpg_ctx* ctx, const hpg_plan_table* plans, const hpg_cost_config* cfg,
                int which, int32_t* out_stage_layers, double* out_weights, double* out_e2e,
                char* err, size_t errlen);

/* ---- cost-model primitives, one call each (cost_model.hpp:49-111) ---- */

/* ResolvedTask (plan.hpp:125-133): a task's layout, its micro-batches per
 * replica (nm_replica, from resolve_plan's apportionment) and its flat
 * (replica, stage, shard) device assignment as topology indices. */
typedef struct {
  int32_t task_slot;             /* workflow task index (id order) */
  int32_t dp, pp, tp;
  const int32_t* stage_layers;   /* [pp] */
  const int64_t* nm_replica;     /* [dp] */
  const int32_t* devices;        /* [dp * pp * tp] */
} hpg_resolved_task;

/* task_cost_detail / task_cost (cost_model.hpp:103-111). agg[7] = TaskCost
 * (comp, tp, pp, dp, bubble, hbm, total); optional stage[dp * pp * 4] =
 * StagePiece (comp, tp, pp, hbm) in [replica][stage] order; optional
 * bubble[dp] = bubble_replica. resident_weight_bytes: optional [N] per-device
 * residency (end_to_end_cost's path); NULL = the task's own weights (the
 * standalone call, cost_model.cpp:320-323). */
int hpg_task_cost(hpg_ctx* ctx, const hpg_resolved_task* task, const hpg_cost_config* cfg,
                  const double* resident_weight_bytes, double agg[7], double* stage,
                  double* bubble, char* err, size_t errlen);
/* min_ring_bottleneck (cost_model.hpp:49-52): InputError for an empty set or
 * an index outside the topology, 0 for one device. */
int hpg_ring_bottleneck(hpg_ctx* ctx, const int32_t* devices, int32_t n, double volume_bytes,
                        double* out, char* err, size_t errlen);
/* min_pair_cost (cost_model.hpp:54-56): +inf when either set is empty. */
int hpg_pair_cost(hpg_ctx* ctx, const int32_t* src, int32_t n_src, const int32_t* dst,
                  int32_t n_dst, double volume_bytes, double* out, char* err, size_t errlen);

/* nested_sha_search (search.hpp:115-118). */
int hpg_search(hpg_ctx* ctx, const hpg_knobs* knobs, hpg_search_result** out, char* err,
               size_t errlen);
/* Multi-GPU: one context per rank, same problem and knobs on every rank; the
 * arms of every halving round are sharded across ranks and per-arm records
 * are all-gathered (NCCL) after each round. nccl_id is the 128-byte
 * ncclUniqueId produced by hpg_nccl_unique_id on rank 0 and broadcast; it is
 * consumed by the first sharded search of the context (the communicator is
 * kept and reused; later ids are ignored unless rank/world change). */
int hpg_nccl_unique_id(uint8_t id_out[128], char* err, size_t errlen);
int hpg_search_dist(hpg_ctx* ctx, const hpg_knobs* knobs, int rank, int world,
                    const uint8_t nccl_id[128], hpg_search_result** out, char* err,
                    size_t errlen);

/* The per-round exchange hpg_search_dist performs after every SHA round
 * (SURVEY.md §8 E1), over a caller-supplied all-gather instead of NCCL, for
 * launchers with their own process group (and the CPU tests, over gloo).
 * allgather(user, send, recv, bytes): every rank sends `bytes`, recv gets
 * world * bytes in rank order; returns 0 on success. The runs of the round
 * are dealt to ranks by budget (owner[r]: longest slice first to the
 * least-loaded rank); used[r] / best[r] are inputs for the caller's own runs
 * and outputs for all; mine[] holds the improvements (run, 1-based local
 * evaluation index, cost) of the caller's runs; all[] receives every run's
 * improvements, by run, each run's in its owner's order (*n_all = count;
 * HPG_USAGE if cap is too small). Every rank ends with identical outputs. */
typedef int (*hpg_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);
typedef struct {
  int64_t run;
  int64_t local_idx;
  double cost;
} hpg_improvement;
int hpg_dist_exchange(int rank, int world, hpg_allgather_fn allgather, void* user,
                      int32_t n_runs, const int64_t* slices, int32_t* owner, int64_t* used,
                      double* best, const hpg_improvement* mine, int64_t n_mine,
                      hpg_improvement* all, int64_t cap, int64_t* n_all, char* err,
                      size_t errlen);

/* ga_search (search.hpp:132-135): one (task grouping, GPU grouping) arm.
 * task_group[T] and gpu_counts[n_groups]; rng_seed is the Rng seed. */
int hpg_ga_search(hpg_ctx* ctx, const int32_t* task_group, int32_t n_groups,
                  const int32_t* gpu_counts, int64_t budget_slice, uint64_t rng_seed,
                  const hpg_knobs* knobs, hpg_search_result** out, char* err, size_t errlen);

/* exhaustive_search (search.hpp:137-150, search.cpp:884-1031): every task
 * grouping x composition x layout x device assignment, deduplicated by
 * identical-device symmetry, evaluated on the device. Throws (HPG_INPUT) when
 * exhaustive_space_estimate exceeds knobs->exhaustive_cap. The result's
 * info.consumed = ExhaustiveResult::explored (unique plans evaluated),
 * info.budget = raw candidates enumerated; plan/breakdown as for a search
 * (HPG_INFEASIBLE from hpg_result_plan when no plan fits memory). */
int hpg_exhaustive(hpg_ctx* ctx, const hpg_knobs* knobs, hpg_search_result** out, char* err,
                   size_t errlen);
/* exhaustive_space_estimate (search.hpp:153-155, search.cpp:851-882) */
int hpg_exhaustive_estimate(hpg_ctx* ctx, const hpg_knobs* knobs, double* estimate, char* err,
                            size_t errlen);

/* SearchResult / SearchState accessors (search.hpp:79-111) */
typedef struct {
  int64_t budget, consumed;
  uint64_t seed;
  int32_t has_plan;
  int32_t n_b_m, n_trace, n_arms, n_halvings, n_survivor_sets;
  int64_t task_groupings;
  double wall_s;            /* engine wall time of the search */
  double time_to_best_s;    /* engine wall time until the final incumbent */
  int64_t gpu_launches;     /* kernel launches issued by the search */
  int64_t waves;            /* lockstep evaluation waves */
  int64_t plans_evaluated_gpu; /* plans scored on the device (incl. speculative) */
  int64_t h2d_bytes;        /* host->device bytes moved by the search */
  int64_t d2h_bytes;        /* device->host bytes moved by the search */
  double eval_kernel_ms;    /* CUDA-event time of all eval_kernel launches */
  int64_t eval_launches;
  int64_t canonical_bytes;  /* SURVEY.md §8 D1 canonical bytes of all scored plans */
  double host_ms;           /* host GA time (candidate generation, bookkeeping) */
  double batch_ms;          /* wall time of the evaluation waves (pack, copies, kernel, sync) */
} hpg_search_info;

int hpg_result_info(const hpg_search_result* r, hpg_search_info* info);
int hpg_result_b_m(const hpg_search_result* r, int64_t* b_m);
int hpg_result_trace(const hpg_search_result* r, int64_t* consumed, double* cost);
/* ArmRecord: tg_index, gg_index, best_cost, evals */
int hpg_result_arms(const hpg_search_result* r, int64_t* tg_index, int64_t* gg_index,
                    double* best_cost, int64_t* evals);
/* HalvingEvent: level, before, after, survivor_worst, eliminated_best */
int hpg_result_halvings(const hpg_search_result* r, int32_t* level, int64_t* before,
                        int64_t* after, double* survivor_worst, double* eliminated_best);
/* survivor set after every halving (same order as halvings): sizes, then the
 * concatenated survivor indices (gg indices for level 2, tg for level 1) */
int hpg_result_survivor_sizes(const hpg_search_result* r, int32_t* sizes);
int hpg_result_survivors(const hpg_search_result* r, int64_t* idx);
/* chosen plan as a one-plan table: the arrays are owned by the result */
int hpg_result_plan(const hpg_search_result* r, hpg_plan_table* plan, int32_t* groups_flat,
                    double* estimated_cost_s, uint64_t* prov_seed, int64_t* prov_budget);
/* breakdown of the chosen plan */
int hpg_result_breakdown(const hpg_search_result* r, double* per_task, double* reshard_s,
                         double* sync_s, double* end_to_end_s, uint8_t* memory_feasible);
void hpg_result_free(hpg_search_result* r);

/* Config-5 sweep: plans k in [k0, k0+count) from
 * the counter-based generator Rng(seed).fork(k), scored with
 * end_to_end_cost(CostModelConfig{}). costs/feasible optional [count];
 * best = argmin over memory-feasible plans by (cost, k). */
int hpg_sweep(hpg_ctx* ctx, uint64_t seed, uint64_t k0, uint64_t count, double* costs,
              uint8_t* feasible, double* best_cost, uint64_t* best_k, uint64_t* n_feasible,
              char* err, size_t errlen);

/* Device-resident variant for throughput measurement: the plan table and the
 * per-plan results stay in HBM, only the reduction comes back. Times are
 * CUDA-event durations on the context's launch stream. */
typedef struct {
  double best_cost;
  uint64_t best_k;
  uint64_t n_feasible;
  uint64_t xor_bits;         /* XOR of the e2e bit patterns (order-free checksum) */
  uint64_t canonical_bytes;  /* sum of SURVEY.md §8 D1 canonical bytes per plan */
  double total_ms;           /* gen + eval + reduce */
  double eval_ms;            /* eval_kernel only */
  double gen_ms;
  int64_t launches;
  uint64_t global_slab_plans; /* plans whose scratch did not fit the warp's shared slab */
} hpg_sweep_stats;

int hpg_sweep_resident(hpg_ctx* ctx, uint64_t seed, uint64_t k0, uint64_t count,
                       hpg_sweep_stats* stats, char* err, size_t errlen);

/* Sharded config-5 sweep: plans [0, total) split into one
 * contiguous plan-index range per rank; each rank sweeps its range resident in
 * HBM, then one NCCL all-gather of the 32-byte (cost, k, feasible count,
 * checksum) partials gives every rank the global argmin by (cost, lowest k).
 * Uses the context's communicator (created on first use from nccl_id, as in
 * hpg_search_dist). stats: best_cost/best_k/n_feasible/xor_bits are global;
 * canonical_bytes and the times are this rank's. world == 1 needs no nccl_id. */
int hpg_sweep_dist(hpg_ctx* ctx, uint64_t seed, uint64_t total, int rank, int world,
                   const uint8_t nccl_id[128], hpg_sweep_stats* stats, char* err,
                   size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* HPG_H_ */
