/* hp_oracle — CPU restatement of the reference planner's evaluation path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker. The
 * product (paper_2512_12476_b200/libhpg.so) never links or calls it.
 *
 * Restates, in plain C and in the reference's operation order, the functions
 * of /root/reference/proj on the north-star path:
 *   end_to_end_cost       cost_model.cpp:431-487
 *   task_cost_detail      cost_model.cpp:270-396
 *   min_ring_bottleneck   cost_model.cpp:179-207 (heuristic_ring :27-90,
 *                         RingSearch::dfs :94-125)
 *   min_pair_cost         cost_model.cpp:209-218
 *   check_memory          plan.cpp:351-380 (memory model :160-220)
 *   apportion             plan.cpp:222-255, derive_num_microbatches
 *                         workflow.cpp:148-157
 *   balance_data          balance.cpp:14-56
 *   balance_layers        balance.cpp:58-167
 * Parity is pinned: tests/test_oracle.py checks it bit-for-bit against the
 * golden vectors of the compiled reference (tests/golden/, oracle/ref_dump).
 */
#ifndef HP_ORACLE_H_
#define HP_ORACLE_H_

#ifdef __cplusplus
extern "C" {
#endif

#define HPO_MAX_TASKS 6

typedef struct {
  int id, kind, prec, emb; /* kind: 0 generation, 1 inference, 2 training */
  long long h1, h2, nl, vocab;
} hpo_task;

typedef struct {
  int n_dev;
  const double* comp; /* FLOP/s */
  const double* mem;  /* bytes */
  const double* hbm;  /* bytes/s */
  const double* lat;  /* n_dev*n_dev seconds */
  const double* bw;   /* n_dev*n_dev bytes/s */
  int n_tasks;
  hpo_task tasks[HPO_MAX_TASKS];
  int mode; /* 0 sync 1 async */
  double eta;
  long long global_batch, rpp, seq_in, seq_out, mbs;
} hpo_problem;

typedef struct {
  int recompute;
  double reshard_override, sync_override, dbs_override;
  double train_bpp, infer_bpp, kv_bpe;
  int dbs_cap;
  double act_factor;
} hpo_cfg;

/* one plan; per task slot (workflow order) */
typedef struct {
  int dp[HPO_MAX_TASKS], pp[HPO_MAX_TASKS], tp[HPO_MAX_TASKS];
  int* sl[HPO_MAX_TASKS];    /* pp entries */
  double* w[HPO_MAX_TASKS];  /* dp entries */
  int* dev[HPO_MAX_TASKS];   /* dp*pp*tp entries, flat (replica, stage, shard) */
} hpo_plan;

typedef struct {
  double per_task[HPO_MAX_TASKS][7]; /* comp, tp, pp, dp, bubble, hbm, total */
  double reshard, sync, e2e;
  int feasible;
} hpo_breakdown;

double hpo_ring(const hpo_problem* p, const int* devs, int n, double volume);
int hpo_check_memory(const hpo_problem* p, const hpo_cfg* c, const hpo_plan* plan,
                     double* required /* optional n_dev */);
void hpo_end_to_end(const hpo_problem* p, const hpo_cfg* c, const hpo_plan* plan,
                    hpo_breakdown* out);
/* in place; return 1 when the returned plan differs from the input */
int hpo_balance_data(const hpo_problem* p, const hpo_cfg* c, hpo_plan* plan);
int hpo_balance_layers(const hpo_problem* p, const hpo_cfg* c, hpo_plan* plan);
/* the search's evaluate() chain: balance_data -> balance_layers -> e2e */
void hpo_evaluate(const hpo_problem* p, const hpo_cfg* c, hpo_plan* plan, hpo_breakdown* out);

#ifdef __cplusplus
}
#endif

#endif
