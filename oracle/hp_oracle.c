/* hp_oracle.c — TEST INFRASTRUCTURE ONLY (see hp_oracle.h).
 *
 * Straight restatement of the reference's evaluation path in plain C,
 * keeping the reference's loop structure and floating-point operation order
 * (build with -ffp-contract=off). No memoisation, no parallelism: this is the
 * checker, not the product. Line citations are to /root/reference/proj.
 */
#include "hp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXD 256
#define INF_ (1.0 / 0.0)

static double smax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double smin(double a, double b) { return (b < a) ? b : a; } /* std::min */

typedef struct { /* owned plan copy */
  int dp[HPO_MAX_TASKS], pp[HPO_MAX_TASKS], tp[HPO_MAX_TASKS];
  int sl[HPO_MAX_TASKS][MAXD];
  double w[HPO_MAX_TASKS][MAXD];
  int dev[HPO_MAX_TASKS][MAXD];
} oplan;

static void own(const hpo_problem* p, const hpo_plan* in, oplan* o) {
  for (int t = 0; t < p->n_tasks; ++t) {
    o->dp[t] = in->dp[t];
    o->pp[t] = in->pp[t];
    o->tp[t] = in->tp[t];
    memcpy(o->sl[t], in->sl[t], sizeof(int) * in->pp[t]);
    memcpy(o->w[t], in->w[t], sizeof(double) * in->dp[t]);
    memcpy(o->dev[t], in->dev[t], sizeof(int) * in->dp[t] * in->pp[t] * in->tp[t]);
  }
}

static void give(const hpo_problem* p, const oplan* o, hpo_plan* out) {
  for (int t = 0; t < p->n_tasks; ++t) {
    memcpy(out->sl[t], o->sl[t], sizeof(int) * o->pp[t]);
    memcpy(out->w[t], o->w[t], sizeof(double) * o->dp[t]);
  }
}

/* ---- links and rings (cost_model.cpp:18-125, 179-218) ---- */

static double edge(const hpo_problem* p, int a, int b, double v) {
  return p->lat[a * p->n_dev + b] + v / p->bw[a * p->n_dev + b];
}

/* heuristic_ring, cost_model.cpp:27-90 */
static double heuristic_ring(const hpo_problem* p, const int* devices, int n, double v) {
  int tour[MAXD], used[MAXD];
  double e[MAXD];
  memset(used, 0, sizeof(used));
  tour[0] = devices[0];
  used[0] = 1;
  for (int step = 1; step < n; ++step) {
    int best = -1;
    double bc = INF_;
    for (int i = 0; i < n; ++i) {
      if (!used[i]) {
        const double c = edge(p, tour[step - 1], devices[i], v);
        if (c < bc) {
          bc = c;
          best = i;
        }
      }
    }
    used[best] = 1;
    tour[step] = devices[best];
  }
  double bott = 0.0;
  for (int i = 0; i < n; ++i) {
    e[i] = edge(p, tour[i], tour[(i + 1) % n], v);
    bott = i == 0 ? e[i] : smax(bott, e[i]);
  }
  for (int pass = 0; pass < 8 && bott > 0; ++pass) {
    int improved = 0;
    for (int i = 1; i < n - 1; ++i) {
      for (int j = i + 1; j < n; ++j) {
        const double new1 = edge(p, tour[i - 1], tour[j], v);
        const double new2 = edge(p, tour[i], tour[(j + 1) % n], v);
        /* multiset minus the two boundary edges: max of the rest */
        double rest = 0.0;
        int any = 0;
        for (int k = 0; k < n; ++k) {
          if (k == i - 1 || k == j) continue;
          rest = any ? smax(rest, e[k]) : e[k];
          any = 1;
        }
        const double cand = smax(smax(new1, new2), rest);
        if (cand < bott) {
          for (int a = i, b = j; a < b; ++a, --b) {
            const int x = tour[a];
            tour[a] = tour[b];
            tour[b] = x;
          }
          for (int a = i, b = j - 1; a < b; ++a, --b) {
            const double x = e[a];
            e[a] = e[b];
            e[b] = x;
          }
          e[i - 1] = new1;
          e[j] = new2;
          bott = cand;
          improved = 1;
        }
      }
    }
    if (!improved) break;
  }
  return bott;
}

typedef struct {
  const hpo_problem* p;
  const int* devices;
  int n;
  double v, best;
  int path[MAXD], len, used[MAXD];
} ringsearch;

/* RingSearch::dfs, cost_model.cpp:94-125 */
static void dfs(ringsearch* r, double cur) {
  if (cur >= r->best) return;
  if (r->len == r->n) {
    r->best = smin(r->best, smax(cur, edge(r->p, r->path[r->len - 1], r->path[0], r->v)));
    return;
  }
  for (int i = 1; i < r->n; ++i) {
    if (!r->used[i]) {
      r->used[i] = 1;
      r->path[r->len++] = r->devices[i];
      dfs(r, smax(cur, edge(r->p, r->path[r->len - 2], r->path[r->len - 1], r->v)));
      --r->len;
      r->used[i] = 0;
    }
  }
}

double hpo_ring(const hpo_problem* p, const int* devices, int n, double v) {
  if (n <= 1) return 0.0;
  if (n == 2) return edge(p, devices[0], devices[1], v);
  const double ub = heuristic_ring(p, devices, n, v);
  if (n > 8) return ub;
  ringsearch r;
  memset(&r, 0, sizeof(r));
  r.p = p;
  r.devices = devices;
  r.n = n;
  r.v = v;
  r.best = ub;
  r.path[0] = devices[0];
  r.len = 1;
  r.used[0] = 1;
  dfs(&r, 0.0);
  return r.best;
}

static double min_pair(const hpo_problem* p, const int* a, int na, const int* b, int nb,
                       double v) {
  double best = INF_;
  for (int x = 0; x < na; ++x)
    for (int y = 0; y < nb; ++y) best = smin(best, edge(p, a[x], b[y], v));
  return best;
}

/* ---- memory model (plan.cpp:160-220) ---- */

static double params_on_device(const hpo_task* t, const oplan* l, int s, int stage) {
  const long long layer_params = 4 * t->h1 * t->h1 + 3 * t->h1 * t->h2;
  double pr = (double)l->sl[s][stage] * (double)layer_params / l->tp[s];
  if (t->emb) {
    const double emb = (double)t->vocab * (double)t->h1 / l->tp[s];
    if (stage == 0) pr += emb;
    if (stage == l->pp[s] - 1) pr += emb;
  }
  return pr;
}

static double kv_bytes(const hpo_problem* p, const hpo_cfg* c, const hpo_task* t,
                       const oplan* l, int s, int stage) {
  return (double)(p->seq_in + p->seq_out) * 2.0 * (double)t->h1 * (double)l->sl[s][stage] *
         c->kv_bpe / l->tp[s];
}

static double model_mem(const hpo_problem* p, const hpo_cfg* c, const oplan* l, int s,
                        int stage) {
  const hpo_task* t = &p->tasks[s];
  const double pr = params_on_device(t, l, s, stage);
  if (t->kind == 2) return pr * c->train_bpp;
  if (t->kind == 1) return pr * c->infer_bpp;
  return pr * c->infer_bpp + (double)p->mbs * c->dbs_cap * kv_bytes(p, c, t, l, s, stage);
}

static double weights_mem(const hpo_cfg* c, const hpo_task* t, const oplan* l, int s,
                          int stage) {
  const double pr = params_on_device(t, l, s, stage);
  return t->kind == 2 ? pr * c->train_bpp : pr * c->infer_bpp;
}

static double working_mem(const hpo_problem* p, const hpo_cfg* c, const oplan* l, int s,
                          int stage) {
  return (double)p->mbs * (double)(p->seq_in + p->seq_out) * (double)p->tasks[s].h1 *
         (double)l->sl[s][stage] * 2.0 * c->act_factor / l->tp[s];
}

/* check_memory, plan.cpp:351-380 */
static int check_mem(const hpo_problem* p, const hpo_cfg* c, const oplan* l, double* req) {
  double ms[MAXD], wm[MAXD];
  for (int d = 0; d < p->n_dev; ++d) ms[d] = wm[d] = 0.0;
  for (int s = 0; s < p->n_tasks; ++s)
    for (int i = 0; i < l->dp[s]; ++i)
      for (int j = 0; j < l->pp[s]; ++j)
        for (int k = 0; k < l->tp[s]; ++k) {
          const int d = l->dev[s][(i * l->pp[s] + j) * l->tp[s] + k];
          ms[d] += model_mem(p, c, l, s, j);
          wm[d] = smax(wm[d], working_mem(p, c, l, s, j));
        }
  int ok = 1;
  for (int d = 0; d < p->n_dev; ++d) {
    const double r = ms[d] + wm[d];
    if (req) req[d] = r;
    if (r > p->mem[d]) ok = 0;
  }
  return ok;
}

/* ---- resolve: nm_base + apportion (workflow.cpp:148-157, plan.cpp:222-255) ---- */

typedef struct {
  double rem;
  int idx;
} remi;

static int cmp_rem(const void* a, const void* b) {
  const remi* x = (const remi*)a;
  const remi* y = (const remi*)b;
  if (x->rem != y->rem) return x->rem > y->rem ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static void apportion(const hpo_problem* p, const oplan* l, int s, long long* out) {
  const int dp = l->dp[s];
  const long long samples = p->global_batch * p->rpp;
  const long long denom = (long long)dp * p->mbs;
  const long long nm_base = (samples + denom - 1) / denom;
  const long long total = nm_base * dp;
  double wsum = 0.0;
  for (int i = 0; i < dp; ++i) wsum += l->w[s][i];
  remi rema[MAXD];
  long long assigned = 0;
  for (int i = 0; i < dp; ++i) {
    const double quota = (double)total * l->w[s][i] / wsum;
    out[i] = (long long)floor(quota);
    rema[i].rem = quota - (double)out[i];
    rema[i].idx = i;
    assigned += out[i];
  }
  qsort(rema, dp, sizeof(remi), cmp_rem);
  for (int r = 0; assigned < total; ++assigned, ++r) ++out[rema[r % dp].idx];
  for (int i = 0; i < dp; ++i) {
    while (out[i] == 0) {
      int donor = 0;
      for (int k = 1; k < dp; ++k)
        if (out[donor] < out[k]) donor = k;
      --out[donor];
      ++out[i];
    }
  }
}

/* ---- task_cost_detail (cost_model.cpp:270-396) ---- */

typedef struct {
  double agg[7];
  double sum4[MAXD]; /* per (replica, stage) cell: comp + tp + pp + hbm */
} tdetail;

static void task_detail(const hpo_problem* p, const hpo_cfg* c, const oplan* l, int s,
                        const double* resident, tdetail* out) {
  const hpo_task* t = &p->tasks[s];
  const int dp = l->dp[s], pp = l->pp[s], tp = l->tp[s];
  long long nm[MAXD];
  apportion(p, l, s, nm);
  const long long seq_total = p->seq_in + p->seq_out;
  const double cv_tp = (double)t->prec * (double)p->mbs * (double)seq_total * (double)t->h1 *
                       (2.0 * (tp - 1) / tp);
  const double cv_pp = (double)t->prec * (double)p->mbs * (double)seq_total * (double)t->h1;
  const double tpf = t->kind != 2 ? 2.0 : (c->recompute ? 6.0 : 4.0);
  const double ppf = t->kind == 2 ? 2.0 : 1.0;
  const double cpf = t->kind == 2 ? 3.0 : 1.0;
  const long long sq = t->kind == 0 ? p->seq_in : p->seq_in + p->seq_out;
  const double sd = (double)sq, h1d = (double)t->h1, h2d = (double)t->h2;
  const double flops = 2.0 * 4.0 * sd * h1d * h1d + 2.0 * 2.0 * sd * sd * h1d +
                       2.0 * 3.0 * sd * h1d * h2d;
  double comp_[MAXD], tp_[MAXD], pp_[MAXD], hbm_[MAXD], bub[MAXD];
  for (int i = 0; i < dp; ++i) {
    for (int j = 0; j < pp; ++j) {
      const int cell = i * pp + j;
      const int* sd_ = &l->dev[s][cell * tp];
      const long long nl_j = l->sl[s][j];
      comp_[cell] = tp_[cell] = pp_[cell] = hbm_[cell] = 0.0;
      tp_[cell] = tp > 1 ? tpf * (double)nm[i] * (double)nl_j * hpo_ring(p, sd_, tp, cv_tp) : 0.0;
      for (int k = 0; k < tp; ++k) {
        const int d = sd_[k];
        comp_[cell] = smax(comp_[cell], cpf * (double)nm[i] * (double)p->mbs * (double)nl_j *
                                            flops / (p->comp[d] * tp));
        if (t->kind == 0 && p->seq_out > 0) {
          double dbs = c->dbs_override;
          if (dbs <= 0) {
            const double kv_seq = kv_bytes(p, c, t, l, s, j);
            const double res = resident ? resident[d] : weights_mem(c, t, l, s, j);
            const double free_b = p->mem[d] - res;
            dbs = floor(free_b / kv_seq);
            const double hi = (double)(nm[i] * p->mbs);
            dbs = (dbs < 1.0) ? 1.0 : ((hi < dbs) ? hi : dbs);
          }
          const double wb = (double)t->prec * (double)nl_j *
                            (4.0 * (double)t->h1 * (double)t->h1 +
                             3.0 * (double)t->h1 * (double)t->h2);
          hbm_[cell] = smax(hbm_[cell], (double)p->seq_out * (double)nm[i] * (double)p->mbs *
                                            wb / (dbs * p->hbm[d] * tp));
        }
      }
      if (j + 1 < pp) {
        pp_[cell] = ppf * (double)nm[i] * min_pair(p, sd_, tp, &l->dev[s][(cell + 1) * tp], tp, cv_pp);
      }
    }
    bub[i] = 0.0;
    if (t->kind == 2 && pp > 1) {
      double sum = 0.0;
      for (int j = 1; j < pp; ++j) {
        const int cell = i * pp + j;
        sum += comp_[cell] + tp_[cell] + pp_[cell];
      }
      bub[i] = sum / (double)nm[i];
    }
  }
  double* a = out->agg;
  for (int x = 0; x < 7; ++x) a[x] = 0.0;
  if (t->kind == 2 && dp > 1) {
    int peers[MAXD];
    for (int j = 0; j < pp; ++j) {
      const double cv_dp = (double)t->prec * (double)l->sl[s][j] *
                           (4.0 * (double)t->h1 * (double)t->h1 +
                            3.0 * (double)t->h1 * (double)t->h2) *
                           (2.0 * (dp - 1) / ((double)dp * tp));
      for (int k = 0; k < tp; ++k) {
        for (int i = 0; i < dp; ++i) peers[i] = l->dev[s][(i * pp + j) * tp + k];
        a[3] = smax(a[3], hpo_ring(p, peers, dp, cv_dp));
      }
    }
  }
  double total = 0.0;
  for (int i = 0; i < dp; ++i) {
    double stage_max = 0.0;
    for (int j = 0; j < pp; ++j) {
      const int cell = i * pp + j;
      a[0] = smax(a[0], comp_[cell]);
      a[1] = smax(a[1], tp_[cell]);
      a[2] = smax(a[2], pp_[cell]);
      a[5] = smax(a[5], hbm_[cell]);
      out->sum4[cell] = comp_[cell] + tp_[cell] + pp_[cell] + hbm_[cell];
      stage_max = smax(stage_max, out->sum4[cell]);
    }
    a[4] = smax(a[4], bub[i]);
    total = smax(total, t->kind == 2 ? stage_max + bub[i] : stage_max);
  }
  if (t->kind == 2) total += a[3];
  a[6] = total;
}

static double phi(const double* v, int n, double eta) {
  double mx = -INF_, sum = 0.0;
  for (int i = 0; i < n; ++i) {
    mx = smax(mx, v[i]);
    sum += v[i];
  }
  return mx + (1.0 - eta) * (sum - mx);
}

/* end_to_end_cost, cost_model.cpp:431-487 */
static void e2e(const hpo_problem* p, const hpo_cfg* c, const oplan* l, hpo_breakdown* bd) {
  double resident[MAXD];
  for (int d = 0; d < p->n_dev; ++d) resident[d] = 0.0;
  for (int s = 0; s < p->n_tasks; ++s)
    for (int i = 0; i < l->dp[s]; ++i)
      for (int j = 0; j < l->pp[s]; ++j)
        for (int k = 0; k < l->tp[s]; ++k)
          resident[l->dev[s][(i * l->pp[s] + j) * l->tp[s] + k]] +=
              weights_mem(c, &p->tasks[s], l, s, j);
  double tot[HPO_MAX_TASKS];
  int gen = -1, tr6 = -1;
  static tdetail det; /* large; not re-entrant (test infrastructure) */
  for (int s = 0; s < p->n_tasks; ++s) {
    task_detail(p, c, l, s, resident, &det);
    memcpy(bd->per_task[s], det.agg, sizeof(det.agg));
    tot[s] = det.agg[6];
    if (p->tasks[s].id == 1) gen = s;
    if (p->tasks[s].id == 6) tr6 = s;
  }
  double transfer = 0.0;
  const double ov = p->mode == 0 ? c->reshard_override : c->sync_override;
  if (ov >= 0) {
    transfer = ov;
  } else if (gen >= 0 && tr6 >= 0) {
    const hpo_task* g = &p->tasks[gen];
    const long long layer_params = 4 * g->h1 * g->h1 + 3 * g->h1 * g->h2;
    const long long pc = g->nl * layer_params + (g->emb ? 2 * g->vocab * g->h1 : 0);
    const double bytes = (double)pc * g->prec;
    transfer = min_pair(p, l->dev[gen], l->dp[gen] * l->pp[gen] * l->tp[gen], l->dev[tr6],
                        l->dp[tr6] * l->pp[tr6] * l->tp[tr6], bytes);
  }
  bd->reshard = p->mode == 0 ? transfer : 0.0;
  bd->sync = p->mode == 0 ? 0.0 : transfer;
  double gens[6], infs[6], trs[6];
  int ng = 0, ni = 0, nt = 0;
  for (int s = 0; s < p->n_tasks; ++s) {
    if (p->tasks[s].kind == 0) gens[ng++] = tot[s];
    else if (p->tasks[s].kind == 1) infs[ni++] = tot[s];
    else trs[nt++] = tot[s];
  }
  const double gv = ng ? phi(gens, ng, p->eta) : 0.0;
  const double iv = ni ? phi(infs, ni, p->eta) : 0.0;
  const double tv = nt ? phi(trs, nt, p->eta) : 0.0;
  bd->e2e = p->mode == 0 ? gv + iv + tv + transfer : smax(gv, iv + tv) + transfer;
  bd->feasible = check_mem(p, c, l, NULL);
}

int hpo_check_memory(const hpo_problem* p, const hpo_cfg* c, const hpo_plan* plan,
                     double* required) {
  static oplan l;
  own(p, plan, &l);
  return check_mem(p, c, &l, required);
}

void hpo_end_to_end(const hpo_problem* p, const hpo_cfg* c, const hpo_plan* plan,
                    hpo_breakdown* out) {
  static oplan l;
  own(p, plan, &l);
  e2e(p, c, &l, out);
}

/* ---- balancing (balance.cpp) ---- */

static int bal_data(const hpo_problem* p, const hpo_cfg* c, oplan* plan) {
  static oplan cand;
  cand = *plan;
  int touched = 0;
  for (int s = 0; s < p->n_tasks; ++s) {
    if (p->tasks[s].kind != 0 || plan->dp[s] < 2) continue;
    /* rate_weights, balance.cpp:14-35 (task_cost_detail without residency) */
    static tdetail det;
    task_detail(p, c, plan, s, NULL, &det);
    long long nm[MAXD];
    apportion(p, plan, s, nm);
    const int dp = plan->dp[s], pp = plan->pp[s];
    double rates[MAXD];
    for (int i = 0; i < dp; ++i) {
      double b = 0.0;
      for (int j = 0; j < pp; ++j) b = smax(b, det.sum4[i * pp + j]);
      const double per_mb = b / (double)nm[i];
      rates[i] = per_mb > 0 ? 1.0 / per_mb : 1.0;
    }
    double sum = 0.0;
    for (int i = 0; i < dp; ++i) sum += rates[i];
    for (int i = 0; i < dp; ++i) cand.w[s][i] = (double)dp * rates[i] / sum;
    touched = 1;
  }
  if (!touched) return 0;
  hpo_breakdown b0, b1;
  e2e(p, c, plan, &b0);
  e2e(p, c, &cand, &b1);
  if (b1.e2e < b0.e2e) {
    *plan = cand;
    return 1;
  }
  return 0;
}

/* task_total_with_split, balance.cpp:61-77 */
static double total_with_split(const hpo_problem* p, const hpo_cfg* c, const oplan* cand, int s,
                               const int* split) {
  static oplan trial;
  trial = *cand;
  memcpy(trial.sl[s], split, sizeof(int) * trial.pp[s]);
  if (!check_mem(p, c, &trial, NULL)) return INF_;
  static tdetail det;
  task_detail(p, c, &trial, s, NULL, &det);
  return det.agg[6];
}

static int next_comp(int* v, int parts) {
  int tail = v[parts - 1];
  for (int i = parts - 2; i >= 0; --i) {
    if (tail > parts - 1 - i) {
      ++v[i];
      for (int k = i + 1; k < parts - 1; ++k) v[k] = 1;
      v[parts - 1] = tail - 1 - (parts - 2 - i);
      return 1;
    }
    tail += v[i];
  }
  return 0;
}

static int bal_layers(const hpo_problem* p, const hpo_cfg* c, oplan* plan) {
  static oplan cand;
  cand = *plan;
  int touched = 0;
  for (int s = 0; s < p->n_tasks; ++s) {
    const long long nl = p->tasks[s].nl;
    const int pp = cand.pp[s];
    if (pp < 2 || nl == pp) continue;
    int best_split[MAXD];
    memcpy(best_split, cand.sl[s], sizeof(int) * pp);
    double best = total_with_split(p, c, &cand, s, best_split);
    if ((long long)pp * nl <= 64) {
      int split[MAXD];
      for (int k = 0; k < pp - 1; ++k) split[k] = 1;
      split[pp - 1] = (int)nl - (pp - 1);
      do {
        const double v = total_with_split(p, c, &cand, s, split);
        if (v < best) {
          best = v;
          memcpy(best_split, split, sizeof(int) * pp);
        }
      } while (next_comp(split, pp));
    } else {
      while (1) {
        static tdetail det;
        task_detail(p, c, &cand, s, NULL, &det);
        int bn = 0;
        double worst = -1.0;
        for (int j = 0; j < pp; ++j) {
          double load = 0.0;
          for (int i = 0; i < cand.dp[s]; ++i) load = smax(load, det.sum4[i * pp + j]);
          if (load > worst) {
            worst = load;
            bn = j;
          }
        }
        if (best_split[bn] <= 1) break;
        double step_best = best;
        int have = 0, step_split[MAXD];
        for (int side = 0; side < 2; ++side) {
          const int nb = side == 0 ? bn - 1 : bn + 1;
          if (nb < 0 || nb >= pp) continue;
          int split[MAXD];
          memcpy(split, best_split, sizeof(int) * pp);
          --split[bn];
          ++split[nb];
          const double v = total_with_split(p, c, &cand, s, split);
          if (v < step_best) {
            step_best = v;
            memcpy(step_split, split, sizeof(int) * pp);
            have = 1;
          }
        }
        if (!have) break;
        best = step_best;
        memcpy(best_split, step_split, sizeof(int) * pp);
        /* the candidate's layout is the loop's `layout` (balance.cpp:85, 150) */
        memcpy(cand.sl[s], best_split, sizeof(int) * pp);
      }
    }
    if (memcmp(best_split, cand.sl[s], sizeof(int) * pp) != 0) {
      memcpy(cand.sl[s], best_split, sizeof(int) * pp);
      touched = 1;
    }
  }
  if (!touched) return 0;
  if (!check_mem(p, c, &cand, NULL)) return 0;
  hpo_breakdown b0, b1;
  e2e(p, c, plan, &b0);
  e2e(p, c, &cand, &b1);
  if (b1.e2e < b0.e2e) {
    *plan = cand;
    return 1;
  }
  return 0;
}

int hpo_balance_data(const hpo_problem* p, const hpo_cfg* c, hpo_plan* plan) {
  static oplan l;
  own(p, plan, &l);
  const int ch = bal_data(p, c, &l);
  give(p, &l, plan);
  return ch;
}

int hpo_balance_layers(const hpo_problem* p, const hpo_cfg* c, hpo_plan* plan) {
  static oplan l;
  own(p, plan, &l);
  const int ch = bal_layers(p, c, &l);
  give(p, &l, plan);
  return ch;
}

void hpo_evaluate(const hpo_problem* p, const hpo_cfg* c, hpo_plan* plan, hpo_breakdown* out) {
  static oplan l;
  own(p, plan, &l);
  bal_data(p, c, &l);
  bal_layers(p, c, &l);
  e2e(p, c, &l, out);
  give(p, &l, plan);
}
