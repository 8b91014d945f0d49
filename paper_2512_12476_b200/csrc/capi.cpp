// extern "C" entry points of include/hpg.h. Exceptions never cross the
// boundary: they become HPG_* status codes plus a message (the mapping of
// run_guarded, proj/src/cli.cpp:55-68).
#include <cstdio>
#include <cstring>

#include "engine.hpp"
#include "search.hpp"

using namespace hpg;

struct hpg_ctx {
  Ctx* impl;
};

namespace {

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::snprintf(err, errlen, "%s", msg.c_str());
  }
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    set_err(err, errlen, "");
    return HPG_OK;
  } catch (const UsageError& e) {
    set_err(err, errlen, e.what());
    return HPG_USAGE;
  } catch (const InputError& e) {
    set_err(err, errlen, e.what());
    return HPG_INPUT;
  } catch (const InfeasibleError& e) {
    set_err(err, errlen, e.what());
    return HPG_INFEASIBLE;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return HPG_INTERNAL;
  } catch (...) {
    set_err(err, errlen, "unknown engine failure");
    return HPG_INTERNAL;
  }
}

void check_ctx(const hpg_ctx* c) {
  if (c == nullptr || c->impl == nullptr) throw UsageError("null engine context");
}

}  // namespace

extern "C" {

int hpg_abi_version(void) { return HPG_ABI_VERSION; }

void hpg_cost_config_default(hpg_cost_config* cfg) {
  if (cfg) *cfg = default_cost_config();
}

void hpg_knobs_default(hpg_knobs* k) {
  if (!k) return;
  std::memset(k, 0, sizeof(*k));
  k->budget = 1000;
  k->seed = 0;
  k->population = 16;
  k->locality_bias = 0.8;
  k->quantize_gpu_counts = 1;
  k->level1_filter_adjacent = 0;
  k->level1_cap = 0;
  k->gg_arm_cap = 64;
  k->swap_pair_sample = 8;
  k->balance_data = 1;
  k->balance_layers = 1;
  k->balance_seqlen = 1;
  k->recompute = 1;
  k->reshard_override = -1.0;
  k->sync_override = -1.0;
  k->n_tg_override = 0;
  k->tg_override = nullptr;
  k->exhaustive_cap = 1e6;
}

int hpg_create(const hpg_problem* problem, int cuda_device, hpg_ctx** out, char* err,
               size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!problem || !out) throw UsageError("hpg_create: null argument");
    *out = nullptr;
    Ctx* c = create_ctx(*problem, cuda_device);
    *out = new hpg_ctx{c};
  });
}

void hpg_destroy(hpg_ctx* ctx) {
  if (!ctx) return;
  if (ctx->impl) {
    const DeviceScope on_device(ctx->impl->device);
    delete ctx->impl;
  }
  delete ctx;
}

int hpg_max_devices_per_node(const hpg_ctx* ctx) {
  return ctx && ctx->impl ? ctx->impl->prob.max_node_size : -1;
}

int hpg_restage(hpg_ctx* ctx, const hpg_problem* problem, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_ctx(ctx);
    if (!problem) throw UsageError("hpg_restage: null problem");
    const DeviceScope on_device(ctx->impl->device);
    restage(*ctx->impl, *problem);
  });
}

int hpg_link(const hpg_ctx* ctx, int a, int b, double* latency_s, double* bandwidth_bps) {
  if (!ctx || !ctx->impl) return HPG_USAGE;
  const Problem& P = ctx->impl->prob;
  if (a < 0 || b < 0 || a >= P.N || b >= P.N) return HPG_INPUT;
  const int c = P.cls[static_cast<size_t>(a) * P.N + b];
  if (latency_s) *latency_s = P.lat[c];
  if (bandwidth_bps) *bandwidth_bps = P.bw[c];
  return HPG_OK;
}

int hpg_eval(hpg_ctx* ctx, const hpg_plan_table* plans, const hpg_cost_config* cfg,
             hpg_eval_out* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_ctx(ctx);
    if (!plans || !out) throw UsageError("hpg_eval: null argument");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const hpg_cost_config c = cfg ? *cfg : default_cost_config();
    std::vector<TablePlan> tps = unpack_table(C.prob, *plans);
    Batch b;
    for (auto& tp : tps) {
      b.cands.push_back(&tp.cand);
      b.modes.push_back(kModeE2E);
    }
    BatchOut bo;
    run_batch(C, b, to_dev_cfg(c), 0, false, out->per_task != nullptr, false, bo);
    const int T = C.prob.T;
    for (size_t i = 0; i < tps.size(); ++i) {
      if (out->end_to_end_s) out->end_to_end_s[i] = bo.res[i].cost;
      if (out->memory_feasible) out->memory_feasible[i] = (bo.res[i].flags & kResFeasOut) ? 1 : 0;
      if (out->reshard_s) out->reshard_s[i] = bo.res[i].reshard_s;
      if (out->sync_s) out->sync_s[i] = bo.res[i].sync_s;
    }
    if (out->per_task) std::memcpy(out->per_task, bo.per_task.data(), 8 * tps.size() * T * 7);
  });
}

int hpg_check_memory(hpg_ctx* ctx, const hpg_plan_table* plans, const hpg_cost_config* cfg,
                     uint8_t* feasible, double* required, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    check_ctx(ctx);
    if (!plans) throw UsageError("hpg_check_memory: null argument");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const hpg_cost_config c = cfg ? *cfg : default_cost_config();
    std::vector<TablePlan> tps = unpack_table(C.prob, *plans);
    Batch b;
    for (auto& tp : tps) {
      b.cands.push_back(&tp.cand);
      b.modes.push_back(kModeMemcheck);
    }
    BatchOut bo;
    run_batch(C, b, to_dev_cfg(c), 0, false, false, required != nullptr, bo);
    for (size_t i = 0; i < tps.size(); ++i) {
      if (feasible) feasible[i] = (bo.res[i].flags & kResFeasIn) ? 1 : 0;
    }
    if (required) std::memcpy(required, bo.required.data(), 8 * bo.required.size());
  });
}

int hpg_balance(hpg_ctx* ctx, const hpg_plan_table* plans, const hpg_cost_config* cfg, int which,
                int32_t* out_stage_layers, double* out_weights, double* out_e2e, char* err,
                size_t errlen) {
  return guarded(err, errlen, [&] {
    check_ctx(ctx);
    if (!plans) throw UsageError("hpg_balance: null argument");
    if (which < 1 || which > 3) throw UsageError("hpg_balance: which must be 1, 2 or 3");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const hpg_cost_config c = cfg ? *cfg : default_cost_config();
    std::vector<TablePlan> tps = unpack_table(C.prob, *plans);
    Batch b;
    const int mode = which == 1 ? kModeBalanceData : (which == 2 ? kModeBalanceLayers : kModeChain);
    for (auto& tp : tps) {
      b.cands.push_back(&tp.cand);
      b.modes.push_back(mode);
    }
    BatchOut bo;
    run_batch(C, b, to_dev_cfg(c), which == 3 ? 3 : 0, true, false, false, bo);
    const int T = C.prob.T;
    for (size_t i = 0; i < tps.size(); ++i) {
      Cand& in = tps[i].cand;
      apply_ws(C.prob, in, bo.out_ws + bo.ws_off[i]);
      const double* w = in.w();
      const int32_t* sl = in.sl();
      for (int s = 0; s < T; ++s) {
        if (out_stage_layers) {
          const int64_t so = plans->sl_off[static_cast<int64_t>(i) * T + s];
          for (int j = 0; j < in.hdr().pp[s]; ++j) out_stage_layers[so + j] = sl[in.o.sl[s] + j];
        }
        if (out_weights) {
          const int64_t wo = plans->w_off[static_cast<int64_t>(i) * T + s];
          for (int k = 0; k < in.hdr().dp[s]; ++k) out_weights[wo + k] = w[in.o.w[s] + k];
        }
      }
      if (out_e2e) out_e2e[i] = bo.res[i].cost;
    }
  });
}

}  // extern "C"
