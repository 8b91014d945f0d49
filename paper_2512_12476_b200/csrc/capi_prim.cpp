// C ABI of the cost-model primitives (include/hpg.h): task_cost_detail /
// task_cost, min_ring_bottleneck and min_pair_cost, one GPU call each
// (prim_kernels.cuh). The reference-side adapter (integration/) maps the
// reference's ResolvedTask / std::span arguments onto these.
#include <cstdio>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "eval_launch.hpp"

using namespace hpg;

struct hpg_ctx {
  Ctx* impl;
};

namespace {

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (err && errlen > 0) std::snprintf(err, errlen, "%s", msg.c_str());
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
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return HPG_INTERNAL;
  } catch (...) {
    set_err(err, errlen, "unknown engine failure");
    return HPG_INTERNAL;
  }
}

// device-index list -> u8 (the engine's slot type), validated against N
std::vector<uint8_t> to_slots(const int32_t* d, int n, int N, const char* what) {
  std::vector<uint8_t> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    if (d[i] < 0 || d[i] >= N) throw InputError(what);
    v[i] = static_cast<uint8_t>(d[i]);
  }
  return v;
}

// one staging area in HBM for a primitive call: [inputs | outputs]
uint8_t* stage(Ctx& C, const std::vector<std::pair<const void*, size_t>>& parts, size_t out_bytes,
               std::vector<size_t>& offs, size_t& out_off) {
  size_t total = 0;
  offs.clear();
  for (const auto& p : parts) {
    offs.push_back(total);
    total += (p.second + 15) & ~size_t(15);
  }
  out_off = total;
  total += out_bytes;
  C.d_prim.reserve(total);
  std::vector<uint8_t> h(total - out_bytes);
  for (size_t i = 0; i < parts.size(); ++i)
    if (parts[i].second) std::memcpy(h.data() + offs[i], parts[i].first, parts[i].second);
  if (!h.empty())
    cuda_check(cudaMemcpyAsync(C.d_prim.p, h.data(), h.size(), cudaMemcpyHostToDevice, C.stream),
               "H2D primitive inputs");
  C.h2d_bytes += static_cast<int64_t>(h.size());
  return C.d_prim.p;
}

}  // namespace

extern "C" {

int hpg_task_cost(hpg_ctx* ctx, const hpg_resolved_task* task, const hpg_cost_config* cfg,
                  const double* resident_weight_bytes, double agg[7], double* stage_out,
                  double* bubble_out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !task || !agg) throw UsageError("hpg_task_cost: null argument");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const Problem& P = C.prob;
    const int t = task->task_slot;
    if (t < 0 || t >= P.T) throw InputError("task slot outside the workflow");
    const int dp = task->dp, pp = task->pp, tp = task->tp;
    if (dp < 1 || pp < 1 || tp < 1) throw InputError("layout degrees must be >= 1");
    if (static_cast<int64_t>(dp) * pp * tp > P.N)
      throw InputError("layout needs more devices than the topology has");
    if (!task->stage_layers || !task->nm_replica || !task->devices)
      throw UsageError("hpg_task_cost: null layout array");
    for (int i = 0; i < dp; ++i)
      if (task->nm_replica[i] < 1) throw InputError("nm_replica entries must be >= 1");
    const std::vector<uint8_t> devs =
        to_slots(task->devices, dp * pp * tp, P.N, "device index outside the topology");
    RecHeader h{};
    h.n_tasks = P.T;
    h.dp[t] = dp;
    h.pp[t] = pp;
    h.tp[t] = tp;
    const size_t out_doubles = 7 + 4 * static_cast<size_t>(dp) * pp + dp;
    std::vector<size_t> off;
    size_t out_off = 0;
    uint8_t* D = stage(C,
                       {{task->stage_layers, 4 * static_cast<size_t>(pp)},
                        {task->nm_replica, 8 * static_cast<size_t>(dp)},
                        {devs.data(), devs.size()},
                        {resident_weight_bytes, resident_weight_bytes ? 8 * static_cast<size_t>(P.N) : 0}},
                       8 * out_doubles, off, out_off);
    const hpg_cost_config c = cfg ? *cfg : default_cost_config();
    cuda_check(launch_task_cost(C.dprob, to_dev_cfg(c), t, h, reinterpret_cast<int32_t*>(D + off[0]),
                                reinterpret_cast<int64_t*>(D + off[1]), D + off[2],
                                resident_weight_bytes ? reinterpret_cast<double*>(D + off[3]) : nullptr,
                                reinterpret_cast<double*>(D + out_off), C.stream),
               "task_cost_kernel");
    std::vector<double> out(out_doubles);
    cuda_check(cudaMemcpyAsync(out.data(), D + out_off, 8 * out_doubles, cudaMemcpyDeviceToHost,
                               C.stream), "D2H task cost");
    cuda_check(cudaStreamSynchronize(C.stream), "task_cost_kernel");
    ++C.launches;
    C.d2h_bytes += static_cast<int64_t>(8 * out_doubles);
    std::memcpy(agg, out.data(), 7 * 8);
    if (stage_out) std::memcpy(stage_out, out.data() + 7, 8 * 4 * static_cast<size_t>(dp) * pp);
    if (bubble_out) std::memcpy(bubble_out, out.data() + 7 + 4 * dp * pp, 8 * static_cast<size_t>(dp));
  });
}

int hpg_ring_bottleneck(hpg_ctx* ctx, const int32_t* devices, int32_t n, double volume_bytes,
                        double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !out) throw UsageError("hpg_ring_bottleneck: null argument");
    // min_ring_bottleneck's own checks (cost_model.cpp:181-188)
    if (n < 1) throw InputError("ring over an empty device set");
    if (!devices) throw UsageError("hpg_ring_bottleneck: null device list");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    const std::vector<uint8_t> a =
        to_slots(devices, n, C.prob.N, "ring over a device index outside the topology");
    std::vector<size_t> off;
    size_t out_off = 0;
    uint8_t* D = stage(C, {{a.data(), a.size()}}, 8, off, out_off);
    cuda_check(launch_ring(C.dprob, 0, D + off[0], n, nullptr, 0, volume_bytes,
                           reinterpret_cast<double*>(D + out_off), C.stream),
               "ring_kernel");
    cuda_check(cudaMemcpyAsync(out, D + out_off, 8, cudaMemcpyDeviceToHost, C.stream), "D2H ring");
    cuda_check(cudaStreamSynchronize(C.stream), "ring_kernel");
    ++C.launches;
  });
}

int hpg_pair_cost(hpg_ctx* ctx, const int32_t* src, int32_t n_src, const int32_t* dst,
                  int32_t n_dst, double volume_bytes, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!ctx || !ctx->impl || !out) throw UsageError("hpg_pair_cost: null argument");
    if (n_src < 0 || n_dst < 0) throw UsageError("hpg_pair_cost: negative set size");
    Ctx& C = *ctx->impl;
    const DeviceScope on_device(C.device);
    if (n_src == 0 || n_dst == 0) {
      *out = kInf;  // no pair: the reference's loop leaves +inf
      return;
    }
    if (!src || !dst) throw UsageError("hpg_pair_cost: null device list");
    const std::vector<uint8_t> a = to_slots(src, n_src, C.prob.N, "device index outside the topology");
    const std::vector<uint8_t> b = to_slots(dst, n_dst, C.prob.N, "device index outside the topology");
    std::vector<size_t> off;
    size_t out_off = 0;
    uint8_t* D = stage(C, {{a.data(), a.size()}, {b.data(), b.size()}}, 8, off, out_off);
    cuda_check(launch_ring(C.dprob, 1, D + off[0], n_src, D + off[1], n_dst, volume_bytes,
                           reinterpret_cast<double*>(D + out_off), C.stream),
               "ring_kernel");
    cuda_check(cudaMemcpyAsync(out, D + out_off, 8, cudaMemcpyDeviceToHost, C.stream), "D2H pair");
    cuda_check(cudaStreamSynchronize(C.stream), "ring_kernel");
    ++C.launches;
  });
}

}  // extern "C"
