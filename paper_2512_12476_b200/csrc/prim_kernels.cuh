// Cost-model primitives exported one call at a time through the C ABI:
//
//   task_cost_kernel  task_cost_detail / task_cost (cost_model.hpp:103-111,
//                     cost_model.cpp:270-401) of ONE resolved task
//   ring_kernel       min_ring_bottleneck (cost_model.hpp:51-52,
//                     cost_model.cpp:179-207) and min_pair_cost (:55-56,
//                     :209-218)
//
// One warp each, on the same device functions as end_to_end (eval_device.cuh),
// so the bits are those of the batched path. Scratch is carved per call from
// dynamic shared memory exactly like the sweep kernel's (carve_e2e).
#pragma once

namespace hpg {
namespace dev {

// out: agg[7] (comp, tp, pp, dp, bubble, hbm, total) | pieces [dp][pp][4]
// (comp, tp, pp, hbm) | bubble [dp]
__global__ void __launch_bounds__(32, 1)
task_cost_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ DevCostConfig cfg,
                 int t, const __grid_constant__ RecHeader h,
                 const int32_t* __restrict__ sl_in, const int64_t* __restrict__ nm_in,
                 const uint8_t* __restrict__ dev_in, const double* __restrict__ resident_in,
                 double* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ws ws[1];
  Ws& s = ws[0];
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev, T = P.n_tasks;
  if (lane == 0) {
    s.h = h;
    rec_offsets(s.h, s.o);
    carve_e2e(s, smem, e2e_sizes(s.o, s.h, T), N, T);
    s.prof = nullptr;
    s.team = &s;
    s.n_warps = 1;
    s.job_words[0] = s.job_words[1] = 0;
    s.job = s.job_words;
    s.dtab_stride = 0;
    s.cls = P.cls;
    s.cta_sync = 0;
    s.memo_tp_ok = s.memo_pp_ok = s.memo_cm_ok = 0;
    s.agg_ok = s.resident_ok = s.memv_ok = s.bridge_ok = 0;
  }
  __syncwarp();
  const int dp = h.dp[t], pp = h.pp[t], tp = h.tp[t];
  for (int j = lane; j < pp; j += 32) s.sl[s.o.sl[t] + j] = sl_in[j];
  for (int i = lane; i < dp; i += 32) {
    s.nm[s.o.w[t] + i] = nm_in[i];
    s.w[s.o.w[t] + i] = 1.0;
  }
  for (int e = lane; e < dp * pp * tp; e += 32) s.dev[s.o.dev[t] + e] = dev_in[e];
  for (int i = lane; i < s.o.dpk[T]; i += 32) s.dpr_sl[i] = -1;
  if (resident_in)
    for (int d = lane; d < N; d += 32) s.resident[d] = resident_in[d];
  __syncwarp();
  task_cost(P, cfg, s, t, resident_in != nullptr, s.agg);
  // the cells of task t are still in the cell-piece scratch
  double* pieces = out + 7;
  double* bubble = out + 7 + 4 * dp * pp;
  for (int i = lane; i < 7; i += 32) out[i] = s.agg[i];
  for (int c = lane; c < dp * pp; c += 32) {
    pieces[4 * c + 0] = s.c_comp[c];
    pieces[4 * c + 1] = s.c_tp[c];
    pieces[4 * c + 2] = s.c_pp[c];
    pieces[4 * c + 3] = s.c_hbm[c];
  }
  // bubble_cost per replica (cost_model.cpp:243-249, 343-349): training, pp > 1
  const bool bub = P.task[t].kind == kTraining && pp > 1;
  for (int i = lane; i < dp; i += 32) {
    double b = 0.0;
    if (bub) {
      double sum = 0.0;
      for (int j = 1; j < pp; ++j) {
        const int c = i * pp + j;
        sum += s.c_comp[c] + s.c_tp[c] + s.c_pp[c];
      }
      b = sum / static_cast<double>(nm_in[i]);
    }
    bubble[i] = b;
  }
}

// mode 0: min_ring_bottleneck over a[0..na); mode 1: min_pair_cost a x b
__global__ void __launch_bounds__(32, 1)
ring_kernel(const __grid_constant__ DevProblem P, int mode, const uint8_t* __restrict__ a_in, int na,
            const uint8_t* __restrict__ b_in, int nb, double volume, double* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ws ws[1];
  Ws& s = ws[0];
  const int lane = threadIdx.x & 31;
  const int N = P.n_dev, T = P.n_tasks;
  uint8_t* a = smem;
  uint8_t* b = smem + carve_round(na);
  if (lane == 0) {
    E2ESizes z{};
    z.cell_max = 1;
    z.ring_max = na > 8 ? na : 8;
    carve_e2e(s, b + carve_round(nb > 0 ? nb : 1), z, N, T);
    s.cls = P.cls;
    s.n_warps = 1;
    s.cta_sync = 0;
  }
  for (int i = lane; i < na; i += 32) a[i] = a_in[i];
  for (int i = lane; i < nb; i += 32) b[i] = b_in[i];
  __syncwarp();
  class_costs(P, s, volume);
  double r;
  if (mode == 0) {
    r = ring_bottleneck_impl(P, s, a, na, volume);
  } else {
    double best = kInf;
    for (int e = lane; e < na * nb; e += 32) best = smin(best, ecost(P, s, a[e / nb], b[e % nb]));
    r = warp_min(best);
  }
  if (lane == 0) *out = r;
}

}  // namespace dev

// dynamic shared memory of task_cost_kernel for one task header
int task_cost_smem(const RecHeader& h, int N, int T) {
  RecOffsets o;
  rec_offsets(h, o);
  return e2e_carve_bytes(e2e_sizes(o, h, T), N, T);
}

cudaError_t launch_task_cost(const DevProblem& P, const DevCostConfig& cfg, int t,
                             const RecHeader& h, const int32_t* d_sl, const int64_t* d_nm,
                             const uint8_t* d_dev, const double* d_resident, double* d_out,
                             cudaStream_t st) {
  const int bytes = task_cost_smem(h, P.n_dev, P.n_tasks);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(dev::task_cost_kernel), bytes);
  if (e != cudaSuccess) return e;
  DevProblem p = P;
  p.ring_cache = nullptr;
  dev::task_cost_kernel<<<1, 32, bytes, st>>>(p, cfg, t, h, d_sl, d_nm, d_dev, d_resident, d_out);
  return cudaGetLastError();
}

cudaError_t launch_ring(const DevProblem& P, int mode, const uint8_t* d_a, int na,
                        const uint8_t* d_b, int nb, double volume, double* d_out, cudaStream_t st) {
  E2ESizes z{};
  z.cell_max = 1;
  z.ring_max = na > 8 ? na : 8;
  const int bytes = carve_round(na) + carve_round(nb > 0 ? nb : 1) +
                    e2e_carve_bytes(z, P.n_dev, P.n_tasks);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(dev::ring_kernel), bytes);
  if (e != cudaSuccess) return e;
  DevProblem p = P;
  p.ring_cache = nullptr;
  dev::ring_kernel<<<1, 32, bytes, st>>>(p, mode, d_a, na, d_b, nb, volume, d_out);
  return cudaGetLastError();
}

}  // namespace hpg
