// Config-5 sweep scoring kernel: end_to_end_cost of
// every generated plan, many plan-warps per SM.
//
// The general eval_kernel carves one worst-case scratch area per warp (every
// array sized for sum_t dp*pp*tp = T*N), which caps a c4 sweep at a few warps
// per SM: the kernel is latency-bound (dependent FP64 chains, shuffles,
// gathers), so resident warps are its throughput. Here every warp carves
// exactly what ITS plan needs for end_to_end_cost (common.hpp e2e_sizes) out
// of a per-warp shared-memory slab, and falls back to a per-warp slab in
// global memory (L1/L2-resident) for the rare plan that does not fit. The CTA's
// warps share one shared-memory copy of the N x N link-class matrix.
//
// Each warp folds its plans into a running (min cost, lowest k) over the
// memory-feasible plans, a feasible count and an XOR of the cost bits; the
// per-warp partials persist across chunks (merged in place), so a whole sweep
// needs no host round trip until the end.
#pragma once

namespace hpg {
namespace dev {

__device__ __forceinline__ void carve_e2e(Ws& s, uint8_t* base, const E2ESizes& z, int N, int T) {
  uint8_t* p = base;
  s.w = reinterpret_cast<double*>(carve_ptr(p, 8 * z.w));
  s.nm = reinterpret_cast<int64_t*>(carve_ptr(p, 8 * z.w));
  s.rtp = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cells));
  s.ppp = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cells));
  s.cmin = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cells));
  s.dpr = reinterpret_cast<double*>(carve_ptr(p, 8 * z.dpk));
  s.dpr_sl = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * z.dpk));
  s.resident = reinterpret_cast<double*>(carve_ptr(p, 8 * N));
  s.c_comp = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cell_max));
  s.c_tp = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cell_max));
  s.c_pp = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cell_max));
  s.c_hbm = reinterpret_cast<double*>(carve_ptr(p, 8 * z.cell_max));
  s.edge = reinterpret_cast<double*>(carve_ptr(p, 8 * z.ring_max));
  s.cc = reinterpret_cast<double*>(carve_ptr(p, 8 * kMaxClasses));
  s.rm = reinterpret_cast<double*>(carve_ptr(p, 8 * 64));
  s.agg = reinterpret_cast<double*>(carve_ptr(p, 8 * T * 7));
  s.sl = reinterpret_cast<int32_t*>(carve_ptr(p, 4 * z.sl));
  s.mmt = reinterpret_cast<double*>(carve_ptr(p, 8 * z.sl));
  s.wmt = reinterpret_cast<double*>(carve_ptr(p, 8 * z.sl));
  s.dev = carve_ptr(p, z.slots);
  s.dstage = carve_ptr(p, T * N);
  s.tour = carve_ptr(p, z.ring_max);
  s.peers = carve_ptr(p, z.ring_max);
  // balancer state: never touched by end_to_end_cost
  s.wnew = s.wsave = nullptr;
  s.sl_save = s.sl_save2 = s.split_best = nullptr;
  s.dtab = nullptr;
  s.cflag = nullptr;
  s.ccell = nullptr;
}

// kWarps plan-warps per CTA, kBlocks CTAs per SM (the register budget)
template <int kWarps, int kBlocks>
__global__ void __launch_bounds__(32 * kWarps, kBlocks)
sweep_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ DevCostConfig cfg,
             const uint8_t* __restrict__ recs, int64_t stride,
             int64_t n, uint64_t k0, int slab_bytes, int cls_smem, uint8_t* __restrict__ gslab,
             int64_t gslab_bytes, EvalResult* __restrict__ res, SweepPartial* __restrict__ part,
             unsigned long long* __restrict__ n_global, int sync,
             const uint32_t* __restrict__ order) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Ws ws[kWarps];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int N = P.n_dev, T = P.n_tasks;
  const int cls_bytes = cls_smem ? carve_round(N * N) : 0;
  if (cls_smem) {
    // the CTA's copy of the link-class matrix (every ring, pair and bridge
    // edge cost is a lookup into it)
    const int nn = N * N;
    if ((nn & 15) == 0 && (reinterpret_cast<uintptr_t>(P.cls) & 15) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(P.cls);
      uint4* dst = reinterpret_cast<uint4*>(smem);
      for (int i = threadIdx.x; i < nn / 16; i += blockDim.x) dst[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < nn; i += blockDim.x) smem[i] = P.cls[i];
    }
  }
  Ws& s = ws[warp];
  if (lane == 0) {
    s.prof = nullptr;
    s.team = &s;
    s.n_warps = 1;
    s.job_words[0] = s.job_words[1] = 0;
    s.job = s.job_words;
    s.dtab_stride = 0;
    s.cls = cls_smem ? smem : P.cls;
    s.cta_sync = sync == 1 ? static_cast<int32_t>(blockDim.x) : 0;  // per-task barriers

  }
  __syncthreads();
  uint8_t* const slab = smem + cls_bytes + warp * slab_bytes;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  uint8_t* const gbase = gslab + gw * gslab_bytes;
  SweepPartial acc = part[gw];
  unsigned long long spilled = 0;
  // with sync, every warp runs the same number of rounds (one plan or an idle
  // pass each) so the CTA's barriers line up: one at the start of a plan
  // (sync >= 1) and one before each task's cost (end_to_end; sync == 1)
  const int64_t step = static_cast<int64_t>(gridDim.x) * kWarps;
  const int64_t rounds = sync ? (n + step - 1) / step : 0;
  for (int64_t p = gw, rd = 0; sync ? rd < rounds : p < n; p += step, ++rd) {
    if (sync) bar_sync(5, blockDim.x);
    if (p >= n) {
      if (sync == 1)
        for (int t = 0; t < T; ++t) bar_sync(5, blockDim.x);
      continue;
    }
    // the chunk's plans in work-class order: consecutive plans (one round of
    // a CTA) have similar per-task shapes
    const int64_t q = order ? static_cast<int64_t>(__ldg(order + p)) : p;
    const uint8_t* rec = recs + q * stride;
    // the header and offsets go straight into the warp's shared Ws (eval_one
    // restages them): no per-thread copies in local memory
    if (lane < 20) reinterpret_cast<int32_t*>(&s.h)[lane] = __ldcg(reinterpret_cast<const int32_t*>(rec) + lane);
    __syncwarp();
    if (lane == 0) {
      rec_offsets(s.h, s.o);
      const E2ESizes z = e2e_sizes(s.o, s.h, T);
      const int need = e2e_carve_bytes(z, N, T);
      const bool fits = need <= slab_bytes;
      spilled += fits ? 0 : 1;
      HPG_DCHECK(fits || need <= gslab_bytes);
      carve_e2e(s, fits ? slab : gbase, z, N, T);
    }
    __syncwarp();
    const EvalResult r =
        eval_one(P, cfg, s, 0, rec, kModeE2E, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (lane == 0) {
      if (res) res[q] = r;
      const uint64_t k = k0 + static_cast<uint64_t>(q);
      acc.xor_bits ^= static_cast<unsigned long long>(__double_as_longlong(r.cost));
      if (r.flags & kResFeasOut) {
        ++acc.n_feasible;
        if (r.cost < acc.best || (r.cost == acc.best && k < acc.best_k)) {
          acc.best = r.cost;
          acc.best_k = k;
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    part[gw] = acc;
    if (spilled) atomicAdd(n_global, spilled);
  }
}

}  // namespace dev

namespace {
template <int kWarps, int kBlocks>
cudaError_t sweep_launch_impl(const DevProblem& P, const DevCostConfig& cfg, const uint8_t* d_recs,
                              int64_t stride, int64_t n, uint64_t k0, SweepLaunch& L,
                              const uint32_t* d_order, EvalResult* d_res, cudaStream_t st) {
  auto kern = dev::sweep_kernel<kWarps, kBlocks>;
  const int dyn = L.cls_bytes + kWarps * L.slab_bytes;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), dyn);
  if (e != cudaSuccess) return e;
  kern<<<L.grid, 32 * kWarps, dyn, st>>>(P, cfg, d_recs, stride, n, k0, L.slab_bytes,
                                         L.cls_bytes > 0 ? 1 : 0, L.gslab, L.gslab_bytes, d_res,
                                         L.part, L.n_global, L.sync, d_order);
  return cudaGetLastError();
}

template <int kWarps, int kBlocks>
cudaError_t sweep_plan_impl(int N, int T, int n_sm, int slab_req, SweepLaunch& L) {
  auto kern = dev::sweep_kernel<kWarps, kBlocks>;
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return e;
  int dev = 0, smem_sm = 0, smem_blk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  L.warps = kWarps;
  L.blocks = kBlocks;
  L.cls_bytes = N * N <= kClsSweepMax ? carve_round(N * N) : 0;
  // per-CTA budget: the SM's shared memory split over the resident CTAs, less
  // the static Ws array and the 1 KB the driver reserves per CTA
  int per_cta = smem_sm / kBlocks - static_cast<int>(fa.sharedSizeBytes) - 1024;
  if (per_cta > smem_blk - static_cast<int>(fa.sharedSizeBytes)) per_cta = smem_blk - static_cast<int>(fa.sharedSizeBytes);
  int slab = ((per_cta - L.cls_bytes) / kWarps) & ~15;
  if (slab_req > 0 && slab_req < slab) slab = slab_req & ~15;
  if (slab < 1024) return cudaErrorInvalidConfiguration;
  L.slab_bytes = slab;
  L.gslab_bytes = carve_round(e2e_carve_bytes(e2e_sizes_max(N, T), N, T));
  // the occupancy query needs the dynamic shared-memory opt-in first
  e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), L.cls_bytes + kWarps * L.slab_bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = occupancy_per_sm(reinterpret_cast<const void*>(kern), 32 * kWarps,
                       L.cls_bytes + kWarps * L.slab_bytes, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  L.grid = n_sm * per_sm;
  return cudaSuccess;
}
}  // namespace

// shapes (warps x CTAs per SM): 8x2 (default), 16x1 and 8x1 (every warp of
// an SM in one CTA, phase-aligned), 4x4, 2x8
cudaError_t sweep_plan(int N, int T, int n_sm, int warps, int slab_req, SweepLaunch& L) {
  switch (warps) {
    case 16: return sweep_plan_impl<16, 1>(N, T, n_sm, slab_req, L);
    case 81: return sweep_plan_impl<8, 1>(N, T, n_sm, slab_req, L);
    case 4: return sweep_plan_impl<4, 4>(N, T, n_sm, slab_req, L);
    case 2: return sweep_plan_impl<2, 8>(N, T, n_sm, slab_req, L);
    default: return sweep_plan_impl<8, 2>(N, T, n_sm, slab_req, L);
  }
}

cudaError_t launch_sweep(const DevProblem& P, const DevCostConfig& cfg, const uint8_t* d_recs,
                         int64_t stride, int64_t n, uint64_t k0, SweepLaunch& L,
                         const uint32_t* d_order, EvalResult* d_res, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (L.warps == 16)
    return sweep_launch_impl<16, 1>(P, cfg, d_recs, stride, n, k0, L, d_order, d_res, st);
  if (L.warps == 8 && L.blocks == 1)
    return sweep_launch_impl<8, 1>(P, cfg, d_recs, stride, n, k0, L, d_order, d_res, st);
  if (L.warps == 4)
    return sweep_launch_impl<4, 4>(P, cfg, d_recs, stride, n, k0, L, d_order, d_res, st);
  if (L.warps == 2)
    return sweep_launch_impl<2, 8>(P, cfg, d_recs, stride, n, k0, L, d_order, d_res, st);
  return sweep_launch_impl<8, 2>(P, cfg, d_recs, stride, n, k0, L, d_order, d_res, st);
}

}  // namespace hpg
