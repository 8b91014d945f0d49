// Config-5 sweep: 10^8-scale exhaustive cost-model
// sweep over synthetic candidates from a counter-based generator.
//
//   gen_kernel     one thread per plan k: stream Rng(seed).fork(k) (rng.hpp:64)
//                  -> task grouping, sample_composition (combinatorics.cpp:115-146),
//                  layouts (enumerate_layouts order, search.cpp:127-150), a device
//                  permutation and one shuffle per task; writes a compact plan
//                  record into the HBM plan table
//   sweep_kernel   end_to_end_cost per plan (one warp per plan, many plan-warps
//                  per SM; sweep_kernel.cuh) folded into per-warp partials:
//                  argmin over memory-feasible plans by (cost, k), feasible
//                  count, XOR checksum of the cost bit patterns
#include <cuda_runtime.h>

#include "common.hpp"
#include "eval_launch.hpp"
#include "rng.hpp"
#include "sweep.hpp"

namespace hpg {
namespace dev {

// Work estimate of one task of a plan (end_to_end_cost's phases: cell
// pieces, TP ring bounds, PP pairs, DP rings) and its class on a log2 scale
// with `halves` sub-steps per octave, clamped to `levels` classes
__device__ __forceinline__ uint32_t work_estimate(int dp, int pp, int tp, bool train) {
  const int ncell = dp * pp;
  uint32_t w = 2u * ((ncell + 31) >> 5) + static_cast<uint32_t>(((dp + 31) >> 5) * pp);
  if (tp > 1) w += static_cast<uint32_t>(((ncell * tp + 31) >> 5) * tp);
  if (pp > 1) w += static_cast<uint32_t>((ncell * tp * tp + 31) >> 5);
  if (train && dp > 1) w += static_cast<uint32_t>(pp * tp * (dp == 2 ? 1 : (dp <= 8 ? 24 : 4 * dp)));
  return w;
}
__device__ __forceinline__ uint32_t work_class(uint32_t w, int halves, int levels) {
  // floor(halves * log2(w)) from the leading bit and the next one
  const int lg = 31 - __clz(w | 1u);
  int c = halves * lg;
  if (halves == 2 && lg > 0 && ((w >> (lg - 1)) & 1u)) ++c;
  c -= 3 * halves;  // w < 8: class 0
  return static_cast<uint32_t>(c < 0 ? 0 : (c >= levels ? levels - 1 : c));
}

__global__ void gen_kernel(SweepTablesDev tb, uint64_t seed, uint64_t k0, int64_t n,
                           uint8_t* __restrict__ recs, int64_t stride,
                           unsigned long long* __restrict__ bytes_acc,
                           uint32_t* __restrict__ keys, uint32_t* __restrict__ hist) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t my_bytes = 0;
  if (idx < n) {
    const uint64_t k = k0 + static_cast<uint64_t>(idx);
    Rng rng = Rng(seed).fork(k);
    const int N = tb.n_dev, T = tb.n_tasks;
    const int ti = static_cast<int>(rng.bounded(static_cast<uint64_t>(tb.n_tgs)));
    const int8_t* grp = tb.tg_group + ti * kMaxTasks;
    const int ng = tb.tg_ng[ti];
    // sample_composition(N, ng, 1): distinct cut points by rejection, sorted
    int cuts[kMaxTasks];
    int nc = 0;
    while (nc < ng - 1) {
      const int c = 1 + static_cast<int>(rng.bounded(static_cast<uint64_t>(N - 1)));
      bool dup = false;
      for (int i = 0; i < nc; ++i) dup |= cuts[i] == c;
      if (!dup) cuts[nc++] = c;
    }
    for (int i = 1; i < nc; ++i) {
      const int v = cuts[i];
      int j = i - 1;
      while (j >= 0 && cuts[j] > v) {
        cuts[j + 1] = cuts[j];
        --j;
      }
      cuts[j + 1] = v;
    }
    int counts[kMaxTasks];
    int prev = 0;
    for (int i = 0; i < nc; ++i) {
      counts[i] = cuts[i] - prev;
      prev = cuts[i];
    }
    counts[nc] = N - prev;
    // layouts, per group then per task in the group
    RecHeader h;
    h.n_tasks = T | kRecCompact;
    for (int g = 0; g < ng; ++g) {
      for (int s = 0; s < T; ++s) {
        if (grp[s] != g) continue;
        const int o = tb.opt_off[s * (tb.n_dev + 1) + counts[g]];
        const int no = tb.opt_off[s * (tb.n_dev + 1) + counts[g] + 1] - o;
        const int pick = static_cast<int>(rng.bounded(static_cast<uint64_t>(no)));
        h.dp[s] = tb.opt[3 * (o + pick)];
        h.pp[s] = tb.opt[3 * (o + pick) + 1];
        h.tp[s] = tb.opt[3 * (o + pick) + 2];
      }
    }
    for (int s = T; s < kMaxTasks; ++s) h.dp[s] = h.pp[s] = h.tp[s] = 0;
    RecOffsets ro;
    rec_offsets(h, ro);
    h.bytes = ro.bytes;
    uint8_t* rec = recs + idx * stride;
    int32_t* hw = reinterpret_cast<int32_t*>(rec);
    const int32_t* hs = reinterpret_cast<const int32_t*>(&h);
#pragma unroll
    for (int i = 0; i < 20; ++i) hw[i] = hs[i];
    // device permutation, then one shuffle per task over its group's devices
    uint8_t perm[kMaxDevices];
    for (int i = 0; i < N; ++i) perm[i] = static_cast<uint8_t>(i);
    rng.shuffle(perm, N);
    uint8_t* dv = rec + ro.dev_byte;
    int cursor = 0;
    for (int g = 0; g < ng; ++g) {
      for (int s = 0; s < T; ++s) {
        if (grp[s] != g) continue;
        uint8_t* a = dv + ro.dev[s];
        for (int i = 0; i < counts[g]; ++i) a[i] = perm[cursor + i];
        rng.shuffle(a, counts[g]);
      }
      cursor += counts[g];
    }
    // canonical bytes/plan: tg id + k counts +
    // sum_t (3 + pp_t + slots_t) + 9 result bytes
    my_bytes = 1 + ng + 9;
    for (int s = 0; s < T; ++s) my_bytes += 3 + h.pp[s] + ro.dev[s + 1] - ro.dev[s];
    if (keys) {
      // most significant first: the training tasks (DP rings: the largest and
      // most variable share of a plan; 16 half-octave classes each), the
      // generation -> actor-training bridge (na * nb edge costs; 8 classes),
      // the generation task (8 classes), the inference tasks (4 classes each)
      uint32_t key = 0;
      for (int s = 0; s < T; ++s)
        if ((tb.train_mask >> s) & 1)
          key = (key << 4) | work_class(work_estimate(h.dp[s], h.pp[s], h.tp[s], true), 2, 16);
      if (tb.gen_slot >= 0 && tb.train6_slot >= 0) {
        const int g = tb.gen_slot, a = tb.train6_slot;
        const uint32_t na = static_cast<uint32_t>(h.dp[g] * h.pp[g] * h.tp[g]);
        const uint32_t nb = static_cast<uint32_t>(h.dp[a] * h.pp[a] * h.tp[a]);
        key = (key << 3) | work_class((na * nb + 31) >> 5, 1, 8);
      }
      for (int s = 0; s < T; ++s) {
        if ((tb.train_mask >> s) & 1) continue;
        const bool gen = s == tb.gen_slot;
        key = (key << (gen ? 3 : 2)) |
              work_class(work_estimate(h.dp[s], h.pp[s], h.tp[s], false), 1, gen ? 8 : 4);
      }
      key &= (1u << kSweepKeyBits) - 1u;
      keys[idx] = key;
      atomicAdd(&hist[key], 1u);
    }
  }
  for (int o = 16; o > 0; o >>= 1) my_bytes += __shfl_xor_sync(0xffffffffu, my_bytes, o);
  if ((threadIdx.x & 31) == 0 && my_bytes) atomicAdd(bytes_acc, static_cast<unsigned long long>(my_bytes));
}

// exclusive scan of the key histogram in place (one CTA of 1024 threads)
__global__ void __launch_bounds__(1024) order_scan_kernel(uint32_t* __restrict__ hist, int bins) {
  __shared__ uint32_t warp_tot[32];
  const int per = bins / blockDim.x;
  uint32_t* h = hist + threadIdx.x * per;
  uint32_t sum = 0;
  for (int i = 0; i < per; ++i) sum += h[i];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = warp_tot[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  uint32_t run = x - sum + (w > 0 ? warp_tot[w - 1] : 0u);
  for (int i = 0; i < per; ++i) {
    const uint32_t c = h[i];
    h[i] = run;
    run += c;
  }
}

__global__ void order_scatter_kernel(const uint32_t* __restrict__ keys, uint32_t* __restrict__ off,
                                     uint32_t* __restrict__ order, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) order[atomicAdd(&off[keys[i]], 1u)] = static_cast<uint32_t>(i);
}

}  // namespace dev

cudaError_t launch_order(const SweepOrder& ord, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  dev::order_scan_kernel<<<1, 1024, 0, st>>>(ord.hist, 1 << kSweepKeyBits);
  const int threads = 256;
  dev::order_scatter_kernel<<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, st>>>(
      ord.keys, ord.hist, ord.order, n);
  return cudaGetLastError();
}

cudaError_t launch_gen(const SweepTablesDev& tb, uint64_t seed, uint64_t k0, int64_t n,
                       uint8_t* d_recs, int64_t stride, unsigned long long* d_bytes,
                       const SweepOrder* ord, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (ord) {
    const cudaError_t e = cudaMemsetAsync(ord->hist, 0, sizeof(uint32_t) << kSweepKeyBits, st);
    if (e != cudaSuccess) return e;
  }
  const int threads = 128;
  const int64_t blocks = (n + threads - 1) / threads;
  dev::gen_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(tb, seed, k0, n, d_recs,
                                                                     stride, d_bytes,
                                                                     ord ? ord->keys : nullptr,
                                                                     ord ? ord->hist : nullptr);
  return cudaGetLastError();
}

}  // namespace hpg
