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

__global__ void gen_kernel(SweepTablesDev tb, uint64_t seed, uint64_t k0, int64_t n,
                           uint8_t* __restrict__ recs, int64_t stride,
                           unsigned long long* __restrict__ bytes_acc) {
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
  }
  for (int o = 16; o > 0; o >>= 1) my_bytes += __shfl_xor_sync(0xffffffffu, my_bytes, o);
  if ((threadIdx.x & 31) == 0 && my_bytes) atomicAdd(bytes_acc, static_cast<unsigned long long>(my_bytes));
}

}  // namespace dev

cudaError_t launch_gen(const SweepTablesDev& tb, uint64_t seed, uint64_t k0, int64_t n,
                       uint8_t* d_recs, int64_t stride, unsigned long long* d_bytes,
                       cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int threads = 128;
  const int64_t blocks = (n + threads - 1) / threads;
  dev::gen_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(tb, seed, k0, n, d_recs,
                                                                     stride, d_bytes);
  return cudaGetLastError();
}

}  // namespace hpg
