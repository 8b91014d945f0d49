// GA initial candidates on the device (first step of SURVEY.md §8 F1):
// make_candidate's device assignment (random_medium_assignment +
// random_fine_assignment, search.cpp:152-234, 318-334) with the reference's
// RNG stream replayed bit for bit (rng.hpp:10-65).
//
// A run's candidates come from one sequential stream, but every candidate
// draws the same number of values (gen_draws_per_candidate), so the host
// steps the stream to each candidate's start state and one thread per
// candidate replays its draws. Record headers, weights and stage splits come
// from the host (they depend on the layout combination only); the kernel
// writes the device slots into the packed record and a compact copy.
#include <cuda_runtime.h>

#include "devstate.hpp"

#include "gen_ga.hpp"
#include "rng.hpp"

namespace hpg {
namespace dev {

// next() % n, exactly, through a 128-bit reciprocal (Lemire, Kaser & Kurz
// 2019; the host uses the same identity, rng.hpp fastmod_u64)
__device__ __forceinline__ uint64_t bounded_fast(Rng& rng, uint64_t n, const GenTablesDev& tb) {
  const uint64_t a = rng.next();
  if (n > static_cast<uint64_t>(kGenFastModMax)) return a % n;
  const uint64_t mlo = tb.fastmod[2 * n], mhi = tb.fastmod[2 * n + 1];
  // low = (M * a) mod 2^128
  const uint64_t low_lo = mlo * a;
  const uint64_t low_hi = __umul64hi(mlo, a) + mhi * a;
  // ((low_lo * n) >> 64) + low_hi * n, then >> 64
  const uint64_t bottom = __umul64hi(low_lo, n);
  const uint64_t top_lo = low_hi * n;
  const uint64_t top_hi = __umul64hi(low_hi, n);
  const uint64_t sum_lo = top_lo + bottom;
  return top_hi + (sum_lo < top_lo ? 1 : 0);
}

template <typename T>
__device__ __forceinline__ void shuffle_fast(Rng& rng, T* v, int n, const GenTablesDev& tb) {
  for (int i = n; i > 1; --i) {
    const int j = static_cast<int>(bounded_fast(rng, static_cast<uint64_t>(i), tb));
    const T tmp = v[i - 1];
    v[i - 1] = v[j];
    v[j] = tmp;
  }
}

__global__ void gen_ga_kernel(GenTablesDev tb, const GenItem* __restrict__ items,
                              const int32_t* __restrict__ cand_item, const Rng* __restrict__ starts,
                              int n_cands, uint8_t* __restrict__ recs,
                              const int64_t* __restrict__ off,
                              const int64_t* __restrict__ dev_out_off,
                              uint8_t* __restrict__ dev_out) {
  const int jdx = blockIdx.x * blockDim.x + threadIdx.x;
  if (jdx >= n_cands) return;
  const GenItem& g = items[cand_item[jdx]];
  const int idx = g.first + (jdx - g.first_out);
  Rng rng = starts[jdx];
  // per-thread scratch in shared memory, sized to the problem (gen_smem_per_thread)
  extern __shared__ __align__(16) uint8_t gsm[];
  uint8_t* my = gsm + static_cast<size_t>(threadIdx.x) * tb.smem_per_thread;
  int16_t* regions = reinterpret_cast<int16_t*>(my);
  int16_t* nodes = regions + tb.n_regions;
  int16_t* cnt = nodes + tb.max_nodes_per_region;
  int16_t* start = cnt + tb.n_nodes;
  int16_t* fill = start + tb.n_nodes;
  int16_t* ranks = fill + tb.n_nodes;
  uint8_t* flat = reinterpret_cast<uint8_t*>(ranks + tb.n_nodes);
  uint8_t* bucket = flat + tb.n_dev;
  uint8_t* rec = recs + off[idx];
  RecHeader h;
  for (int i = 0; i < 20; ++i) reinterpret_cast<int32_t*>(&h)[i] = reinterpret_cast<const int32_t*>(rec)[i];
  RecOffsets o;
  rec_offsets(h, o);
  uint8_t* dv = rec + o.dev_byte;
  // random_medium_assignment: regions shuffled, nodes shuffled per region,
  // devices in node order, then the locality-bias scramble
  for (int r = 0; r < tb.n_regions; ++r) regions[r] = static_cast<int16_t>(r);
  shuffle_fast(rng, regions, tb.n_regions, tb);
  int nf = 0;
  for (int ri = 0; ri < tb.n_regions; ++ri) {
    const int reg = regions[ri];
    const int n0 = tb.region_off[reg], nn = tb.region_off[reg + 1] - n0;
    for (int k = 0; k < nn; ++k) nodes[k] = static_cast<int16_t>(k);
    shuffle_fast(rng, nodes, nn, tb);
    for (int k = 0; k < nn; ++k) {
      const int node = n0 + nodes[k];
      for (int e = tb.node_off[node]; e < tb.node_off[node + 1]; ++e) flat[nf++] = tb.node_devs[e];
    }
  }
  for (int i = nf; i > 1; --i) {
    const bool scramble = rng.uniform() < (1.0 - g.bias);
    const uint64_t pick = bounded_fast(rng, static_cast<uint64_t>(i), tb);
    if (scramble) {
      const uint8_t tmp = flat[i - 1];
      flat[i - 1] = flat[pick];
      flat[pick] = tmp;
    }
  }
  // random_fine_assignment per task of each group, over the group's devices
  int cursor = 0, pos_order = 0;
  for (int grp = 0; grp < g.n_groups; ++grp) {
    const int n = g.counts[grp];
    const uint8_t* gd = flat + cursor;
    for (; pos_order < g.n_order && g.order_group[pos_order] == grp; ++pos_order) {
      const int s = g.order_slot[pos_order];
      for (int r = 0; r < tb.n_nodes; ++r) cnt[r] = 0;
      for (int i = 0; i < n; ++i) ++cnt[tb.node_rank[gd[i]]];
      int nr = 0, acc = 0;
      for (int r = 0; r < tb.n_nodes; ++r) {
        if (!cnt[r]) continue;
        ranks[nr++] = static_cast<int16_t>(r);
        start[r] = static_cast<int16_t>(acc);
        acc += cnt[r];
      }
      for (int k = 0; k < nr; ++k) fill[ranks[k]] = start[ranks[k]];
      for (int i = 0; i < n; ++i) bucket[fill[tb.node_rank[gd[i]]]++] = gd[i];
      shuffle_fast(rng, ranks, nr, tb);
      uint8_t* out = dv + o.dev[s];
      int pos = 0;
      for (int k = 0; k < nr; ++k) {
        uint8_t* b = bucket + start[ranks[k]];
        const int nb = cnt[ranks[k]];
        shuffle_fast(rng, b, nb, tb);
        for (int i = 0; i < nb; ++i) out[pos++] = b[i];
      }
    }
    cursor += n;
  }
  // compact copy of the slots for the host
  uint8_t* co = dev_out + dev_out_off[jdx];
  for (int i = 0; i < o.dev[h.n_tasks & 0xffff]; ++i) co[i] = dv[i];
}

}  // namespace dev

cudaError_t launch_gen_ga(const GenTablesDev& tb, const GenItem* d_items,
                          const int32_t* d_cand_item, const Rng* d_starts, int n_cands,
                          uint8_t* d_recs, const int64_t* d_off, const int64_t* d_dev_out_off,
                          uint8_t* d_dev_out, cudaStream_t st) {
  if (n_cands <= 0) return cudaSuccess;
  const int threads = 64;
  const size_t smem = static_cast<size_t>(threads) * tb.smem_per_thread;
  if (smem > 48 * 1024) {
    const cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(dev::gen_ga_kernel),
                                          static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  dev::gen_ga_kernel<<<(n_cands + threads - 1) / threads, threads, smem, st>>>(
      tb, d_items, d_cand_item, d_starts, n_cands, d_recs, d_off, d_dev_out_off, d_dev_out);
  return cudaGetLastError();
}

}  // namespace hpg
