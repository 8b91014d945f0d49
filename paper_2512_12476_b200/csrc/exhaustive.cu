// Device kernels of exhaustive_search (see exhaustive.hpp). One thread per
// raw candidate; the candidates of a block are tiny (<= 20 devices), so the
// work is the index decode, a key of a few dozen bytes and one hash probe.
#include <cuda_runtime.h>

#include "exhaustive.hpp"

namespace hpg {
namespace dev {

// canonical key (search.cpp:950-977): option index per position, then per
// position and device the code class << 8 | first-appearance rank in class
__device__ void exh_key(const ExhBlock& B, uint64_t idx, uint8_t* key) {
  int oi[kMaxTasks];
  uint8_t devs[kMaxTasks * kExhMaxDevices];
  exh_decode(B, idx, oi, devs);
  uint16_t code[kExhMaxDevices];
  uint8_t seen_cnt[kExhMaxDevices];
  for (int i = 0; i < B.n; ++i) {
    code[i] = 0xffff;
    seen_cnt[i] = 0;
  }
  int w = 0;
  for (int t = 0; t < B.T; ++t) key[w++] = static_cast<uint8_t>(oi[t]);
  for (int t = 0; t < B.T; ++t) {
    const int m = B.comp[B.grp[t]];
    for (int i = 0; i < m; ++i) {
      const int d = devs[t * B.n + i];
      if (code[d] == 0xffff) {
        const int c = B.cls[d];
        code[d] = static_cast<uint16_t>((c << 8) | seen_cnt[c]++);
      }
      key[w++] = static_cast<uint8_t>(code[d] & 0xff);
      key[w++] = static_cast<uint8_t>(code[d] >> 8);
    }
  }
  while (w < B.key_bytes) key[w++] = 0;
}

__global__ void exh_key_kernel(ExhBlock B, uint64_t n, uint8_t* __restrict__ keys) {
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  exh_key(B, idx, keys + idx * B.key_bytes);
}

__device__ __forceinline__ uint64_t exh_hash(const uint64_t* k, int words) {
  uint64_t h = 0x9e3779b97f4a7c15ull;
  for (int i = 0; i < words; ++i) {
    uint64_t x = k[i] + h;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    h = x ^ (x >> 31);
  }
  return h;
}

__device__ __forceinline__ bool exh_key_eq(const uint64_t* a, const uint64_t* b, int words) {
  for (int i = 0; i < words; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// slot value = smallest raw index with this exact key. A slot is claimed with
// a CAS of the inserter's index (keys were all written by the previous
// kernel), and only lowered with atomicMin by indices of the same key.
__global__ void exh_insert_kernel(ExhBlock B, uint64_t n, const uint8_t* __restrict__ keys,
                                  unsigned long long* __restrict__ table, uint64_t mask,
                                  unsigned long long* __restrict__ slot) {
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int words = B.key_bytes / 8;
  const uint64_t* mine = reinterpret_cast<const uint64_t*>(keys + idx * B.key_bytes);
  uint64_t h = exh_hash(mine, words) & mask;
  while (true) {
    unsigned long long cur = table[h];
    if (cur == ~0ull) {
      cur = atomicCAS(&table[h], ~0ull, static_cast<unsigned long long>(idx));
      if (cur == ~0ull) {
        slot[idx] = h;
        return;
      }
    }
    const uint64_t* other = reinterpret_cast<const uint64_t*>(keys + cur * B.key_bytes);
    if (exh_key_eq(mine, other, words)) {
      atomicMin(&table[h], static_cast<unsigned long long>(idx));
      slot[idx] = h;
      return;
    }
    h = (h + 1) & mask;
  }
}

// first occurrences -> compact plan records (unit weights, make_layout split)
// in their own slot; every other slot is marked skip
__global__ void exh_rep_kernel(ExhBlock B, uint64_t n, const unsigned long long* __restrict__ table,
                               const unsigned long long* __restrict__ slot,
                               uint8_t* __restrict__ recs, int32_t* __restrict__ modes,
                               unsigned long long* __restrict__ count) {
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool rep = idx < n && table[slot[idx]] == idx;
  const unsigned ballot = __ballot_sync(0xffffffffu, rep);
  if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(count, static_cast<unsigned long long>(__popc(ballot)));
  if (idx >= n) return;
  modes[idx] = rep ? kModeE2E : kModeSkip;
  if (!rep) return;
  const uint64_t pos = idx;
  int oi[kMaxTasks];
  uint8_t devs[kMaxTasks * kExhMaxDevices];
  exh_decode(B, idx, oi, devs);
  RecHeader h;
  h.n_tasks = B.T | kRecCompact;
  for (int s = 0; s < kMaxTasks; ++s) h.dp[s] = h.pp[s] = h.tp[s] = 0;
  for (int t = 0; t < B.T; ++t) {
    const int s = B.order[t];
    h.dp[s] = B.opt[t][oi[t]][0];
    h.pp[s] = B.opt[t][oi[t]][1];
    h.tp[s] = B.opt[t][oi[t]][2];
  }
  RecOffsets ro;
  rec_offsets(h, ro);
  h.bytes = ro.bytes;
  uint8_t* rec = recs + pos * static_cast<unsigned long long>(B.rec_stride);
  int32_t* hw = reinterpret_cast<int32_t*>(rec);
  const int32_t* hs = reinterpret_cast<const int32_t*>(&h);
#pragma unroll
  for (int i = 0; i < 20; ++i) hw[i] = hs[i];
  uint8_t* dv = rec + ro.dev_byte;
  for (int t = 0; t < B.T; ++t) {
    const int s = B.order[t];
    const int m = B.comp[B.grp[t]];
    for (int i = 0; i < m; ++i) dv[ro.dev[s] + i] = devs[t * B.n + i];
  }
}

// argmin over memory-feasible representatives by (cost, raw index)
__global__ void exh_reduce_kernel(const EvalResult* __restrict__ res, int64_t n,
                                  ExhPartial* __restrict__ out) {
  double best = kInf;
  unsigned long long bi = ~0ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const EvalResult r = res[i];
    if (!(r.flags & kResFeasIn)) continue;
    const unsigned long long k = static_cast<unsigned long long>(i);
    if (r.cost < best || (r.cost == best && k < bi)) {
      best = r.cost;
      bi = k;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob < best || (ob == best && ok < bi)) {
      best = ob;
      bi = ok;
    }
  }
  __shared__ ExhPartial part[32];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) part[warp] = ExhPartial{best, bi};
  __syncthreads();
  if (threadIdx.x == 0) {
    ExhPartial b = part[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      const ExhPartial& p = part[w];
      if (p.best < b.best || (p.best == b.best && p.best_idx < b.best_idx)) b = p;
    }
    out[blockIdx.x] = b;
  }
}

}  // namespace dev

namespace {
unsigned blocks_for(uint64_t n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}
}  // namespace

cudaError_t launch_exh_keys(const ExhBlock& B, uint64_t n, uint8_t* d_keys, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  dev::exh_key_kernel<<<blocks_for(n, 128), 128, 0, st>>>(B, n, d_keys);
  return cudaGetLastError();
}

cudaError_t launch_exh_insert(const ExhBlock& B, uint64_t n, const uint8_t* d_keys,
                              unsigned long long* d_table, uint64_t mask,
                              unsigned long long* d_slot, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  dev::exh_insert_kernel<<<blocks_for(n, 256), 256, 0, st>>>(B, n, d_keys, d_table, mask, d_slot);
  return cudaGetLastError();
}

cudaError_t launch_exh_reps(const ExhBlock& B, uint64_t n, const unsigned long long* d_table,
                            const unsigned long long* d_slot, uint8_t* d_recs, int32_t* d_modes,
                            unsigned long long* d_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  dev::exh_rep_kernel<<<blocks_for(n, 128), 128, 0, st>>>(B, n, d_table, d_slot, d_recs, d_modes,
                                                          d_count);
  return cudaGetLastError();
}

cudaError_t launch_exh_reduce(const EvalResult* d_res, int64_t n, ExhPartial* d_out, int blocks,
                              cudaStream_t st) {
  dev::exh_reduce_kernel<<<blocks, 256, 0, st>>>(d_res, n, d_out);
  return cudaGetLastError();
}

}  // namespace hpg
