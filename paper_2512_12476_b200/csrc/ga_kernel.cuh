// Device-resident GA offspring loop, included by eval.cu so
// that the workers share eval_one with eval_kernel.
//
// ga_run's offspring loop (reference search.cpp:471-563; the host coroutine in
// search.cpp is the same algorithm with the same speculation) runs as a state
// machine per run in global memory. A persistent grid of one-warp workers
// takes tasks from a ticketed ring: "evaluate candidate i of run r" or "step
// run r". The worker that finishes the last evaluation of a wave continues
// that run's GA step itself, which draws the next wave's candidates (record
// copies + device-slot moves with the run's RNG stream, replayed bit for bit),
// publishes all but one of them and evaluates the last one directly. No host
// round trip and no lockstep: each run waits only for its own candidates.
//
// GA control flow is computed redundantly by all 32 lanes (same loads, same
// draws); lane 0 writes, and every write other lanes read back is followed
// by __syncwarp. Everything another SM may have written in this launch is
// read with ld.global.cg.
#pragma once

#include "ga_dev.hpp"
#include "gen_ga.hpp"
#include "rng_jump.hpp"
#include "devstate.hpp"

#define GA_BOUNDED(r, n) ga_bounded(r, n)

namespace hpg {
namespace dev {

// the launch's parameters: passed by value to every launch (a __grid_constant__
// kernel argument) and copied once into this per-CTA shared copy, which every
// GA function reads. A launch carries its own parameters, so contexts on the
// same device (and threads driving them) never share mutable device state.
__shared__ GaParams c_ga;

__device__ __forceinline__ unsigned long long ga_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// next() % n, exactly: for n <= kGaModMax, (hi * 2^32 + lo) % n =
// ((hi % n) * (2^32 % n) + lo % n) % n, each 32-bit remainder by Lemire's
// direct method (M = floor((2^64 - 1) / n) + 1; x % n = mulhi(M * x, n),
// exact for every 32-bit x) from a constant-bank table: no divide, no L2
// round trip (the workers' L1 is mostly shared memory)
constexpr int kGaModMax = 1024;
struct GaModTables {
  uint64_t m[kGaModMax + 1];    // M per divisor
  uint32_t p32[kGaModMax + 1];  // 2^32 mod n
};
constexpr GaModTables ga_mod_tables() {
  GaModTables t{};
  for (int d = 1; d <= kGaModMax; ++d) {
    t.m[d] = ~uint64_t(0) / static_cast<uint64_t>(d) + 1;
    t.p32[d] = static_cast<uint32_t>((uint64_t(1) << 32) % static_cast<uint64_t>(d));
  }
  return t;
}
// initialised at compile time: part of the module image on every device
__constant__ GaModTables c_mod = ga_mod_tables();

__device__ __forceinline__ uint32_t ga_mod32(uint32_t x, uint32_t n, uint64_t m) {
  return static_cast<uint32_t>(__umul64hi(m * x, n));
}

__device__ __forceinline__ uint64_t ga_bounded(Rng& rng, uint64_t n) {
  const uint64_t a = rng.next();
  if (n > static_cast<uint64_t>(kGaModMax)) return a % n;
  const uint32_t d = static_cast<uint32_t>(n);
  const uint64_t m = c_mod.m[d];
  const uint32_t hi = static_cast<uint32_t>(a >> 32), lo = static_cast<uint32_t>(a);
  return ga_mod32(ga_mod32(hi, d, m) * c_mod.p32[d] + ga_mod32(lo, d, m), d, m);
}

__device__ __forceinline__ Rng ga_ld_rng(const Rng* p) {
  Rng r;
  r.seed = __ldcg(&p->seed);
  for (int i = 0; i < 4; ++i) r.s[i] = __ldcg(&p->s[i]);
  return r;
}

__device__ __forceinline__ void ga_st_rng(Rng* p, const Rng& r) {
  if ((threadIdx.x & 31) == 0) *p = r;
}

__device__ __forceinline__ bool ga_same_rng(const Rng& a, const Rng& b) {
  return a.seed == b.seed && a.s[0] == b.s[0] && a.s[1] == b.s[1] && a.s[2] == b.s[2] &&
         a.s[3] == b.s[3];
}

// Per-warp shared-memory scratch of a GA step: the child and a parent record,
// the trial being built, the finished wave's results and the population, so
// that drawing a wave costs a handful of L2 round trips, not one per move.
struct GaSm {
  // problem tables staged once per worker (dependent lookups in the draws)
  const uint8_t* id_rank;     // [N] device -> id rank
  const uint8_t* by_id_rank;  // [N] id rank -> device
  const uint8_t* node_rank;   // [N] device -> node rank
  const uint8_t* node_devs;   // [N] devices in region / node order
  const int16_t* region_off;  // [regions + 1]
  const int16_t* node_off;    // [nodes + 1]
  uint8_t* gen;  // init generation scratch (aliases the evaluation carve)
  uint32_t* gw;  // rank set per task group of the current source [kMaxTasks][8]
  uint8_t* child;
  uint8_t* par;
  uint8_t* tmp;
  EvalResult* res;
  int32_t* pslot;
  double* pcost;
  uint64_t* pseq;
  struct GaInitJob* ijob;  // team job slot for init chunks (teams only)
  int n_warps;             // warps per worker
};

__host__ __device__ inline int ga_tables_bytes(int n_dev, int n_regions, int n_nodes) {
  return (4 * n_dev + 2 * (n_regions + 1) + 2 * (n_nodes + 1) + 15) & ~15;
}

__host__ __device__ inline int ga_smem_bytes(int stride, int max_wave, int n_dev, int n_regions,
                                             int n_nodes) {
  return 3 * stride + 32 * max_wave + kGaMaxPop * (4 + 8 + 8) + 32 * kMaxTasks +
         ga_tables_bytes(n_dev, n_regions, n_nodes);
}

struct GaView {
  GaRun* R;
  int run;
  uint8_t* pool;
  int stride;
  int ng;
  int gstart[kMaxTasks + 1];
  int gslot[kMaxTasks];
  int counts[kMaxTasks];
  int opt_off[kMaxTasks + 1];
  int64_t opt_base;
  GaSm sm;
  __device__ uint8_t* slot(int k) const {
    HPG_DCHECK(k >= 0 && k < 2 + c_ga.pop_cap + c_ga.res_per_run);
    return pool + static_cast<int64_t>(k) * stride;
  }
  __device__ uint8_t* wave_slot(int buf, int i) const {
    HPG_DCHECK(buf >= 0 && buf <= 1 && i >= 0 && buf * c_ga.max_wave + i < c_ga.res_per_run);
    return slot(2 + c_ga.pop_cap + buf * c_ga.max_wave + i);
  }
};

// an init chunk posted to the team's helper warps (kJobGaInit)
constexpr int kJobGaInit = 16;
struct GaInitJob {
  GaView v;
  Rng rng;
  int64_t combo0;
  int n, kind;
};

// global record -> shared (one round trip: the whole slot)
__device__ __forceinline__ void ga_ld_rec(uint8_t* dst, const uint8_t* src, int stride) {
  const int lane = threadIdx.x & 31;
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = lane; i < (stride >> 4); i += 32) d[i] = __ldcg(s + i);
  __syncwarp();
}

// shared record -> global (the record's own bytes)
__device__ __forceinline__ void ga_st_rec(uint8_t* dst, const uint8_t* src) {
  const int lane = threadIdx.x & 31;
  const int n16 = (*reinterpret_cast<const int32_t*>(src) + 15) >> 4;
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = lane; i < n16; i += 32) d[i] = s[i];
  __syncwarp();
}

__device__ __forceinline__ void ga_sm_copy(uint8_t* dst, const uint8_t* src) {
  const int lane = threadIdx.x & 31;
  const int n16 = (*reinterpret_cast<const int32_t*>(src) + 15) >> 4;
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = lane; i < n16; i += 32) d[i] = s[i];
  __syncwarp();
}

// global record -> global (improvement / best-member copies)
__device__ __forceinline__ void ga_rec_copy(uint8_t* dst, const uint8_t* src) {
  const int lane = threadIdx.x & 31;
  const int bytes = __ldcg(reinterpret_cast<const int32_t*>(src));
  const int n16 = (bytes + 15) >> 4;
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = lane; i < n16; i += 32) d[i] = __ldcg(s + i);
  __syncwarp();
}

// device-slot geometry of a (shared-memory) record
struct GaGeo {
  int dev_byte;
  int off[kMaxTasks + 1];
};

__device__ __forceinline__ void ga_geo(const uint8_t* rec, int T, GaGeo& g) {
  const RecHeader& h = *reinterpret_cast<const RecHeader*>(rec);
  int sw = 0, ssl = 0;
  g.off[0] = 0;
  for (int t = 0; t < T; ++t) {
    sw += h.dp[t];
    ssl += h.pp[t];
    g.off[t + 1] = g.off[t] + h.dp[t] * h.pp[t] * h.tp[t];
  }
  g.dev_byte = static_cast<int>(sizeof(RecHeader)) + 8 * sw + 4 * ssl;
}

// group_device_set as a bitmask over id ranks (search.cpp:336-341)
__device__ __forceinline__ void ga_rank_set(const uint8_t* id_rank, const uint8_t* d, int n,
                                            uint32_t (&w)[8]) {
  const int lane = threadIdx.x & 31;
  uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = lane; i < n; i += 32) {
    const int r = id_rank[d[i]];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if ((r >> 5) == k) m[k] |= 1u << (r & 31);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = __reduce_or_sync(0xffffffffu, m[k]);
}

__device__ __forceinline__ int ga_select_rank(const uint8_t* by_id_rank, const uint32_t (&w)[8],
                                              uint64_t idx) {
  for (int k = 0; k < 8; ++k) {
    const uint64_t pc = static_cast<uint64_t>(__popc(w[k]));
    if (idx >= pc) {
      idx -= pc;
      continue;
    }
    uint32_t x = w[k];
    for (uint64_t i = 0; i < idx; ++i) x &= x - 1;
    return by_id_rank[32 * k + __ffs(x) - 1];
  }
  return -1;
}

// first index i < n with d[i] == v (lane-parallel), or -1
__device__ __forceinline__ int ga_find(const uint8_t* d, int n, int v) {
  const int lane = threadIdx.x & 31;
  for (int b = 0; b < n; b += 32) {
    const int i = b + lane;
    const bool hit = i < n && d[i] == v;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (m) return b + __ffs(m) - 1;
  }
  return -1;
}

// ---- trials drawn lane-parallel ----
// Every trial of a wave starts from the same source record (the child, or the
// parent of a mutation stage) and a move consumes a fixed number of draws
// (level 3: four, level 5: three; a mutation one more for its level), so
// each lane steps the stream to its trial's start, computes the trial's
// device-slot patches against the source, and the warp writes the records.
struct GaSrcInfo {
  GaGeo geo;
  int ne;
  int elig[kMaxTasks];
};

constexpr int kGaMaxPatch = 2 * kMaxTasks;
constexpr int kGaPendBias = 1 << 20;  // pending per share of a wave still being drawn
// ring task kinds (payload index): >= 0 evaluate candidate i; step; draws
constexpr int kGaTaskStep = -1, kGaTaskDraw3 = -15, kGaTaskDraw5 = -14, kGaTaskSpec = -13;

// per-source tables: geometry, eligible tasks, rank set of every group
__device__ void ga_src_info(const GaView& v, const uint8_t* src, GaSrcInfo& si) {
  ga_geo(src, c_ga.n_tasks, si.geo);
  si.ne = 0;
  for (int s = 0; s < c_ga.n_tasks; ++s)
    if (si.geo.off[s + 1] - si.geo.off[s] >= 2) si.elig[si.ne++] = s;
  const uint8_t* dv = src + si.geo.dev_byte;
  for (int g = 0; g < v.ng; ++g) {
    const int s = v.gslot[v.gstart[g]];
    uint32_t w[8];
    ga_rank_set(v.sm.id_rank, dv + si.geo.off[s], si.geo.off[s + 1] - si.geo.off[s], w);
    if ((threadIdx.x & 31) == 0)
      for (int k = 0; k < 8; ++k) v.sm.gw[g * 8 + k] = w[k];
  }
  __syncwarp();
}

// one move of this lane against the source: patches (absolute device-slot
// index, new byte); the draws of random_move (search.cpp:360-421)
__device__ __forceinline__ int ga_lane_move(const GaView& v, const uint8_t* src,
                                            const GaSrcInfo& si, int level, Rng& rng,
                                            int (&pp)[kGaMaxPatch], int (&pv)[kGaMaxPatch]) {
  const uint8_t* dv = src + si.geo.dev_byte;
  int np = 0;
  if (level == 3) {
    const int ng = v.ng;
    const int g1 = static_cast<int>(GA_BOUNDED(rng, static_cast<uint64_t>(ng)));
    int g2 = static_cast<int>(GA_BOUNDED(rng, static_cast<uint64_t>(ng - 1)));
    if (g2 >= g1) ++g2;
    const int s1 = v.gslot[v.gstart[g1]], s2 = v.gslot[v.gstart[g2]];
    const int n1 = si.geo.off[s1 + 1] - si.geo.off[s1], n2 = si.geo.off[s2 + 1] - si.geo.off[s2];
    uint32_t w1[8], w2[8];
    for (int k = 0; k < 8; ++k) {
      w1[k] = v.sm.gw[g1 * 8 + k];
      w2[k] = v.sm.gw[g2 * 8 + k];
    }
    const int b = ga_select_rank(v.sm.by_id_rank, w2, GA_BOUNDED(rng, static_cast<uint64_t>(n2)));
    const int a = ga_select_rank(v.sm.by_id_rank, w1, GA_BOUNDED(rng, static_cast<uint64_t>(n1)));
    for (int side = 0; side < 2; ++side) {
      const int g = side ? g2 : g1, from = side ? b : a, to = side ? a : b;
      for (int k = v.gstart[g]; k < v.gstart[g + 1]; ++k) {
        const int s = v.gslot[k];
        const int o = si.geo.off[s], n = si.geo.off[s + 1] - o;
        for (int i = 0; i < n; ++i)
          if (dv[o + i] == from) {
            pp[np] = o + i;
            pv[np++] = to;
            break;
          }
      }
    }
    return np;
  }
  const int s = si.elig[GA_BOUNDED(rng, static_cast<uint64_t>(si.ne))];
  const int o = si.geo.off[s];
  const uint64_t n = static_cast<uint64_t>(si.geo.off[s + 1] - o);
  const uint64_t p1 = GA_BOUNDED(rng, n);
  uint64_t p2 = GA_BOUNDED(rng, n - 1);
  if (p2 >= p1) ++p2;
  pp[0] = o + static_cast<int>(p1);
  pv[0] = dv[o + p2];
  pp[1] = o + static_cast<int>(p2);
  pv[1] = dv[o + p1];
  return 2;
}

// writes trials [0, n) = the source with lane t's patches, to buffer buf
// from index at: all record chunks of all trials in one pass, then the patches
__device__ __forceinline__ void ga_emit_all(const GaView& v, int buf, int at, int n,
                                            const uint8_t* src, int dev_byte, int np,
                                            const int (&pp)[kGaMaxPatch],
                                            const int (&pv)[kGaMaxPatch]) {
  const int lane = threadIdx.x & 31;
  const int n16 = (*reinterpret_cast<const int32_t*>(src) + 15) >> 4;
  const int4* s = reinterpret_cast<const int4*>(src);
  uint8_t* d0 = v.wave_slot(buf, at);
  for (int k = lane; k < n * n16; k += 32) {
    const int t = k / n16, c = k - t * n16;
    reinterpret_cast<int4*>(d0 + static_cast<int64_t>(t) * v.stride)[c] = s[c];
  }
  __syncwarp();
  if (lane < n) {
    uint8_t* d = d0 + static_cast<int64_t>(lane) * v.stride + dev_byte;
    for (int q = 0; q < np; ++q) d[pp[q]] = static_cast<uint8_t>(pv[q]);
  }
  __syncwarp();
}

// draw_mut: up to kGaTrials mutated copies of the (shared) parent, then the
// parent itself, stored to stage buffer buf from index base
__device__ void ga_draw_mut(const GaView& v, Rng r, const uint8_t* parent, GaStage* st, int buf,
                            int base) {
  const int lane = threadIdx.x & 31;
  GaSrcInfo si;
  ga_src_info(v, parent, si);
  const bool has_l3 = v.ng >= 2, has_l5 = si.ne > 0;
  int ntr = 0;
  Rng mine = r;
  int np = 0, pp[kGaMaxPatch], pv[kGaMaxPatch];
  if (has_l3 || has_l5) {
    // stream positions: every trial is one mutate (level draw + move draws)
    ntr = kGaTrials;
    Rng q = r;
    for (int t = 0; t < kGaTrials; ++t) {
      if (lane == t) mine = q;
      int level;
      if (has_l3 && has_l5) {
        level = GA_BOUNDED(q, 2) == 0 ? 3 : 5;
      } else {
        level = has_l3 ? 3 : 5;
      }
      for (int k = 0; k < (level == 3 ? 4 : 3); ++k) q.next();
    }
    r = q;
    if (lane < kGaTrials) {
      int level;
      if (has_l3 && has_l5) {
        level = GA_BOUNDED(mine, 2) == 0 ? 3 : 5;
      } else {
        level = has_l3 ? 3 : 5;
      }
      np = ga_lane_move(v, parent, si, level, mine, pp, pv);
      st->snaps[lane] = mine;  // the stream after this trial
    }
    __syncwarp();
    ga_emit_all(v, buf, base, ntr, parent, si.geo.dev_byte, np, pp, pv);
  }
  ga_st_rng(&st->after_all, r);
  ga_st_rec(v.wave_slot(buf, base + ntr), parent);
  if (lane == 0) {
    st->buf = buf;
    st->base = base;
    st->ntr = ntr;
  }
  __syncwarp();
}


// ---- init phase: make_candidate on the device (search.cpp:152-234, 283-334) ----

// record layout of combination `combo` (decode_layout_combo): header, unit
// weights, uniform stage split (init_cand, make_layout plan.cpp:89-100)
__device__ void ga_lane_layouts(const GaView& v, int64_t combo, uint8_t* rec, RecOffsets& o) {
    RecHeader h;
  h.bytes = 0;
  h.n_tasks = c_ga.n_tasks;
  for (int t = 0; t < kMaxTasks; ++t) h.dp[t] = h.pp[t] = h.tp[t] = 0;
  for (int k = 0; k < c_ga.n_tasks; ++k) {
    const int s = v.gslot[k];
    const int n_opt = v.opt_off[k + 1] - v.opt_off[k];
    const short4 l = __ldg(c_ga.opts + v.opt_base + v.opt_off[k] + static_cast<int>(combo % n_opt));
    combo /= n_opt;
    h.dp[s] = l.x;
    h.pp[s] = l.y;
    h.tp[s] = l.z;
  }
  rec_offsets(h, o);
  h.bytes = o.bytes;
  int32_t* hw = reinterpret_cast<int32_t*>(rec);
  const int32_t* hs = reinterpret_cast<const int32_t*>(&h);
  for (int i = 0; i < 20; ++i) hw[i] = hs[i];
  double* w = reinterpret_cast<double*>(rec + o.w_byte);
  for (int i = 0; i < o.w[c_ga.n_tasks]; ++i) w[i] = 1.0;
  int32_t* sl = reinterpret_cast<int32_t*>(rec + o.sl_byte);
  for (int t = 0; t < c_ga.n_tasks; ++t) {
    const int64_t nl = c_ga.task_nl[t];
    const int pp = h.pp[t];
    for (int j = 0; j < pp; ++j)
      sl[o.sl[t] + j] = static_cast<int32_t>(nl / pp) + (j < nl % pp ? 1 : 0);
  }
  for (int i = o.dev_byte + o.dev[c_ga.n_tasks]; i < o.bytes; ++i) rec[i] = 0;  // padding
}

// per-lane generation scratch, interleaved across the warp's lanes (element
// i of a lane's array at [i][lane]): in shared memory (aliasing the idle
// evaluation carve) or, for large problems, in the worker's global scratch
struct GaGenScratch {
  int16_t* s16;  // int16 arrays: regions | nodes | cnt | start | fill | ranks
  uint8_t* s8;   // uint8 arrays: flat | bucket
  int lane;
  __device__ int16_t& a16(int i) const { return s16[i * 32 + lane]; }
  __device__ uint8_t& a8(int i) const { return s8[i * 32 + lane]; }
};

// one candidate by this lane: layouts, random_medium_assignment and
// random_fine_assignment per task of each group (the reference's draws)
__device__ void ga_lane_make(const GaView& v, int64_t combo, Rng& rng_io, uint8_t* rec,
                             const GaGenScratch& sc) {
  // everything the loops touch in registers / restrict pointers: the byte
  // stores below would otherwise force reloads of the stream state and of
  // every pointer (char stores alias everything)
  Rng rng = rng_io;
  const int lane = sc.lane;
  int16_t* __restrict__ s16 = sc.s16;
  uint8_t* __restrict__ s8 = sc.s8;
  const uint8_t* __restrict__ node_rank = v.sm.node_rank;
  const uint8_t* __restrict__ node_devs = v.sm.node_devs;
  const int16_t* __restrict__ region_off = v.sm.region_off;
  const int16_t* __restrict__ node_off = v.sm.node_off;
  const int n_regions = c_ga.n_regions, n_nodes = c_ga.n_nodes;
  const double keep = 1.0 - c_ga.bias;
#define A16(i) s16[(i) * 32 + lane]
#define A8(i) s8[(i) * 32 + lane]
  RecOffsets o;
  const long long p0 = c_ga.prof ? clock64() : 0;
  ga_lane_layouts(v, combo, rec, o);
  const long long p1 = c_ga.prof ? clock64() : 0;
  const int o_nodes = n_regions, o_cnt = o_nodes + c_ga.max_nodes_per_region,
            o_start = o_cnt + n_nodes, o_fill = o_start + n_nodes, o_ranks = o_fill + n_nodes;
  const int o_bucket = c_ga.n_dev;
  for (int r = 0; r < n_regions; ++r) A16(r) = static_cast<int16_t>(r);
  for (int i = n_regions; i > 1; --i) {
    const int j = static_cast<int>(ga_bounded(rng, static_cast<uint64_t>(i)));
    const int16_t t = A16(i - 1);
    A16(i - 1) = A16(j);
    A16(j) = t;
  }
  int nf = 0;
  for (int ri = 0; ri < n_regions; ++ri) {
    const int reg = A16(ri);
    const int n0 = region_off[reg], nn = region_off[reg + 1] - n0;
    for (int q = 0; q < nn; ++q) A16(o_nodes + q) = static_cast<int16_t>(q);
    for (int i = nn; i > 1; --i) {
      const int j = static_cast<int>(ga_bounded(rng, static_cast<uint64_t>(i)));
      const int16_t t = A16(o_nodes + i - 1);
      A16(o_nodes + i - 1) = A16(o_nodes + j);
      A16(o_nodes + j) = t;
    }
    for (int q = 0; q < nn; ++q) {
      const int node = n0 + A16(o_nodes + q);
      for (int e = node_off[node]; e < node_off[node + 1]; ++e) A8(nf++) = node_devs[e];
    }
  }
  for (int i = nf; i > 1; --i) {
    const bool scramble = (static_cast<double>(rng.next() >> 11) * 0x1.0p-53) < keep;
    const int pick = static_cast<int>(ga_bounded(rng, static_cast<uint64_t>(i)));
    if (scramble) {
      const uint8_t t = A8(i - 1);
      A8(i - 1) = A8(pick);
      A8(pick) = t;
    }
  }
  uint8_t* __restrict__ dv = rec + o.dev_byte;
  int dev_off[kMaxTasks + 1];
  for (int t = 0; t <= kMaxTasks; ++t) dev_off[t] = o.dev[t];
  const long long p2 = c_ga.prof ? clock64() : 0;
  int cursor = 0;
  for (int g = 0; g < v.ng; ++g) {
    const int n = v.counts[g];
    for (int k = v.gstart[g]; k < v.gstart[g + 1]; ++k) {
      const int s = v.gslot[k];
      for (int r = 0; r < n_nodes; ++r) A16(o_cnt + r) = 0;
      for (int i = 0; i < n; ++i) ++A16(o_cnt + node_rank[A8(cursor + i)]);
      int nr = 0, acc = 0;
      for (int r = 0; r < n_nodes; ++r) {
        const int c = A16(o_cnt + r);
        if (!c) continue;
        A16(o_ranks + nr++) = static_cast<int16_t>(r);
        A16(o_start + r) = static_cast<int16_t>(acc);
        acc += c;
      }
      for (int q = 0; q < nr; ++q) {
        const int rk = A16(o_ranks + q);
        A16(o_fill + rk) = A16(o_start + rk);
      }
      for (int i = 0; i < n; ++i) {
        const uint8_t d = A8(cursor + i);
        const int fi = o_fill + node_rank[d];
        const int f = A16(fi);
        A8(o_bucket + f) = d;
        A16(fi) = static_cast<int16_t>(f + 1);
      }
      for (int i = nr; i > 1; --i) {
        const int j = static_cast<int>(ga_bounded(rng, static_cast<uint64_t>(i)));
        const int16_t t = A16(o_ranks + i - 1);
        A16(o_ranks + i - 1) = A16(o_ranks + j);
        A16(o_ranks + j) = t;
      }
      uint8_t* __restrict__ out = dv + dev_off[s];
      int pos = 0;
      for (int q = 0; q < nr; ++q) {
        const int rk = A16(o_ranks + q);
        const int b0 = o_bucket + A16(o_start + rk);
        const int nb = A16(o_cnt + rk);
        for (int i = nb; i > 1; --i) {
          const int j = static_cast<int>(ga_bounded(rng, static_cast<uint64_t>(i)));
          const uint8_t t = A8(b0 + i - 1);
          A8(b0 + i - 1) = A8(b0 + j);
          A8(b0 + j) = t;
        }
        for (int i = 0; i < nb; ++i) out[pos++] = A8(b0 + i);
      }
    }
    cursor += n;
  }
#undef A16
#undef A8
  rng_io = rng;
  if (c_ga.prof && lane == 1) {  // diagnostics: layouts, medium, fine
    atomicAdd(&c_ga.ctl[99], static_cast<unsigned long long>(p1 - p0));
    atomicAdd(&c_ga.ctl[125], static_cast<unsigned long long>(p2 - p1));
    atomicAdd(&c_ga.ctl[126], static_cast<unsigned long long>(clock64() - p2));
    atomicAdd(&c_ga.ctl[127], 1ull);
  }
}

// an init chunk's candidates on team lane tl of L (tl = 32 * warp + lane):
// candidates combo0 + c for c = tl, tl + L, ... < n from stream state rng
// (lane tl steps the stream tl * gen_draws values ahead, then L - 1
// candidates ahead after each of its candidates); the stream after candidate
// c is kept for the chunk's walk. base: this warp's generation scratch.
__device__ void ga_init_part(const GaView& v, const Rng& rng, int64_t combo0, int n, int tl, int L,
                             uint8_t* base) {
  const int lane = threadIdx.x & 31;
  const uint64_t* jumps = c_ga.jumps + 4 * static_cast<int64_t>(__ldcg(&v.R->jump_off));
  Rng* snaps = c_ga.init_snaps + static_cast<int64_t>(v.run) * c_ga.init_cap;
  GaGenScratch sc;
  sc.s16 = reinterpret_cast<int16_t*>(base);
  sc.s8 = base + 64 * (c_ga.n_regions + c_ga.max_nodes_per_region + 4 * c_ga.n_nodes);
  sc.lane = lane;
  Rng r = rng;
  const long long t0 = c_ga.prof ? clock64() : 0;
  if (tl > 0 && tl < n) rng_apply_jump(r, jumps + 4 * (tl - 1));
  const long long t1 = c_ga.prof ? clock64() : 0;
  long long tj = 0;
  for (int c = tl; c < n; c += L) {
    const long long a = c_ga.prof ? clock64() : 0;
    if (c > tl) rng_apply_jump(r, jumps + 4 * (L - 2));
    if (c_ga.prof) tj += clock64() - a;
    HPG_DCHECK(c < c_ga.init_cap);
    ga_lane_make(v, combo0 + c, r, v.wave_slot(0, c), sc);
    snaps[c] = r;
  }
  if (c_ga.prof && tl == 1 && n > 1) {  // diagnostics: first jump, later jumps, total
    atomicAdd(&c_ga.ctl[111], static_cast<unsigned long long>(t1 - t0));
    atomicAdd(&c_ga.ctl[97], static_cast<unsigned long long>(tj));
    atomicAdd(&c_ga.ctl[98], static_cast<unsigned long long>(clock64() - t0));
  }
}

// a helper warp's generation scratch (global; warp 0 keeps its own slot)
__device__ __forceinline__ uint8_t* ga_helper_gen(int w, int n_warps) {
  const int64_t slot = gridDim.x + static_cast<int64_t>(blockIdx.x) * (n_warps - 1) + (w - 1);
  return c_ga.gen_scratch + slot * c_ga.gen_smem * 32;
}

// an init chunk (warp 0 of a worker): one candidate per lane, over the whole
// team when the chunk is wider than a warp (the helpers wait on the team's
// job barrier between evaluations)
__device__ void ga_init_chunk(const GaView& v, const Rng& rng, int64_t combo0, int n) {
  const int lane = threadIdx.x & 31;
  uint8_t* base = c_ga.gen_in_smem ? v.sm.gen : c_ga.gen_scratch + static_cast<int64_t>(blockIdx.x) *
                                                                     c_ga.gen_smem * 32;
  const int nw = v.sm.n_warps;
  if (nw > 1 && n > 32) {
    GaInitJob* j = v.sm.ijob;
    if (lane == 0) {
      j->v = v;
      j->rng = rng;
      j->combo0 = combo0;
      j->n = n;
      j->kind = kJobGaInit;
    }
    __syncwarp();
    bar_sync(1, 32 * nw);
    ga_init_part(v, rng, combo0, n, lane, 32 * nw, base);
    __threadfence();
    bar_sync(2, 32 * nw);
    if (lane == 0) j->kind = 0;
  } else {
    ga_init_part(v, rng, combo0, n, lane, 32, base);
  }
  __threadfence_block();
  __syncwarp();
}

// per-run scalar state, identical in every lane during a step
struct GaHot {
  Rng rng;
  int64_t used, streak, seq;
  double best, best_member_cost;
  int n_pop, state, have_spec, best_member_flags, impr_flags;
  int child_buf, child_idx;
  double child_cost;
  int n3, n5, m5;
  Rng before3, before5, b5;
  int64_t n_offspring, n_waves, n_evals;
  unsigned long long impr_time;
  int wave_buf, wave_n;
  bool child_sm;  // sm.child holds the child record
  int64_t init_target, attempt_cap, attempts, combo, chunk;
};

__device__ __forceinline__ void ga_load(const GaRun* R, GaHot& h) {
  h.rng = ga_ld_rng(&R->rng);
  h.used = __ldcg(&R->used);
  h.streak = __ldcg(&R->streak);
  h.seq = __ldcg(&R->seq);
  h.best = __ldcg(&R->best);
  h.best_member_cost = __ldcg(&R->best_member_cost);
  h.n_pop = __ldcg(&R->n_pop);
  h.state = __ldcg(&R->state);
  h.have_spec = __ldcg(&R->have_spec);
  h.best_member_flags = __ldcg(&R->best_member_flags);
  h.impr_flags = __ldcg(&R->impr_flags);
  h.child_buf = __ldcg(&R->child_buf);
  h.child_idx = __ldcg(&R->child_idx);
  h.child_cost = __ldcg(&R->child_cost);
  h.n3 = __ldcg(&R->n3);
  h.n5 = __ldcg(&R->n5);
  h.m5 = __ldcg(&R->m5);
  h.before3 = ga_ld_rng(&R->before3);
  h.before5 = ga_ld_rng(&R->before5);
  h.b5 = ga_ld_rng(&R->b5);
  h.n_offspring = __ldcg(&R->n_offspring);
  h.n_waves = __ldcg(&R->n_waves);
  h.n_evals = __ldcg(&R->n_evals);
  h.impr_time = __ldcg(&R->impr_time);
  h.wave_buf = __ldcg(&R->wave_buf);
  h.wave_n = __ldcg(&R->wave_n);
  h.child_sm = false;
  h.init_target = __ldcg(&R->init_target);
  h.attempt_cap = __ldcg(&R->attempt_cap);
  h.attempts = __ldcg(&R->attempts);
  h.combo = __ldcg(&R->combo);
  h.chunk = __ldcg(&R->chunk);
}

__device__ __forceinline__ void ga_store(GaRun* R, const GaHot& h) {
  if ((threadIdx.x & 31) == 0) {
    R->rng = h.rng;
    R->used = h.used;
    R->streak = h.streak;
    R->seq = h.seq;
    R->best = h.best;
    R->best_member_cost = h.best_member_cost;
    R->n_pop = h.n_pop;
    R->state = h.state;
    R->have_spec = h.have_spec;
    R->best_member_flags = h.best_member_flags;
    R->impr_flags = h.impr_flags;
    R->child_buf = h.child_buf;
    R->child_idx = h.child_idx;
    R->child_cost = h.child_cost;
    R->n3 = h.n3;
    R->n5 = h.n5;
    R->m5 = h.m5;
    R->before3 = h.before3;
    R->before5 = h.before5;
    R->b5 = h.b5;
    R->n_offspring = h.n_offspring;
    R->n_waves = h.n_waves;
    R->n_evals = h.n_evals;
    R->impr_time = h.impr_time;
    R->wave_buf = h.wave_buf;
    R->wave_n = h.wave_n;
    R->attempts = h.attempts;
    R->combo = h.combo;
    R->chunk = h.chunk;
  }
  __syncwarp();
}

// the population to / from shared memory (pop_slot in full: the free slots
// past n_pop are used by insertions)
__device__ __forceinline__ void ga_pop_load(const GaView& v, const GaHot& h) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < c_ga.pop_cap; i += 32) {
    v.sm.pslot[i] = __ldcg(&v.R->pop_slot[i]);
    if (i < h.n_pop) {
      v.sm.pcost[i] = __ldcg(&v.R->pop_cost[i]);
      v.sm.pseq[i] = __ldcg(&v.R->pop_seq[i]);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void ga_pop_store(const GaView& v, const GaHot& h) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < c_ga.pop_cap; i += 32) {
    v.R->pop_slot[i] = v.sm.pslot[i];
    if (i < h.n_pop) {
      v.R->pop_cost[i] = v.sm.pcost[i];
      v.R->pop_seq[i] = v.sm.pseq[i];
    }
  }
  __syncwarp();
}

// the finished wave's results to shared memory
__device__ __forceinline__ void ga_res_load(const GaView& v, const GaHot& h) {
  const int lane = threadIdx.x & 31;
  const double2* s = reinterpret_cast<const double2*>(
      c_ga.res + static_cast<int64_t>(v.run) * c_ga.res_per_run + h.wave_buf * c_ga.max_wave);
  double2* d = reinterpret_cast<double2*>(v.sm.res);
  for (int i = lane; i < 2 * h.wave_n; i += 32) d[i] = __ldcg(s + i);
  __syncwarp();
}

// score (search.cpp:454-461): one budget unit; a new run best is an improvement
__device__ void ga_score(const GaView& v, GaHot& h, const uint8_t* rec_g, double cost) {
  ++h.used;
  if (cost < h.best) {
    h.best = cost;
    h.impr_time = ga_timer();
    if ((threadIdx.x & 31) == 0) {
      const unsigned long long k = atomicAdd(&c_ga.ctl[kGaCtlImpr], 1ull);
      HPG_DCHECK(static_cast<int64_t>(k) < c_ga.impr_cap);
      if (static_cast<int64_t>(k) < c_ga.impr_cap)
        c_ga.impr[k] = GaImpr{v.run, 0, h.used, cost, h.impr_time};
    }
    h.impr_time = __shfl_sync(0xffffffffu, h.impr_time, 0);
    ga_rec_copy(v.slot(1), rec_g);
    h.impr_flags |= 1;
  }
}

__device__ __forceinline__ void ga_child_to_sm(const GaView& v, GaHot& h) {
  if (!h.child_sm) {
    ga_ld_rec(v.sm.child, v.wave_slot(h.child_buf, h.child_idx), v.stride);
    h.child_sm = true;
  }
}

// insert_member (search.cpp:462-470), kept sorted by (cost, insertion seq)
__device__ void ga_insert(const GaView& v, GaHot& h) {
  const int lane = threadIdx.x & 31;
  const int P = c_ga.pop_cap;
  const double cost = h.child_cost;
  ga_child_to_sm(v, h);
  if (cost < h.best_member_cost) {
    h.best_member_cost = cost;
    ga_st_rec(v.slot(0), v.sm.child);
    h.best_member_flags = 3;
  }
  const uint64_t seq = static_cast<uint64_t>(h.seq++);
  int pos = 0;
  while (pos < h.n_pop && !(cost < v.sm.pcost[pos])) ++pos;
  const int last = h.n_pop < P ? h.n_pop : P - 1;
  const int slot = v.sm.pslot[last];
  for (int i = last; i > pos; --i) {
    if (lane == 0) {
      v.sm.pslot[i] = v.sm.pslot[i - 1];
      v.sm.pcost[i] = v.sm.pcost[i - 1];
      v.sm.pseq[i] = v.sm.pseq[i - 1];
    }
    __syncwarp();
  }
  if (lane == 0) {
    v.sm.pslot[pos] = slot;
    v.sm.pcost[pos] = cost;
    v.sm.pseq[pos] = seq;
  }
  __syncwarp();
  if (h.n_pop < P) ++h.n_pop;
  ga_st_rec(v.slot(slot), v.sm.child);
}

__device__ __forceinline__ void ga_insert_if(const GaView& v, GaHot& h) {
  if (h.n_pop < c_ga.pop_cap || h.child_cost < v.sm.pcost[h.n_pop - 1]) ga_insert(v, h);
}

// speculative next mutation stage from state r, assuming the child is
// inserted as it stands (search.cpp ga_run: same parent draw)
__device__ void ga_speculate(const GaView& v, GaHot& h, const Rng& r, int buf, int base) {
  const int P = c_ga.pop_cap;
  const double cc = h.child_cost;
  const bool ins = h.n_pop < P || cc < v.sm.pcost[h.n_pop - 1];
  int pos = h.n_pop, n_spec = h.n_pop;
  if (ins) {
    pos = 0;
    while (pos < h.n_pop && !(v.sm.pcost[pos] > cc)) ++pos;
    n_spec = h.n_pop + 1 < P ? h.n_pop + 1 : P;
  }
  Rng rr = r;
  const int i = static_cast<int>(GA_BOUNDED(rr, static_cast<uint64_t>(n_spec)));
  const uint8_t* parent;
  if (!ins || i < pos || i > pos) {
    ga_ld_rec(v.sm.par, v.slot(v.sm.pslot[!ins || i < pos ? i : i - 1]), v.stride);
    parent = v.sm.par;
  } else {
    ga_child_to_sm(v, h);
    parent = v.sm.child;
  }
  ga_draw_mut(v, rr, parent, &v.R->spec, buf, base);
  ga_st_rng(&v.R->spec.start, r);
  __syncwarp();
}

// swap trials at one level from the child (search.cpp:534-558 draw loop)
__device__ int ga_draw(const GaView& v, GaHot& h, int level, int buf, int at, Rng* sn) {
  const int lane = threadIdx.x & 31;
  ga_child_to_sm(v, h);
  GaSrcInfo si;
  ga_src_info(v, v.sm.child, si);
  const bool ok = level == 3 ? v.ng >= 2 : si.ne > 0;
  if (!ok || c_ga.sps <= 0) return 0;  // random_move fails before any draw
  const int n = c_ga.sps, per = level == 3 ? 4 : 3;
  int np = 0, pp[kGaMaxPatch], pv[kGaMaxPatch];
  Rng mine = h.rng;
  if (lane < n) {
    for (int k = 0; k < per * lane; ++k) mine.next();
    np = ga_lane_move(v, v.sm.child, si, level, mine, pp, pv);
    sn[lane] = mine;
  }
  __syncwarp();
  ga_emit_all(v, buf, at, n, v.sm.child, si.geo.dev_byte, np, pp, pv);
  // the stream after the last trial
  h.rng.seed = __shfl_sync(0xffffffffu, mine.seed, n - 1);
  for (int k = 0; k < 4; ++k) h.rng.s[k] = __shfl_sync(0xffffffffu, mine.s[k], n - 1);
  return n;
}

// the sequential trial walk over scored trials [b, b + n) of the finished
// wave: 1 accepted (new child), 2 budget stop, 0 ran out
__device__ int ga_walk(const GaView& v, GaHot& h, int b, int n, const Rng& before, const Rng* sn) {
  const int64_t slice = __ldcg(&v.R->slice);
  for (int t = 0; t < n; ++t) {
    if (h.used >= slice) {
      h.rng = t == 0 ? before : ga_ld_rng(&sn[t - 1]);
      return 2;
    }
    const EvalResult& e = v.sm.res[b + t];
    if (!(e.flags & kResFeasIn)) continue;
    const double c2 = e.cost;
    ga_score(v, h, v.wave_slot(h.wave_buf, b + t), c2);
    if (c2 < h.child_cost) {
      h.child_buf = h.wave_buf;
      h.child_idx = b + t;
      h.child_cost = c2;
      h.child_sm = false;
      h.rng = ga_ld_rng(&sn[t]);
      return 1;
    }
  }
  if (n > 0) h.rng = ga_ld_rng(&sn[n - 1]);
  return 0;
}

// publishes evaluation tasks (run, i) for i in [i0, i1)
__device__ void ga_publish(int run, int i0, int i1) {
  const int lane = threadIdx.x & 31;
  const int n = i1 - i0;
  if (n <= 0) return;
  __threadfence();  // every lane's record stores before any task is visible
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&c_ga.ctl[kGaCtlTail], static_cast<unsigned long long>(n));
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int k = lane; k < n; k += 32) {
    const unsigned long long t = base + k;
    c_ga.q_pay[t & c_ga.q_mask] = make_uint2(static_cast<unsigned>(run), static_cast<unsigned>(i0 + k));
    __threadfence();
    atomicExch(&c_ga.q_seq[t & c_ga.q_mask], t + 1);
  }
  __syncwarp();
}


// One draw of a swap wave (kGaTaskDraw3 / kGaTaskDraw5 / kGaTaskSpec) from
// the positions the step stored: draws, publishes its candidates and closes
// its share. 1 when the whole wave has been evaluated already (the caller
// continues the run).
__device__ int ga_draw_task(int r, int kind, const GaSm& sm) {
  GaRun* R = c_ga.runs + r;
  GaView v;
  v.R = R;
  v.run = r;
  v.pool = c_ga.pool + __ldcg(&R->pool_off);
  v.stride = __ldcg(&R->rec_stride);
  v.ng = __ldcg(&R->ng);
  for (int k = 0; k <= kMaxTasks; ++k) v.gstart[k] = __ldcg(&R->gstart[k]);
  for (int k = 0; k < kMaxTasks; ++k) v.gslot[k] = __ldcg(&R->gslot[k]);
  v.sm = sm;
  GaHot h;
  ga_load(R, h);
  const int wb = h.wave_buf;
  int i0 = 0, i1 = 0;
  if (kind == kGaTaskDraw3) {
    h.rng = h.before3;
    ga_draw(v, h, 3, wb, 0, R->snaps3);
    i0 = 0;
    i1 = h.n3;
  } else if (kind == kGaTaskDraw5) {
    h.rng = h.before5;
    ga_draw(v, h, 5, wb, h.n3, R->snaps5);
    i0 = h.n3;
    i1 = h.n3 + h.n5;
  } else {
    ga_pop_load(v, h);
    const int base2 = h.n3 + h.n5;
    ga_speculate(v, h, ga_ld_rng(&R->spec_from), wb, base2);
    i0 = base2;
    i1 = base2 + __ldcg(&R->spec.ntr) + 1;
    if ((threadIdx.x & 31) == 0) R->wave_n = i1;
  }
  ga_publish(r, i0, i1);
  __threadfence();
  int done = 0;
  if ((threadIdx.x & 31) == 0)
    done = atomicAdd(&R->pending, (i1 - i0) - kGaPendBias) == kGaPendBias - (i1 - i0);
  done = __shfl_sync(0xffffffffu, done, 0);
  if (done) __threadfence();
  return done;
}

// diagnostics: sub-phase cycles of a GA step (ctl words 100..107)
#define GA_PH(slot, expr)                                                         \
  do {                                                                            \
    const long long ph0_ = c_ga.prof ? clock64() : 0;                               \
    expr;                                                                         \
    if (c_ga.prof && (threadIdx.x & 31) == 0)                                        \
      atomicAdd(&c_ga.ctl[100 + (slot)], static_cast<unsigned long long>(clock64() - ph0_)); \
  } while (0)

// one GA step of run r: runs the state machine until it has published a wave
// that is still being evaluated or the run ends (returns 0); 1 asks the
// worker to step the run again (not used: a finished wave continues here)
__device__ int ga_step(int r, const GaSm& sm) {
  GaRun* R = c_ga.runs + r;
  GaView v;
  v.R = R;
  v.run = r;
  v.pool = c_ga.pool + __ldcg(&R->pool_off);
  v.stride = __ldcg(&R->rec_stride);
  v.ng = __ldcg(&R->ng);
  for (int k = 0; k <= kMaxTasks; ++k) v.gstart[k] = __ldcg(&R->gstart[k]);
  for (int k = 0; k < kMaxTasks; ++k) v.gslot[k] = __ldcg(&R->gslot[k]);
  for (int k = 0; k < kMaxTasks; ++k) v.counts[k] = __ldcg(&R->counts[k]);
  for (int k = 0; k <= kMaxTasks; ++k) v.opt_off[k] = __ldcg(&R->opt_off[k]);
  v.opt_base = __ldcg(&R->opt_base);
  v.sm = sm;
  const int64_t slice = __ldcg(&R->slice);
  GaHot h;
  GA_PH(0, ga_load(R, h); ga_pop_load(v, h);
        if (h.state != kGaLoop && h.state != kGaInit && h.state != kGaInitDone) ga_res_load(v, h));
  // A wave's candidates are published as they are drawn, so evaluation
  // overlaps the rest of the step: pending starts biased and drops to the
  // true count when the step closes the wave.
  auto wave_begin = [&](int buf) {
    h.wave_buf = buf;
    if ((threadIdx.x & 31) == 0) {
      R->wave_buf = buf;
      R->pending = kGaPendBias;
    }
    __threadfence();
    __syncwarp();
  };
  auto wave_cancel = [&]() {
    if ((threadIdx.x & 31) == 0) R->pending = 0;
    __syncwarp();
  };
  // closes the wave of n candidates; 1 when they have all been evaluated
  // already (this warp continues the run), else 0
  auto wave_end = [&](int n) {
    h.wave_n = n;
    ++h.n_waves;
    h.n_evals += n;
    int done = 0;
    GA_PH(1, ga_pop_store(v, h); ga_store(R, h); __threadfence();
          if ((threadIdx.x & 31) == 0) done = atomicAdd(&R->pending, n - kGaPendBias) == kGaPendBias - n;
          done = __shfl_sync(0xffffffffu, done, 0));
    if (done) {
      __threadfence();
      if (h.state != kGaInitDone) ga_res_load(v, h);
    }
    return done;
  };
  auto finish = [&]() {
    h.state = kGaDone;
    ga_pop_store(v, h);
    ga_store(R, h);
    __threadfence();
    if ((threadIdx.x & 31) == 0) {
      const unsigned long long d = atomicAdd(&c_ga.ctl[kGaCtlDone], 1ull) + 1;
      if (d == static_cast<unsigned long long>(c_ga.n_runs)) atomicExch(&c_ga.ctl[kGaCtlStop], 1ull);
    }
    __syncwarp();
    return 0;
  };
  while (true) {
    if (h.state == kGaInit) {
      // init: cycle layout combinations in doubling chunks until init_target
      // members (search.cpp:437-450 as restated in ga_run)
      if (!(h.n_pop < h.init_target && h.used < slice && h.attempts < h.attempt_cap)) {
        if (h.n_pop == 0) return finish();
        h.state = kGaLoop;
        continue;
      }
      const int64_t need = h.init_target - h.n_pop;
      const int64_t grow = h.chunk * 2 > 2 * need + 2 ? h.chunk * 2 : 2 * need + 2;
      h.chunk = h.attempt_cap - h.attempts < grow ? h.attempt_cap - h.attempts : grow;
      wave_begin(0);
      GA_PH(8, ga_init_chunk(v, h.rng, h.combo, static_cast<int>(h.chunk)));
      if (c_ga.prof && (threadIdx.x & 31) == 0) {
        atomicAdd(&c_ga.ctl[109], 1ull);
        atomicAdd(&c_ga.ctl[110], static_cast<unsigned long long>(h.chunk));
      }
      h.state = kGaInitDone;
      ga_publish(r, 0, static_cast<int>(h.chunk));
      if (wave_end(static_cast<int>(h.chunk))) continue;
      return 0;
    }
    if (h.state == kGaInitDone) {
      const int lane = threadIdx.x & 31;
      const int n = h.wave_n;
      const int64_t combo0 = h.combo;
      h.combo += n;
      const Rng* snaps = c_ga.init_snaps + static_cast<int64_t>(r) * c_ga.init_cap;
      h.rng = ga_ld_rng(&snaps[n - 1]);
      const EvalResult* res = c_ga.res + static_cast<int64_t>(r) * c_ga.res_per_run;
      bool stop = false;
      for (int b = 0; b < n && !stop; b += 32) {
        int fl = 0;
        double co = 0.0;
        if (b + lane < n) {
          fl = __ldcg(&res[b + lane].flags);
          co = __ldcg(&res[b + lane].cost);
        }
        for (int j = 0; j < 32 && b + j < n; ++j) {
          const int f = __shfl_sync(0xffffffffu, fl, j);
          const double cj = __shfl_sync(0xffffffffu, co, j);
          ++h.attempts;
          if (!(f & kResFeasIn)) continue;
          const int c = b + j;
          ga_score(v, h, v.wave_slot(0, c), cj);
          h.child_buf = 0;
          h.child_idx = c;
          h.child_cost = cj;
          h.child_sm = false;
          ga_insert(v, h);
          if (h.n_pop >= h.init_target) {
            h.rng = ga_ld_rng(&snaps[c]);
            h.combo = combo0 + c + 1;
            stop = true;
            break;
          }
        }
      }
      h.state = kGaInit;
      continue;
    }
    if (h.state == kGaLoop) {
      if (!(h.used < slice && h.streak < kGaStreakCap)) return finish();
      ++h.n_offspring;
      if (h.have_spec && ga_same_rng(ga_ld_rng(&R->spec.start), h.rng)) {
        // the speculative stage drawn with the finished wave is this one
        const int4* s = reinterpret_cast<const int4*>(&R->spec);
        int4* d = reinterpret_cast<int4*>(&R->cur);
        const int lane = threadIdx.x & 31;
        GA_PH(3, for (int i = lane; i < static_cast<int>(sizeof(GaStage) / 16); i += 32) d[i] = __ldcg(s + i);
              __syncwarp());
        h.have_spec = 0;
        h.state = kGaMut;
        continue;
      }
      h.have_spec = 0;
      Rng r2 = h.rng;
      const int i = static_cast<int>(GA_BOUNDED(r2, static_cast<uint64_t>(h.n_pop)));
      wave_begin(0);
      GA_PH(6, ga_ld_rec(sm.par, v.slot(sm.pslot[i]), v.stride);
            ga_draw_mut(v, r2, sm.par, &R->cur, 0, 0));
      h.state = kGaMut;
      const int nm = __ldcg(&R->cur.ntr) + 1;
      ga_publish(r, 0, nm);
      if (wave_end(nm)) continue;
      return 0;
    }
    if (h.state == kGaMut) {
      // the stage's results are in sm.res (its wave just finished)
      const int buf = __ldcg(&R->cur.buf), base = __ldcg(&R->cur.base), ntr = __ldcg(&R->cur.ntr);
      int chosen = -1;
      for (int i = 0; i < ntr; ++i)
        if (sm.res[base + i].flags & kResFeasIn) {
          chosen = i;
          break;
        }
      if (chosen >= 0) {
        h.rng = ga_ld_rng(&R->cur.snaps[chosen]);
        h.child_idx = base + chosen;
      } else {
        h.rng = ga_ld_rng(&R->cur.after_all);
        if (!(sm.res[base + ntr].flags & kResFeasIn)) {
          ++h.streak;
          h.state = kGaLoop;
          continue;
        }
        h.child_idx = base + ntr;
      }
      h.child_buf = buf;
      h.child_sm = false;
      h.child_cost = sm.res[h.child_idx].cost;
      h.streak = 0;
      GA_PH(7, ga_score(v, h, v.wave_slot(buf, h.child_idx), h.child_cost));
      if (h.used < slice) {
        // the swap wave: L3 trials, L5 trials and the speculative stage.
        // Their stream positions are fixed in advance (a level-3 move draws
        // four values, a level-5 move three), so other workers draw two of
        // the three at the same time (ga_draw_task) while this one draws the
        // first; each publishes its candidates and closes its share of the wave
        const int wb = 1 - h.child_buf;
        ga_child_to_sm(v, h);
        GaGeo geo;
        ga_geo(sm.child, c_ga.n_tasks, geo);
        int ne = 0;
        for (int s = 0; s < c_ga.n_tasks; ++s) ne += geo.off[s + 1] - geo.off[s] >= 2;
        const int sps = c_ga.sps;
        h.n3 = v.ng >= 2 && sps > 0 ? sps : 0;
        h.n5 = ne > 0 && sps > 0 ? sps : 0;
        h.before3 = h.rng;
        // throughput mode (many live runs: the GPU is busy with evaluations):
        // the L3 trials alone first; L5 and the speculative stage follow only
        // if no L3 trial is accepted (as a redraw wave from the same stream
        // position), which spends fewer evaluations per offspring
        const bool split = h.n3 > 0 && static_cast<long long>(c_ga.n_runs) -
                                               static_cast<long long>(__ldcg(&c_ga.ctl[kGaCtlDone])) >
                                           c_ga.split_runs;
        if (split) {
          Rng q = h.rng;
          for (int k2 = 0; k2 < 4 * h.n3; ++k2) q.next();
          h.before5 = q;
          h.wave_buf = wb;
          ++h.n_waves;
          h.state = kGaSwap3;
          ga_pop_store(v, h);
          ga_store(R, h);
          if ((threadIdx.x & 31) == 0) {
            R->wave_buf = wb;
            R->wave_n = h.n3;
            R->pending = kGaPendBias;
          }
          __threadfence();
          __syncwarp();
          int dn = 0;
          GA_PH(2, dn = ga_draw_task(r, kGaTaskDraw3, sm));
          if (dn) {
            ga_load(R, h);
            ga_pop_load(v, h);
            ga_res_load(v, h);
            continue;
          }
          return 0;
        }
        if (h.n3 + h.n5 > 0) {
          Rng q = h.rng;
          for (int k2 = 0; k2 < 4 * h.n3; ++k2) q.next();
          h.before5 = q;
          for (int k2 = 0; k2 < 3 * h.n5; ++k2) q.next();
          h.rng = q;
          const int first = h.n3 > 0 ? kGaTaskDraw3 : kGaTaskDraw5;
          const int shares = (h.n3 > 0) + (h.n5 > 0) + 1;
          h.wave_buf = wb;
          ++h.n_waves;
          h.state = kGaSwap;
          ga_pop_store(v, h);
          ga_store(R, h);
          if ((threadIdx.x & 31) == 0) {
            R->wave_buf = wb;
            R->spec_from = q;
            R->pending = shares * kGaPendBias;
          }
          __threadfence();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) {
            // the other draws go to the ring
            const int n_t = shares - 1;
            const unsigned long long base = atomicAdd(&c_ga.ctl[kGaCtlTail],
                                                      static_cast<unsigned long long>(n_t));
            // first = L3 when there are L3 trials, else L5; the rest: L5
            // (when both levels draw) and the speculative stage
            int kinds[2], nk = 0;
            if (first == kGaTaskDraw3 && h.n5 > 0) kinds[nk++] = kGaTaskDraw5;
            kinds[nk++] = kGaTaskSpec;
            for (int k3 = 0; k3 < nk; ++k3) {
              const unsigned long long t = base + k3;
              c_ga.q_pay[t & c_ga.q_mask] =
                  make_uint2(static_cast<unsigned>(r), static_cast<unsigned>(kinds[k3]));
              __threadfence();
              atomicExch(&c_ga.q_seq[t & c_ga.q_mask], t + 1);
            }
          }
          __syncwarp();
          int dn = 0;
          GA_PH(2, dn = ga_draw_task(r, first, sm));
          if (dn) {
            ga_load(R, h);
            ga_pop_load(v, h);
            ga_res_load(v, h);
            continue;
          }
          return 0;
        }
        h.before5 = h.rng;
      }
      GA_PH(5, ga_insert_if(v, h));
      h.state = kGaLoop;
      continue;
    }
    if (h.state == kGaSwap) {
      h.rng = h.before5;
      int w3 = 0;
      GA_PH(4, w3 = ga_walk(v, h, 0, h.n3, h.before3, R->snaps3));
      if (w3 == 0 && h.used < slice) {
        h.rng = h.before5;
        int w5 = 0;
        GA_PH(4, w5 = ga_walk(v, h, h.n3, h.n5, h.before5, R->snaps5));
        if (w5 == 0) h.have_spec = 1;
      } else if (w3 == 1 && h.used < slice) {
        const int wb2 = 1 - h.child_buf;
        h.b5 = h.rng;
        wave_begin(wb2);
        h.m5 = ga_draw(v, h, 5, wb2, 0, R->snaps5);
        ga_publish(r, 0, h.m5);
        if (h.m5 > 0) {
          ga_speculate(v, h, ga_ld_rng(&R->snaps5[h.m5 - 1]), wb2, h.m5);
          h.state = kGaRedraw;
          const int nw = h.m5 + __ldcg(&R->spec.ntr) + 1;
          ga_publish(r, h.m5, nw);
          if (wave_end(nw)) continue;
          return 0;
        }
        wave_cancel();
      }
      GA_PH(5, ga_insert_if(v, h));
      h.state = kGaLoop;
      continue;
    }
    if (h.state == kGaSwap3) {
      // the L3-only wave: then the L5 trials (+ speculation) from the child,
      // whichever it is now, at the stream position the walk leaves: the
      // L3 walk's acceptance point, or the end of the L3 draws
      h.rng = h.before5;
      int w3 = 0;
      GA_PH(4, w3 = ga_walk(v, h, 0, h.n3, h.before3, R->snaps3));
      if ((w3 == 0 || w3 == 1) && h.used < slice) {
        const int wb2 = 1 - h.child_buf;
        h.b5 = h.rng;
        wave_begin(wb2);
        h.m5 = ga_draw(v, h, 5, wb2, 0, R->snaps5);
        ga_publish(r, 0, h.m5);
        if (h.m5 > 0) {
          ga_speculate(v, h, ga_ld_rng(&R->snaps5[h.m5 - 1]), wb2, h.m5);
          h.state = kGaRedraw;
          const int nw = h.m5 + __ldcg(&R->spec.ntr) + 1;
          ga_publish(r, h.m5, nw);
          if (wave_end(nw)) continue;
          return 0;
        }
        wave_cancel();
      }
      GA_PH(5, ga_insert_if(v, h));
      h.state = kGaLoop;
      continue;
    }
    if (h.state == kGaRedraw) {
      if (ga_walk(v, h, 0, h.m5, h.b5, R->snaps5) == 0) h.have_spec = 1;
      ga_insert_if(v, h);
      h.state = kGaLoop;
      continue;
    }
    return 0;  // kGaDone: not reached
  }
}

// canonical bytes of one plan (engine.cpp wave_stage)
__device__ __forceinline__ long long ga_canonical(const DevProblem& P, const uint8_t* rec, int ng) {
  const int32_t* h = reinterpret_cast<const int32_t*>(rec);
  long long cb = 1 + ng + 9;
  int sw = 0, wg = 0;
  for (int t = 0; t < P.n_tasks; ++t) {
    const int dp = __ldcg(h + 2 + t), pp = __ldcg(h + 2 + kMaxTasks + t),
              tp = __ldcg(h + 2 + 2 * kMaxTasks + t);
    cb += 3 + pp + dp * pp * tp;
    if (t == P.gen_slot) wg = sw;
    sw += dp;
  }
  if (P.gen_slot >= 0) {
    const int dpg = __ldcg(h + 2 + P.gen_slot);
    const double* w = reinterpret_cast<const double*>(rec + sizeof(RecHeader)) + wg;
    bool unit = true;
    for (int k = 0; k < dpg; ++k)
      if (__ldcg(w + k) != 1.0) unit = false;
    if (!unit) cb += 8 * dpg;
  }
  return cb;
}

// helper warps of a GA worker: init-chunk candidates (kJobGaInit) and the
// per-task parts of the lead's evaluations (team_helper's jobs)
__device__ __noinline__ void ga_team_helper(const DevProblem& P, const DevCostConfig& cfg, Ws* team,
                                            int w, const GaInitJob* ij) {
  const int lane = threadIdx.x & 31;
  Ws& s = team[w];
  const Ws& s0 = team[0];
  const int threads = 32 * s.n_warps;
  uint8_t* gen = ga_helper_gen(w, s.n_warps);
  while (true) {
    bar_sync(1, threads);
    if (ij->kind == kJobGaInit) {
      ga_init_part(ij->v, ij->rng, ij->combo0, ij->n, 32 * w + lane, threads, gen);
      __threadfence();
      bar_sync(2, threads);
      continue;
    }
    const int kind = s0.job[0], mask = s0.job[1];
    if (kind == kJobExit) return;
    {  // the lead's current plan view
      const int32_t* hs = reinterpret_cast<const int32_t*>(&s0.h);
      int32_t* hd = reinterpret_cast<int32_t*>(&s.h);
      for (int i = lane; i < static_cast<int>(sizeof(RecHeader) / 4); i += 32) hd[i] = hs[i];
      const int32_t* os = reinterpret_cast<const int32_t*>(&s0.o);
      int32_t* od = reinterpret_cast<int32_t*>(&s.o);
      for (int i = lane; i < static_cast<int>(sizeof(RecOffsets) / 4); i += 32) od[i] = os[i];
      if (lane == 0) {
        s.memo_tp_ok = s0.memo_tp_ok;
        s.memo_pp_ok = s0.memo_pp_ok;
        s.memo_cm_ok = s0.memo_cm_ok;
      }
      __syncwarp();
    }
    team_share(P, cfg, s, kind, mask, w);
    bar_sync(2, threads);
  }
}

// kTeam = 1: one-warp workers (busy rounds); kTeam = 2: each worker has a
// helper warp for the per-task parts of an evaluation (eval_kernel's teams),
// for rounds with few live runs where an evaluation's latency is the chain;
// kTeam = 4: three helpers, registers uncapped (the last, narrowest rounds)
template <int kTeam>
__global__ void __launch_bounds__(32 * kTeam, kTeam == 4 ? 2 : 16 / kTeam)
ga_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ DevCostConfig cfg,
          const __grid_constant__ Carve cv, double* __restrict__ gscratch,
          int64_t gscratch_doubles, const __grid_constant__ GaParams ga_in) {
  extern __shared__ __align__(16) uint8_t smem[];
  {
    static_assert(sizeof(GaParams) % 8 == 0, "GaParams copy granule");
    const uint64_t* src = reinterpret_cast<const uint64_t*>(&ga_in);
    uint64_t* dst = reinterpret_cast<uint64_t*>(&c_ga);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(GaParams) / 8); i += blockDim.x)
      dst[i] = src[i];
    __syncthreads();
  }
  __shared__ Ws team[kTeam];
  __shared__ GaInitJob ijob[1];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  GaSm sm;
  sm.ijob = ijob;
  sm.n_warps = kTeam;
  if (warp == 0) {
    // GA scratch after the evaluation carve (launch_ga_offspring sizes it)
    uint8_t* p = smem + carve2_bytes(cv);
    const int stride = c_ga.max_stride;
    sm.child = p;
    sm.par = p + stride;
    sm.tmp = p + 2 * stride;
    sm.res = reinterpret_cast<EvalResult*>(p + 3 * stride);
    sm.pcost = reinterpret_cast<double*>(p + 3 * stride + 32 * c_ga.max_wave);
    sm.pseq = reinterpret_cast<uint64_t*>(sm.pcost + kGaMaxPop);
    sm.pslot = reinterpret_cast<int32_t*>(sm.pseq + kGaMaxPop);
    sm.gw = reinterpret_cast<uint32_t*>(sm.pslot + kGaMaxPop);
    sm.gen = smem;
    uint8_t* tb = reinterpret_cast<uint8_t*>(sm.gw + 8 * kMaxTasks);
    const int N = c_ga.n_dev;
    uint8_t* id_rank = tb;
    uint8_t* by_id_rank = tb + N;
    uint8_t* node_rank = tb + 2 * N;
    uint8_t* node_devs = tb + 3 * N;
    int16_t* region_off = reinterpret_cast<int16_t*>(tb + 4 * N);
    int16_t* node_off = region_off + c_ga.n_regions + 1;
    const int lane0 = threadIdx.x & 31;
    for (int i = lane0; i < N; i += 32) {
      id_rank[i] = static_cast<uint8_t>(c_ga.id_rank[i]);
      by_id_rank[i] = static_cast<uint8_t>(c_ga.by_id_rank[i]);
      node_rank[i] = static_cast<uint8_t>(c_ga.node_rank[i]);
      node_devs[i] = c_ga.node_devs[i];
    }
    for (int i = lane0; i <= c_ga.n_regions; i += 32) region_off[i] = static_cast<int16_t>(c_ga.region_off[i]);
    for (int i = lane0; i <= c_ga.n_nodes; i += 32) node_off[i] = static_cast<int16_t>(c_ga.node_off[i]);
    sm.id_rank = id_rank;
    sm.by_id_rank = by_id_rank;
    sm.node_rank = node_rank;
    sm.node_devs = node_devs;
    sm.region_off = region_off;
    sm.node_off = node_off;
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    Ws& l = team[0];
    uint8_t* p = carve(l, smem, cv);
    l.dtab = gscratch + static_cast<int64_t>(blockIdx.x) * gscratch_doubles;
    l.dtab_stride = 0;
    l.prof = g_plan_prof;  // diagnostics only (HPG_GA_LOG): a shared dummy slot block
    l.team = team;
    l.n_warps = kTeam;
    l.job_words[0] = l.job_words[1] = 0;
    l.job = l.job_words;
    l.cta_sync = 0;
    if (!cv.cls_smem) l.cls = P.cls;  // else carved last (the init scratch stays below it)
    for (int w = 1; w < kTeam; ++w) {
      team[w] = l;
      p = carve_team_scratch(team[w], p, cv);
    }
    if (blockIdx.x == 0) atomicCAS(&c_ga.ctl[kGaCtlT0], 0ull, ga_timer());
    ijob[0].kind = 0;
  }
  __syncthreads();
  Ws& s = team[0];
  // persistent workers: the link-class matrix is staged once
  if (warp == 0 && cv.cls_smem) stage_link_classes(P, s);
  __syncthreads();
  if (warp > 0) {  // helper: init chunks and per-task jobs of warp 0's evaluations
    ga_team_helper(P, cfg, team, warp, ijob);
    return;
  }
  while (true) {
    // take a ticket, wait for its task (or for the end of the launch)
    unsigned long long t = 0;
    uint2 pay = make_uint2(0, 0);
    int stop = 0;
    if (lane == 0) {
      t = atomicAdd(&c_ga.ctl[kGaCtlHead], 1ull);
      volatile unsigned long long* seq = c_ga.q_seq + (t & c_ga.q_mask);
      volatile unsigned long long* stopw = c_ga.ctl + kGaCtlStop;
      unsigned ns = 32;
      while (*seq != t + 1) {
        if (*stopw) {
          stop = 1;
          break;
        }
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
      }
      if (!stop) {
        __threadfence();
        pay = __ldcg(c_ga.q_pay + (t & c_ga.q_mask));
      }
    }
    stop = __shfl_sync(0xffffffffu, stop, 0);
    if (stop) break;
    int run = static_cast<int>(__shfl_sync(0xffffffffu, pay.x, 0));
    int idx = static_cast<int>(__shfl_sync(0xffffffffu, pay.y, 0));
    while (true) {
      if (idx <= kGaTaskSpec) {  // one draw of a swap wave
        if (!ga_draw_task(run, idx, sm)) break;
        idx = kGaTaskStep;
        continue;
      }
      if (idx < 0) {  // GA step (again while its waves finish before it closes them)
        const long long c0 = c_ga.prof ? clock64() : 0;
        const int again = ga_step(run, sm);
        if (c_ga.prof && lane == 0) {
          atomicAdd(&c_ga.ctl[kGaCtlProf], static_cast<unsigned long long>(clock64() - c0));
          atomicAdd(&c_ga.ctl[kGaCtlProf + 1], 1ull);
        }
        if (!again) break;
        continue;
      }
      const long long c1 = c_ga.prof ? clock64() : 0;
      GaRun* R = c_ga.runs + run;
      const int buf = __ldcg(&R->wave_buf);
      uint8_t* rec = c_ga.pool + __ldcg(&R->pool_off) +
                     static_cast<int64_t>(2 + c_ga.pop_cap + buf * c_ga.max_wave + idx) *
                         __ldcg(&R->rec_stride);
      long long cb = 0;
      if (lane == 0) cb = ga_canonical(P, rec, __ldcg(&R->ng));
      const EvalResult e = eval_one(P, cfg, s, c_ga.kb_flags, rec, kModeEvaluate, nullptr, nullptr,
                                    nullptr, nullptr, rec);
      int last = 0;
      if (lane == 0) {
        HPG_DCHECK(run >= 0 && run < c_ga.n_runs && buf * c_ga.max_wave + idx < c_ga.res_per_run);
        c_ga.res[static_cast<int64_t>(run) * c_ga.res_per_run + buf * c_ga.max_wave + idx] = e;
        atomicAdd(&c_ga.ctl[kGaCtlEvals], 1ull);
        atomicAdd(&c_ga.ctl[kGaCtlBytes], static_cast<unsigned long long>(cb));
        __threadfence();
        last = atomicSub(&R->pending, 1) == 1;
        if (last) __threadfence();
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (c_ga.prof && lane == 0) {
        atomicAdd(&c_ga.ctl[kGaCtlProf + 2], static_cast<unsigned long long>(clock64() - c1));
        atomicAdd(&c_ga.ctl[kGaCtlProf + 3], 1ull);
      }
      if (!last) break;
      idx = -1;  // this warp finished the wave: continue the run
    }
  }
  team_exit(s);
}

}  // namespace dev

namespace {
template <int kTeam>
cudaError_t ga_launch_team(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                           const GaParams& G, double* gscratch, int64_t gscratch_doubles,
                           int n_sm, int& grid, cudaStream_t st) {
  auto kern = dev::ga_kernel<kTeam>;
  cv.n_warps = kTeam;
  // the N x N link-class matrix in each worker's shared memory: small
  // problems always; up to 128 devices (16 KB) for the helper-warp teams of
  // the narrow, latency-bound rounds (HPG_GA_CLS_TEAM=0 turns that off)
  static const int cls_team = [] {
    const char* v = std::getenv("HPG_GA_CLS_TEAM");  // 0: off, 1: teams, 2: every worker
    return v ? std::atoi(v) : 1;
  }();
  const int nn = P.n_dev * P.n_dev;
  cv.cls_smem = nn <= 4096 || ((kTeam > 1 ? cls_team >= 1 : cls_team >= 2) && nn <= kClsSmemMax) ? 1 : 0;
  cv.bytes = carve2_bytes(cv) + dev::ga_smem_bytes(G.max_stride, G.max_wave, G.n_dev, G.n_regions,
                                                    G.n_nodes);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), cv.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = occupancy_per_sm(reinterpret_cast<const void*>(kern), 32 * kTeam, cv.bytes, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  grid = n_sm * per_sm;
  // the workers' generation scratch (gen_scratch) has 16 warp slots per SM:
  // clamp every team size before the launch
  if (grid * kTeam > 16 * n_sm) grid = 16 * n_sm / kTeam;
  GaParams g2 = G;
  if (g2.split_runs < 0) g2.split_runs = grid / 16;  // ~one swap wave per run fills the workers
  kern<<<grid, 32 * kTeam, cv.bytes, st>>>(P, cfg, cv, gscratch, gscratch_doubles, g2);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_ga_offspring(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                                const GaParams& G, double* gscratch, int64_t gscratch_doubles,
                                int n_sm, int& grid, cudaStream_t st) {
  // few live runs (at most one per SM): workers with helper warps, which
  // shorten each evaluation (measured per SHA round on c1-c4: teams of four
  // win whenever runs <= SMs and lose throughput in the wide early rounds)
  static const int team_env = [] {
    const char* v = std::getenv("HPG_GA_TEAM");  // diagnostics: 1, 2 or 4 forces the team size
    return v ? std::atoi(v) : 0;
  }();
  int team = 1;
  if (team_env == 1 || team_env == 2 || team_env == 4)
    team = team_env;
  else if (P.n_tasks >= 2 && G.n_runs <= n_sm)
    team = P.n_tasks >= 3 ? 4 : 2;
  if (team == 4) {
    const cudaError_t e = ga_launch_team<4>(P, cfg, cv, G, gscratch, gscratch_doubles, n_sm, grid, st);
    if (e != cudaErrorInvalidConfiguration) return e;
    (void)cudaGetLastError();
  }
  if (team >= 2) {
    const cudaError_t e = ga_launch_team<2>(P, cfg, cv, G, gscratch, gscratch_doubles, n_sm, grid, st);
    if (e != cudaErrorInvalidConfiguration) return e;
    (void)cudaGetLastError();
  }
  return ga_launch_team<1>(P, cfg, cv, G, gscratch, gscratch_doubles, n_sm, grid, st);
}

}  // namespace hpg
