// Problem staging, plan validation/packing and the batched device call.
#include "engine.hpp"

#include <immintrin.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>

#include "eval_launch.hpp"
#include "host_pool.hpp"

namespace hpg {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw InternalError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}


namespace {

std::string str_or_empty(const char* s) { return s ? std::string(s) : std::string(); }

int task_kind_of(int id) { return id == 1 ? kGeneration : (id <= 4 ? kInference : kTraining); }

}  // namespace

Problem build_problem(const hpg_problem& p) {
  Problem P;
  // ---- workflow (build_workflow, workflow.cpp:97-146; validators :16-33) ----
  if (p.eta < 0.0 || p.eta > 1.0) throw InputError("eta must be within [0, 1]");
  if (p.global_batch < 1 || p.responses_per_prompt < 1 || p.micro_batch_size < 1)
    throw InputError("batch sizes must be >= 1");
  if (p.seq_in < 1 || p.seq_out < 0) throw InputError("seq_in must be >= 1 and seq_out >= 0");
  if (p.n_tasks < 1 || p.n_tasks > kMaxTasks || p.tasks == nullptr)
    throw InputError("workflow must list 1..6 tasks");
  P.algorithm = p.algorithm;
  P.mode = p.mode;
  P.eta = p.eta;
  P.global_batch = p.global_batch;
  P.rpp = p.responses_per_prompt;
  P.seq_in = p.seq_in;
  P.seq_out = p.seq_out;
  P.mbs = p.micro_batch_size;
  std::fill(std::begin(P.slot_of_id), std::end(P.slot_of_id), -1);
  int prev = 0;
  for (int t = 0; t < p.n_tasks; ++t) {
    const hpg_task& in = p.tasks[t];
    if (in.id < 1 || in.id > 6) throw InputError("unknown task id " + std::to_string(in.id));
    if (in.id <= prev) throw InputError("workflow tasks must be ordered by id");
    prev = in.id;
    if (in.kind < 0 || in.kind > 2) throw InputError("unknown task kind");
    if (in.hidden_size < 1 || in.intermediate_size < 1 || in.num_layers < 1)
      throw InputError(
          "model spec requires hidden_size, intermediate_size and num_layers >= 1");
    if (in.include_embedding && in.vocab_size < 1)
      throw InputError("include_embedding requires vocab_size >= 1");
    HostTask h;
    h.id = in.id;
    h.kind = in.kind;
    h.h1 = in.hidden_size;
    h.h2 = in.intermediate_size;
    h.nl = in.num_layers;
    h.emb = in.include_embedding != 0;
    h.vocab = in.vocab_size;
    h.prec = in.precision_bytes;
    h.layer_params = 4 * h.h1 * h.h1 + 3 * h.h1 * h.h2;
    h.param_count = h.nl * h.layer_params + (h.emb ? 2 * h.vocab * h.h1 : 0);
    P.slot_of_id[in.id] = t;
    P.tasks.push_back(h);
  }
  (void)task_kind_of;
  P.T = p.n_tasks;
  for (int e = 0; e < p.n_dep_edges; ++e) {
    P.dep_edges.emplace(p.dep_edges[2 * e], p.dep_edges[2 * e + 1]);
  }

  // ---- topology (DeviceTopology::make, topology.cpp:44-113) ----
  if (p.n_devices < 1 || p.devices == nullptr)
    throw InputError("topology must list at least one device");
  if (p.n_devices > kMaxDevices)
    throw InputError("engine limit: at most 256 devices per topology");
  if (p.intra_region_latency_ms < 0 || p.intra_region_bandwidth_gbps <= 0)
    throw InputError(
        "intra-region defaults must be non-negative latency and positive bandwidth");
  P.def_lat_ms = p.intra_region_latency_ms;
  P.def_bw_gbps = p.intra_region_bandwidth_gbps;
  const int N = p.n_devices;
  P.N = N;
  std::map<std::string, int> index;
  std::map<std::string, int> node_sizes;
  for (int i = 0; i < N; ++i) {
    const hpg_device& d = p.devices[i];
    const std::string id = str_or_empty(d.id);
    if (id.empty()) throw InputError("device id must be non-empty");
    if (d.comp_tflops <= 0 || d.mem_gb <= 0 || d.hbm_gbps <= 0 || d.intra_node_gbps <= 0)
      throw InputError("device '" + id + "' has a non-positive attribute (comp/mem/hbm/intra)");
    const std::string node = str_or_empty(d.node), region = str_or_empty(d.region);
    if (node.empty() || region.empty())
      throw InputError("device '" + id + "' needs node and region labels");
    if (!index.emplace(id, i).second) throw InputError("duplicate device id '" + id + "'");
    P.max_node_size = std::max(P.max_node_size, ++node_sizes[node]);
    P.dev_id.push_back(id);
    P.dev_node.push_back(node);
    P.dev_region.push_back(region);
    P.dev_model.push_back(str_or_empty(d.gpu_model));
    P.comp_tflops.push_back(d.comp_tflops);
    P.mem_gb.push_back(d.mem_gb);
    P.hbm_gbps.push_back(d.hbm_gbps);
    P.intra_gbps.push_back(d.intra_node_gbps);
    P.comp.push_back(d.comp_tflops * 1e12);  // kTflops
    P.mem.push_back(d.mem_gb * 1e9);         // kGigabyte
    P.hbm.push_back(d.hbm_gbps * 1e9);
  }
  auto ordered = [](const std::string& a, const std::string& b) {
    return a <= b ? std::make_pair(a, b) : std::make_pair(b, a);
  };
  std::map<std::pair<std::string, std::string>, std::pair<double, double>> region_matrix;
  for (int e = 0; e < p.n_region_links; ++e) {
    const hpg_region_link& rl = p.region_links[e];
    const std::string src = str_or_empty(rl.src), dst = str_or_empty(rl.dst);
    if (rl.latency_ms < 0 || rl.bandwidth_gbps <= 0)
      throw InputError("region link " + src + "<->" + dst +
                       " must have latency >= 0 and bandwidth > 0");
    if (!region_matrix
             .emplace(ordered(src, dst), std::make_pair(rl.latency_ms * 1e-3,
                                                        rl.bandwidth_gbps * 1.25e8))
             .second)
      throw InputError("duplicate region link " + src + "<->" + dst);
    P.rl_src.push_back(src);
    P.rl_dst.push_back(dst);
    P.rl_lat_ms.push_back(rl.latency_ms);
    P.rl_bw_gbps.push_back(rl.bandwidth_gbps);
  }
  // link classes: distinct (latency, bandwidth) bit patterns; class 0 = self
  std::map<std::pair<uint64_t, uint64_t>, int> cls_of;
  auto class_id = [&](double lat, double bw) {
    uint64_t a, b;
    std::memcpy(&a, &lat, 8);
    std::memcpy(&b, &bw, 8);
    auto it = cls_of.find({a, b});
    if (it != cls_of.end()) return it->second;
    const int id = static_cast<int>(P.lat.size());
    if (id >= kMaxClasses) throw InputError("engine limit: more than 64 distinct link classes");
    cls_of.emplace(std::make_pair(a, b), id);
    P.lat.push_back(lat);
    P.bw.push_back(bw);
    return id;
  };
  class_id(0.0, std::numeric_limits<double>::infinity());
  P.cls.assign(static_cast<size_t>(N) * N, 0);
  for (int a = 0; a < N; ++a) {
    for (int b = 0; b < N; ++b) {
      double lat, bw;
      if (a == b) {
        lat = 0.0;
        bw = std::numeric_limits<double>::infinity();
      } else if (P.dev_node[a] == P.dev_node[b] && P.dev_region[a] == P.dev_region[b]) {
        lat = 5e-6;  // kIntraNodeLatencyS
        bw = std::min(P.intra_gbps[a] * 1e9, P.intra_gbps[b] * 1e9);
      } else if (P.dev_region[a] == P.dev_region[b]) {
        lat = p.intra_region_latency_ms * 1e-3;
        bw = p.intra_region_bandwidth_gbps * 1.25e8;
      } else {
        auto it = region_matrix.find(ordered(P.dev_region[a], P.dev_region[b]));
        if (it == region_matrix.end())
          throw InputError("no link rule between regions '" + P.dev_region[a] + "' and '" +
                           P.dev_region[b] + "' (devices " + P.dev_id[a] + ", " + P.dev_id[b] +
                           ")");
        lat = it->second.first;
        bw = it->second.second;
      }
      P.cls[static_cast<size_t>(a) * N + b] = static_cast<uint8_t>(class_id(lat, bw));
    }
  }
  // lexicographic orders of the std::string keys the reference iterates
  std::vector<int> order(N);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(),
            [&](int x, int y) { return P.dev_id[x] < P.dev_id[y]; });
  P.id_rank.assign(N, 0);
  for (int r = 0; r < N; ++r) P.id_rank[order[r]] = r;
  P.by_id_rank = order;
  std::map<std::string, int> node_names;
  for (int i = 0; i < N; ++i) node_names.emplace(P.dev_node[i], 0);
  int r = 0;
  for (auto& kv : node_names) kv.second = r++;
  P.n_nodes = r;
  P.node_rank.assign(N, 0);
  for (int i = 0; i < N; ++i) P.node_rank[i] = node_names[P.dev_node[i]];
  std::map<std::string, std::map<std::string, std::vector<int>>> by_region;
  for (int i = 0; i < N; ++i) by_region[P.dev_region[i]][P.dev_node[i]].push_back(i);
  for (auto& [reg, nodes] : by_region) {
    std::vector<std::vector<int>> v;
    for (auto& [nd, devs] : nodes) v.push_back(devs);
    P.region_nodes.push_back(std::move(v));
  }
  return P;
}

DevCostConfig to_dev_cfg(const hpg_cost_config& c) {
  DevCostConfig d;
  d.recompute = c.recompute;
  d.dbs_cap = c.dbs_cap;
  d.reshard_override = c.reshard_override;
  d.sync_override = c.sync_override;
  d.dbs_override = c.dbs_override;
  d.train_bytes_per_param = c.train_bytes_per_param;
  d.infer_bytes_per_param = c.infer_bytes_per_param;
  d.kv_bytes_per_elem = c.kv_bytes_per_elem;
  d.act_factor = c.act_factor;
  return d;
}

hpg_cost_config default_cost_config() {
  hpg_cost_config c;
  c.recompute = 1;
  c.reshard_override = -1.0;
  c.sync_override = -1.0;
  c.dbs_override = -1.0;
  c.train_bytes_per_param = 18.0;
  c.infer_bytes_per_param = 2.0;
  c.kv_bytes_per_elem = 2.0;
  c.dbs_cap = 1;
  c.act_factor = 4.0;
  return c;
}

void init_cand(Cand& c, int T, const int* dp, const int* pp, const int* tp, const Problem& P) {
  RecHeader h{};
  h.n_tasks = T;
  for (int t = 0; t < T; ++t) {
    h.dp[t] = dp[t];
    h.pp[t] = pp[t];
    h.tp[t] = tp[t];
  }
  rec_offsets(h, c.o);
  h.bytes = c.o.bytes;
  c.rec.assign(c.o.bytes, 0);
  std::memcpy(c.rec.data(), &h, sizeof(h));
  double* w = c.w();
  for (int i = 0; i < c.o.w[T]; ++i) w[i] = 1.0;
  int32_t* sl = c.sl();
  for (int t = 0; t < T; ++t) {
    const int64_t nl = P.tasks[t].nl;
    for (int j = 0; j < pp[t]; ++j) {
      sl[c.o.sl[t] + j] = static_cast<int32_t>(nl / pp[t]) + (j < nl % pp[t] ? 1 : 0);
    }
  }
}

Ctx::~Ctx() {
  if (dist.comm) dist_destroy(dist);
  if (d_blob) cudaFree(d_blob);
  if (d_sweep_tables) cudaFree(d_sweep_tables);
  if (d_gen_tables) cudaFree(d_gen_tables);
  for (cudaEvent_t e : {ev0, ev1, ev2, ev3, ev_done[0], ev_done[1], ev_x[0], ev_x[1], ev_x[2], ev_x[3],
                        ev_x[4], ev_x[5]})
    if (e) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
}

Ctx* create_ctx(const hpg_problem& hp, int device) {
  Problem P = build_problem(hp);
  int n_dev = 0;
  cuda_check(cudaGetDeviceCount(&n_dev), "cudaGetDeviceCount (no CUDA device: the engine has "
                                         "no CPU fallback)");
  if (device < 0 || device >= n_dev) throw InternalError("CUDA device index out of range");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major < 10) {
    throw InternalError(std::string("engine is built for sm_100a; device is ") + prop.name);
  }
  auto* ctx = new Ctx();
  try {
    ctx->device = device;
    ctx->n_sm = prop.multiProcessorCount;
    cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreate(&ctx->ev0), "event");
    cuda_check(cudaEventCreate(&ctx->ev1), "event");
    cuda_check(cudaEventCreate(&ctx->ev2), "event");
    cuda_check(cudaEventCreate(&ctx->ev3), "event");
    cuda_check(cudaEventCreateWithFlags(&ctx->ev_done[0], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ctx->ev_done[1], cudaEventDisableTiming), "event");
    for (cudaEvent_t& e : ctx->ev_x) cuda_check(cudaEventCreate(&e), "event");
    stage_problem(*ctx, std::move(P));
    if (std::getenv("HPG_BW_TEST")) {  // diagnostics: copy bandwidth through the wave buffers
      for (const size_t mb : {1, 8, 64}) {
        const size_t n = mb << 20;
        ctx->h_recs.reserve(n);
        ctx->d_recs.reserve(n);
        std::memset(ctx->h_recs.p, 1, n);
        float ms_h = 0.f, ms_d = 0.f;
        for (int rep = 0; rep < 3; ++rep) {
          if (std::getenv("HPG_BW_DIRTY")) std::memset(ctx->h_recs.p, rep, n);  // hot, dirty lines
          cudaEventRecord(ctx->ev0, ctx->stream);
          cudaMemcpyAsync(ctx->d_recs.p, ctx->h_recs.p, n, cudaMemcpyHostToDevice, ctx->stream);
          cudaEventRecord(ctx->ev1, ctx->stream);
          cudaMemcpyAsync(ctx->h_recs.p, ctx->d_recs.p, n, cudaMemcpyDeviceToHost, ctx->stream);
          cudaEventRecord(ctx->ev2, ctx->stream);
          cudaStreamSynchronize(ctx->stream);
          cudaEventElapsedTime(&ms_h, ctx->ev0, ctx->ev1);
          cudaEventElapsedTime(&ms_d, ctx->ev1, ctx->ev2);
        }
        unsigned int flags = 0;
        cudaHostGetFlags(&flags, ctx->h_recs.p);
        std::fprintf(stderr, "hpg bw %zu MB: H2D %.1f GB/s D2H %.1f GB/s (host flags %u)\n", mb,
                     n / ms_h / 1e6, n / ms_d / 1e6, flags);
      }
    }
  } catch (...) {
    delete ctx;
    throw;
  }
  return ctx;
}

void restage(Ctx& ctx, const hpg_problem& hp) {
  Problem P = build_problem(hp);
  cuda_check(cudaSetDevice(ctx.device), "cudaSetDevice");
  stage_problem(ctx, std::move(P));
}

// Uploads the flattened problem (device attributes, link classes) and fills
// the by-value kernel header. Validation already happened in build_problem.
void stage_problem(Ctx& ctxr, Problem&& P) {
  Ctx* ctx = &ctxr;
  {
    // sweep / generator tables belong to the previous problem
    if (ctx->d_sweep_tables) {
      cudaFree(ctx->d_sweep_tables);
      ctx->d_sweep_tables = nullptr;
    }
    if (ctx->d_gen_tables) {
      cudaFree(ctx->d_gen_tables);
      ctx->d_gen_tables = nullptr;
    }
    ctx->prob = std::move(P);
    const Problem& Q = ctx->prob;
    const int N = Q.N, C = static_cast<int>(Q.lat.size());
    const size_t bytes = 8 * (3 * N + 2 * C) + static_cast<size_t>(N) * N;
    ctx->h_blob.reserve(bytes);
    double* dd = reinterpret_cast<double*>(ctx->h_blob.p);
    std::memcpy(dd, Q.comp.data(), 8 * N);
    std::memcpy(dd + N, Q.mem.data(), 8 * N);
    std::memcpy(dd + 2 * N, Q.hbm.data(), 8 * N);
    std::memcpy(dd + 3 * N, Q.lat.data(), 8 * C);
    std::memcpy(dd + 3 * N + C, Q.bw.data(), 8 * C);
    std::memcpy(ctx->h_blob.p + 8 * (3 * N + 2 * C), Q.cls.data(), static_cast<size_t>(N) * N);
    if (bytes > ctx->blob_bytes) {
      if (ctx->d_blob) cudaFree(ctx->d_blob);
      ctx->d_blob = nullptr;
      cuda_check(cudaMalloc(&ctx->d_blob, bytes), "cudaMalloc problem");
      ctx->blob_bytes = bytes;
    }
    cuda_check(cudaMemcpyAsync(ctx->d_blob, ctx->h_blob.p, bytes, cudaMemcpyHostToDevice,
                               ctx->stream), "H2D problem");
    cuda_check(cudaStreamSynchronize(ctx->stream), "H2D problem");
    ctx->h2d_bytes += static_cast<int64_t>(bytes);
    ctx->max_nl = 1;
    DevProblem& D = ctx->dprob;
    const double* db = reinterpret_cast<const double*>(ctx->d_blob);
    D.n_dev = N;
    D.n_tasks = Q.T;
    D.n_classes = C;
    D.mode = Q.mode;
    D.algorithm = Q.algorithm;
    D.gen_slot = Q.slot_of_id[1];
    D.train6_slot = Q.slot_of_id[6];
    D.max_tp = Q.max_node_size;
    D.eta = Q.eta;
    D.global_batch = Q.global_batch;
    D.rpp = Q.rpp;
    D.seq_in = Q.seq_in;
    D.seq_out = Q.seq_out;
    D.mbs = Q.mbs;
    D.total_seq = Q.global_batch * Q.rpp;
    for (const HostTask& h : Q.tasks) ctx->max_nl = std::max(ctx->max_nl, h.nl);
    for (int t = 0; t < Q.T; ++t) {
      const HostTask& h = Q.tasks[t];
      DevTask& d = D.task[t];
      d.id = h.id;
      d.kind = h.kind;
      d.precision_bytes = h.prec;
      d.include_embedding = h.emb ? 1 : 0;
      d.h1 = h.h1;
      d.h2 = h.h2;
      d.nl = h.nl;
      d.vocab = h.vocab;
      d.layer_params = h.layer_params;
      d.param_count = h.param_count;
    }
    D.comp = db;
    D.mem = db + N;
    D.hbm = db + 2 * N;
    D.lat = db + 3 * N;
    D.bw = db + 3 * N + C;
    D.cls = reinterpret_cast<const uint8_t*>(ctx->d_blob) + 8 * (3 * N + 2 * C);
    // device-wide ring memo: 2^20 slots (48 MiB), cleared per problem.
    // HPG_RING_CACHE=0 disables it (A/B measurements).
    const char* rc = std::getenv("HPG_RING_CACHE");
    const bool use_rc = !(rc && rc[0] == '0');
    constexpr size_t kSlots = size_t(1) << 20;
    D.ring_cache = nullptr;
    D.ring_mask = kSlots - 1;
    D.ring_arena = nullptr;
    D.ring_arena_cap = 0;
    if (use_rc) {
      // slots, then the sequence arena (64 MiB; its first word counts the
      // bytes handed out, starting after itself)
      constexpr size_t kArena = size_t(64) << 20;
      const size_t slot_bytes = kSlots * sizeof(RingSlot);
      ctx->d_ring.reserve(slot_bytes + kArena);
      cuda_check(cudaMemsetAsync(ctx->d_ring.p, 0, slot_bytes, ctx->stream), "ring cache clear");
      const unsigned long long start = 16;
      cuda_check(cudaMemcpyAsync(ctx->d_ring.p + slot_bytes, &start, 8, cudaMemcpyHostToDevice,
                                 ctx->stream), "ring arena reset");
      cuda_check(cudaStreamSynchronize(ctx->stream), "ring cache clear");
      D.ring_cache = reinterpret_cast<RingSlot*>(ctx->d_ring.p);
      D.ring_arena = ctx->d_ring.p + slot_bytes;
      D.ring_arena_cap = kArena;
    }
  }
}

// Empties the device-wide ring memo and its sequence arena (on the context's
// stream): every search starts cold, so no ring value is carried from one
// search to the next (the memo is a within-search cache).
void reset_ring_memo(Ctx& ctx) {
  const DevProblem& D = ctx.dprob;
  if (!D.ring_cache) return;
  cuda_check(cudaMemsetAsync(D.ring_cache, 0, (D.ring_mask + 1) * sizeof(RingSlot), ctx.stream),
             "ring memo reset");
  static const unsigned long long start = 16;
  cuda_check(cudaMemcpyAsync(D.ring_arena, &start, 8, cudaMemcpyHostToDevice, ctx.stream),
             "ring arena reset");
}

namespace {

// What balancing can change: the generation task's replica weights
// (balance_data) and every task's stage split (balance_layers); the other
// weights stay 1.0 and devices never move. A wave returns [gen weights |
// stage layers] per plan, 8-aligned.
inline int64_t ws_bytes_of(const Problem& P, const Cand& c) {
  const int g = P.slot_of_id[1];
  const int64_t wg = g >= 0 ? 8 * static_cast<int64_t>(c.hdr().dp[g]) : 0;
  return (wg + 4 * static_cast<int64_t>(c.o.sl[P.T]) + 7) & ~int64_t(7);
}

// Copy into pinned staging with non-temporal stores: the H2D DMA then reads
// DRAM instead of snooping lines left dirty in 16 cores' private caches
// (measured: 5 GB/s with dirty lines vs 50+ GB/s).
inline void nt_copy(uint8_t* dst, const uint8_t* src, size_t n) {
  while (n && (reinterpret_cast<uintptr_t>(dst) & 15)) {
    *dst++ = *src++;
    --n;
  }
  for (; n >= 16; n -= 16, dst += 16, src += 16)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst),
                     _mm_loadu_si128(reinterpret_cast<const __m128i*>(src)));
  while (n--) *dst++ = *src++;
}

// one wave = one eval_kernel launch; staged (packed + enqueued) and finished
// (synchronised + unpacked) separately so consecutive chunks of a very large
// wave overlap host packing with the device work of the previous chunk
struct WaveBufs {
  HostBuf<uint8_t>* h_in;
  DevBuf<uint8_t>* d_in;
  DevBuf<uint8_t>* d_out;
  HostBuf<uint8_t>* h_out;
  cudaEvent_t e0, e1, done, eh, ed, ex;
};

struct WaveJob {
  int n = 0;
  int64_t in_bytes = 0, out_bytes = 0, ws_total = 0;
  long long* d_prof = nullptr;
  WaveBufs buf{};
  std::chrono::steady_clock::time_point t0, t1, t2;
};

WaveBufs wave_bufs(Ctx& ctx, int set) {
  if (set == 0)
    return {&ctx.h_recs, &ctx.d_recs, &ctx.d_out, &ctx.h_out, ctx.ev0, ctx.ev1, ctx.ev_done[0],
            ctx.ev_x[0], ctx.ev_x[1], ctx.ev_x[4]};
  return {&ctx.h_recs2, &ctx.d_recs2, &ctx.d_out2, &ctx.h_out2, ctx.ev2, ctx.ev3, ctx.ev_done[1],
          ctx.ev_x[2], ctx.ev_x[3], ctx.ev_x[5]};
}

void wave_stage(Ctx& ctx, const Batch& b, const DevCostConfig& cfg, int kb_flags, bool want_out,
                bool want_per_task, bool want_required, const WaveBufs& buf, BatchOut& out,
                WaveJob& job) {
  const int n = static_cast<int>(b.cands.size());
  job = WaveJob{};
  job.n = n;
  job.buf = buf;
  out.res.resize(n);
  out.off.resize(n);
  out.ws_off.resize(n);
  if (n == 0) return;
  job.t0 = std::chrono::steady_clock::now();
  const Problem& P = ctx.prob;
  Carve cv{};
  cv.n_dev = P.N;
  cv.n_tasks = P.T;
  int64_t total = 0, ws_total = 0;
  for (int i = 0; i < n; ++i) {
    const Cand& c = *b.cands[i];
    out.off[i] = total;
    total += c.o.bytes;
    out.ws_off[i] = ws_total;
    ws_total += ws_bytes_of(P, c);
    const int T = P.T;
    cv.max_w = std::max(cv.max_w, c.o.w[T]);
    cv.max_sl = std::max(cv.max_sl, c.o.sl[T]);
    cv.max_slots = std::max(cv.max_slots, c.o.dev[T]);
    cv.max_cells = std::max(cv.max_cells, c.o.cell[T]);
    cv.max_dpk = std::max(cv.max_dpk, c.o.dpk[T]);
  }
  job.ws_total = ws_total;
  // device-generated candidates: compact offsets of their device slots
  const int n_items = static_cast<int>(b.gen.size());
  const int64_t n_gen = b.n_gen;
  out.gen_dev_off.assign(n_gen, 0);
  int64_t dev_total = 0;
  for (const GenItem& it : b.gen)
    for (int c = 0; c < it.count; ++c) {
      out.gen_dev_off[it.first_out + c] = dev_total;
      dev_total += b.cands[it.first + c]->o.dev[P.T];
    }
  // one input transfer: [offsets i64 | out offsets i64 | modes i32 (8-aligned) |
  // generator: items | item per candidate i32 | start states | slot offsets i64 |
  // records]
  const int64_t nn = static_cast<int64_t>(n);
  auto al8 = [](int64_t x) { return (x + 7) & ~int64_t(7); };
  const int64_t in_off = 0, in_ooff = 8 * nn, in_modes = 16 * nn,
                in_items = in_modes + al8(4 * nn),
                in_citem = in_items + al8(static_cast<int64_t>(sizeof(GenItem)) * n_items),
                in_starts = in_citem + al8(4 * n_gen),
                in_goff = in_starts + static_cast<int64_t>(sizeof(Rng)) * n_gen,
                in_recs = in_goff + 8 * n_gen;
  const int64_t in_bytes = in_recs + total;
  job.in_bytes = in_bytes;
  buf.h_in->reserve(in_bytes);
  int64_t* h_off = reinterpret_cast<int64_t*>(buf.h_in->p + in_off);
  int64_t* h_ooff = reinterpret_cast<int64_t*>(buf.h_in->p + in_ooff);
  int32_t* h_modes = reinterpret_cast<int32_t*>(buf.h_in->p + in_modes);
  uint8_t* h_rec = buf.h_in->p + in_recs;
  if (n_items) {
    std::memcpy(buf.h_in->p + in_items, b.gen.data(), sizeof(GenItem) * n_items);
    std::memcpy(buf.h_in->p + in_citem, b.gen_item.data(), 4 * n_gen);
    std::memcpy(buf.h_in->p + in_starts, b.gen_starts.data(), sizeof(Rng) * n_gen);
    std::memcpy(buf.h_in->p + in_goff, out.gen_dev_off.data(), 8 * n_gen);
  }
  // canonical bytes: tg id + k counts + per task
  // (3 + pp + slots) + 9 result bytes (+ 8*dp for a weighted generation task)
  auto canonical = [&](const Cand& c) {
    int64_t cb = 1 + c.ng + 9;
    for (int t = 0; t < P.T; ++t) cb += 3 + c.hdr().pp[t] + c.size(t);
    const int g = P.slot_of_id[1];
    if (g >= 0) {
      const double* w = c.w() + c.o.w[g];
      for (int k = 0; k < c.hdr().dp[g]; ++k)
        if (w[k] != 1.0) {
          cb += 8 * c.hdr().dp[g];
          break;
        }
    }
    return cb;
  };
  const int n_chunks = n >= 256 ? 16 : 1;
  int64_t cb_part[16] = {};
  host_parallel_for(n_chunks, n_chunks > 1, [&](int ch) {
    const int i0 = static_cast<int>(static_cast<int64_t>(n) * ch / n_chunks);
    const int i1 = static_cast<int>(static_cast<int64_t>(n) * (ch + 1) / n_chunks);
    int64_t cb = 0;
    for (int i = i0; i < i1; ++i) {
      const Cand& c = *b.cands[i];
      nt_copy(h_rec + out.off[i], c.rec.data(), c.o.bytes);
      h_off[i] = out.off[i];
      h_ooff[i] = out.ws_off[i];
      h_modes[i] = b.modes[i];
      cb += canonical(c);
    }
    _mm_sfence();
    cb_part[ch] = cb;
  });
  for (int ch = 0; ch < n_chunks; ++ch) ctx.canonical_bytes += cb_part[ch];
  // one output transfer: [results 32 B each | balanced weight / split sections |
  // generated device slots]
  const int64_t out_res = 0, out_ws = 32 * nn;
  const int64_t out_gdev = out_ws + (want_out ? ws_total : 0);
  const int64_t out_bytes = out_gdev + ((dev_total + 7) & ~int64_t(7));
  job.out_bytes = out_bytes;
  buf.d_in->reserve(in_bytes);
  buf.d_out->reserve(out_bytes);
  if (want_per_task) ctx.d_per_task.reserve(static_cast<size_t>(n) * P.T * 7);
  if (want_required) ctx.d_required.reserve(static_cast<size_t>(n) * P.N);
  cudaStream_t st = ctx.stream;
  job.t1 = std::chrono::steady_clock::now();
  static const bool batch_log = std::getenv("HPG_BATCH_LOG") != nullptr;  // diagnostics only
  if (batch_log) cuda_check(cudaEventRecord(buf.eh, st), "event");
  cuda_check(cudaMemcpyAsync(buf.d_in->p, buf.h_in->p, in_bytes, cudaMemcpyHostToDevice, st),
             "H2D wave");
  if (batch_log) cuda_check(cudaEventRecord(buf.ex, st), "event");
  const int64_t* d_off = reinterpret_cast<const int64_t*>(buf.d_in->p + in_off);
  const int64_t* d_ooff = reinterpret_cast<const int64_t*>(buf.d_in->p + in_ooff);
  const int32_t* d_modes = reinterpret_cast<const int32_t*>(buf.d_in->p + in_modes);
  const uint8_t* d_rec = buf.d_in->p + in_recs;
  EvalResult* d_res = reinterpret_cast<EvalResult*>(buf.d_out->p + out_res);
  uint8_t* d_ows = want_out ? buf.d_out->p + out_ws : nullptr;
  if (n_items) {
    cuda_check(launch_gen_ga(gen_tables(ctx), reinterpret_cast<const GenItem*>(buf.d_in->p + in_items),
                             reinterpret_cast<const int32_t*>(buf.d_in->p + in_citem),
                             reinterpret_cast<const Rng*>(buf.d_in->p + in_starts),
                             static_cast<int>(n_gen), buf.d_in->p + in_recs, d_off,
                             reinterpret_cast<const int64_t*>(buf.d_in->p + in_goff),
                             buf.d_out->p + out_gdev, st),
               "gen_ga_kernel");
    ++ctx.launches;
  }
  // small waves are latency-bound on cold SMs: stage the class matrix in smem
  cv.cls_smem = (n <= 2 * ctx.n_sm && P.N * P.N <= kClsSmemMax) ? 1 : 0;
  // ... and get helper warps for the per-task costs of each plan
  static const int team_policy = [] {
    const char* v = std::getenv("HPG_TEAM_POLICY");  // diagnostics: 0 off, 1 small only
    return v ? std::atoi(v) : 2;
  }();
  // the largest team with which the whole wave is resident in one round
  cv.n_warps = 1;
  if (P.T >= 2 && team_policy >= 1) {
    for (const int w : {std::min(kMaxTeamWarps, P.T), 2}) {
      if (w == 2 && team_policy < 2) continue;
      Carve ct = cv;
      ct.n_warps = w;
      int g = 0;
      const cudaError_t e = eval_grid(ct, n, ctx.n_sm, g);  // too much smem: no team
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        continue;
      }
      if (g >= n) {
        cv.n_warps = w;
        break;
      }
    }
  }
  int grid = 0;
  {
    const cudaError_t e = eval_grid(cv, n, ctx.n_sm, grid);
    if (e != cudaSuccess)
      throw InternalError(std::string("eval_kernel occupancy (") + std::to_string(carve2_bytes(cv)) +
                          " B smem, " + std::to_string(cv.n_warps) + " warps, " +
                          std::to_string(n) + " plans): " + cudaGetErrorString(e));
  }
  const int64_t scratch = eval_scratch_doubles(P.N, ctx.max_nl);
  // sized once for the largest possible persistent grid (32 CTAs per SM)
  ctx.d_scratch.reserve(static_cast<size_t>(std::max(grid, 32 * ctx.n_sm)) * scratch);
  static const char* plan_prof_log = std::getenv("HPG_PLAN_PROFILE");  // diagnostics only
  if (plan_prof_log) {
    cuda_check(cudaMalloc(&job.d_prof, sizeof(long long) * kPlanProfSlots * n), "profile alloc");
    cuda_check(cudaMemsetAsync(job.d_prof, 0, sizeof(long long) * kPlanProfSlots * n, st),
               "profile clear");
    cuda_check(eval_set_plan_profile(job.d_prof), "profile symbol");
  }
  cuda_check(cudaEventRecord(buf.e0, st), "event");
  cuda_check(launch_eval(ctx.dprob, cfg, cv, kb_flags, d_rec, d_off, d_modes, 0, n, 0, d_ows,
                         d_ooff, d_res, want_per_task ? ctx.d_per_task.p : nullptr,
                         want_required ? ctx.d_required.p : nullptr, ctx.d_scratch.p, scratch,
                         grid, st),
             "eval_kernel launch");
  cuda_check(cudaEventRecord(buf.e1, st), "event");
  ++ctx.launches;
  ++ctx.eval_launches;
  ctx.plans_evaluated += n;
  ctx.h2d_bytes += in_bytes;
  ctx.d2h_bytes += out_bytes + (want_per_task ? 8 * static_cast<int64_t>(n) * P.T * 7 : 0) +
                   (want_required ? 8 * static_cast<int64_t>(n) * P.N : 0);
  buf.h_out->reserve(out_bytes);
  cuda_check(cudaMemcpyAsync(buf.h_out->p, buf.d_out->p, out_bytes, cudaMemcpyDeviceToHost, st),
             "D2H wave");
  out.out_ws = want_out ? buf.h_out->p + out_ws : nullptr;
  out.ws_bytes = want_out ? ws_total : 0;
  out.gen_devs = n_gen ? buf.h_out->p + out_gdev : nullptr;
  if (want_per_task) out.per_task.resize(static_cast<size_t>(n) * P.T * 7);
  if (want_required) out.required.resize(static_cast<size_t>(n) * P.N);
  if (want_per_task)
    cuda_check(cudaMemcpyAsync(out.per_task.data(), ctx.d_per_task.p, 8 * out.per_task.size(),
                               cudaMemcpyDeviceToHost, st), "D2H per-task");
  if (want_required)
    cuda_check(cudaMemcpyAsync(out.required.data(), ctx.d_required.p, 8 * out.required.size(),
                               cudaMemcpyDeviceToHost, st), "D2H required");
  if (batch_log) cuda_check(cudaEventRecord(buf.ed, st), "event");
  cuda_check(cudaEventRecord(buf.done, st), "event");
  job.t2 = std::chrono::steady_clock::now();
}

void wave_finish(Ctx& ctx, const Batch& b, WaveJob& job, BatchOut& out) {
  const int n = job.n;
  if (n == 0) return;
  const Problem& P = ctx.prob;
  cuda_check(cudaEventSynchronize(job.buf.done), "eval_kernel");
  const auto t3 = std::chrono::steady_clock::now();
  float ms = 0.f;
  cuda_check(cudaEventElapsedTime(&ms, job.buf.e0, job.buf.e1), "event time");
  ctx.eval_ms += ms;
  static const char* wave_log = std::getenv("HPG_WAVE_LOG");  // diagnostics only
  if (wave_log) {
    if (FILE* f = std::fopen(wave_log, "a")) {
      int nev = 0;
      for (int i = 0; i < n; ++i) nev += b.modes[i] == kModeEvaluate;
      std::fprintf(f, "%d %d %.4f\n", n, nev, ms);
      std::fclose(f);
    }
  }
  if (job.d_prof) {
    static const char* plan_prof_log = std::getenv("HPG_PLAN_PROFILE");
    std::vector<long long> pr(static_cast<size_t>(kPlanProfSlots) * n);
    cuda_check(cudaMemcpy(pr.data(), job.d_prof, sizeof(long long) * kPlanProfSlots * n,
                          cudaMemcpyDeviceToHost),
               "profile D2H");
    cuda_check(eval_set_plan_profile(nullptr), "profile symbol");
    cudaFree(job.d_prof);
    job.d_prof = nullptr;
    static int wave_no = 0;
    if (FILE* f = std::fopen(plan_prof_log, "a")) {
      // wave n ms | per plan: mode stage bal_data bal_layers e2e | dp,pp,tp per task
      for (int i = 0; i < n; ++i) {
        const long long* q = &pr[kPlanProfSlots * static_cast<size_t>(i)];
        const long long t1 = q[1] ? q[1] : q[0], t2 = q[2] ? q[2] : t1, t3_ = q[3] ? q[3] : t2;
        std::fprintf(f, "%d %d %.4f %d %lld %lld %lld %lld", wave_no, n, ms, b.modes[i], t1 - q[0],
                     t2 - t1, t3_ - t2, q[4] - t3_);
        const RecHeader& h = b.cands[i]->hdr();
        for (int t = 0; t < P.T; ++t) std::fprintf(f, " %d,%d,%d", h.dp[t], h.pp[t], h.tp[t]);
        std::fprintf(f, " |");
        for (int k = 5; k < kPlanProfSlots; ++k) std::fprintf(f, " %lld", q[k]);
        std::fputc('\n', f);
      }
      std::fclose(f);
    }
    unsigned long long acc[32];
    cuda_check(eval_phase_acc(acc), "phase acc");
    const std::string acc_path = std::string(plan_prof_log) + ".phases";
    if (FILE* f = std::fopen(acc_path.c_str(), "w")) {
      for (int k = 0; k < 32; ++k) std::fprintf(f, "%d %llu\n", k, acc[k]);
      std::fclose(f);
    }
    ++wave_no;
  }
  std::memcpy(out.res.data(), job.buf.h_out->p, sizeof(EvalResult) * n);
  static const char* batch_log = std::getenv("HPG_BATCH_LOG");  // diagnostics only
  if (batch_log) {
    const auto t4 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b_) {
      return std::chrono::duration<double, std::micro>(b_ - a).count();
    };
    float h2d = 0.f, d2h = 0.f, gap = 0.f;
    cudaEventElapsedTime(&h2d, job.buf.eh, job.buf.ex);
    cudaEventElapsedTime(&gap, job.buf.ex, job.buf.e0);
    cudaEventElapsedTime(&d2h, job.buf.e1, job.buf.ed);
    if (FILE* f = std::fopen(batch_log, "a")) {
      // n in_bytes out_bytes pack_us enqueue_us sync_us post_us kernel_ms h2d_ms d2h_ms
      std::fprintf(f, "%d %lld %lld %.1f %.1f %.1f %.1f %.4f %.4f %.4f %.4f\n", n,
                   static_cast<long long>(job.in_bytes), static_cast<long long>(job.out_bytes),
                   us(job.t0, job.t1), us(job.t1, job.t2), us(job.t2, t3), us(t3, t4), ms, h2d,
                   d2h, gap);
      std::fclose(f);
    }
  }
}

}  // namespace

// Very large waves (the first SHA rounds of a 10^5-10^6 budget on 10^4 arms)
// run as consecutive launches of at most kMaxWavePlans plans, double-buffered:
// chunk k is packed and enqueued while the device works on chunk k-1, and
// pinned staging stays bounded instead of growing to gigabytes.
void run_batch(Ctx& ctx, const Batch& b, const DevCostConfig& cfg, int kb_flags, bool want_out,
               bool want_per_task, bool want_required, BatchOut& out) {
  constexpr int kMaxWavePlans = 32768;
  const int n = static_cast<int>(b.cands.size());
  if (n <= kMaxWavePlans || want_per_task || want_required) {
    WaveJob job;
    wave_stage(ctx, b, cfg, kb_flags, want_out, want_per_task, want_required, wave_bufs(ctx, 0),
               out, job);
    wave_finish(ctx, b, job, out);
    return;
  }
  out.res.clear();
  out.off.clear();
  out.ws_off.clear();
  out.per_task.clear();
  out.required.clear();
  out.ws_store.clear();
  Batch sub[2];
  BatchOut part[2];
  WaveJob job[2];
  auto collect = [&](int set) {
    wave_finish(ctx, sub[set], job[set], part[set]);
    const BatchOut& p = part[set];
    out.res.insert(out.res.end(), p.res.begin(), p.res.end());
    const int64_t base = static_cast<int64_t>(out.ws_store.size());
    for (int64_t o : p.ws_off) out.ws_off.push_back(base + o);
    for (int64_t o : p.off) out.off.push_back(o);
    if (want_out) out.ws_store.insert(out.ws_store.end(), p.out_ws, p.out_ws + p.ws_bytes);
  };
  int k = 0;
  for (int i0 = 0; i0 < n; i0 += kMaxWavePlans, ++k) {
    const int i1 = std::min(n, i0 + kMaxWavePlans);
    const int set = k & 1;
    sub[set].cands.assign(b.cands.begin() + i0, b.cands.begin() + i1);
    sub[set].modes.assign(b.modes.begin() + i0, b.modes.begin() + i1);
    wave_stage(ctx, sub[set], cfg, kb_flags, want_out, false, false, wave_bufs(ctx, set),
               part[set], job[set]);
    if (k >= 1) collect(set ^ 1);
  }
  collect((k - 1) & 1);
  out.out_ws = want_out ? out.ws_store.data() : nullptr;
  out.ws_bytes = static_cast<int64_t>(out.ws_store.size());
}

const GenTablesDev& gen_tables(Ctx& ctx) {
  if (ctx.d_gen_tables) return ctx.gen_tb;
  const Problem& P = ctx.prob;
  std::vector<int32_t> region_off{0}, node_off{0};
  std::vector<uint8_t> node_devs;
  for (const auto& nodes : P.region_nodes) {
    for (const auto& devs : nodes) {
      for (int d : devs) node_devs.push_back(static_cast<uint8_t>(d));
      node_off.push_back(static_cast<int32_t>(node_devs.size()));
    }
    region_off.push_back(static_cast<int32_t>(node_off.size() - 1));
  }
  std::vector<int16_t> node_rank(P.N);
  for (int i = 0; i < P.N; ++i) node_rank[i] = static_cast<int16_t>(P.node_rank[i]);
  std::vector<uint64_t> fm(2 * (kGenFastModMax + 1), 0);
  for (int d = 1; d <= kGenFastModMax; ++d) {
    const unsigned __int128 m = ~static_cast<unsigned __int128>(0) / d + 1;
    fm[2 * d] = static_cast<uint64_t>(m);
    fm[2 * d + 1] = static_cast<uint64_t>(m >> 64);
  }
  auto round16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  const size_t b_fm = round16(8 * fm.size()), b_ro = round16(4 * region_off.size()),
               b_no = round16(4 * node_off.size()), b_nr = round16(2 * node_rank.size()),
               b_nd = round16(node_devs.size() + 1);
  std::vector<uint8_t> blob(b_fm + b_ro + b_no + b_nr + b_nd, 0);
  size_t at = 0;
  std::memcpy(blob.data() + at, fm.data(), 8 * fm.size());
  const size_t o_ro = (at += b_fm);
  std::memcpy(blob.data() + at, region_off.data(), 4 * region_off.size());
  const size_t o_no = (at += b_ro);
  std::memcpy(blob.data() + at, node_off.data(), 4 * node_off.size());
  const size_t o_nr = (at += b_no);
  std::memcpy(blob.data() + at, node_rank.data(), 2 * node_rank.size());
  const size_t o_nd = (at += b_nr);
  std::memcpy(blob.data() + at, node_devs.data(), node_devs.size());
  cuda_check(cudaMalloc(&ctx.d_gen_tables, blob.size()), "cudaMalloc generator tables");
  cuda_check(cudaMemcpy(ctx.d_gen_tables, blob.data(), blob.size(), cudaMemcpyHostToDevice),
             "H2D generator tables");
  const uint8_t* b = static_cast<const uint8_t*>(ctx.d_gen_tables);
  GenTablesDev& t = ctx.gen_tb;
  t.n_dev = P.N;
  t.n_regions = static_cast<int32_t>(P.region_nodes.size());
  t.n_nodes = P.n_nodes;
  t.max_nodes_per_region = 0;
  for (const auto& rn : P.region_nodes)
    t.max_nodes_per_region = std::max(t.max_nodes_per_region, static_cast<int32_t>(rn.size()));
  // int16 regions / nodes / 4 x node-rank arrays, then u8 flat + bucket
  t.smem_per_thread = static_cast<int32_t>(
      (2 * (t.n_regions + t.max_nodes_per_region + 4 * t.n_nodes) + 2 * P.N + 15) & ~15);
  t.fastmod = reinterpret_cast<const uint64_t*>(b);
  t.region_off = reinterpret_cast<const int32_t*>(b + o_ro);
  t.node_off = reinterpret_cast<const int32_t*>(b + o_no);
  t.node_rank = reinterpret_cast<const int16_t*>(b + o_nr);
  t.node_devs = b + o_nd;
  return t;
}

void apply_ws(const Problem& P, Cand& c, const uint8_t* ws) {
  const int g = P.slot_of_id[1];
  int64_t at = 0;
  if (g >= 0) {
    const int64_t wg = 8 * static_cast<int64_t>(c.hdr().dp[g]);
    std::memcpy(c.w() + c.o.w[g], ws, wg);
    at = wg;
  }
  std::memcpy(c.sl(), ws + at, 4 * static_cast<size_t>(c.o.sl[P.T]));
}

std::vector<TablePlan> unpack_table(const Problem& P, const hpg_plan_table& t) {
  std::vector<TablePlan> out;
  if (t.n_plans < 0) throw UsageError("negative plan count");
  const int T = P.T, N = P.N;
  out.resize(t.n_plans);
  for (int p = 0; p < t.n_plans; ++p) {
    TablePlan& tp = out[p];
    const int ng = t.n_groups[p];
    if (ng < 1) throw InputError("task grouping must contain at least one group");
    if (ng > T) throw InputError("task groups must be non-empty");
    tp.groups.assign(ng, {});
    for (int s = 0; s < T; ++s) {
      const int g = t.task_group[static_cast<int64_t>(p) * T + s];
      if (g < 0 || g >= ng) throw InputError("task grouping must cover every workflow task");
      tp.groups[g].push_back(s);
    }
    for (const auto& g : tp.groups)
      if (g.empty()) throw InputError("task groups must be non-empty");
    int64_t count_sum = 0;
    for (int g = 0; g < ng; ++g) {
      const int c = t.gpu_counts[static_cast<int64_t>(p) * T + g];
      if (c < 1) throw InputError("gpu_counts entries must be >= 1");
      tp.counts.push_back(c);
      count_sum += c;
    }
    if (count_sum != N)
      throw InputError("gpu_counts must sum to the device count (" + std::to_string(N) + ")");
    int dp[kMaxTasks], pp[kMaxTasks], tpp[kMaxTasks];
    for (int s = 0; s < T; ++s) {
      dp[s] = t.dp[static_cast<int64_t>(p) * T + s];
      pp[s] = t.pp[static_cast<int64_t>(p) * T + s];
      tpp[s] = t.tp[static_cast<int64_t>(p) * T + s];
      if (dp[s] < 1 || pp[s] < 1 || tpp[s] < 1) throw InputError("dp, pp and tp must be >= 1");
    }
    init_cand(tp.cand, T, dp, pp, tpp, P);
    Cand& c = tp.cand;
    c.ng = ng;
    std::vector<std::vector<int>> group_sets(ng);
    std::vector<bool> group_set_init(ng, false);
    for (int g = 0; g < ng; ++g) {
      for (int s : tp.groups[g]) {
        const HostTask& task = P.tasks[s];
        const std::string tid = std::to_string(task.id);
        // ParallelLayout::validate (plan.cpp:54-87)
        if (pp[s] > task.nl) throw InputError("pp exceeds layer count");
        const int64_t so = t.sl_off[static_cast<int64_t>(p) * T + s];
        int64_t total = 0;
        for (int j = 0; j < pp[s]; ++j) {
          const int v = t.stage_layers[so + j];
          if (v < 1) throw InputError("every pipeline stage needs at least one layer");
          total += v;
          c.sl()[c.o.sl[s] + j] = v;
        }
        if (total != task.nl) throw InputError("stage_layers must sum to the model layer count");
        const int64_t wo = t.w_off[static_cast<int64_t>(p) * T + s];
        double wsum = 0;
        for (int i = 0; i < dp[s]; ++i) {
          const double w = t.weights[wo + i];
          if (!(w > 0)) throw InputError("replica batch weights must be positive");
          wsum += w;
          c.w()[c.o.w[s] + i] = w;
        }
        if (std::abs(wsum - dp[s]) > 1e-6 * dp[s])
          throw InputError("replica batch weights must sum to dp");
        const int size = dp[s] * pp[s] * tpp[s];
        if (size != tp.counts[g])
          throw InputError("task " + tid + ": dp*pp*tp must equal its group's GPU count");
        const int64_t dof = t.dev_off[static_cast<int64_t>(p) * T + s];
        std::vector<int> used;
        for (int e = 0; e < size; ++e) {
          const int d = t.devices[dof + e];
          if (d < 0 || d >= N) throw InputError("unknown device index " + std::to_string(d));
          if (std::find(used.begin(), used.end(), d) != used.end())
            throw InputError("task " + tid + ": device '" + P.dev_id[d] +
                             "' hosts more than one tasklet");
          used.push_back(d);
          c.dev()[c.o.dev[s] + e] = static_cast<uint8_t>(d);
        }
        std::sort(used.begin(), used.end());
        if (!group_set_init[g]) {
          group_sets[g] = used;
          group_set_init[g] = true;
        } else if (group_sets[g] != used) {
          throw InputError("co-located tasks in group " + std::to_string(g) +
                           " must share the same device set");
        }
      }
    }
    std::vector<int> seen(N, 0);
    for (int g = 0; g < ng; ++g) {
      for (int d : group_sets[g]) {
        if (seen[d]++) throw InputError("device '" + P.dev_id[d] + "' appears in more than one GPU group");
      }
    }
  }
  return out;
}

}  // namespace hpg
