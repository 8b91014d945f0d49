// C ABI of the sharded search's per-round exchange over a caller-supplied
// all-gather (include/hpg.h hpg_dist_exchange): the same deal_runs +
// exchange_round that hpg_search_dist runs over NCCL (dist_exchange.cpp).
// Host-only: launchers (and the CPU test suite, over torch.distributed/gloo)
// drive it without a GPU.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hpg.h"
#include "dist_exchange.hpp"

namespace {

class CallbackTransport : public hpg::Transport {
 public:
  CallbackTransport(int rank, int world, hpg_allgather_fn fn, void* user)
      : rank_(rank), world_(world), fn_(fn), user_(user) {}
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void allgather(const void* send, void* recv, size_t bytes) override {
    if (fn_(user_, send, recv, bytes) != 0) throw std::runtime_error("all-gather callback failed");
  }

 private:
  int rank_, world_;
  hpg_allgather_fn fn_;
  void* user_;
};

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (err && errlen > 0) std::snprintf(err, errlen, "%s", msg.c_str());
}

}  // namespace

extern "C" int hpg_dist_exchange(int rank, int world, hpg_allgather_fn allgather, void* user,
                                 int32_t n_runs, const int64_t* slices, int32_t* owner_out,
                                 int64_t* used, double* best, const hpg_improvement* mine,
                                 int64_t n_mine, hpg_improvement* all, int64_t cap, int64_t* n_all,
                                 char* err, size_t errlen) {
  try {
    if (world < 1 || rank < 0 || rank >= world || n_runs < 0 || !allgather || !n_all ||
        (n_runs > 0 && (!slices || !used || !best)) || (n_mine > 0 && !mine)) {
      set_err(err, errlen, "hpg_dist_exchange: bad argument");
      return HPG_USAGE;
    }
    const size_t R = static_cast<size_t>(n_runs);
    const std::vector<int> owner = hpg::deal_runs(std::vector<int64_t>(slices, slices + R), world);
    std::vector<hpg::RunRecord> rec(R);
    std::vector<std::vector<hpg::ImprRecord>> imp(R);
    for (size_t r = 0; r < R; ++r) rec[r] = hpg::RunRecord{used[r], best[r]};
    for (int64_t e = 0; e < n_mine; ++e) {
      const hpg_improvement& x = mine[e];
      if (x.run < 0 || static_cast<size_t>(x.run) >= R || owner[x.run] != rank) {
        set_err(err, errlen, "hpg_dist_exchange: improvement of a run this rank does not own");
        return HPG_USAGE;
      }
      imp[x.run].push_back(hpg::ImprRecord{x.run, x.local_idx, x.cost});
    }
    CallbackTransport tr(rank, world, allgather, user);
    hpg::exchange_round(tr, owner, rec, imp);
    int64_t total = 0;
    for (size_t r = 0; r < R; ++r) total += static_cast<int64_t>(imp[r].size());
    *n_all = total;
    if (total > cap || (total > 0 && !all)) {
      set_err(err, errlen, "hpg_dist_exchange: improvement buffer too small (need " +
                               std::to_string(total) + ")");
      return HPG_USAGE;
    }
    int64_t k = 0;
    for (size_t r = 0; r < R; ++r) {
      if (owner_out) owner_out[r] = owner[r];
      used[r] = rec[r].used;
      best[r] = rec[r].best;
      for (const hpg::ImprRecord& x : imp[r]) all[k++] = hpg_improvement{x.run, x.local_idx, x.cost};
    }
    set_err(err, errlen, "");
    return HPG_OK;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return HPG_INTERNAL;
  }
}
