// Per-round record exchange of the sharded search.
//
// The runs of one SHA round are dealt to the ranks (deal_runs); each rank
// runs its own, then one exchange gives every rank every run's record
// (evaluations used, best cost) and incumbent-improvement list, so every rank
// then takes identical best_half decisions (search.cpp:590-620) and rebuilds
// the same global incumbent trace. The transport is an interface: NCCL over
// the context's communicator inside hpg_search_dist, or any caller-supplied
// all-gather (hpg_dist_exchange in include/hpg.h, e.g. torch.distributed/gloo).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace hpg {

struct RunRecord {
  int64_t used;
  double best;
};

struct ImprRecord {
  int64_t run;
  int64_t local_idx;  // 1-based evaluation index inside the run
  double cost;
};

class Transport {
 public:
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // every rank contributes `bytes` bytes; recv gets world * bytes in rank order
  virtual void allgather(const void* send, void* recv, size_t bytes) = 0;
};

// Owner rank of every run of a round: longest slice first (stable by run
// index), each to the rank with the least budget so far (ties: lowest rank).
// Deterministic, so every rank computes the same deal.
std::vector<int> deal_runs(const std::vector<int64_t>& slices, int world);

// rec[r] / impr[r] are inputs for the runs this rank owns and outputs for all
// runs; impr lists keep the owner's order. Two all-gathers: the fixed-size
// records (plus each rank's improvement count), then the improvements padded
// to the largest count.
void exchange_round(Transport& tr, const std::vector<int>& owner, std::vector<RunRecord>& rec,
                    std::vector<std::vector<ImprRecord>>& impr);

}  // namespace hpg
