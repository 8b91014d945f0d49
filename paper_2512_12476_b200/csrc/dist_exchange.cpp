// See dist_exchange.hpp. Host-only (no CUDA): the C-ABI hook hpg_dist_exchange
// runs this same code over a caller's all-gather, which is how the gloo
// world-size-2 tests drive it on machines without GPUs.
#include "dist_exchange.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <stdexcept>

namespace hpg {

std::vector<int> deal_runs(const std::vector<int64_t>& slices, int world) {
  const size_t R = slices.size();
  std::vector<int> owner(R, 0);
  if (world <= 1) return owner;
  std::vector<size_t> order(R);
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return slices[a] > slices[b]; });
  std::vector<int64_t> load(static_cast<size_t>(world), 0);
  for (size_t r : order) {
    int best = 0;
    for (int k = 1; k < world; ++k)
      if (load[k] < load[best]) best = k;
    owner[r] = best;
    load[best] += std::max<int64_t>(slices[r], 1);
  }
  return owner;
}

void exchange_round(Transport& tr, const std::vector<int>& owner, std::vector<RunRecord>& rec,
                    std::vector<std::vector<ImprRecord>>& impr) {
  const int world = tr.world(), me = tr.rank();
  const size_t R = owner.size();
  if (rec.size() != R || impr.size() != R) throw std::invalid_argument("exchange_round: sizes");
  if (world <= 1) return;
  // 1. [n_impr | records of all runs (own entries meaningful)]
  std::vector<ImprRecord> mine;
  for (size_t r = 0; r < R; ++r)
    if (owner[r] == me) mine.insert(mine.end(), impr[r].begin(), impr[r].end());
  const size_t b1 = 8 + sizeof(RunRecord) * R;
  std::vector<uint8_t> s1(b1, 0), g1(b1 * world);
  const int64_t nm = static_cast<int64_t>(mine.size());
  std::memcpy(s1.data(), &nm, 8);
  for (size_t r = 0; r < R; ++r)
    if (owner[r] == me) std::memcpy(s1.data() + 8 + sizeof(RunRecord) * r, &rec[r], sizeof(RunRecord));
  tr.allgather(s1.data(), g1.data(), b1);
  std::vector<int64_t> cnt(world);
  int64_t mx = 0;
  for (int k = 0; k < world; ++k) {
    std::memcpy(&cnt[k], g1.data() + b1 * k, 8);
    mx = std::max(mx, cnt[k]);
  }
  for (size_t r = 0; r < R; ++r) {
    const int k = owner[r];
    if (k < 0 || k >= world) throw std::invalid_argument("exchange_round: owner out of range");
    if (k == me) continue;
    std::memcpy(&rec[r], g1.data() + b1 * k + 8 + sizeof(RunRecord) * r, sizeof(RunRecord));
  }
  // 2. improvements, padded to the largest count
  if (mx == 0) {
    for (size_t r = 0; r < R; ++r)
      if (owner[r] != me) impr[r].clear();
    return;
  }
  const size_t b2 = sizeof(ImprRecord) * static_cast<size_t>(mx);
  std::vector<uint8_t> s2(b2, 0), g2(b2 * world);
  if (!mine.empty()) std::memcpy(s2.data(), mine.data(), sizeof(ImprRecord) * mine.size());
  tr.allgather(s2.data(), g2.data(), b2);
  for (size_t r = 0; r < R; ++r)
    if (owner[r] != me) impr[r].clear();
  for (int k = 0; k < world; ++k) {
    if (k == me) continue;
    const ImprRecord* p = reinterpret_cast<const ImprRecord*>(g2.data() + b2 * k);
    for (int64_t e = 0; e < cnt[k]; ++e) {
      const ImprRecord& x = p[e];
      if (x.run < 0 || static_cast<size_t>(x.run) >= R || owner[x.run] != k)
        throw std::runtime_error("exchange_round: improvement of a run the sender does not own");
      impr[x.run].push_back(x);
    }
  }
}

}  // namespace hpg
