#include "devstate.hpp"

#include <map>
#include <mutex>
#include <tuple>

namespace hpg {
namespace {

std::mutex g_mu;
std::map<std::pair<int, const void*>, int>& smem_limits() {
  static std::map<std::pair<int, const void*>, int> m;
  return m;
}
std::map<std::tuple<int, const void*, int, int>, int>& occupancy() {
  static std::map<std::tuple<int, const void*, int, int>, int> m;
  return m;
}

}  // namespace

cudaError_t ensure_dyn_smem(const void* fn, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  int& cur = smem_limits()[{dev, fn}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

cudaError_t occupancy_per_sm(const void* fn, int threads, int bytes, int* per_sm) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(dev, fn, threads, bytes);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    const auto it = occupancy().find(key);
    if (it != occupancy().end()) {
      *per_sm = it->second;
      return cudaSuccess;
    }
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, fn, threads, static_cast<size_t>(bytes));
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  occupancy()[key] = *per_sm;
  return cudaSuccess;
}

}  // namespace hpg
