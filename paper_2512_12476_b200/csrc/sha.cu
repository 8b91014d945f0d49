// sha_best_half: one successive-halving step for many segments at once
// (best_half, search.cpp:590-620). Survivors are the ceil(n/2) arms with the
// smallest (score, arm index) — the order of the reference's stable_sort —
// computed as a rank count per arm (exact, order-independent). One CTA per
// segment; the event values are the scores at ranks keep-1 and keep.
#include <cuda_runtime.h>

#include "eval_launch.hpp"

namespace hpg {
namespace dev {

__global__ void best_half_kernel(const double* __restrict__ scores,
                                 const int32_t* __restrict__ seg_off,
                                 const int32_t* __restrict__ arm_idx, int32_t* __restrict__ keep,
                                 double* __restrict__ events) {
  const int s = blockIdx.x;
  const int b = seg_off[s], e = seg_off[s + 1];
  const int n = e - b;
  const int k = (n + 1) / 2;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double si = scores[b + i];
    const int ii = arm_idx[b + i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double sj = scores[b + j];
      const int ij = arm_idx[b + j];
      // comparator of search.cpp:598-605
      const bool less = (sj != si) ? (sj < si) : (ij < ii);
      rank += less ? 1 : 0;
    }
    keep[b + i] = rank < k ? 1 : 0;
    if (rank == k - 1) events[2 * s] = si;
    if (rank == k) events[2 * s + 1] = si;
  }
}

}  // namespace dev

cudaError_t launch_best_half(const double* d_scores, const int32_t* d_seg_off,
                             const int32_t* d_arm_idx, int n_seg, int32_t* d_keep,
                             double* d_events, cudaStream_t st) {
  if (n_seg <= 0) return cudaSuccess;
  dev::best_half_kernel<<<n_seg, 128, 0, st>>>(d_scores, d_seg_off, d_arm_idx, d_keep, d_events);
  return cudaGetLastError();
}

}  // namespace hpg
