// Host-side launch entry points of the CUDA kernels (implemented in *.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace hpg {

int eval_smem_bytes(const Carve& c);

cudaError_t launch_eval(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                        int32_t kb_flags, const uint8_t* d_recs, const int64_t* d_off,
                        const int32_t* d_modes, int32_t uniform_mode, int n, int64_t stride,
                        uint8_t* d_out,
                        EvalResult* d_res, double* d_per_task, double* d_required, int n_sm,
                        cudaStream_t st);

// Segmented best-half selection (search.cpp:590-620) for one SHA level.
cudaError_t launch_best_half(const double* d_scores, const int32_t* d_seg_off,
                             const int32_t* d_arm_idx, int n_seg, int32_t* d_keep_flags,
                             double* d_events, cudaStream_t st);

}  // namespace hpg
