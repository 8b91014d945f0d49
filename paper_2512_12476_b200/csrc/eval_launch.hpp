// Host-side launch entry points of the CUDA kernels (implemented in *.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"
#include "ga_dev.hpp"

namespace hpg {

int eval_smem_bytes(const Carve& c);
// diagnostics: per-plan clock64 phase stamps (5) + sub-phase
// cycles (27), or nullptr
constexpr int kPlanProfSlots = 32;
cudaError_t eval_set_plan_profile(long long* d_buf);
// diagnostics: cumulative balance_layers phase cycles / counters (32 slots)
cudaError_t eval_phase_acc(unsigned long long* out16);
// global scratch (doubles) per CTA of eval_kernel
int64_t eval_scratch_doubles(int n_dev, int64_t max_nl);
// persistent grid size for n plans (occupancy-limited, multiple of the SMs)
cudaError_t eval_grid(Carve cv, int n, int n_sm, int& grid);

cudaError_t launch_eval(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                        int32_t kb_flags, const uint8_t* d_recs, const int64_t* d_off,
                        const int32_t* d_modes, int32_t uniform_mode, int n, int64_t stride,
                        uint8_t* d_out, const int64_t* d_out_off, EvalResult* d_res,
                        double* d_per_task,
                        double* d_required, double* d_scratch, int64_t scratch_doubles,
                        int grid, cudaStream_t st);

// Device-resident GA offspring loop of many runs (ga_kernel.cuh): one
// persistent launch, grid = SMs x resident one-warp workers
cudaError_t launch_ga_offspring(const DevProblem& P, const DevCostConfig& cfg, Carve cv,
                                const GaParams& G, double* gscratch, int64_t gscratch_doubles,
                                int n_sm, int& grid, cudaStream_t st);

// Segmented best-half selection (search.cpp:590-620) for one SHA level.
cudaError_t launch_best_half(const double* d_scores, const int32_t* d_seg_off,
                             const int32_t* d_arm_idx, int n_seg, int32_t* d_keep_flags,
                             double* d_events, cudaStream_t st);

// cost-model primitives, one call each (prim_kernels.cuh)
int task_cost_smem(const RecHeader& h, int N, int T);
cudaError_t launch_task_cost(const DevProblem& P, const DevCostConfig& cfg, int t,
                             const RecHeader& h, const int32_t* d_sl, const int64_t* d_nm,
                             const uint8_t* d_dev, const double* d_resident, double* d_out,
                             cudaStream_t st);
cudaError_t launch_ring(const DevProblem& P, int mode, const uint8_t* d_a, int na,
                        const uint8_t* d_b, int nb, double volume, double* d_out, cudaStream_t st);

}  // namespace hpg
