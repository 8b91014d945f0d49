// FP64 DFMA peak microbenchmark (sm_100a): independent FMA chains per thread,
// full-occupancy grid, timed with CUDA events. Prints one JSON line with the
// measured DFMA TFLOP/s (2 flops per FMA), so FP64 pipe utilisation of the
// engine's kernels can be quoted against a measured number.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8;
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fmas = static_cast<double>(blocks) * threads * kIters * kChains;
  const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  std::printf("{\"kernel\": \"dfma_kernel\", \"sms\": %d, \"best_ms\": %.4f, \"fp64_fma_tflops\": %.3f, "
              "\"dfma_per_sm_per_clk_at_1965mhz\": %.2f}\n",
              sms, best, tflops, fmas / (best * 1e-3) / sms / 1.965e9);
  return 0;
}
