// FP64 pipe peak microbenchmarks (the roofline denominator of seg_kernel).
//
// MEASURED_PEAKS.json holds HBM and bf16 figures only; the fused bucket
// kernel is bound by FP64 issue (DMUL / DADD, no FMA contraction: every
// complex product is rounded like std::complex<double>), so its roofline
// needs the FP64 rate of THIS part at its current clocks.  Two kernels:
//   mul_add: 8 independent chains per thread, each step one DMUL and one
//            DADD (x = x*a; y = y+b) -- the instruction mix seg_kernel issues;
//   fma:     8 independent DFMA chains (2 flops each) -- NVIDIA's FP64 figure.
// Grid: 4 x SMs CTAs of 256 threads (every SMSP holds 16 warps); timed with
// CUDA events, best of 5 launches.
#include <cuda_runtime.h>

#include <algorithm>

namespace qtng {
namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) fp64_mul_add_kernel(double a, double b, double* sink) {
  double x[kChains], y[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
    y[c] = 1e-3 * c;
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      x[c] = __dmul_rn(x[c], a);
      y[c] = __dadd_rn(y[c], b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c] + y[c];
  if (s == 12345.678) sink[0] = s;  // never true; keeps the chains live
}

__global__ void __launch_bounds__(256) fp64_fma_kernel(double a, double b, double* sink) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) sink[0] = s;
}

template <class K>
float best_ms(K kernel, int grid, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  kernel<<<grid, 256>>>(0.9999999, 1e-9, sink);  // warm-up
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kernel<<<grid, 256>>>(0.9999999, 1e-9, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

}  // namespace

// Returns cudaSuccess and the two rates (operations per second: one DMUL or
// DADD = 1 op; one DFMA = 2 flops).
cudaError_t fp64_peak(int device, double* mul_add_ops_per_s, double* fma_flops_per_s) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int grid = 4 * sms;
  double* sink = nullptr;
  if ((e = cudaMalloc(&sink, sizeof(double))) != cudaSuccess) return e;
  const double threads = static_cast<double>(grid) * 256.0;
  const float ms_ma = best_ms(fp64_mul_add_kernel, grid, sink);
  const float ms_fma = best_ms(fp64_fma_kernel, grid, sink);
  e = cudaGetLastError();
  cudaFree(sink);
  if (e != cudaSuccess) return e;
  *mul_add_ops_per_s = threads * kIters * kChains * 2.0 / (ms_ma * 1e-3);
  *fma_flops_per_s = threads * kIters * kChains * 2.0 / (ms_fma * 1e-3);
  return cudaSuccess;
}

}  // namespace qtng
