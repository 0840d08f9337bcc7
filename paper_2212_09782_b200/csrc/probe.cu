// FP64 peak probes for the roofline denominator:
// MEASURED_PEAKS.json carries HBM and bf16 only, so the DMMA and DFMA
// peaks of this B200 are measured here with register-resident operands.
#include <cuda_runtime.h>

#include "common.cuh"

namespace qt {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* sink, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(double* sink, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

}  // namespace

// Returns measured TFLOP/s (2 flops per FMA) of the DMMA (kind=0) or DFMA
// (kind=1) pipe over the whole GPU, best of `reps` launches.
double fp64_peak_tflops(int kind, int reps, cudaStream_t st) {
  int dev = 0, sms = 0;
  QT_CUDA(cudaGetDevice(&dev));
  QT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* sink = nullptr;
  QT_CUDA(cudaMalloc(&sink, 256 * sizeof(double)));
  cudaEvent_t e0, e1;
  QT_CUDA(cudaEventCreate(&e0));
  QT_CUDA(cudaEventCreate(&e1));
  const int iters = kind == 0 ? 4096 : 16384;
  const int blocks = sms * 4;
  double best = 0.0;
  for (int r = 0; r < reps + 1; ++r) {
    QT_CUDA(cudaEventRecord(e0, st));
    if (kind == 0)
      dmma_peak_kernel<<<blocks, 256, 0, st>>>(sink, iters);
    else
      dfma_peak_kernel<<<blocks, 256, 0, st>>>(sink, iters);
    QT_CUDA(cudaEventRecord(e1, st));
    QT_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    QT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double warps = blocks * 256.0 / 32.0;
    const double flops = kind == 0 ? warps * iters * kChains * 512.0            // 8x8x4 FMA x2
                                   : blocks * 256.0 * iters * kChains * 2.0;  // per thread FMA
    if (r > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return best;
}

}  // namespace qt
