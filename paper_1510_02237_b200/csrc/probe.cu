// fp64 pipe probe: the fp64 half of the roofline (MEASURED_PEAKS.json only
// carries HBM and bf16 figures; SURVEY.md 8(d) asks for min(HBM, fp64)).
// Every thread runs 8 independent DFMA chains, so the pipe, not latency,
// bounds the kernel; the grid is 8 CTAs x 256 threads per SM.
#include "pw_internal.h"

namespace pw {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_probe_kernel(int iters, double a, double b, double* sink) {
  double x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 16; ++rep)
#pragma unroll
      for (int k = 0; k < kChains; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == 12345.678) sink[threadIdx.x] = s;  // never true; keeps the chains live
}

}  // namespace
}  // namespace pw

namespace pw {

double probe_fp64_tflops(Ctx& c, int iters) {
  {
    const int blocks = c.num_sms * 8, threads = 256;
    double* sink = nullptr;
    PW_CUDA(cudaMallocAsync(&sink, threads * sizeof(double), c.stream));
    cudaEvent_t e0, e1;
    PW_CUDA(cudaEventCreate(&e0));
    PW_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {  // first launch warms clocks; keep the best
      PW_CUDA(cudaEventRecord(e0, c.stream));
      dfma_probe_kernel<<<blocks, threads, 0, c.stream>>>(iters, 0.999999, 1e-7, sink);
      PW_CUDA(cudaEventRecord(e1, c.stream));
      PW_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      PW_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
      c.launches += 1;
    }
    PW_CUDA(cudaGetLastError());
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    PW_CUDA(cudaFreeAsync(sink, c.stream));
    const double flops = 2.0 * kChains * 16.0 * (double)iters * blocks * threads;
    return flops / (best * 1e-3) / 1e12;
  }
}

}  // namespace pw

