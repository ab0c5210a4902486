// Is the fp64 MMA (mma.sync m8n8k4 f64) a separate pipe from DFMA on B200?
// One CTA of W warps per SM, all SMs: DMMA alone, DFMA alone, both interleaved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_dmma scripts/ubench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* o, int n) {
  double a = o[threadIdx.x] + 1.0, b = o[threadIdx.x + 1] + 0.5;
  double c[8][2] = {};
  double f[8];
  for (int q = 0; q < 8; ++q) f[q] = a + q;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE != 1) dmma(c[q][0], c[q][1], a, b);
      if (MODE != 0) f[q] = fma(f[q], a, b);
      if (MODE == 2) f[q] = fma(f[q], b, a);
    }
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + f[q];
  if (s == 12345.678) o[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 4096 * 8); cudaMemset(o, 0, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 20000, blocks = 148;
  for (int w : {4, 8, 16}) {
    float ms[3];
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<blocks, 32 * w>>>(o, n);
        if (mode == 1) k<1><<<blocks, 32 * w>>>(o, n);
        if (mode == 2) k<2><<<blocks, 32 * w>>>(o, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms[mode], e0, e1);
      }
    }
    const double warps = (double)blocks * w, iters = (double)n * 8;
    // DMMA m8n8k4: 256 FMA per warp-instr = 512 flop; DFMA: 32 FMA per warp-instr = 64 flop
    printf("%2d warps/SM: DMMA alone %.1f TFLOP/s | DFMA alone %.1f TFLOP/s | DMMA+2xDFMA %.2f ms vs %.2f + %.2f\n",
           w, warps * iters * 512 / (ms[0] * 1e-3) / 1e12, warps * iters * 64 / (ms[1] * 1e-3) / 1e12,
           ms[2], ms[0], 2 * ms[1]);
  }
  return 0;
}
