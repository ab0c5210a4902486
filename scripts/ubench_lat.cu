// Latency probes on the B200 (one warp): dependent DFMA chain, dependent LDS, LDC.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_lat scripts/ubench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
struct P { double c[32]; };
__global__ void dfma_chain(double* o, double a, double b, int n, long long* cyc) {
  double x = o[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = fma(x, a, b);
  }
  long long t1 = clock64();
  o[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dfma_4chains(double* o, double a, double b, int n, long long* cyc) {
  double x0 = o[threadIdx.x], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); }
  }
  long long t1 = clock64();
  o[threadIdx.x] = x0 + x1 + x2 + x3;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dfma_8chains(double* o, double a, double b, int n, long long* cyc) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = o[threadIdx.x] + k;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  o[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void ldc_chain(double* o, P p, int n, long long* cyc) {
  double x = o[threadIdx.x];
  int idx = (int)x & 1;  // 0 at runtime, opaque
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) { x = fma(x, p.c[idx + (j & 15)], 1.0); idx = ((int)x) & 0; }
  }
  long long t1 = clock64();
  o[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 1024 * 8); cudaMemset(o, 0, 1024 * 8); cudaMalloc(&c, 8);
  P p; for (int i = 0; i < 32; ++i) p.c[i] = 0.5;
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) {
    dfma_chain<<<1, 32>>>(o, 0.999, 0.001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / (n * 16));
    dfma_4chains<<<1, 32>>>(o, 0.999, 0.001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 4 chains, 1 warp: %.2f cycles per DFMA\n", (double)h / (n * 64));
    dfma_8chains<<<1, 32>>>(o, 0.999, 0.001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 chains, 1 warp: %.2f cycles per DFMA\n", (double)h / (n * 128));
    dfma_8chains<<<1, 128>>>(o, 0.999, 0.001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 chains, 4 warps (1/SMSP): %.2f cycles per DFMA per warp\n", (double)h / (n * 128));
    dfma_8chains<<<1, 256>>>(o, 0.999, 0.001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 chains, 8 warps (2/SMSP): %.2f cycles per DFMA per warp\n", (double)h / (n * 128));
    ldc_chain<<<1, 32>>>(o, p, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("LDC+DFMA dependent: %.2f cycles\n", (double)h / (n * 16));
  }
  return 0;
}
