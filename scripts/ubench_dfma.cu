// DFMA issue rate with the operand kinds of the stencil kernel (one warp per SMSP):
// coefficient in a uniform register vs in a per-thread register (LDC), window in registers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_dfma scripts/ubench_dfma.cu
#include <cstdio>
#include <cuda_runtime.h>
struct P { double c[8]; };
template <int MODE>
__global__ void stencil(double* o, P p, int n, long long* cyc, int idx0) {
  double w[12], acc[4] = {0, 0, 0, 0};
  for (int k = 0; k < 12; ++k) w[k] = o[threadIdx.x + k];
  int idx = idx0 + (threadIdx.x & 0);  // 0, runtime
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double c[7];
#pragma unroll
    for (int m = 0; m < 7; ++m) c[m] = MODE == 0 ? p.c[m] : p.c[m + idx];
#pragma unroll
    for (int m = 0; m < 7; ++m)
#pragma unroll
      for (int x = 0; x < 4; ++x) acc[x] = fma(c[m], w[x + 1 + m], acc[x]);
    idx = (int)acc[0] & 0;
  }
  long long t1 = clock64();
  o[threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 4096 * 8); cudaMemset(o, 0, 4096 * 8); cudaMalloc(&c, 8);
  P p; for (int i = 0; i < 8; ++i) p.c[i] = 0.1 * i;
  const int n = 2000;
  for (int warps : {1, 4, 8, 12}) {
    stencil<0><<<1, 32 * warps>>>(o, p, n, c, 0); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%2d warps: coef in param/UR : %.2f cycles per DFMA per SMSP\n", warps, (double)h / (n * 28.0 * ((warps + 3) / 4)));
    stencil<1><<<1, 32 * warps>>>(o, p, n, c, 0); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%2d warps: coef via LDC (R)  : %.2f cycles per DFMA per SMSP\n", warps, (double)h / (n * 28.0 * ((warps + 3) / 4)));
  }
  return 0;
}
