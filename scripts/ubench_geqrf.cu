// cuSOLVER 64-bit Xgeqrf time vs panel width on tall panels (the incremental subspace QR)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_geqrf scripts/ubench_geqrf.cu -lcusolver -lcublas
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <curand_kernel.h>
__global__ void fill(double* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = (double)((i * 2654435761ULL) % 1000003) / 1000003.0 - 0.5;
}
int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
  long long rows_list[2] = {786432, 3145728};
  int cols_list[5] = {16, 32, 64, 128, 256};
  double* a; cudaMalloc(&a, sizeof(double) * 3145728LL * 256);
  double* tau; cudaMalloc(&tau, sizeof(double) * 256);
  int* info; cudaMalloc(&info, sizeof(int));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (long long rows : rows_list) {
    for (int cols : cols_list) {
      size_t dws = 0, hws = 0;
      cusolverDnXgeqrf_bufferSize(h, prm, rows, cols, CUDA_R_64F, a, rows, CUDA_R_64F, tau, CUDA_R_64F, &dws, &hws);
      void* dw; cudaMalloc(&dw, dws + 8);
      std::vector<char> hw(hws + 8);
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        fill<<<1024, 256>>>(a, rows * cols);
        cudaEventRecord(e0);
        cusolverDnXgeqrf(h, prm, rows, cols, CUDA_R_64F, a, rows, CUDA_R_64F, tau, CUDA_R_64F, dw, dws, hw.data(), hws, info);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("Xgeqrf %8lld x %3d: %8.2f ms  (%.1f GB/s of the panel per pass)\n", rows, cols, best,
             rows * cols * 8.0 / (best * 1e-3) / 1e9);
      cudaFree(dw);
    }
  }
  return 0;
}
