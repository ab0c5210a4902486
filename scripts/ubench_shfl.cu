// Microbenchmark: do SHFL and LDS share on-chip bandwidth on B200?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_shfl ubench_shfl.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_lds(double* out, int mode) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0), acc2 = make_double2(0, 0);
  double s = threadIdx.x, s2 = threadIdx.x * 0.5;
  int idx = threadIdx.x & 31;
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    if (mode & 1) {  // LDS.128, conflict-free (consecutive 16-B per lane)
      const double2 a = sm[(idx + it * 32) & 1023];
      const double2 b = sm[(idx + it * 32 + 512) & 1023];
      acc.x += a.x; acc.y += a.y; acc2.x += b.x; acc2.y += b.y;
    }
    if (mode & 2) {  // 4 x SHFL.32 pairs (2 doubles)
      s = __shfl_xor_sync(0xffffffff, s, 1) + 1.0;
      s2 = __shfl_xor_sync(0xffffffff, s2, 2) + 1.0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc2.x + acc2.y + s + s2;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 1; mode <= 3; ++mode) {
    k_lds<<<148 * 8, 256>>>(out, mode);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_lds<<<148 * 8, 256>>>(out, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    const double warps = 148.0 * 8 * 8;
    // bytes moved per iteration per warp: LDS 2 x 512 B; SHFL 2 x 2 x 128 B (two doubles)
    double lds_b = (mode & 1) ? warps * ITERS * 1024.0 : 0;
    double shf_b = (mode & 2) ? warps * ITERS * 512.0 : 0;
    printf("mode %d (%s): %.3f ms  LDS %.1f TB/s  SHFL %.1f TB/s  total %.1f TB/s\n", mode,
           mode == 1 ? "LDS.128" : mode == 2 ? "SHFL" : "both", ms, lds_b / ms / 1e9,
           shf_b / ms / 1e9, (lds_b + shf_b) / ms / 1e9);
  }
  return 0;
}
