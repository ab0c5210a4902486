// Serial-step GEMV microbenchmark: pw::launch_combine_gemv at c3 size
// (d = 3 * 512^2) for the ranks of the c3 window, over grid sizes.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1510_02237_b200/csrc
//        scripts/ubench_gemv.cu -o scripts/ubench_gemv -Lpaper_1510_02237_b200 -lpitwave_b200
//        -Xlinker -rpath,'$ORIGIN/../paper_1510_02237_b200'
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pw_internal.h"

int main(int argc, char** argv) {
  const long long d = argc > 1 ? atoll(argv[1]) : 3LL * 512 * 512;
  pw::Ctx c{};
  c.device = 0;
  cudaStreamCreate(&c.stream);
  cudaDeviceProp p{};
  cudaGetDeviceProperties(&p, 0);
  c.num_sms = p.multiProcessorCount;
  const int rmax = 320;
  double *D, *Q, *g, *cv, *al, *y, *an, *part;
  cudaMalloc(&D, sizeof(double) * d * rmax);
  cudaMalloc(&Q, sizeof(double) * d * rmax);
  cudaMalloc(&g, sizeof(double) * d);
  cudaMalloc(&cv, sizeof(double) * d);
  cudaMalloc(&y, sizeof(double) * d);
  cudaMalloc(&al, sizeof(double) * rmax);
  cudaMalloc(&an, sizeof(double) * rmax);
  cudaMalloc(&part, sizeof(double) * pw::combine_part_doubles(d, rmax) * 4);
  cudaMemset(D, 0, sizeof(double) * d * rmax);
  cudaMemset(Q, 0, sizeof(double) * d * rmax);
  cudaMemset(g, 0, sizeof(double) * d);
  cudaMemset(cv, 0, sizeof(double) * d);
  cudaMemset(al, 0, sizeof(double) * rmax);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ranks[] = {64, 127, 189, 250, 310};
  const int grids[] = {0};
  for (int r : ranks) {
    for (int nb : grids) {
      try {
        for (int w = 0; w < 3; ++w)
          pw::launch_combine_gemv(c, c.stream, g, D, r, cv, al, Q, r, d, y, an, part, nb);
        const int reps = 20;
        cudaEventRecord(e0, c.stream);
        for (int k = 0; k < reps; ++k)
          pw::launch_combine_gemv(c, c.stream, g, D, r, cv, al, Q, r, d, y, an, part, nb);
        cudaEventRecord(e1, c.stream);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double t = ms * 1e-3 / reps;
        const double bytes = 2.0 * r * d * 8 + 4.0 * d * 8;
        printf("r=%3d grid=%4d  %8.1f us  %7.1f GB/s\n", r, nb, t * 1e6, bytes / t / 1e9);
      } catch (pw::Error& e) {
        printf("error %s\n", e.msg.c_str());
        return 1;
      }
    }
  }
  // pure streaming-read ceiling: copy D -> Q (read + write)
  cudaEventRecord(e0, c.stream);
  cudaMemcpyAsync(Q, D, sizeof(double) * d * 310, cudaMemcpyDeviceToDevice, c.stream);
  cudaEventRecord(e1, c.stream);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("memcpy D->Q r=310: %.1f GB/s\n", 2.0 * 310 * d * 8 / (ms * 1e-3) / 1e9);
  return 0;
}
