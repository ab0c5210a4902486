// fp64 tensor-core GEMM for the Krylov subspace (sm_100a, mma.sync m8n8k4 f64 = DMMA).
//
//   C (m x n) = alpha * op(A) * B[ :, ] + beta * C       column-major, 64-bit sizes
//   op(A) = A (m x k, ld lda) or A^T (A stored k x m)
//
// Every product of the subspace refactorisation and of the sweep's batched projections
// goes through here (api.cu gemm()): the compact-WY applications Q1^T N = N - V T^T V^T N
// and Q = Q1 [Q2; 0], the image product Y = M scatter(R11^-1), the Gram blocks of larft,
// the TSQR panel's trailing updates and Q^T qk / Y alpha.  The shapes are extreme: either
// m = d (3.1M rows at c4) with n, k <= 1024 ("tall": many output tiles, B stays in L2), or
// m, n <= 1024 with k = d ("reduction": few output tiles, so the k range is split over
// grid.z and the partial tiles are summed by a second kernel in a fixed order -- the
// result does not depend on the launch).
//
// B200 has no fp64 tcgen05 kind; fp64 tensor throughput is the warp-level DMMA
// (scripts/ubench_dmma.cu: 37 TFLOP/s, sharing the pipe with DFMA).  CTA tile 128 x 64,
// 8 warps of 32 x 32 (16 DMMA per k4 step), k tiles of 16 staged by cp.async in a
// 3-deep ring (72 KB, two CTAs per SM).  Shared layouts follow the global one so every
// 16-byte copy is a contiguous run; the row padding (+4 doubles) makes the fragment
// loads of both A layouts and of B bank-conflict free per half warp.
//
// Options used by the subspace: `acol` gathers A's columns (op N: column kk of the
// operand is A[:, acol[kk]]) and `b_upper` declares B upper triangular (only k < n0 + 64
// contributes to output tile column block n0) -- together Y = M[:, piv] R11^-1 costs
// d r^2 flops instead of the 2 d m r of a dense product with the scattered inverse.
#include "pw_internal.h"

namespace pw {
namespace {

constexpr int BK = 16, NST = 3, NTH = 256;
constexpr int PADK = BK + 4;  // rows of [m][k] / [n][k] tiles

// CTA tile (32 WM) x (32 WN) with 8 warps of 32 x 32: WM = 4 (128 x 64, the default) or
// WM = 1 (32 x 256, for the 32-row outputs of the TSQR trailing reductions V^T A)
template <int WM_>
struct Cfg {
  static constexpr int WM = WM_, WN = 8 / WM_;
  static constexpr int BM = 32 * WM, BN = 32 * WN;
  static constexpr int PADM = BM + 4;  // rows of the [k][m] tile
  static constexpr int A_STAGE_N = BK * PADM;  // op(A) = A: [k][m]
  static constexpr int A_STAGE_T = BM * PADK;  // op(A) = A^T: [m][k]
  static constexpr int B_STAGE = BN * PADK;    // [n][k]
  static constexpr int A_STAGE = A_STAGE_N > A_STAGE_T ? A_STAGE_N : A_STAGE_T;
  static constexpr size_t SMEM_PIPE = sizeof(double) * (size_t)NST * (A_STAGE + B_STAGE);
  static constexpr size_t SMEM_EPI = sizeof(double) * (size_t)BN * (BM + 1);  // staged C tile
  static constexpr size_t SMEM = SMEM_PIPE > SMEM_EPI ? SMEM_PIPE : SMEM_EPI;
};

__host__ __device__ __forceinline__ long long lmin(long long a, long long b) { return a < b ? a : b; }

__device__ __forceinline__ void cp16(double* s, const double* g, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp8(double* s, const double* g, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct GemmArgs {
  long long m, n, k;
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
  double alpha, beta;
  const int* acol;   // op N only: operand column kk is A[:, acol[kk]] (nullable)
  int b_upper;       // B upper triangular: skip k >= n0 + BN
  int ktiles_per_split;
  int nfast;         // blockIdx.x walks the n tiles (concurrent CTAs share A's rows in L2)
  double* part;      // split-K partial tiles (m x n each, ld m), or nullptr: direct epilogue
};

// Stage k tile kt (global k in [kt*BK, kt*BK+BK)) of op(A) and B into ring slot `st`.
// VEC: 16-byte copies (pointers 16-byte aligned, leading dimensions even); else 8-byte.
template <class K, bool TA, bool VEC>
__device__ __forceinline__ void load_tile(const GemmArgs& g, double* As, double* Bs, long long m0, long long n0,
                                          long long kt) {
  constexpr int BM = K::BM, BN = K::BN, PADM = K::PADM;
  const int tid = threadIdx.x;
  const long long k0 = kt * BK;
  constexpr int W = VEC ? 2 : 1;  // doubles per copy
  if constexpr (!TA) {
    // A is m x k, contiguous in m: [k][m] tile, copies along m
    constexpr int PER_ROW = BM / W, TOTAL = BK * PER_ROW;
#pragma unroll
    for (int j = 0; j < TOTAL / NTH; ++j) {
      const int c = tid + j * NTH;
      const int kl = c / PER_ROW, il = (c - kl * PER_ROW) * W;
      const long long gi = m0 + il, gk = k0 + kl;
      int bytes = 0;
      const double* src = g.A;
      if (gk < g.k && gi < g.m) {
        const long long col = g.acol ? (long long)__ldg(g.acol + gk) : gk;
        src = g.A + gi + col * g.lda;
        bytes = (int)(8 * lmin(W, g.m - gi));
      }
      if constexpr (VEC) cp16(As + kl * PADM + il, src, bytes);
      else cp8(As + kl * PADM + il, src, bytes);
    }
  } else {
    // A is k x m (op = A^T), contiguous in k: [m][k] tile, copies along k
    constexpr int PER_ROW = BK / W, TOTAL = BM * PER_ROW;
#pragma unroll
    for (int j = 0; j < TOTAL / NTH; ++j) {
      const int c = tid + j * NTH;
      const int il = c / PER_ROW, kl = (c - il * PER_ROW) * W;
      const long long gi = m0 + il, gk = k0 + kl;
      int bytes = 0;
      const double* src = g.A;
      if (gk < g.k && gi < g.m) {
        src = g.A + gk + gi * g.lda;
        bytes = (int)(8 * lmin(W, g.k - gk));
      }
      if constexpr (VEC) cp16(As + il * PADK + kl, src, bytes);
      else cp8(As + il * PADK + kl, src, bytes);
    }
  }
  {
    // B is k x n, contiguous in k: [n][k] tile
    constexpr int PER_ROW = BK / W, TOTAL = BN * PER_ROW;
#pragma unroll
    for (int j = 0; j < (TOTAL + NTH - 1) / NTH; ++j) {
      const int c = tid + j * NTH;
      if (TOTAL % NTH == 0 || c < TOTAL) {
        const int jl = c / PER_ROW, kl = (c - jl * PER_ROW) * W;
        const long long gj = n0 + jl, gk = k0 + kl;
        int bytes = 0;
        const double* src = g.B;
        if (gk < g.k && gj < g.n) {
          src = g.B + gk + gj * g.ldb;
          bytes = (int)(8 * lmin(W, g.k - gk));
        }
        if constexpr (VEC) cp16(Bs + jl * PADK + kl, src, bytes);
        else cp8(Bs + jl * PADK + kl, src, bytes);
      }
    }
  }
}

template <class K, bool TA, bool VEC>
__global__ void __launch_bounds__(NTH, 2) dgemm_kernel(GemmArgs g) {
  constexpr int BM = K::BM, BN = K::BN, PADM = K::PADM, A_STAGE = K::A_STAGE, B_STAGE = K::B_STAGE;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + NST * A_STAGE;
  const long long m0 = (long long)(g.nfast ? blockIdx.y : blockIdx.x) * BM;
  const long long n0 = (long long)(g.nfast ? blockIdx.x : blockIdx.y) * BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp % K::WM) * 32, wn = (warp / K::WM) * 32;
  // k tiles of this split; an upper-triangular B ends at the tile's last column
  long long kend = g.k;
  if (g.b_upper) kend = lmin(kend, n0 + BN);
  const long long nkt_all = (kend + BK - 1) / BK;
  const long long kt0 = (long long)blockIdx.z * g.ktiles_per_split;
  const long long kt1 = lmin(nkt_all, kt0 + g.ktiles_per_split);
  const int nkt = kt1 > kt0 ? (int)(kt1 - kt0) : 0;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < NST - 1; ++s) {
    if (s < nkt) load_tile<K, TA, VEC>(g, As + s * A_STAGE, Bs + s * B_STAGE, m0, n0, kt0 + s);
    cp_commit();
  }
  const int ar = lane >> 2, ak = lane & 3;  // fragment row / k of this lane
  for (int t = 0; t < nkt; ++t) {
    cp_wait<NST - 2>();
    __syncthreads();  // tile t landed for all; slot (t-1) % NST is free again
    {
      const int tn = t + NST - 1;
      if (tn < nkt) load_tile<K, TA, VEC>(g, As + (tn % NST) * A_STAGE, Bs + (tn % NST) * B_STAGE, m0, n0, kt0 + tn);
      cp_commit();
    }
    const double* a_s = As + (t % NST) * A_STAGE;
    const double* b_s = Bs + (t % NST) * B_STAGE;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = wm + i * 8 + ar;
        a[i] = TA ? a_s[row * PADK + ks + ak] : a_s[(ks + ak) * PADM + row];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = b_s[(wn + j * 8 + ar) * PADK + ks + ak];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_wait<0>();

  __syncthreads();  // the pipeline buffers become the C tile
  // epilogue: lane holds C[row][col], C[row][col + 1] of each 8 x 8 fragment; stage the
  // tile in shared memory ([col][row], ld BM + 1) and write it column by column with
  // consecutive threads on consecutive rows (coalesced read-modify-write of C)
  double* Cs = smem;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) Cs[(wn + j * 8 + 2 * ak + h) * (BM + 1) + wm + i * 8 + ar] = acc[i][j][h];
  __syncthreads();
  const long long mrem = lmin(BM, g.m - m0), nrem = lmin(BN, g.n - n0);
  double* P = g.part ? g.part + (long long)blockIdx.z * g.m * g.n : nullptr;
  for (int e = threadIdx.x; e < BM * BN; e += NTH) {
    const int cl = e / BM, rl = e - cl * BM;
    if (rl < mrem && cl < nrem) {
      const double v = Cs[cl * (BM + 1) + rl];
      const long long r = m0 + rl, cc = n0 + cl;
      if (P) {
        P[r + cc * g.m] = v;
      } else {
        double* p = g.C + r + cc * g.ldc;
        *p = (g.beta == 0.0) ? g.alpha * v : fma(g.beta, *p, g.alpha * v);
      }
    }
  }
}

// C = alpha * sum_z part[z] + beta * C, summed in split order (deterministic)
__global__ void splitk_reduce_kernel(const double* __restrict__ part, int splits, long long m, long long n,
                                     double alpha, double beta, double* C, long long ldc) {
  const long long total = m * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(long long)z * total + e];
    const long long c = e / m, r = e - c * m;
    double* p = C + r + c * ldc;
    const double v = alpha * s;
    *p = (beta == 0.0) ? v : fma(beta, *p, v);
  }
}

template <class K, bool TA, bool VEC>
void launch_cfg(Ctx& c, const GemmArgs& g, dim3 grid) {
  auto kern = dgemm_kernel<K, TA, VEC>;
  kernel_setup(c, kern, NTH, K::SMEM);
  kern<<<grid, NTH, K::SMEM, c.stream>>>(g);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

template <class K>
void launch_any(Ctx& c, const GemmArgs& g, dim3 grid, bool ta, bool vec) {
  if (ta) {
    if (vec) launch_cfg<K, true, true>(c, g, grid);
    else launch_cfg<K, true, false>(c, g, grid);
  } else {
    if (vec) launch_cfg<K, false, true>(c, g, grid);
    else launch_cfg<K, false, false>(c, g, grid);
  }
}

}  // namespace

void dgemm(Ctx& c, bool ta, long long m, long long n, long long k, double alpha, const double* A, long long lda,
           const double* B, long long ldb, double beta, double* C, long long ldc, const int* acol, bool b_upper) {
  if (m <= 0 || n <= 0) return;
  PW_CHECK(!(ta && acol), PW_ERR_VALUE, "dgemm: column gather needs op(A) = A");
  if (k <= 0) {
    PW_CHECK(beta == 1.0 || beta == 0.0, PW_ERR_STATE, "gemm with k=0 and beta not in {0,1}");
    if (beta == 0.0) PW_CUDA(cudaMemset2DAsync(C, ldc * sizeof(double), 0, m * sizeof(double), n, c.stream));
    return;
  }
  GemmArgs g{};
  g.m = m;
  g.n = n;
  g.k = k;
  g.A = A;
  g.lda = lda;
  g.B = B;
  g.ldb = ldb;
  g.C = C;
  g.ldc = ldc;
  g.alpha = alpha;
  g.beta = beta;
  g.acol = acol;
  g.b_upper = b_upper ? 1 : 0;
  // 32 x 256 tiles for short outputs (m <= 32: the TSQR's V^T A), else 128 x 64
  const bool narrow = m <= 32 && n > 64;
  const long long BMc = narrow ? Cfg<1>::BM : Cfg<4>::BM, BNc = narrow ? Cfg<1>::BN : Cfg<4>::BN;
  const long long tm = (m + BMc - 1) / BMc, tn = (n + BNc - 1) / BNc;
  const long long nkt = (k + BK - 1) / BK;
  // split the k range when the output tiles cannot fill the GPU (two CTAs per SM), keeping
  // at least 16 k tiles per split; the partials cost splits x m x n doubles
  const long long slots = 2LL * (c.num_sms > 0 ? c.num_sms : 148);
  long long splits = 1;
  if (2 * tm * tn <= slots && !b_upper) {
    // one wave: splits x tiles <= slots (a second, partial wave would double the time)
    splits = slots / (tm * tn);
    splits = std::min<long long>(splits, std::max<long long>(1, nkt / 16));
  }
  g.ktiles_per_split = (int)((nkt + splits - 1) / splits);
  splits = (nkt + g.ktiles_per_split - 1) / g.ktiles_per_split;
  double* part = nullptr;
  if (splits > 1) {
    PW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * (size_t)(splits * m * n), c.stream));
    g.part = part;
  }
  const bool vec = ((((uintptr_t)A | (uintptr_t)B) & 15) == 0) && !(lda & 1) && !(ldb & 1);
  // tall products (many m tiles, several n tiles): n fastest, so the CTAs in flight work on
  // few row blocks of A and read each from HBM once; B (k x n <= 8 MB) stays in L2
  g.nfast = (tn > 1 && tm >= 4 * tn && tm < 65536) ? 1 : 0;
  PW_CHECK(splits < 65536 && (g.nfast ? (tn < (1LL << 31) && tm < 65536) : (tm < (1LL << 31) && tn < 65536)),
           PW_ERR_VALUE, "dgemm: grid too large");
  dim3 grid(g.nfast ? (unsigned)tn : (unsigned)tm, g.nfast ? (unsigned)tm : (unsigned)tn, (unsigned)splits);
  if (narrow) launch_any<Cfg<1>>(c, g, grid, ta, vec);
  else launch_any<Cfg<4>>(c, g, grid, ta, vec);
  if (part) {
    const long long total = m * n;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 4LL * slots);
    splitk_reduce_kernel<<<blocks, 256, 0, c.stream>>>(part, (int)splits, m, n, alpha, beta, C, ldc);
    c.launches += 1;
    PW_LAUNCH_CHECK();
    PW_CUDA(cudaFreeAsync(part, c.stream));
  }
}

}  // namespace pw
