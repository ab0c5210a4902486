// Tall-skinny Householder QR of the subspace panel (sm_100a, fp64): the drop-in for LAPACK
// geqrf on the d x P blocks the Krylov basis appends (reference subspace.py:66-68 factors
// all snapshots with scipy qr -> dgeqp3; api.cu keeps the factorisation incremental and
// factors only each update's new block, so this is the O(d P^2) kernel of the update).
//
// Output is geqrf's format (R in the upper triangle, the unit-lower reflectors V below
// the diagonal, tau), so the compact-WY machinery around it (larft, Q1^T N, Q = Q1 Q2)
// is unchanged.  The panel is factored in sub-panels of TB = 32 columns; each one:
//
//   1. TSQR (tsqr_qr_kernel): leaves of TL = 128 rows, one CTA each, Householder QR in
//      shared memory (reflectors stored back in place, the leaf R to a buffer); then a
//      4-ary tree over the stacked R factors (same kernel, one launch per level).
//      One read of the sub-panel.
//   2. Explicit Q (tsqr_expand_kernel): top-down, Q_node [C; 0] for each node, C being
//      the parent's output block; at the leaves that is the sub-panel's Q, written in
//      place over the leaf reflectors.
//   3. Householder reconstruction (Ballard et al., "Reconstructing Householder vectors
//      from tall-skinny QR"): the LU of Q_top - S with s_i = -sign of the running pivot
//      (recon_lu_kernel) gives V = [L1; Q_bot U^-1] (recon_solve_kernel, one pass),
//      T = -U S L1^-T, tau_i = T_ii and R_householder = S R_tsqr -- the same reflectors
//      LAPACK's dgeqrf produces (up to rounding), built from a stable TSQR.
//   4. The sub-panel's reflectors update the panel's remaining columns:
//      A <- A - V T^T (V^T A), three DMMA GEMMs (dgemm.cu).
//
// Why: cuSOLVER's geqrf on these panels runs ~0.37 ms per column at c4 (3.1M rows;
// ~60 GB/s per pass, column by column), 182 ms per 256-column update.  Here each
// 32-column sub-panel costs a few passes over d x 32 doubles plus its trailing GEMMs.
#include "pw_internal.h"

namespace pw {
namespace {

constexpr int TB = 32;   // sub-panel width (columns)
constexpr int TL = 128;  // rows per TSQR leaf / tree node (4 child R's of <= 32 rows)
constexpr int TTH = 128; // threads per block (4 warps)

struct TsqrArgs {
  double* panel;        // sub-panel (rows x b, column-major, ld lda)
  long long lda;
  long long rows;
  int b;
  int nin;              // node levels: R factors at the level below
  const double* rin;    // node levels: those R factors (b x b each, ld b)
  double* vnode;        // node levels: reflectors [node][TB * TL] (column-major, ld TL)
  double* tau;          // [node][TB]
  double* rout;         // [node][b * b] R factors of this level
  const double* cin;    // expand: the parent level's output blocks [node][TB * TL], or null (root: C = I)
  double* xout;         // expand, node levels: this level's output blocks [node][TB * TL]
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Householder QR (LAPACK dlarfg convention) of X (TL x b, column-major ld TL) in shared
// memory: R in the upper triangle, v_j (implicit unit) below the diagonal, tau[j].
__device__ void block_house_qr(double* X, double* tau, int b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double s_tau;
  for (int j = 0; j < b; ++j) {
    double* xj = X + j * TL;
    if (warp == 0) {
      double ss = 0.0;
#pragma unroll
      for (int k = 0; k < TL / 32; ++k) {
        const int r = lane + 32 * k;
        const double v = (r > j) ? xj[r] : 0.0;
        ss = fma(v, v, ss);
      }
      ss = warp_sum_d(ss);
      const double alpha = xj[j];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (ss > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      __syncwarp();
      if (ss > 0.0) {
#pragma unroll
        for (int k = 0; k < TL / 32; ++k) {
          const int r = lane + 32 * k;
          if (r > j) xj[r] *= scale;
        }
      }
      if (lane == 0) {
        xj[j] = beta;
        tau[j] = t;
        s_tau = t;
      }
    }
    __syncthreads();
    const double t = s_tau;
    if (t != 0.0) {
      for (int c = j + 1 + warp; c < b; c += TTH / 32) {
        double* xc = X + c * TL;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < TL / 32; ++k) {
          const int r = lane + 32 * k;
          if (r > j) acc = fma(xj[r], xc[r], acc);
        }
        acc = warp_sum_d(acc);
        const double w = t * (xc[j] + acc);
#pragma unroll
        for (int k = 0; k < TL / 32; ++k) {
          const int r = lane + 32 * k;
          if (r > j) xc[r] = fma(-w, xj[r], xc[r]);
        }
        if (lane == 0) xc[j] -= w;
      }
    }
    __syncthreads();
  }
}

// X <- Q X with Q = H_0 H_1 ... H_{b-1} (reflectors V, tau); X is TL x b, each warp owns
// whole columns of X, so no barrier is needed between reflectors.
__device__ void block_apply_q(const double* V, const double* tau, double* X, int b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < b; c += TTH / 32) {
    double* xc = X + c * TL;
    double x[TL / 32];
#pragma unroll
    for (int k = 0; k < TL / 32; ++k) x[k] = xc[lane + 32 * k];
    for (int j = b - 1; j >= 0; --j) {
      const double t = tau[j];
      if (t == 0.0) continue;
      const double* vj = V + j * TL;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < TL / 32; ++k) {
        const int r = lane + 32 * k;
        if (r > j) acc = fma(vj[r], x[k], acc);
      }
      acc = warp_sum_d(acc);
      // x_j sits in lane j % 32, slot j / 32
      const double xj = __shfl_sync(0xffffffffu, x[0], j & 31);  // j < 32: slot 0
      const double w = t * (xj + acc);
#pragma unroll
      for (int k = 0; k < TL / 32; ++k) {
        const int r = lane + 32 * k;
        if (r > j) x[k] = fma(-w, vj[r], x[k]);
        else if (r == j) x[k] -= w;
      }
    }
#pragma unroll
    for (int k = 0; k < TL / 32; ++k) xc[lane + 32 * k] = x[k];
  }
}

// Level 0 (LEAF): block i = panel rows [i TL, i TL + TL); level >= 1: block i = the stacked
// R factors 4i .. 4i+3 of the level below.  Writes this block's R, tau and reflectors.
template <bool LEAF>
__global__ void __launch_bounds__(TTH) tsqr_qr_kernel(TsqrArgs a) {
  __shared__ __align__(16) double X[TB * TL];
  __shared__ double tau[TB];
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  for (int e = threadIdx.x; e < TB * TL; e += TTH) {
    const int c = e / TL, r = e - c * TL;
    double v = 0.0;
    if (c < b) {
      if (LEAF) {
        if (r0 + r < a.rows) v = a.panel[r0 + r + (long long)c * a.lda];
      } else {
        const long long child = 4 * i + r / b;
        if (r < 4 * b && child < a.nin) v = a.rin[child * b * b + (r % b) + (long long)c * b];
      }
    }
    X[e] = v;
  }
  __syncthreads();
  block_house_qr(X, tau, b);
  // R (b x b, zero below the diagonal), tau, reflectors
  for (int e = threadIdx.x; e < b * b; e += TTH) {
    const int c = e / b, r = e - c * b;
    a.rout[i * b * b + e] = (r <= c) ? X[c * TL + r] : 0.0;
  }
  if (threadIdx.x < TB) a.tau[i * TB + threadIdx.x] = threadIdx.x < b ? tau[threadIdx.x] : 0.0;
  for (int e = threadIdx.x; e < b * TL; e += TTH) {
    const int c = e / TL, r = e - c * TL;
    if (LEAF) {
      if (r0 + r < a.rows) a.panel[r0 + r + (long long)c * a.lda] = X[e];
    } else {
      a.vnode[i * (TB * TL) + e] = X[e];
    }
  }
}

// Top-down explicit Q: block i's output = Q_i [C_i; 0], C_i = rows (i % 4) b.. of the parent's
// output block (or I at the root).  Leaves write their rows of the sub-panel's Q in place.
template <bool LEAF>
__global__ void __launch_bounds__(TTH) tsqr_expand_kernel(TsqrArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* V = sm;
  double* X = sm + TB * TL;
  __shared__ double tau[TB];
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  for (int e = threadIdx.x; e < TB * TL; e += TTH) {
    const int c = e / TL, r = e - c * TL;
    double v = 0.0, x = 0.0;
    if (c < b) {
      if (LEAF) {
        if (r0 + r < a.rows) v = a.panel[r0 + r + (long long)c * a.lda];
      } else {
        v = a.vnode[i * (TB * TL) + e];
      }
      if (r < b) {
        x = a.cin ? a.cin[(i / 4) * (TB * TL) + (long long)c * TL + (i % 4) * b + r] : (r == c ? 1.0 : 0.0);
      }
    }
    V[e] = v;
    X[e] = x;
  }
  if (threadIdx.x < TB) tau[threadIdx.x] = threadIdx.x < b ? a.tau[i * TB + threadIdx.x] : 0.0;
  __syncthreads();
  block_apply_q(V, tau, X, b);
  __syncthreads();
  for (int e = threadIdx.x; e < b * TL; e += TTH) {
    const int c = e / TL, r = e - c * TL;
    if (LEAF) {
      if (r0 + r < a.rows) a.panel[r0 + r + (long long)c * a.lda] = X[e];
    } else {
      a.xout[i * (TB * TL) + e] = X[e];
    }
  }
}

// Modified LU of Q_top - S (one warp; lane = row): U, s, L1 -> tau, T = -U S L1^-T, the
// explicit unit-lower V_top for the trailing GEMMs, and the panel's top block
// (strict lower = L1, upper = S R).  small: [U (b x b) | Vtop (b x b) | T (b x b)].
__global__ void recon_lu_kernel(double* panel, long long lda, int b, const double* R, double* tau_out,
                                double* small) {
  __shared__ double M[TB][TB + 1];
  __shared__ double Li[TB][TB + 1];  // L1^-1
  __shared__ double s[TB];
  const int lane = threadIdx.x;
  for (int c = 0; c < b; ++c) M[lane][c] = lane < b ? panel[lane + (long long)c * lda] : 0.0;
  __syncwarp();
  for (int i = 0; i < b; ++i) {
    if (lane == 0) {
      const double si = M[i][i] >= 0.0 ? -1.0 : 1.0;  // s_i = -sign(running pivot)
      s[i] = si;
      M[i][i] -= si;
    }
    __syncwarp();
    if (lane > i && lane < b) {
      const double l = M[lane][i] / M[i][i];
      M[lane][i] = l;
      for (int c = i + 1; c < b; ++c) M[lane][c] = fma(-l, M[i][c], M[lane][c]);
    }
    __syncwarp();
  }
  // L1^-1 (unit lower) by columns: lane = column
  if (lane < b) {
    for (int r = 0; r < b; ++r) {
      double v = (r == lane) ? 1.0 : 0.0;
      for (int k = lane; k < r; ++k) v = fma(-M[r][k], Li[k][lane], v);
      Li[r][lane] = (r < lane) ? 0.0 : v;
    }
  }
  __syncwarp();
  double* U = small;
  double* Vt = small + b * b;
  double* T = small + 2 * b * b;
  if (lane < b) {
    const int r = lane;
    for (int c = 0; c < b; ++c) {
      U[r + c * b] = (r <= c) ? M[r][c] : 0.0;
      Vt[r + c * b] = (r > c) ? M[r][c] : (r == c ? 1.0 : 0.0);
      // T[r][c] = -sum_k U[r][k] s_k Li[c][k]   (U upper: k >= r; Li lower: k <= c)
      double t = 0.0;
      for (int k = r; k <= c; ++k) t = fma(M[r][k] * s[k], Li[c][k], t);
      T[r + c * b] = (r <= c) ? -t : 0.0;
    }
    tau_out[r] = -M[r][r] * s[r];
    // panel top block: L1 strictly below the diagonal, S R on and above it
    for (int c = 0; c < b; ++c)
      panel[r + (long long)c * lda] = (r > c) ? M[r][c] : s[r] * R[r + c * b];
  }
}

// V_bot = Q_bot U^-1, one row per thread (rows b .. rows-1), in place.
__global__ void __launch_bounds__(128) recon_solve_kernel(double* panel, long long lda, long long rows, int b,
                                                         const double* U) {
  __shared__ double Us[TB * TB];
  __shared__ double inv[TB];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) Us[e] = U[e];
  __syncthreads();
  if (threadIdx.x < b) inv[threadIdx.x] = 1.0 / Us[threadIdx.x * (b + 1)];
  __syncthreads();
  for (long long r = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    double x[TB];
#pragma unroll
    for (int c = 0; c < TB; ++c)
      if (c < b) x[c] = panel[r + (long long)c * lda];
#pragma unroll
    for (int c = 0; c < TB; ++c) {
      if (c < b) {
        double v = x[c];
#pragma unroll
        for (int k = 0; k < c; ++k) v = fma(-x[k], Us[k + c * b], v);
        x[c] = v * inv[c];
      }
    }
#pragma unroll
    for (int c = 0; c < TB; ++c)
      if (c < b) panel[r + (long long)c * lda] = x[c];
  }
}

size_t expand_smem() { return sizeof(double) * 2 * TB * TL; }

}  // namespace

// geqrf of A (rows x p, ld lda) -> R / V in place, tau (min(rows, p)); see the header.
void tsqr_geqrf(Ctx& c, long long rows, int p, double* A, long long lda, double* tau) {
  const long long kmax = std::min<long long>(rows, p);
  if (kmax <= 0) return;
  // per sub-panel scratch: level sizes of the tree over the leaves
  const long long n0 = (rows + TL - 1) / TL;
  std::vector<long long> nl{n0};
  while (nl.back() > 1) nl.push_back((nl.back() + 3) / 4);
  const int levels = (int)nl.size();
  long long nodes_above = 0;
  for (int l = 1; l < levels; ++l) nodes_above += nl[l];
  // layout: R of every level, tau of every level, node reflectors and node outputs (levels >= 1),
  // small blocks (U, Vtop, T), and the trailing GEMM temporaries (W, X: TB x p each)
  long long total_nodes = n0 + nodes_above;
  const size_t n_r = (size_t)total_nodes * TB * TB;
  const size_t n_tau = (size_t)total_nodes * TB;
  const size_t n_v = (size_t)nodes_above * TB * TL;
  const size_t n_small = 3 * TB * TB;
  const size_t n_w = 2 * (size_t)TB * p;
  double* scr = nullptr;
  const size_t n_all = n_r + n_tau + 2 * n_v + n_small + n_w;
  PW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scr), sizeof(double) * n_all, c.stream));
  double* Rb = scr;
  double* Tb = Rb + n_r;
  double* Vb = Tb + n_tau;
  double* Xb = Vb + n_v;
  double* small = Xb + n_v;
  double* Wt = small + n_small;
  double* Xt = Wt + (size_t)TB * p;
  // offsets of level l in the per-node arrays
  std::vector<long long> off(levels, 0), voff(levels, 0);
  for (int l = 1; l < levels; ++l) {
    off[l] = off[l - 1] + nl[l - 1];
    voff[l] = (l == 1) ? 0 : voff[l - 1] + nl[l - 1];
  }
  kernel_setup(c, tsqr_expand_kernel<true>, TTH, expand_smem());
  kernel_setup(c, tsqr_expand_kernel<false>, TTH, expand_smem());
  for (long long j0 = 0; j0 < kmax; j0 += TB) {
    const int b = (int)std::min<long long>(TB, kmax - j0);
    const long long mrows = rows - j0;
    double* P = A + j0 + j0 * lda;
    // the tree shape depends on mrows: recompute (fewer leaves for later sub-panels)
    std::vector<long long> ml{(mrows + TL - 1) / TL};
    while (ml.back() > 1) ml.push_back((ml.back() + 3) / 4);
    const int L = (int)ml.size();
    TsqrArgs a{};
    a.panel = P;
    a.lda = lda;
    a.rows = mrows;
    a.b = b;
    // 1. TSQR up the tree
    for (int l = 0; l < L; ++l) {
      a.tau = Tb + off[l] * TB;
      a.rout = Rb + off[l] * TB * TB;
      if (l == 0) {
        tsqr_qr_kernel<true><<<(unsigned)ml[0], TTH, 0, c.stream>>>(a);
      } else {
        a.rin = Rb + off[l - 1] * TB * TB;
        a.nin = (int)ml[l - 1];
        a.vnode = Vb + voff[l] * TB * TL;
        tsqr_qr_kernel<false><<<(unsigned)ml[l], TTH, 0, c.stream>>>(a);
      }
      c.launches += 1;
      PW_LAUNCH_CHECK();
    }
    const double* Rroot = Rb + off[L - 1] * TB * TB;
    // 2. explicit Q down the tree
    for (int l = L - 1; l >= 0; --l) {
      a.tau = Tb + off[l] * TB;
      a.cin = (l == L - 1) ? nullptr : Xb + voff[l + 1] * TB * TL;
      if (l == 0) {
        tsqr_expand_kernel<true><<<(unsigned)ml[0], TTH, expand_smem(), c.stream>>>(a);
      } else {
        a.vnode = Vb + voff[l] * TB * TL;
        a.xout = Xb + voff[l] * TB * TL;
        tsqr_expand_kernel<false><<<(unsigned)ml[l], TTH, expand_smem(), c.stream>>>(a);
      }
      c.launches += 1;
      PW_LAUNCH_CHECK();
    }
    // 3. reconstruction
    recon_lu_kernel<<<1, 32, 0, c.stream>>>(P, lda, b, Rroot, tau + j0, small);
    const long long nb = std::max<long long>(1, std::min<long long>((mrows + 127) / 128, 8LL * std::max(c.num_sms, 1)));
    recon_solve_kernel<<<(unsigned)nb, 128, 0, c.stream>>>(P, lda, mrows, b, small);
    c.launches += 2;
    PW_LAUNCH_CHECK();
    // 4. trailing columns: A <- A - V T^T (V^T A),  V = [Vtop; panel rows b..]
    const long long nrest = p - j0 - b;
    if (nrest > 0) {
      double* Ar = A + j0 + (j0 + b) * lda;
      const double* Vtop = small + (size_t)b * b;
      const double* T = small + 2 * (size_t)b * b;
      dgemm(c, true, b, nrest, b, 1.0, Vtop, b, Ar, lda, 0.0, Wt, b);
      if (mrows > b) dgemm(c, true, b, nrest, mrows - b, 1.0, P + b, lda, Ar + b, lda, 1.0, Wt, b);
      dgemm(c, true, b, nrest, b, 1.0, T, b, Wt, b, 0.0, Xt, b);
      dgemm(c, false, b, nrest, b, -1.0, Vtop, b, Xt, b, 1.0, Ar, lda);
      if (mrows > b) dgemm(c, false, mrows - b, nrest, b, -1.0, P + b, lda, Xt, b, 1.0, Ar + b, lda);
    }
  }
  PW_CUDA(cudaFreeAsync(scr, c.stream));
}

}  // namespace pw
