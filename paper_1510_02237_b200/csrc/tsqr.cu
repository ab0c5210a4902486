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
  double* tau;          // [node][TB]  (unused by the kernels: T carries tau on its diagonal)
  double* tnode;        // [node][TB * TB] compact-WY T of every block (b x b, ld b)
  double* rout;         // [node][b * b] R factors of this level
  const double* cin;    // expand: the parent level's output blocks [node][TB * TL], or null (root: C = I)
  double* xout;         // expand, node levels: this level's output blocks [node][TB * TL]
};

constexpr int LD = TL + 1;  // shared row stride of a TL x TB block (odd: lane = column is conflict free)

// Thread layout of every block kernel here: lane = column c (0..31), warp = row chunk q
// (rows 32q .. 32q+31 of the 128-row block).  A column's dot product is four per-warp
// partials summed through shared memory -- no shuffle reductions on the critical path.

// Householder QR (LAPACK dlarfg convention) of X (TL x b, column-major, ld LD) in shared
// memory.  Thread (c, q) keeps its 32 entries of column c in registers for the whole
// factorisation; per column j the owner threads (j, q) publish column j through a
// shared buffer (read back as broadcasts), so the shared-memory traffic per step is one
// column instead of the whole block.  Column j stays unscaled while later columns are
// updated (v_r = x_r * scale[j]); one barrier pair per column: partial dots x_j . x_c
// for every c >= j (which include ||x_j||), then every thread derives beta, tau, scale
// and its column's w itself.  The j loop is unrolled so register indices stay static.
__device__ void block_house_qr(double* X, double* tau, double* scale, double (*part)[TB][4], double (*xb)[TL],
                               double* xcj_s, int b) {
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  double x[32];
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) x[rr] = X[c * LD + q * 32 + rr];
  if (c == 0) {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) xb[0][q * 32 + rr] = x[rr];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    if (j >= b) break;
    double (*pd)[4] = part[j & 1];
    const double* xjs = xb[j & 1];
    double xj[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) xj[rr] = xjs[q * 32 + rr];
    const double alpha = xjs[j];
    double acc = 0.0;
    if (c >= j && c < b) {
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (q > 0 || rr > j) a4[rr & 3] = fma(xj[rr], x[rr], a4[rr & 3]);
      acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    }
    pd[c][q] = acc;
    if (q == 0) xcj_s[c] = x[j];
    __syncthreads();
    const double dj = (pd[j][0] + pd[j][1]) + (pd[j][2] + pd[j][3]);
    double t = 0.0, beta = alpha, sc = 0.0;
    if (dj > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, dj)), alpha);
      t = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    if (c > j && c < b && t != 0.0) {
      const double dc = (pd[c][0] + pd[c][1]) + (pd[c][2] + pd[c][3]);
      const double xcj = xcj_s[c];
      const double w = t * fma(sc, dc, xcj);
      const double ws = w * sc;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (q > 0 || rr > j) x[rr] = fma(-ws, xj[rr], x[rr]);
      if (q == 0) x[j] = xcj - w;  // row j (< 32) lives in chunk 0
    }
    if (c == j) {
      if (q == 0) {
        x[j] = beta;
        tau[j] = t;
        scale[j] = sc;
      }
    }
    if (c == j + 1 && j + 1 < b) {  // publish the next column (updated above)
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) xb[(j + 1) & 1][q * 32 + rr] = x[rr];
    }
    __syncthreads();
  }
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) X[c * LD + q * 32 + rr] = x[rr];
  __syncthreads();
}

// After block_house_qr: R (upper b x b) out, X turned into the explicit unit-lower V in
// place, and the compact-WY T (Q = I - V T V^T, larft) of the block into Tout (b x b).
__device__ void block_finish(double* X, const double* tau, const double* scale, double* Rout, double* Tout,
                             double (*G)[TB + 1], int b) {
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < b * b; e += TTH) {
    const int cc = e / b, r = e - cc * b;
    Rout[e] = (r <= cc) ? X[cc * LD + r] : 0.0;
  }
  __syncthreads();
  if (c < b) {
    const double sc = scale[c];
    for (int rr = 0; rr < 32; ++rr) {
      const int r = q * 32 + rr;
      double* p = X + c * LD + r;
      *p = (r > c) ? *p * sc : (r == c ? 1.0 : 0.0);
    }
  }
  __syncthreads();
  // G = V^T V on the fp64 tensor cores: warp q computes rows 8q .. 8q+7 of G (four 8 x 8
  // fragments), k over the TL block rows in steps of 4 (m8n8k4: A = V^T rows, B = V cols)
  {
    const int ar = c >> 2, ak = c & 3;
    double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
    for (int k0 = 0; k0 < TL; k0 += 4) {
      const double av = X[(q * 8 + ar) * LD + k0 + ak];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const double bv = X[(f * 8 + ar) * LD + k0 + ak];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[f][0]), "+d"(acc[f][1])
                     : "d"(av), "d"(bv));
      }
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      G[q * 8 + ar][f * 8 + 2 * ak] = acc[f][0];
      G[q * 8 + ar][f * 8 + 2 * ak + 1] = acc[f][1];
    }
  }
  __syncthreads();
  // T by the UT transform: T = S^-1, S = strict_upper(G) + diag(1 / tau) (T^-1 + T^-T =
  // V^T V for I - V T V^T = H_0 ... H_{b-1}).  Warp 0, lane = column c of T, back
  // substitution bottom-up with the column in registers (no serial chain across lanes).
  // A reflector with tau = 0 (H = I: a zero column in this block) has a zero row and column
  // in T: its S row / column are masked out of the solve.
  if (q == 0) {
    double tcol[TB];
    const bool live_c = c < b && tau[c] != 0.0;
#pragma unroll
    for (int r = TB - 1; r >= 0; --r) {
      double v = 0.0;
      if (live_c && r <= c && r < b && tau[r] != 0.0) {
        if (r == c) {
          v = tau[c];
        } else {
          double a2[2] = {0.0, 0.0};
#pragma unroll
          for (int k = r + 1; k < TB; ++k)
            if (k <= c) a2[k & 1] = fma(G[r][k], tcol[k], a2[k & 1]);
          v = -tau[r] * (a2[0] + a2[1]);
        }
      }
      tcol[r] = v;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < TB; ++r)
      if (r < c) G[c][r] = tcol[r];  // T's strict upper part, transposed into G's strict lower part
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b * b; e += TTH) {
    const int cc = e / b, r = e - cc * b;
    Tout[e] = (r < cc) ? G[cc][r] : (r == cc ? tau[r] : 0.0);
  }
}

// Level 0 (LEAF): block i = panel rows [i TL, i TL + TL); level >= 1: block i = the stacked
// R factors 4i .. 4i+3 of the level below.  Writes this block's R, T and explicit V.
template <bool LEAF>
__global__ void __launch_bounds__(TTH) tsqr_qr_kernel(TsqrArgs a) {
  extern __shared__ __align__(16) double X[];  // TB x LD
  __shared__ double tau[TB], scale[TB];
  __shared__ double part[2][TB][4];
  __shared__ double G[TB][TB + 1];
  __shared__ double xb[2][TL];
  __shared__ double xcj_s[TB];
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  static_assert(TTH == TL, "one block row per thread in the load / store phases");
  {
    // thread = row: all 32 loads in flight before the first shared store (coalesced per column)
    const int r = threadIdx.x;
    double v[TB];
    const double* src = nullptr;
    long long ld = 0;
    if (LEAF) {
      if (r0 + r < a.rows) {
        src = a.panel + r0 + r;
        ld = a.lda;
      }
    } else {
      const long long child = 4 * i + r / b;
      if (r < 4 * b && child < a.nin) {
        src = a.rin + child * b * b + (r % b);
        ld = b;
      }
    }
#pragma unroll
    for (int c = 0; c < TB; ++c) v[c] = (src && c < b) ? src[c * ld] : 0.0;
#pragma unroll
    for (int c = 0; c < TB; ++c) X[c * LD + r] = v[c];
  }
  __syncthreads();
  block_house_qr(X, tau, scale, part, xb, xcj_s, b);
  block_finish(X, tau, scale, a.rout + i * b * b, a.tnode + i * TB * TB, G, b);
  __syncthreads();
  {
    const int r = threadIdx.x;
    double* dst = LEAF ? ((r0 + r < a.rows) ? a.panel + r0 + r : nullptr) : a.vnode + i * (TB * TL) + r;
    const long long ld = LEAF ? a.lda : TL;
    if (dst) {
#pragma unroll
      for (int c = 0; c < TB; ++c)
        if (c < b) dst[c * ld] = X[c * LD + r];
    }
  }
}

// Top-down explicit Q: block i's output = Q_i [C_i; 0] = [C_i; 0] - V (T (V_top^T C_i)),
// C_i = rows (i % 4) b .. of the parent's output block (I at the root): two b x b products
// and one TL x b x b product per block, no reductions over rows.  Leaves write their rows
// of the sub-panel's Q in place.
template <bool LEAF>
__global__ void __launch_bounds__(TTH) tsqr_expand_kernel(TsqrArgs a) {
  extern __shared__ __align__(16) double V[];  // TB x LD, then reused for the output
  __shared__ double C[TB][TB + 1], Y[TB][TB + 1], T[TB][TB + 1];
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  {
    const int r = threadIdx.x;
    const double* src = LEAF ? ((r0 + r < a.rows) ? a.panel + r0 + r : nullptr) : a.vnode + i * (TB * TL) + r;
    const long long ld = LEAF ? a.lda : TL;
    double v[TB];
#pragma unroll
    for (int cc = 0; cc < TB; ++cc) v[cc] = (src && cc < b) ? src[cc * ld] : 0.0;
#pragma unroll
    for (int cc = 0; cc < TB; ++cc) V[cc * LD + r] = v[cc];
  }
  for (int e = threadIdx.x; e < TB * TB; e += TTH) {
    const int cc = e / TB, r = e - cc * TB;
    double x = 0.0, t = 0.0;
    if (cc < b && r < b) {
      x = a.cin ? a.cin[(i / 4) * (TB * TL) + (long long)cc * TL + (i % 4) * b + r] : (r == cc ? 1.0 : 0.0);
      t = a.tnode[i * TB * TB + r + cc * b];
    }
    C[r][cc] = x;  // C[row][col]
    T[r][cc] = t;
  }
  __syncthreads();
  // Y = V_top^T C  (thread (c, q): rows 8q .. 8q+7 of Y, column c)
  double y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int row = q * 8 + k;
    double acc = 0.0;
    for (int kk = 0; kk < b; ++kk) acc = fma(V[row * LD + kk], C[kk][c], acc);
    y[k] = acc;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) Y[q * 8 + k][c] = y[k];
  __syncthreads();
  // Y2 = T Y   (same ownership; T upper triangular)
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int row = q * 8 + k;
    double acc = 0.0;
    for (int kk = row; kk < b; ++kk) acc = fma(T[row][kk], Y[kk][c], acc);
    y[k] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; ++k) Y[q * 8 + k][c] = y[k];
  __syncthreads();
  // X = [C; 0] - V Y2: thread (c, q) computes rows 32q .. 32q+31 of column c
  double x[32];
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    const int r = q * 32 + rr;
    x[rr] = (r < TB) ? C[r][c] : 0.0;
  }
  for (int kk = 0; kk < b; ++kk) {
    const double ykk = Y[kk][c];
    const double* vk = V + kk * LD + q * 32;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) x[rr] = fma(-vk[rr], ykk, x[rr]);
  }
  __syncthreads();  // everyone done reading V: reuse it for the output
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) V[c * LD + q * 32 + rr] = x[rr];
  __syncthreads();
  {
    const int r = threadIdx.x;
    double* dst = LEAF ? ((r0 + r < a.rows) ? a.panel + r0 + r : nullptr) : a.xout + i * (TB * TL) + r;
    const long long ld = LEAF ? a.lda : TL;
    if (dst) {
#pragma unroll
      for (int cc = 0; cc < TB; ++cc)
        if (cc < b) dst[cc * ld] = V[cc * LD + r];
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

size_t block_smem() { return sizeof(double) * TB * LD; }

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
  const size_t n_tau = (size_t)total_nodes * TB * TB;  // T of every block
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
  kernel_setup(c, tsqr_qr_kernel<true>, TTH, block_smem());
  kernel_setup(c, tsqr_qr_kernel<false>, TTH, block_smem());
  kernel_setup(c, tsqr_expand_kernel<true>, TTH, block_smem());
  kernel_setup(c, tsqr_expand_kernel<false>, TTH, block_smem());
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
      a.tnode = Tb + off[l] * TB * TB;
      a.rout = Rb + off[l] * TB * TB;
      if (l == 0) {
        tsqr_qr_kernel<true><<<(unsigned)ml[0], TTH, block_smem(), c.stream>>>(a);
      } else {
        a.rin = Rb + off[l - 1] * TB * TB;
        a.nin = (int)ml[l - 1];
        a.vnode = Vb + voff[l] * TB * TL;
        tsqr_qr_kernel<false><<<(unsigned)ml[l], TTH, block_smem(), c.stream>>>(a);
      }
      c.launches += 1;
      PW_LAUNCH_CHECK();
    }
    const double* Rroot = Rb + off[L - 1] * TB * TB;
    // 2. explicit Q down the tree
    for (int l = L - 1; l >= 0; --l) {
      a.tnode = Tb + off[l] * TB * TB;
      a.cin = (l == L - 1) ? nullptr : Xb + voff[l + 1] * TB * TL;
      if (l == 0) {
        tsqr_expand_kernel<true><<<(unsigned)ml[0], TTH, block_smem(), c.stream>>>(a);
      } else {
        a.vnode = Vb + voff[l] * TB * TL;
        a.xout = Xb + voff[l] * TB * TL;
        tsqr_expand_kernel<false><<<(unsigned)ml[l], TTH, block_smem(), c.stream>>>(a);
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
