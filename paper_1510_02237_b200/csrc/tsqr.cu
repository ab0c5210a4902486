// Tall-skinny Householder QR of the subspace panel (sm_100a, fp64): the drop-in for LAPACK
// geqrf on the d x P blocks the Krylov basis appends (reference subspace.py:66-68 factors
// all snapshots with scipy qr -> dgeqp3; api.cu keeps the factorisation incremental and
// factors only each update's new block, so this is the O(d P^2) kernel of the update).
//
// Output is geqrf's format (R in the upper triangle, the unit-lower reflectors V below
// the diagonal, tau), so the compact-WY machinery around it (larft, Q1^T N, Q = Q1 Q2)
// is unchanged.  The panel is factored in sub-panels of TB = 32 columns; each one:
//
//   1. TSQR (tsqr_qr_kernel): leaves of 128 rows (4 warps), one CTA each, Householder QR
//      in shared memory (reflectors stored back in place, the leaf R to a buffer); then an
//      8-ary tree over the stacked R factors (8-warp nodes, one launch per level).  Per
//      column one CTA barrier: the column is broadcast inside each warp, only the per-warp
//      partial dot products cross warps (the previous layout published each column through
//      shared memory with two barriers: ~100 us per tree node, latency-bound).
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

constexpr int TB = 32;    // sub-panel width (columns)
constexpr int NWL = 4;    // leaf blocks: 4 warps, 128 rows
constexpr int NWN = 8;    // tree nodes: 8 warps, fan-in 8 (8 stacked child R's of <= 32 rows; 16 warps would spill)
constexpr int TLN = 32 * NWN;

template <int NW>
struct Blk {
  static constexpr int TL = 32 * NW;     // rows per block
  static constexpr int LD = TL + 1;      // shared row stride (odd: lane = column is conflict free)
  static constexpr int NT = 32 * NW;     // threads (one block row each in the load / store phases)
  static constexpr size_t SMEM = sizeof(double) * TB * LD;
};

struct TsqrArgs {
  double* panel;        // sub-panel (rows x b, column-major, ld lda)
  long long lda;
  long long rows;
  int b;
  int nin;              // node levels: R factors at the level below
  const double* rin;    // node levels: those R factors (b x b each, ld b)
  double* vnode;        // node levels: reflectors [node][TB * TLN] (column-major, ld TLN)
  double* tnode;        // [node][TB * TB] compact-WY T of every block (b x b, ld b)
  double* rout;         // [node][b * b] R factors of this level
  const double* cin;    // expand: the parent level's output blocks [node][TB * TLN], or null (root: C = I)
  double* xout;         // expand, node levels: this level's output blocks [node][TB * TLN]
  unsigned long long* prof;  // PW_TSQR_PROF=1: block 0's phase timestamps (globaltimer ns), else null
};

__device__ __forceinline__ void prof_mark(unsigned long long* prof, int k) {
  if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    prof[k] = t;
  }
}

// Thread layout of every block kernel here: lane = column c (0..31), warp = row chunk q
// (rows 32q .. 32q+31 of the block).  A column's dot product is NW per-warp partials summed
// through shared memory in a fixed pairwise order (deterministic).
template <int NW>
__device__ __forceinline__ double sum_parts(const double* p) {
  double s[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) s[w] = p[w];
#pragma unroll
  for (int h = 1; h < NW; h *= 2)
#pragma unroll
    for (int w = 0; w + h < NW; w += 2 * h) s[w] = s[w] + s[w + h];
  return s[0];
}

// Householder QR (LAPACK dlarfg convention) of X (TL x b, column-major, ld LD) in shared
// memory.  Thread (c, q) keeps its 32 entries of column c in registers for the whole
// factorisation.  Per column j: lane j of each warp publishes its chunk of column j to a
// per-warp buffer that the warp reads back as broadcasts, every thread forms its partial
// x_j . x_c, ONE barrier,
// then every thread derives beta, tau, scale and its column's w from the summed partials
// and updates its chunk.  Partials and the row-j entries are double-buffered by j & 1, so
// one barrier per column suffices.  Column j stays unscaled while later columns are
// updated (v_r = x_r * scale[j]).  The j loop is unrolled so register indices stay static.
template <int NW>
__device__ void block_house_qr(double* X, double* tau, double* scale, double (*part)[TB][NW],
                               double (*rowj)[TB], double (*xcol)[32], int b) {
  constexpr int LD = Blk<NW>::LD;
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  double x[32];
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) x[rr] = X[c * LD + q * 32 + rr];
#pragma unroll 1
  for (int j = 0; j < b; ++j) {
    // column j's chunk: lane j stores it (16-byte stores), the warp reads it back as
    // broadcasts -- 32 shared-memory instructions instead of 64 32-bit shuffles
    double xj[32];
    double2* xc = reinterpret_cast<double2*>(xcol[q]);
    if (c == j) {
#pragma unroll
      for (int k = 0; k < 16; ++k) xc[k] = make_double2(x[2 * k], x[2 * k + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 t2 = xc[k];
      xj[2 * k] = t2.x;
      xj[2 * k + 1] = t2.y;
    }
    // every lane computes (lanes of finished or absent columns produce values nobody reads):
    // rows > j only -- in chunk 0 a compile-time mask (j, rr unrolled), the other chunks are
    // all below row 31 (a warp-uniform branch, no per-element selects)
    // 8 accumulator chains of 4 (latency: the column loop is a serial chain of these steps)
    double a8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (q == 0) {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (rr > j) a8[rr & 7] = fma(xj[rr], x[rr], a8[rr & 7]);
    } else {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) a8[rr & 7] = fma(xj[rr], x[rr], a8[rr & 7]);
    }
    part[j & 1][c][q] = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    if (q == 0) {  // row j of every column (alpha = column j's): x[j], j not compile-time --
      double s16[16], s8[8], s4[4], s2[2];  // a 5-level select tree on j's bits
#pragma unroll
      for (int k = 0; k < 16; ++k) s16[k] = (j & 16) ? x[k + 16] : x[k];
#pragma unroll
      for (int k = 0; k < 8; ++k) s8[k] = (j & 8) ? s16[k + 8] : s16[k];
#pragma unroll
      for (int k = 0; k < 4; ++k) s4[k] = (j & 4) ? s8[k + 4] : s8[k];
#pragma unroll
      for (int k = 0; k < 2; ++k) s2[k] = (j & 2) ? s4[k + 2] : s4[k];
      rowj[j & 1][c] = (j & 1) ? s2[1] : s2[0];
    }
    __syncthreads();
    const double dj = sum_parts<NW>(part[j & 1][j]);
    const double alpha = rowj[j & 1][j];
    double t = 0.0, beta = alpha, sc = 0.0;
    if (dj > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, dj)), alpha);
      // one division: inv = 1 / (beta (alpha - beta)); t = (beta - alpha) / beta, sc = 1 / (alpha - beta)
      const double amb = alpha - beta;
      const double inv = 1.0 / (beta * amb);
      t = -amb * amb * inv;
      sc = beta * inv;
    }
    // columns c > j take the reflector; the others update with ws = 0 (x + (-0) xj = x)
    const bool upd = c > j && c < b && t != 0.0;
    const double dc = sum_parts<NW>(part[j & 1][c]);
    const double xcj = rowj[j & 1][c];
    const double w = t * fma(sc, dc, xcj);
    const double ws = upd ? w * sc : 0.0;
    if (q == 0) {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (rr > j) x[rr] = fma(-ws, xj[rr], x[rr]);
      // row j (< 32) lives in chunk 0: the reflector's own row (beta) or the R entry
      const double rj = (c == j) ? beta : xcj - w;
      const bool setj = upd || c == j;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (rr == j && setj) x[rr] = rj;
    } else {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) x[rr] = fma(-ws, xj[rr], x[rr]);
    }
    if (c == j && q == 0) {
      tau[j] = t;
      scale[j] = sc;
    }
  }
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) X[c * LD + q * 32 + rr] = x[rr];
  __syncthreads();
}

// After block_house_qr: R (upper b x b) out, X turned into the explicit unit-lower V in
// place, and the compact-WY T (Q = I - V T V^T, larft) of the block into Tout (b x b).
template <int NW>
__device__ void block_finish(double* X, const double* tau, const double* scale, double* Rout, double* Tout,
                             double (*G)[TB + 1], double (*Wm)[TB + 1], double (*Ym)[TB + 1], int b) {
  constexpr int TL = Blk<NW>::TL, LD = Blk<NW>::LD, NT = Blk<NW>::NT;
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < b * b; e += NT) {
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
  // G = V^T V on the fp64 tensor cores: warp q < 4 computes rows 8q .. 8q+7 of G (four 8 x 8
  // fragments), k over the TL block rows in steps of 4 (m8n8k4: A = V^T rows, B = V cols)
  if (q < 4) {
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
  // V^T V for I - V T V^T = H_0 ... H_{b-1}).  A reflector with tau = 0 (H = I: a zero
  // column in this block) or beyond b has a zero row and column in T: its S row and column
  // are the identity's, inverted as such, and its diagonal zeroed afterwards.  The inverse
  // is built by recursive doubling over the diagonal blocks, all threads at once:
  //   [A B; 0 D]^-1 = [A^-1, -A^-1 (B D^-1); 0, D^-1]  for block sizes 1, 2, 4, 8, 16.
  {
    auto live = [&](int r) { return r < b && tau[r] != 0.0; };
    for (int e = threadIdx.x; e < TB * TB; e += NT) {
      const int r = e / TB, k = e - r * TB;
      Wm[r][k] = (r == k) ? (live(r) ? tau[r] : 1.0) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int sz = 1; sz < TB; sz *= 2) {
      // Y = B D^-1 for every pair of diagonal blocks (o = 2 sz p): B = S[o:o+sz, o+sz:o+2sz]
      for (int e = threadIdx.x; e < (TB / 2) * sz; e += NT) {
        const int pr = e / (sz * sz), rem = e - pr * sz * sz, r = rem / sz, cc = rem - r * sz;
        const int o = 2 * sz * pr, row = o + r, col = o + sz + cc;
        double acc = 0.0;
        for (int k = 0; k <= cc; ++k) {
          const int kk = o + sz + k;  // D^-1 upper triangular
          const double bv = (live(row) && live(kk)) ? G[row][kk] : 0.0;
          acc = fma(bv, Wm[kk][col], acc);
        }
        Ym[row][col] = acc;
      }
      __syncthreads();
      // X = -A^-1 Y into the upper-right block
      for (int e = threadIdx.x; e < (TB / 2) * sz; e += NT) {
        const int pr = e / (sz * sz), rem = e - pr * sz * sz, r = rem / sz, cc = rem - r * sz;
        const int o = 2 * sz * pr, row = o + r, col = o + sz + cc;
        double acc = 0.0;
        for (int k = r; k < sz; ++k) acc = fma(Wm[row][o + k], Ym[o + k][col], acc);  // A^-1 upper
        Wm[row][col] = -acc;
      }
      __syncthreads();
    }
    if (threadIdx.x < TB && !live(threadIdx.x)) Wm[threadIdx.x][threadIdx.x] = 0.0;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += NT) {
    const int cc = e / b, r = e - cc * b;
    Tout[e] = (r <= cc) ? Wm[r][cc] : 0.0;
  }
}

// LEAF (NW = NWL): block i = panel rows [i TL, i TL + TL); nodes (NW = NWN): block i = the
// stacked R factors NW i .. NW i + NW - 1 of the level below.  Writes this block's R, T and
// explicit V.
template <bool LEAF, int NW>
__global__ void __launch_bounds__(32 * NW) tsqr_qr_kernel(TsqrArgs a) {
  constexpr int TL = Blk<NW>::TL, LD = Blk<NW>::LD;
  extern __shared__ __align__(16) double X[];  // TB x LD
  __shared__ double tau[TB], scale[TB];
  __shared__ double part[2][TB][NW];
  __shared__ double rowj[2][TB];
  __shared__ __align__(16) double xcol[NW][32];
  __shared__ double G[TB][TB + 1], Wm[TB][TB + 1], Ym[TB][TB + 1];
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  prof_mark(a.prof, 0);
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
      const long long child = NW * i + r / b;
      if (r < NW * b && child < a.nin) {
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
  prof_mark(a.prof, 1);
  block_house_qr<NW>(X, tau, scale, part, rowj, xcol, b);
  prof_mark(a.prof, 2);
  block_finish<NW>(X, tau, scale, a.rout + i * b * b, a.tnode + i * TB * TB, G, Wm, Ym, b);
  __syncthreads();
  prof_mark(a.prof, 3);
  {
    const int r = threadIdx.x;
    double* dst = LEAF ? ((r0 + r < a.rows) ? a.panel + r0 + r : nullptr) : a.vnode + i * (TB * TLN) + r;
    const long long ld = LEAF ? a.lda : TLN;
    if (dst) {
#pragma unroll
      for (int c = 0; c < TB; ++c)
        if (c < b) dst[c * ld] = X[c * LD + r];
    }
  }
  prof_mark(a.prof, 4);
}

// Top-down explicit Q: block i's output = Q_i [C_i; 0] = [C_i; 0] - V (T (V_top^T C_i)),
// C_i = rows (i % NWN) b .. of the parent's output block (I at the root): two b x b
// products and one TL x b x b product per block, no reductions over rows.  Leaves write
// their rows of the sub-panel's Q in place.
template <bool LEAF, int NW>
__global__ void __launch_bounds__(32 * NW) tsqr_expand_kernel(TsqrArgs a) {
  constexpr int TL = Blk<NW>::TL, LD = Blk<NW>::LD, NT = Blk<NW>::NT;
  constexpr int RPW = TB / NW;  // rows of the b x b products per warp
  extern __shared__ __align__(16) double V[];  // TB x LD, then reused for the output
  __shared__ double C[TB][TB + 1], Y[TB][TB + 1], T[TB][TB + 1];
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  {
    const int r = threadIdx.x;
    const double* src = LEAF ? ((r0 + r < a.rows) ? a.panel + r0 + r : nullptr) : a.vnode + i * (TB * TLN) + r;
    const long long ld = LEAF ? a.lda : TLN;
    double v[TB];
#pragma unroll
    for (int cc = 0; cc < TB; ++cc) v[cc] = (src && cc < b) ? src[cc * ld] : 0.0;
#pragma unroll
    for (int cc = 0; cc < TB; ++cc) V[cc * LD + r] = v[cc];
  }
  for (int e = threadIdx.x; e < TB * TB; e += NT) {
    const int cc = e / TB, r = e - cc * TB;
    double x = 0.0, t = 0.0;
    if (cc < b && r < b) {
      x = a.cin ? a.cin[(i / NWN) * (TB * TLN) + (long long)cc * TLN + (i % NWN) * b + r] : (r == cc ? 1.0 : 0.0);
      t = a.tnode[i * TB * TB + r + cc * b];
    }
    C[r][cc] = x;  // C[row][col]
    T[r][cc] = t;
  }
  __syncthreads();
  // Y = V_top^T C  (thread (c, q): rows RPW q .. RPW q + RPW - 1 of Y, column c)
  double y[RPW];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int row = q * RPW + k;
    double acc = 0.0;
    for (int kk = 0; kk < b; ++kk) acc = fma(V[row * LD + kk], C[kk][c], acc);
    y[k] = acc;
  }
#pragma unroll
  for (int k = 0; k < RPW; ++k) Y[q * RPW + k][c] = y[k];
  __syncthreads();
  // Y2 = T Y   (same ownership; T upper triangular)
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int row = q * RPW + k;
    double acc = 0.0;
    for (int kk = row; kk < b; ++kk) acc = fma(T[row][kk], Y[kk][c], acc);
    y[k] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < RPW; ++k) Y[q * RPW + k][c] = y[k];
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
    double* dst = LEAF ? ((r0 + r < a.rows) ? a.panel + r0 + r : nullptr) : a.xout + i * (TB * TLN) + r;
    const long long ld = LEAF ? a.lda : TLN;
    if (dst) {
#pragma unroll
      for (int cc = 0; cc < TB; ++cc)
        if (cc < b) dst[cc * ld] = V[cc * LD + r];
    }
  }
}

// The leaf level of the explicit-Q pass, thread = row: X = [C; 0] - V (T (V_top^T C)) for the
// 128-row leaf i, written over the leaf's reflectors.  A thread keeps its row of V in registers
// (32 coalesced loads) and forms its 32 outputs against Y2 = T V_top^T C broadcast from shared
// memory -- no staging of the 128 x 32 block through shared memory, six leaves per SM.  Every
// element is accumulated in the order of tsqr_expand_kernel<true> (k ascending, the same fma),
// so the two are bitwise equal (PW_TSQR_EXPAND=1 selects the staged kernel for A/B runs).
__global__ void __launch_bounds__(32 * NWL) tsqr_expand_leaf_rows_kernel(TsqrArgs a) {
  constexpr int TL = Blk<NWL>::TL, NT = Blk<NWL>::NT;
  __shared__ double C[TB][TB + 1], Y[TB][TB + 1], T[TB][TB + 1], Vt[TB][TB + 1];
  __shared__ __align__(16) double Y2t[TB][TB];  // [col][k]: the k pairs a thread walks are 16-byte loads
  const int b = a.b;
  const long long i = blockIdx.x;
  const long long r0 = i * TL;
  const int r = threadIdx.x;
  double* const row = (r0 + r < a.rows) ? a.panel + r0 + r : nullptr;
  double v[TB];
#pragma unroll
  for (int cc = 0; cc < TB; ++cc) v[cc] = (row && cc < b) ? row[cc * a.lda] : 0.0;
  if (r < TB) {
#pragma unroll
    for (int cc = 0; cc < TB; ++cc) Vt[r][cc] = v[cc];
  }
  for (int e = threadIdx.x; e < TB * TB; e += NT) {
    const int cc = e / TB, rr = e - cc * TB;
    double x = 0.0, t = 0.0;
    if (cc < b && rr < b) {
      x = a.cin ? a.cin[(i / NWN) * (TB * TLN) + (long long)cc * TLN + (i % NWN) * b + rr] : (rr == cc ? 1.0 : 0.0);
      t = a.tnode[i * TB * TB + rr + cc * b];
    }
    C[rr][cc] = x;
    T[rr][cc] = t;
  }
  __syncthreads();
  // Y = V_top^T C
  for (int e = threadIdx.x; e < TB * TB; e += NT) {
    const int yr = e / TB, c = e - yr * TB;
    double acc = 0.0;
    for (int kk = 0; kk < b; ++kk) acc = fma(Vt[kk][yr], C[kk][c], acc);
    Y[yr][c] = acc;
  }
  __syncthreads();
  // Y2 = T Y (T upper triangular), stored transposed
  for (int e = threadIdx.x; e < TB * TB; e += NT) {
    const int yr = e / TB, c = e - yr * TB;
    double acc = 0.0;
    for (int kk = yr; kk < b; ++kk) acc = fma(T[yr][kk], Y[kk][c], acc);
    Y2t[c][yr] = acc;
  }
  __syncthreads();
  if (!row) return;
#pragma unroll 1
  for (int c0 = 0; c0 < TB; c0 += 4) {
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = (r < TB) ? C[r][c0 + u] : 0.0;
#pragma unroll
    for (int k2 = 0; k2 < TB / 2; ++k2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 y2 = *reinterpret_cast<const double2*>(&Y2t[c0 + u][2 * k2]);
        x[u] = fma(-v[2 * k2], y2.x, x[u]);
        x[u] = fma(-v[2 * k2 + 1], y2.y, x[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < b) row[(long long)(c0 + u) * a.lda] = x[u];
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



// Trailing update of a sub-panel, C (rows x n, ld ldc) -= V (rows x TB, ld ldv) X (TB x n, ld TB):
// the rank-32 GEMM the generic tiles run 3.5x off the HBM roofline (one 128 x 64 tile per CTA
// with a 32-deep k loop is all prologue and epilogue).  Streaming form: a thread owns one row,
// keeps its 32 entries of V in registers, and walks the columns of C (coalesced 256-byte column
// segments per warp) with X broadcast from shared memory; 8 columns in flight per thread.
// Bytes: rows x (2 n + TB) x 8; flops 2 x rows x n x TB on the DFMA pipe -- about balanced.
constexpr int kRkThreads = 256;
__global__ void __launch_bounds__(kRkThreads, 2) rank_tb_update_kernel(const double* __restrict__ V, long long ldv,
                                                                       const double* __restrict__ X, int n,
                                                                       double* __restrict__ C, long long ldc,
                                                                       long long rows) {
  extern __shared__ double xs[];  // TB x n, column-major (ld TB)
  for (int e = threadIdx.x; e < TB * n; e += blockDim.x) xs[e] = X[e];
  __syncthreads();
  for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < rows;
       row += (long long)gridDim.x * blockDim.x) {
    double v[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) v[k] = V[row + k * ldv];
    double* crow = C + row;
    int j = 0;
    for (; j + 8 <= n; j += 8) {
      double cc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cc[u] = crow[(long long)(j + u) * ldc];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2* xc = reinterpret_cast<const double2*>(xs + (size_t)(j + u) * TB);
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < TB / 2; ++k) {
          const double2 x2 = xc[k];
          acc = fma(v[2 * k], x2.x, acc);
          acc = fma(v[2 * k + 1], x2.y, acc);
        }
        cc[u] -= acc;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) crow[(long long)(j + u) * ldc] = cc[u];
    }
    for (; j < n; ++j) {
      const double* xc = xs + (size_t)j * TB;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < TB; ++k) acc = fma(v[k], xc[k], acc);
      crow[(long long)j * ldc] -= acc;
    }
  }
}

void launch_rank_tb_update(Ctx& c, const double* V, long long ldv, const double* X, int n, double* C, long long ldc,
                           long long rows) {
  const size_t smem = sizeof(double) * TB * (size_t)n;
  // set up once for the widest X (n <= 256: 64 KB), whatever this call's n
  const int per_sm = kernel_setup(c, rank_tb_update_kernel, kRkThreads, sizeof(double) * TB * 256);
  const long long want = (rows + kRkThreads - 1) / kRkThreads;
  const int grid = (int)std::max<long long>(1, std::min<long long>(want, (long long)std::max(c.num_sms, 1) * per_sm * 4));
  rank_tb_update_kernel<<<grid, kRkThreads, smem, c.stream>>>(V, ldv, X, n, C, ldc, rows);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

}  // namespace

// geqrf of A (rows x p, ld lda) -> R / V in place, tau (min(rows, p)); see the header.
void tsqr_geqrf(Ctx& c, long long rows, int p, double* A, long long lda, double* tau) {
  const long long kmax = std::min<long long>(rows, p);
  if (kmax <= 0) return;
  // per sub-panel scratch: level sizes of the tree over the leaves (leaves of 128 rows, nodes
  // of fan-in NWN)
  const long long n0 = (rows + Blk<NWL>::TL - 1) / Blk<NWL>::TL;
  std::vector<long long> nl{n0};
  while (nl.back() > 1) nl.push_back((nl.back() + NWN - 1) / NWN);
  const int levels = (int)nl.size();
  long long nodes_above = 0;
  for (int l = 1; l < levels; ++l) nodes_above += nl[l];
  // layout: R of every level, T of every level, node reflectors and node outputs (levels >= 1),
  // small blocks (U, Vtop, T), and the trailing GEMM temporaries (W, X: TB x p each)
  long long total_nodes = n0 + nodes_above;
  const size_t n_r = (size_t)total_nodes * TB * TB;
  const size_t n_tau = (size_t)total_nodes * TB * TB;  // T of every block
  const size_t n_v = (size_t)nodes_above * TB * TLN;
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
  kernel_setup(c, tsqr_qr_kernel<true, NWL>, Blk<NWL>::NT, Blk<NWL>::SMEM);
  kernel_setup(c, tsqr_qr_kernel<false, NWN>, Blk<NWN>::NT, Blk<NWN>::SMEM);
  kernel_setup(c, tsqr_expand_kernel<true, NWL>, Blk<NWL>::NT, Blk<NWL>::SMEM);
  kernel_setup(c, tsqr_expand_kernel<false, NWN>, Blk<NWN>::NT, Blk<NWN>::SMEM);
  // PW_TSQR_PROF=1: phase timestamps of block 0 of the last tree level's QR (debug)
  unsigned long long* prof = nullptr;
  const char* pe = getenv("PW_TSQR_PROF");
  if (pe && *pe == '1') PW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&prof), 8 * 8, c.stream));
  for (long long j0 = 0; j0 < kmax; j0 += TB) {
    const int b = (int)std::min<long long>(TB, kmax - j0);
    const long long mrows = rows - j0;
    double* P = A + j0 + j0 * lda;
    // the tree shape depends on mrows: recompute (fewer leaves for later sub-panels)
    std::vector<long long> ml{(mrows + Blk<NWL>::TL - 1) / Blk<NWL>::TL};
    while (ml.back() > 1) ml.push_back((ml.back() + NWN - 1) / NWN);
    const int L = (int)ml.size();
    TsqrArgs a{};
    a.prof = prof;
    a.panel = P;
    a.lda = lda;
    a.rows = mrows;
    a.b = b;
    // 1. TSQR up the tree
    for (int l = 0; l < L; ++l) {
      a.tnode = Tb + off[l] * TB * TB;
      a.rout = Rb + off[l] * TB * TB;
      if (l == 0) {
        tsqr_qr_kernel<true, NWL><<<(unsigned)ml[0], Blk<NWL>::NT, Blk<NWL>::SMEM, c.stream>>>(a);
      } else {
        a.rin = Rb + off[l - 1] * TB * TB;
        a.nin = (int)ml[l - 1];
        a.vnode = Vb + voff[l] * TB * TLN;
        tsqr_qr_kernel<false, NWN><<<(unsigned)ml[l], Blk<NWN>::NT, Blk<NWN>::SMEM, c.stream>>>(a);
      }
      c.launches += 1;
      PW_LAUNCH_CHECK();
    }
    const double* Rroot = Rb + off[L - 1] * TB * TB;
    // 2. explicit Q down the tree
    for (int l = L - 1; l >= 0; --l) {
      a.tnode = Tb + off[l] * TB * TB;
      a.cin = (l == L - 1) ? nullptr : Xb + voff[l + 1] * TB * TLN;
      if (l == 0) {
        const char* se = getenv("PW_TSQR_EXPAND");
        const bool staged = se && atoi(se) == 1;
        if (staged)
          tsqr_expand_kernel<true, NWL><<<(unsigned)ml[0], Blk<NWL>::NT, Blk<NWL>::SMEM, c.stream>>>(a);
        else
          tsqr_expand_leaf_rows_kernel<<<(unsigned)ml[0], Blk<NWL>::NT, 0, c.stream>>>(a);
      } else {
        a.vnode = Vb + voff[l] * TB * TLN;
        a.xout = Xb + voff[l] * TB * TLN;
        tsqr_expand_kernel<false, NWN><<<(unsigned)ml[l], Blk<NWN>::NT, Blk<NWN>::SMEM, c.stream>>>(a);
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
      if (mrows > b) {
        // b == TB except for a ragged last sub-panel (none follows it: nrest == 0 there)
        const char* ge = getenv("PW_TSQR_TRAIL_GEMM");
        const bool generic = ge && atoi(ge) == 1;
        if (b == TB && nrest <= 256 && !generic)
          launch_rank_tb_update(c, P + b, lda, Xt, (int)nrest, Ar + b, lda, mrows - b);
        else
          dgemm(c, false, mrows - b, nrest, b, -1.0, P + b, lda, Xt, b, 1.0, Ar + b, lda);
      }
    }
  }
  PW_CUDA(cudaFreeAsync(scr, c.stream));
  if (prof) {
    unsigned long long t[8];
    PW_CUDA(cudaMemcpyAsync(t, prof, sizeof(t), cudaMemcpyDeviceToHost, c.stream));
    PW_CUDA(cudaStreamSynchronize(c.stream));
    fprintf(stderr, "[tsqr prof] load %.1f us  house %.1f us  finish %.1f us  store %.1f us\n", (t[1] - t[0]) * 1e-3,
            (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3);
    PW_CUDA(cudaFreeAsync(prof, c.stream));
  }
}

}  // namespace pw
