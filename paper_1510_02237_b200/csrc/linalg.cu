// Krylov-subspace linear algebra for the KSE correction (sm_100a, fp64).
//
//  * pivoted_qr_small   -- column-pivoted Householder QR of the m x m triangular
//                          factor R1 of the snapshot block (one cooperative
//                          launch, 2 grid barriers per column).  Pivoted QR of
//                          R1 has the pivots of dgeqp3 on the snapshots
//                          themselves (subspace.py:67-68), see DESIGN.md.
//  * form_q2            -- explicit Q2[:, :r] from the reflectors (dorgqr role)
//  * tri_inverse_scatter-- scatter(R11^-1) of subspace.py:76-78
//  * larft_cols         -- the dlarft recurrence for the compact-WY T of a new panel
//  * make_unit_lower    -- geqrf output -> explicit unit-lower Householder vectors
//  * combine_tma /      -- the serial correction step of the KSE sweep,
//    combine_gemv          qn[i+1] = G(qn[i]) + D alpha_i + c_i fused with the
//                          next projection coefficients alpha_{i+1} = Q^T qn[i+1]
//                          (one HBM pass over D and Q: 2 r d 8 bytes); the TMA
//                          bulk-copy kernel by default, the LSU kernel otherwise
//  * residual           -- iteration_residual (parareal.py:50-59)
#include <cooperative_groups.h>

#include "pw_internal.h"

namespace cg = cooperative_groups;

namespace pw {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
  return v;
}

// ---------------------------------------------------------------- small pivoted QR
constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;

// A: mr x m column-major (lda = mr), mr = min(d, m) rows of R1.  Steps j < min(mr, m).
__global__ void __launch_bounds__(kQrThreads) pqr_kernel(double* A, int mr, int m, int* piv,
                                                         double* tau, double* norms, double* diag) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned done[64];  // m <= 2048
  __shared__ double red_v[kQrWarps];
  __shared__ int red_i[kQrWarps];
  __shared__ int s_p;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kQrWarps + warp;
  const int nwarps = gridDim.x * kQrWarps;
  const int steps = mr < m ? mr : m;
  for (int k = threadIdx.x; k < 64; k += blockDim.x) done[k] = 0u;
  // initial column norms
  for (int c = gwarp; c < m; c += nwarps) {
    const double* col = A + (size_t)c * mr;
    double s = 0.0;
    for (int i = lane; i < mr; i += 32) s = fma(col[i], col[i], s);
    s = warp_sum(s);
    if (lane == 0) norms[c] = sqrt(s);
  }
  grid.sync();
  for (int j = 0; j < steps; ++j) {
    // pivot: max remaining norm, lowest index on ties (idamax semantics)
    double best = -1.0;
    int bi = m;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      if (done[c >> 5] & (1u << (c & 31))) continue;
      const double v = norms[c];
      if (v > best || (v == best && c < bi)) { best = v; bi = c; }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double ov = __shfl_xor_sync(FULL, best, off);
      const int oi = __shfl_xor_sync(FULL, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = best; red_i[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = red_v[0];
      int bidx = red_i[0];
      for (int w = 1; w < kQrWarps; ++w)
        if (red_v[w] > b || (red_v[w] == b && red_i[w] < bidx)) { b = red_v[w]; bidx = red_i[w]; }
      s_p = bidx;
      done[bidx >> 5] |= (1u << (bidx & 31));
    }
    __syncthreads();
    const int p = s_p;
    // Householder reflector of column p, rows j..mr-1 (dlarfg)
    if (gwarp == p % nwarps) {
      double* col = A + (size_t)p * mr;
      double s = 0.0;
      for (int i = j + 1 + lane; i < mr; i += 32) s = fma(col[i], col[i], s);
      s = warp_sum(s);
      const double alpha = col[j];
      double t = 0.0, beta = alpha;
      if (s != 0.0) {
        const double xnorm = sqrt(s);
        beta = -copysign(hypot(alpha, xnorm), alpha);
        t = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        for (int i = j + 1 + lane; i < mr; i += 32) col[i] *= scal;
      }
      __syncwarp();
      if (lane == 0) {
        col[j] = beta;
        tau[j] = t;
        piv[j] = p;
        diag[j] = fabs(beta);
      }
    }
    grid.sync();
    // apply H_j to the remaining columns; recompute their trailing norms
    const double t = tau[j];
    const double* v = A + (size_t)p * mr;
    for (int c = gwarp; c < m; c += nwarps) {
      if (done[c >> 5] & (1u << (c & 31))) continue;
      double* col = A + (size_t)c * mr;
      double w = 0.0;
      for (int i = j + 1 + lane; i < mr; i += 32) w = fma(v[i], col[i], w);
      w = warp_sum(w) + col[j];
      const double tw = t * w;
      double s = 0.0;
      for (int i = j + 1 + lane; i < mr; i += 32) {
        const double x = col[i] - tw * v[i];
        col[i] = x;
        s = fma(x, x, s);
      }
      s = warp_sum(s);
      if (lane == 0) {
        col[j] -= tw;
        norms[c] = sqrt(s);
      }
    }
    grid.sync();
  }
  // columns never pivoted (m > mr): record them after the pivoted ones
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int k = steps;
    for (int c = 0; c < m && k < m; ++c)
      if (!(done[c >> 5] & (1u << (c & 31)))) piv[k++] = c;
  }
}

// The same factorisation with ONE grid barrier per column (default; PW_PQR=2 selects the
// two-barrier kernel above for A/B runs).  After the barrier that publishes the updated columns
// and norms, EVERY block finds the pivot and forms the reflector of the pivot column itself
// (warp 0, from the unscaled column in global memory into shared memory): the same
// instruction sequence on the same operands in every block, so the blocks agree bit for bit
// and the second barrier (pivot owner -> everyone) disappears.  The owner's in-place write of
// the scaled reflector, beta, tau and the pivot index is deferred until after the next barrier,
// when no block reads the unscaled column any more (the reflector buffer is double-buffered by
// step parity).  Results are bitwise equal to pqr_kernel (tests/test_gpu_tsqr.py).
constexpr int kQrMaxRows = 2048;
__global__ void __launch_bounds__(kQrThreads) pqr1_kernel(double* A, int mr, int m, int* piv,
                                                          double* tau, double* norms, double* diag) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned done[64];  // m <= 2048
  __shared__ double red_v[kQrWarps];
  __shared__ int red_i[kQrWarps];
  __shared__ int s_p;
  __shared__ double s_t[2], s_beta[2];
  __shared__ double vbuf[2][kQrMaxRows];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kQrWarps + warp;
  const int nwarps = gridDim.x * kQrWarps;
  const int steps = mr < m ? mr : m;
  for (int k = threadIdx.x; k < 64; k += blockDim.x) done[k] = 0u;
  for (int c = gwarp; c < m; c += nwarps) {
    const double* col = A + (size_t)c * mr;
    double s = 0.0;
    for (int i = lane; i < mr; i += 32) s = fma(col[i], col[i], s);
    s = warp_sum(s);
    if (lane == 0) norms[c] = sqrt(s);
  }
  grid.sync();
  int p_prev = -1;
  for (int j = 0; j <= steps; ++j) {
    // deferred in-place write of step j-1's reflector by its owner block (the column is done:
    // nobody reads it any more)
    if (j > 0 && (int)blockIdx.x == p_prev % (int)gridDim.x) {
      double* col = A + (size_t)p_prev * mr;
      const double* v = vbuf[(j - 1) & 1];
      for (int i = j + threadIdx.x; i < mr; i += blockDim.x) col[i] = v[i];
      if (threadIdx.x == 0) {
        col[j - 1] = s_beta[(j - 1) & 1];
        tau[j - 1] = s_t[(j - 1) & 1];
        piv[j - 1] = p_prev;
        diag[j - 1] = fabs(s_beta[(j - 1) & 1]);
      }
    }
    if (j == steps) break;
    // pivot: max remaining norm, lowest index on ties (idamax semantics)
    double best = -1.0;
    int bi = m;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      if (done[c >> 5] & (1u << (c & 31))) continue;
      const double v = norms[c];
      if (v > best || (v == best && c < bi)) { best = v; bi = c; }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double ov = __shfl_xor_sync(FULL, best, off);
      const int oi = __shfl_xor_sync(FULL, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = best; red_i[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = red_v[0];
      int bidx = red_i[0];
      for (int w = 1; w < kQrWarps; ++w)
        if (red_v[w] > b || (red_v[w] == b && red_i[w] < bidx)) { b = red_v[w]; bidx = red_i[w]; }
      s_p = bidx;
      done[bidx >> 5] |= (1u << (bidx & 31));
    }
    __syncthreads();
    const int p = s_p;
    double* vj = vbuf[j & 1];
    // Householder reflector of column p, rows j..mr-1 (dlarfg), formed by every block
    if (warp == 0) {
      const double* col = A + (size_t)p * mr;
      double s = 0.0;
      for (int i = j + 1 + lane; i < mr; i += 32) s = fma(col[i], col[i], s);
      s = warp_sum(s);
      const double alpha = col[j];
      double t = 0.0, beta = alpha;
      if (s != 0.0) {
        const double xnorm = sqrt(s);
        beta = -copysign(hypot(alpha, xnorm), alpha);
        t = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        for (int i = j + 1 + lane; i < mr; i += 32) vj[i] = col[i] * scal;
      } else {
        for (int i = j + 1 + lane; i < mr; i += 32) vj[i] = col[i];
      }
      if (lane == 0) {
        s_t[j & 1] = t;
        s_beta[j & 1] = beta;
      }
    }
    __syncthreads();
    // apply H_j to the remaining columns; recompute their trailing norms
    const double t = s_t[j & 1];
    for (int c = gwarp; c < m; c += nwarps) {
      if (done[c >> 5] & (1u << (c & 31))) continue;
      double* col = A + (size_t)c * mr;
      double w = 0.0;
      for (int i = j + 1 + lane; i < mr; i += 32) w = fma(vj[i], col[i], w);
      w = warp_sum(w) + col[j];
      const double tw = t * w;
      double s = 0.0;
      for (int i = j + 1 + lane; i < mr; i += 32) {
        const double x = col[i] - tw * vj[i];
        col[i] = x;
        s = fma(x, x, s);
      }
      s = warp_sum(s);
      if (lane == 0) {
        col[j] -= tw;
        norms[c] = sqrt(s);
      }
    }
    p_prev = p;
    grid.sync();
  }
  // columns never pivoted (m > mr): record them after the pivoted ones
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int k = steps;
    for (int c = 0; c < m && k < m; ++c)
      if (!(done[c >> 5] & (1u << (c & 31)))) piv[k++] = c;
  }
}

// Q2[:, c] = H_0 ... H_c e_c  (c < r), one warp per column, x staged in smem
constexpr int kQ2Warps = 4;
__global__ void __launch_bounds__(kQ2Warps * 32) form_q2_kernel(const double* A, int mr,
                                                                 const int* piv, const double* tau,
                                                                 int r, double* Q2) {
  extern __shared__ double xs[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * kQ2Warps + warp;
  if (c >= r) return;
  double* x = xs + (size_t)warp * mr;
  for (int i = lane; i < mr; i += 32) x[i] = (i == c) ? 1.0 : 0.0;
  __syncwarp();
  for (int j = c; j >= 0; --j) {
    const double* v = A + (size_t)piv[j] * mr;
    double w = 0.0;
    for (int i = j + 1 + lane; i < mr; i += 32) w = fma(v[i], x[i], w);
    w = warp_sum(w) + x[j];
    const double tw = tau[j] * w;
    __syncwarp();
    for (int i = j + 1 + lane; i < mr; i += 32) x[i] -= tw * v[i];
    if (lane == 0) x[j] -= tw;
    __syncwarp();
  }
  for (int i = lane; i < mr; i += 32) Q2[(size_t)c * mr + i] = x[i];
}

// X[piv[k], c] = (R11^-1)[k, c]; R11[i][k] = A[i, piv[k]] (i <= k < r).
// Column-oriented back substitution, one warp per column, b staged in smem.
__global__ void __launch_bounds__(kQ2Warps * 32) tri_inv_kernel(const double* A, int mr, int m,
                                                                 const int* piv, int r, double* X) {
  extern __shared__ double bs[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * kQ2Warps + warp;
  if (c >= r) return;
  double* b = bs + (size_t)warp * mr;
  for (int i = lane; i <= c; i += 32) b[i] = (i == c) ? 1.0 : 0.0;
  __syncwarp();
  for (int l = c; l >= 0; --l) {
    const double* col = A + (size_t)piv[l] * mr;  // R11[:, l]
    const double yl = b[l] / col[l];
    __syncwarp();
    for (int i = lane; i < l; i += 32) b[i] -= yl * col[i];
    if (lane == 0) b[l] = yl;
    __syncwarp();
  }
  for (int k = lane; k <= c; k += 32) X[(size_t)c * m + piv[k]] = b[k];
}

// ---------------------------------------------------------------- fused serial step
// One HBM pass over D and Q per serial correction step (2 r d 8 bytes).  A
// persistent grid of 2 CTAs per SM walks 1024-row tiles: 4 rows per thread and
// 4 columns of D in flight per iteration (16 independent 8-byte loads per
// thread), then 8 columns of Q at a time, reduced inside the warp by an 8-way
// transpose (9 shuffles per 8 columns) and accumulated per warp in shared
// memory; one fixed-order cross-warp sum per CTA, one fixed-order cross-CTA
// sum in reduce_parts_kernel -> deterministic alpha.
constexpr int kCgThreads = 256;
constexpr int kCgWarps = kCgThreads / 32;
constexpr int kCgRpt = 4;  // rows per thread
constexpr int kCgRows = kCgThreads * kCgRpt;

__device__ __forceinline__ double transpose_reduce8(double (&acc)[8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = upper ? acc[i] : acc[i + off];
      const double keep = upper ? acc[i + off] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, off);
    }
  }
  double v = acc[0];  // column lane & 7, summed over the lane's group of 8
  v += __shfl_xor_sync(FULL, v, 8);
  v += __shfl_xor_sync(FULL, v, 16);
  return v;
}

// Row ownership inside a 1024-row tile: scalar layout, row(s) = row0 + tid + 256 s; paired
// layout (V2, d even), row(s) = row0 + 512 (s/2) + 2 tid + (s%2), loaded as 16-byte pairs.
template <bool V2>
__device__ __forceinline__ long long cg_row(long long row0, int s) {
  if constexpr (V2) return row0 + (long long)(s >> 1) * (2 * kCgThreads) + 2 * threadIdx.x + (s & 1);
  else return row0 + threadIdx.x + (long long)s * kCgThreads;
}

// v[s] = col[row(s)] (0 beyond d), streaming (evict-first) loads
template <bool V2>
__device__ __forceinline__ void cg_load(const double* __restrict__ col, long long row0, long long d,
                                        double (&v)[kCgRpt]) {
  if constexpr (V2) {
#pragma unroll
    for (int h = 0; h < kCgRpt / 2; ++h) {
      const long long row = cg_row<true>(row0, 2 * h);
      double2 t = make_double2(0.0, 0.0);
      if (row < d) t = __ldcs(reinterpret_cast<const double2*>(col + row));
      v[2 * h] = t.x;
      v[2 * h + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int s = 0; s < kCgRpt; ++s) {
      const long long row = cg_row<false>(row0, s);
      v[s] = row < d ? __ldcs(col + row) : 0.0;
    }
  }
}

// wpart[warp][k] += sum over this tile's rows of Q[row, k] * y[row]
template <bool V2>
__device__ __forceinline__ void tile_qty(const double* __restrict__ Q, long long ldq, int r, long long d,
                                         long long row0, const double (&y)[kCgRpt],
                                         double* __restrict__ wpart) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k0 = 0; k0 < r; k0 += 8) {
    double acc[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      acc[kk] = 0.0;
      if (k0 + kk < r) {
        double q[kCgRpt];
        cg_load<V2>(Q + (long long)(k0 + kk) * ldq, row0, d, q);
#pragma unroll
        for (int s = 0; s < kCgRpt; ++s) acc[kk] = fma(q[s], y[s], acc[kk]);
      }
    }
    const double v = transpose_reduce8(acc);
    if (lane < 8 && k0 + lane < r) wpart[warp * r + k0 + lane] += v;
  }
}

__device__ __forceinline__ void flush_wpart(const double* wpart, int r, double* __restrict__ part) {
  __syncthreads();
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kCgWarps; ++w) s += wpart[w * r + k];
    part[(long long)blockIdx.x * r + k] = s;
  }
}

// y = [g +] c + D alpha  (rd columns of D)  and  part = Q^T y partials (rq columns of Q);
// g may be NULL, rd or rq may be 0 (the overlapped sweep runs the D pass and the Q pass
// as separate launches, the D pass concurrently with the coarse propagator).
template <int UNR, int MINB, bool V2>
__global__ void __launch_bounds__(kCgThreads, MINB) combine_gemv_kernel(
    const double* __restrict__ g, const double* __restrict__ D, int rd, const double* __restrict__ cvec,
    const double* __restrict__ alpha, const double* __restrict__ Q, int rq, long long d, long long ld,
    double* __restrict__ y_out, double* __restrict__ part, const double* __restrict__ alpha_sub) {
  // d rows starting at the given pointers; D and Q columns are ld apart (ld >= d: a row
  // block of a sharded basis passes its block's first-row pointers)
  extern __shared__ double sh[];
  double* a_s = sh;             // rd
  double* wpart = sh + rd;      // kCgWarps x rq
  for (int k = threadIdx.x; k < rd; k += blockDim.x) a_s[k] = alpha_sub ? alpha[k] - alpha_sub[k] : alpha[k];
  for (int k = threadIdx.x; k < kCgWarps * rq; k += blockDim.x) wpart[k] = 0.0;
  __syncthreads();
  const long long ntiles = (d + kCgRows - 1) / kCgRows;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row0 = tile * kCgRows;
    double y[kCgRpt];
#pragma unroll
    for (int s = 0; s < kCgRpt; ++s) {
      const long long row = cg_row<V2>(row0, s);
      y[s] = row < d ? (g ? g[row] + cvec[row] : cvec[row]) : 0.0;
    }
    // y += D alpha  (column-major D: every column read as one coalesced 8 KB run)
    int k = 0;
    for (; k + UNR <= rd; k += UNR) {
      double t[UNR][kCgRpt];
#pragma unroll
      for (int kk = 0; kk < UNR; ++kk) cg_load<V2>(D + (long long)(k + kk) * ld, row0, d, t[kk]);
#pragma unroll
      for (int kk = 0; kk < UNR; ++kk)
#pragma unroll
        for (int s = 0; s < kCgRpt; ++s) y[s] = fma(t[kk][s], a_s[k + kk], y[s]);
    }
    for (; k < rd; ++k) {
      double t[kCgRpt];
      cg_load<V2>(D + (long long)k * ld, row0, d, t);
#pragma unroll
      for (int s = 0; s < kCgRpt; ++s) y[s] = fma(t[s], a_s[k], y[s]);
    }
#pragma unroll
    for (int s = 0; s < kCgRpt; ++s) {
      const long long row = cg_row<V2>(row0, s);
      if (row < d) y_out[row] = y[s];
    }
    if (rq > 0) tile_qty<V2>(Q, ld, rq, d, row0, y, wpart);
  }
  if (rq > 0) flush_wpart(wpart, rq, part);
}

// ---------------------------------------------------------------- TMA-fed serial step
// Same arithmetic as combine_gemv_kernel<., ., true> (row pairs, fixed-order sums), but the
// D and Q column chunks reach shared memory by 1D bulk copies (cp.async.bulk, the TMA
// engine): one producer lane per CTA keeps kTmaStages x 8 columns x 512 rows (192 KB) in
// flight through full/empty mbarrier pairs, and 8 consumer warps only read shared memory.
// One CTA per SM; tiles of 512 rows, 2 rows (one 16-byte pair) per consumer thread.
constexpr int kTmaRows = 512;                 // rows per tile
constexpr int kTmaCols = 8;                   // columns per stage
constexpr int kTmaStages = 6;                 // ring depth
constexpr int kTmaConsumers = 256;            // 8 warps
constexpr int kTmaThreads = kTmaConsumers + 32;
constexpr size_t kTmaStageBytes = (size_t)kTmaCols * kTmaRows * sizeof(double);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The chunk schedule both sides walk: per tile, ceil(rd/8) D stages then ceil(rq/8) Q stages.
__global__ void __launch_bounds__(kTmaThreads, 1) combine_tma_kernel(
    const double* __restrict__ g, const double* __restrict__ D, int rd, const double* __restrict__ cvec,
    const double* __restrict__ alpha, const double* __restrict__ Q, int rq, long long d, long long ld,
    double* __restrict__ y_out, double* __restrict__ part, int nst, unsigned int* __restrict__ done,
    double* __restrict__ alpha_next, const double* __restrict__ alpha_sub) {
  // nst ring stages (<= kTmaStages: fewer when rd + 8 rq doubles of bookkeeping must fit too).
  // The last CTA to finish sums the per-CTA partials into alpha_next (fixed order).
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);                       // nst x 8 x 512
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + nst * kTmaStageBytes);
  uint64_t* empty = full + nst;
  double* a_s = reinterpret_cast<double*>(empty + nst);                   // rd
  double* wpart = a_s + rd;                                               // 8 warps x rq
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // alpha_sub: the pass applies D (alpha - alpha_sub) (the sweep's folded correction term)
  for (int k = tid; k < rd; k += blockDim.x) a_s[k] = alpha_sub ? alpha[k] - alpha_sub[k] : alpha[k];
  for (int k = tid; k < kCgWarps * rq; k += blockDim.x) wpart[k] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCgWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntiles = (d + kTmaRows - 1) / kTmaRows;
  const int nsd = (rd + kTmaCols - 1) / kTmaCols, nsq = (rq + kTmaCols - 1) / kTmaCols;
  if (warp == kCgWarps) {
    // ---------------- producer: one lane issues every bulk copy
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long row0 = tile * kTmaRows;
        const uint32_t rows = (uint32_t)min((long long)kTmaRows, d - row0);
        for (int q = 0; q < nsd + nsq; ++q) {
          const bool isd = q < nsd;
          const int k0 = (isd ? q : q - nsd) * kTmaCols;
          const int ncol = min(kTmaCols, (isd ? rd : rq) - k0);
          const double* base = (isd ? D : Q) + row0;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_tx(&full[stage], (uint32_t)(ncol * rows * sizeof(double)));
          double* dst = ring + (size_t)stage * kTmaCols * kTmaRows;
          for (int c = 0; c < ncol; ++c)
            bulk_g2s(dst + (size_t)c * kTmaRows, base + (long long)(k0 + c) * ld, rows * sizeof(double),
                     &full[stage]);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ---------------- consumers: rows 2*tid, 2*tid+1 of each tile
    int stage = 0;
    uint32_t phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const long long row0 = tile * kTmaRows;
      const long long row = row0 + 2 * tid;
      const bool ok = row < d;  // d even: both rows of the pair or neither
      double y0 = 0.0, y1 = 0.0;
      if (ok) {
        y0 = g ? g[row] + cvec[row] : cvec[row];
        y1 = g ? g[row + 1] + cvec[row + 1] : cvec[row + 1];
      }
      for (int q = 0; q < nsd; ++q) {
        const int k0 = q * kTmaCols, ncol = min(kTmaCols, rd - k0);
        mbar_wait(&full[stage], phase);
        const double* src = ring + (size_t)stage * kTmaCols * kTmaRows + 2 * tid;
#pragma unroll
        for (int c = 0; c < kTmaCols; ++c) {
          if (c < ncol) {
            const double2 t = *reinterpret_cast<const double2*>(src + (size_t)c * kTmaRows);
            if (ok) {
              y0 = fma(t.x, a_s[k0 + c], y0);
              y1 = fma(t.y, a_s[k0 + c], y1);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == nst) { stage = 0; phase ^= 1; }
      }
      if (ok) *reinterpret_cast<double2*>(y_out + row) = make_double2(y0, y1);
      for (int q = 0; q < nsq; ++q) {
        const int k0 = q * kTmaCols, ncol = min(kTmaCols, rq - k0);
        mbar_wait(&full[stage], phase);
        const double* src = ring + (size_t)stage * kTmaCols * kTmaRows + 2 * tid;
        double acc[8];
#pragma unroll
        for (int c = 0; c < kTmaCols; ++c) {
          acc[c] = 0.0;
          if (c < ncol && ok) {
            const double2 t = *reinterpret_cast<const double2*>(src + (size_t)c * kTmaRows);
            acc[c] = fma(t.x, y0, t.y * y1);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == nst) { stage = 0; phase ^= 1; }
        const double v = transpose_reduce8(acc);
        if (lane < 8 && k0 + lane < rq) wpart[warp * rq + k0 + lane] += v;
      }
    }
  }
  if (rq > 0) {
    flush_wpart(wpart, rq, part);
    int* last = reinterpret_cast<int*>(wpart + kCgWarps * rq);  // one int after the partials
    __threadfence();
    __syncthreads();
    if (tid == 0) *last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (*last) {
      __threadfence();
      for (int k = tid; k < rq; k += blockDim.x) {
        double sum = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) sum += __ldcg(part + (long long)b * rq + k);
        alpha_next[k] = sum;
      }
      if (tid == 0) *done = 0u;  // ready for the next launch on the stream
    }
  }
}

__global__ void __launch_bounds__(kCgThreads, 2) project_partial_kernel(
    const double* __restrict__ Q, int r, long long d, const double* __restrict__ v,
    double* __restrict__ part) {
  extern __shared__ double wpart[];
  for (int k = threadIdx.x; k < kCgWarps * r; k += blockDim.x) wpart[k] = 0.0;
  __syncthreads();
  const long long ntiles = (d + kCgRows - 1) / kCgRows;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row0 = tile * kCgRows;
    double y[kCgRpt];
#pragma unroll
    for (int s = 0; s < kCgRpt; ++s) {
      const long long row = cg_row<false>(row0, s);
      y[s] = row < d ? v[row] : 0.0;
    }
    tile_qty<false>(Q, d, r, d, row0, y, wpart);
  }
  flush_wpart(wpart, r, part);
}

// alpha[k] = sum_b part[b][k]  (fixed order: deterministic); 32 columns x 8 partial streams per CTA
__global__ void __launch_bounds__(256) reduce_parts_kernel(const double* __restrict__ part, int nblk,
                                                           int r, double* __restrict__ alpha) {
  __shared__ double red[8][32];
  const int kk = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + kk;
  double s = 0.0;
  if (k < r)
    for (int b = grp; b < nblk; b += 8) s += part[(long long)b * r + k];
  red[grp][kk] = s;
  __syncthreads();
  if (grp == 0 && k < r) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][kk];
    alpha[k] = t;
  }
}

// ---------------------------------------------------------------- elementwise / residual
__global__ void axpby_kernel(double* __restrict__ y, const double* __restrict__ a,
                             const double* __restrict__ b, double alpha, double beta, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = alpha * a[i] + beta * b[i];
}

constexpr int kResThreads = 256;
__global__ void sqdiff_partial_kernel(const double* __restrict__ a, long long lda,
                                      const double* __restrict__ b, long long ldb, long long nrows,
                                      int chunks, double* __restrict__ part) {
  __shared__ double red[kResThreads / 32];
  const int col = blockIdx.y;
  const long long per = (nrows + chunks - 1) / chunks;
  const long long lo = (long long)blockIdx.x * per;
  const long long hi = lo + per < nrows ? lo + per : nrows;
  const double* ac = a + col * lda;
  const double* bc = b + col * ldb;
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double df = bc[i] - ac[i];
    s = fma(df, df, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kResThreads / 32; ++w) t += red[w];
    part[(long long)col * chunks + blockIdx.x] = t;
  }
}

__global__ void colmax_kernel(const double* __restrict__ part, int ncols, int chunks,
                              double* __restrict__ out) {
  __shared__ double red[256];
  double best = 0.0;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < chunks; ++k) s += part[(long long)c * chunks + k];
    const double nrm = sqrt(s);
    best = fmax(best, nrm);  // fmax ignores NaN like max(r, nan)? see api docs
  }
  red[threadIdx.x] = best;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

__global__ void extract_upper_kernel(const double* __restrict__ W, long long ldw, int mr, int m,
                                     double* __restrict__ R) {
  const long long total = (long long)mr * m;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(idx / mr), row = (int)(idx % mr);
    R[idx] = row <= col ? W[(long long)col * ldw + row] : 0.0;
  }
}

// zero the strict lower triangle of a rows x cols block (leading dim ld)
__global__ void zero_strict_lower_kernel(double* __restrict__ A, long long ld, int rows, int cols) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(idx / rows), row = (int)(idx % rows);
    if (row > col) A[(long long)col * ld + row] = 0.0;
  }
}

__global__ void set_diag_kernel(double* __restrict__ A, long long ld, int k, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) A[(long long)i * ld + i] = v;
}

// Column block of k Householder vectors after geqrf -> explicit unit-lower form:
// column j (0-based in the block) gets zeros in rows [0, off + j) and 1 at row off + j.
__global__ void make_unit_lower_kernel(double* __restrict__ A, long long ld, int off, int k) {
  const long long rows = (long long)off + k;
  const long long total = rows * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(idx / rows);
    const long long row = idx - (long long)col * rows;
    const long long diag = (long long)off + col;
    if (row < diag) A[(long long)col * ld + row] = 0.0;
    else if (row == diag) A[(long long)col * ld + row] = 1.0;
  }
}

// Compact-WY T block of reflector columns col0..col0+p-1 given G = V^T V_new (m x p, ld m,
// m = col0 + p) and tau: the dlarft recurrence restricted to the new block,
//   T[i, i] = tau_i,  T[col0:i, i] = -tau_i T[col0:i, col0:i] G[col0:i, i],
// one CTA, columns in order (each depends on the previous ones); T upper, ld ldt.  The
// coupling block T[0:col0, new] = -T_old (V_old^T V_new) T_new is two GEMMs (api.cu).
__global__ void __launch_bounds__(1024) larft_cols_kernel(double* __restrict__ T, int ldt,
                                                          const double* __restrict__ G,
                                                          const double* __restrict__ tau, int col0,
                                                          int p) {
  const int m = col0 + p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int i = col0; i < m; ++i) {
    const double ti = tau[i];
    const double* g = G + (size_t)(i - col0) * m;
    // one warp per row j, lanes split the l sum (independent L2 loads, then a warp reduction)
    for (int j = col0 + warp; j < i; j += nwarp) {
      double w = 0.0;
      for (int l = j + lane; l < i; l += 32) w = fma(T[(size_t)l * ldt + j], g[l], w);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      if (lane == 0) T[(size_t)i * ldt + j] = -ti * w;
    }
    if (threadIdx.x == 0) T[(size_t)i * ldt + i] = ti;
    __syncthreads();
  }
}

int g_pqr_blocks_per_sm = -1;

}  // namespace

void launch_larft_cols(Ctx& c, double* T, int ldt, const double* G, const double* tau, int col0, int p) {
  if (p <= 0) return;
  larft_cols_kernel<<<1, 1024, 0, c.stream>>>(T, ldt, G, tau, col0, p);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

void launch_make_unit_lower(Ctx& c, double* A, long long ld, int off, int k) {
  const long long total = ((long long)off + k) * k;
  if (k <= 0) return;
  int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)c.num_sms * 8));
  make_unit_lower_kernel<<<blocks, 256, 0, c.stream>>>(A, ld, off, k);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

void launch_axpby_cols(Ctx& c, double* y, const double* a, const double* b, double alpha,
                       double beta, size_t n) {
  if (n == 0) return;
  int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)c.num_sms * 8);
  axpby_kernel<<<blocks, 256, 0, c.stream>>>(y, a, b, alpha, beta, n);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

static void ensure_red(Ctx& c, size_t n) {
  if (c.red_cap >= n) return;
  if (c.red) PW_CUDA(cudaFreeAsync(c.red, c.stream));
  size_t cap = std::max<size_t>(n, 1 << 16);
  PW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c.red), cap * sizeof(double), c.stream));
  c.red_cap = cap;
}

void launch_extract_upper(Ctx& c, const double* W, long long ldw, int mr, int m, double* R) {
  const long long total = (long long)mr * m;
  int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)c.num_sms * 8));
  extract_upper_kernel<<<blocks, 256, 0, c.stream>>>(W, ldw, mr, m, R);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

void launch_zero_strict_lower_block(Ctx& c, double* A, long long ld, int rows, int cols) {
  const long long total = (long long)rows * cols;
  if (total <= 0) return;
  int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)c.num_sms * 8));
  zero_strict_lower_kernel<<<blocks, 256, 0, c.stream>>>(A, ld, rows, cols);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

void launch_set_diag_block(Ctx& c, double* A, long long ld, int k, double v) {
  if (k <= 0) return;
  set_diag_kernel<<<(k + 255) / 256, 256, 0, c.stream>>>(A, ld, k, v);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

size_t residual_scratch_doubles(int ncols, long long nrows) {
  int chunks = (int)std::max<long long>(1, std::min<long long>((nrows + 8191) / 8192, 64));
  return (size_t)ncols * chunks;
}

void launch_residual(Ctx& c, const double* a, long long lda, const double* b, long long ldb,
                     int ncols, long long nrows, double* scratch, double* out_dev) {
  if (ncols <= 0) {
    PW_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), c.stream));
    return;
  }
  int chunks = (int)std::max<long long>(1, std::min<long long>((nrows + 8191) / 8192, 64));
  sqdiff_partial_kernel<<<dim3(chunks, ncols), kResThreads, 0, c.stream>>>(a, lda, b, ldb, nrows,
                                                                          chunks, scratch);
  colmax_kernel<<<1, 256, 0, c.stream>>>(scratch, ncols, chunks, out_dev);
  c.launches += 2;
  PW_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- K7 window diagnostics
// One pass over a window endpoint: max|q| (NaN-propagating like numpy's max), sum q^2 and
// the non-finite count (reference diagnostics.py:20-36 max_norm / total_energy, and the
// all_finite check of parareal.py:316-318).  Per-block partials, then one finishing block.
__device__ __forceinline__ double nanmax2(double a, double b) {
  return (a != a || a > b) ? a : b;  // a NaN on either side wins
}

constexpr int kDiagThreads = 256;
__global__ void window_diag_partial_kernel(const double* __restrict__ q, long long n,
                                           double* __restrict__ part) {
  __shared__ double smax[kDiagThreads / 32], ssum[kDiagThreads / 32], sbad[kDiagThreads / 32];
  double mx = 0.0, s = 0.0, bad = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < n; i += stride) {
    const double x = __ldcs(q + i);
    mx = nanmax2(fabs(x), mx);
    s = fma(x, x, s);
    bad += isfinite(x) ? 0.0 : 1.0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = nanmax2(__shfl_xor_sync(0xffffffffu, mx, o), mx);
    s += __shfl_xor_sync(0xffffffffu, s, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smax[w] = mx;
    ssum[w] = s;
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kDiagThreads / 32; ++k) {
      mx = nanmax2(smax[k], smax[0]);
      smax[0] = mx;
      ssum[0] += ssum[k];
      sbad[0] += sbad[k];
    }
    part[3 * blockIdx.x + 0] = smax[0];
    part[3 * blockIdx.x + 1] = ssum[0];
    part[3 * blockIdx.x + 2] = sbad[0];
  }
}

__global__ void window_diag_finish_kernel(const double* __restrict__ part, int nblk, double cell_area,
                                          const long long* __restrict__ probes, int nprobe,
                                          const double* __restrict__ q, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double mx = 0.0, s = 0.0, bad = 0.0;
  for (int b = 0; b < nblk; ++b) {
    mx = nanmax2(part[3 * b], mx);
    s += part[3 * b + 1];
    bad += part[3 * b + 2];
  }
  out[0] = mx;
  out[1] = s * cell_area;
  out[2] = bad;
  for (int k = 0; k < nprobe; ++k) out[3 + k] = q[probes[k]];
}

size_t window_diag_scratch_doubles(const Ctx& c) { return 3 * (size_t)std::max(c.num_sms, 1) * 2 + 8; }

void launch_window_diag(Ctx& c, const double* q, long long n, double cell_area, const long long* probes_dev,
                        int nprobe, double* scratch, double* out_dev) {
  const int nblk = (int)std::max<long long>(1, std::min<long long>((long long)std::max(c.num_sms, 1) * 2,
                                                                   (n + kDiagThreads - 1) / kDiagThreads));
  window_diag_partial_kernel<<<nblk, kDiagThreads, 0, c.stream>>>(q, n, scratch);
  window_diag_finish_kernel<<<1, 32, 0, c.stream>>>(scratch, nblk, cell_area, probes_dev, nprobe, q, out_dev);
  c.launches += 2;
  PW_LAUNCH_CHECK();
}

int pivoted_qr_small(Ctx& c, double* R, int mr, int m, double rank_tol, int* piv_dev,
                     double* tau_dev, double* diag_dev, int* rank_host) {
  PW_CHECK(m >= 1 && m <= 2048, PW_ERR_VALUE, "pivoted QR supports 1..2048 snapshot columns");
  const int steps = std::min(mr, m);
  if (g_pqr_blocks_per_sm < 0) {
    PW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_pqr_blocks_per_sm, pqr_kernel,
                                                          kQrThreads, 0));
    if (g_pqr_blocks_per_sm < 1) g_pqr_blocks_per_sm = 1;
  }
  ensure_red(c, (size_t)m);
  double* norms = c.red;
  int want = (m + kQrWarps - 1) / kQrWarps;
  int blocks = std::max(1, std::min(want, c.num_sms * std::min(g_pqr_blocks_per_sm, 1)));
  if (const char* be = getenv("PW_PQR_BLOCKS")) blocks = std::max(1, std::min(blocks, atoi(be)));  // tuning hook
  void* args[] = {&R, &mr, &m, &piv_dev, &tau_dev, &norms, &diag_dev};
  const char* pe = getenv("PW_PQR");
  const bool two_barriers = (pe && atoi(pe) == 2) || mr > kQrMaxRows;
  PW_CUDA(cudaLaunchCooperativeKernel(two_barriers ? (void*)pqr_kernel : (void*)pqr1_kernel, dim3(blocks),
                                      dim3(kQrThreads), args, 0, c.stream));
  c.launches += 1;
  // rank = #{ |R_jj| > tol |R_11| } (subspace.py:69-72): host side from the m diagonal values
  std::vector<double> dg(steps);
  PW_CUDA(cudaMemcpyAsync(dg.data(), diag_dev, sizeof(double) * steps, cudaMemcpyDeviceToHost, c.stream));
  PW_CUDA(cudaStreamSynchronize(c.stream));
  int r = 0;
  if (dg[0] != 0.0) {
    for (int k = 0; k < steps; ++k)
      if (dg[k] > rank_tol * dg[0]) ++r;
  }
  *rank_host = r;
  return r;
}

void form_q2(Ctx& c, const double* R, int mr, const int* piv, const double* tau, int r,
             double* Q2) {
  if (r <= 0) return;
  size_t smem = sizeof(double) * mr * kQ2Warps;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    PW_CUDA(cudaFuncSetAttribute(form_q2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  form_q2_kernel<<<(r + kQ2Warps - 1) / kQ2Warps, kQ2Warps * 32, smem, c.stream>>>(R, mr, piv, tau,
                                                                                   r, Q2);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

void tri_inverse_scatter(Ctx& c, const double* R, int mr, int m, const int* piv, int r,
                         double* X) {
  PW_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * (size_t)m * r, c.stream));
  if (r <= 0) return;
  size_t smem = sizeof(double) * mr * kQ2Warps;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    PW_CUDA(cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  tri_inv_kernel<<<(r + kQ2Warps - 1) / kQ2Warps, kQ2Warps * 32, smem, c.stream>>>(R, mr, m, piv, r, X);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

// Xc (r x r, ld r) = rows piv[0..r) of X (m x r, ld m): the compact upper-triangular R11^-1
__global__ void gather_rows_kernel(const double* __restrict__ X, int m, const int* __restrict__ piv, int r,
                                   double* __restrict__ Xc) {
  const long long total = (long long)r * r;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / r), k = (int)(e - (long long)j * r);
    Xc[e] = X[piv[k] + (long long)j * m];
  }
}

void launch_gather_rows(Ctx& c, const double* X, int m, const int* piv, int r, double* Xc) {
  if (r <= 0) return;
  const long long total = (long long)r * r;
  gather_rows_kernel<<<(int)std::min<long long>((total + 255) / 256, 1024), 256, 0, c.stream>>>(X, m, piv, r, Xc);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

// alpha = Q^T s for snapshot columns c0 .. c0 + nc - 1, read off the factorisation:
// S Pi = Q R2 (R2 = the pivoted factor of R1, stored by pqr in place: column piv[k] of Rs holds
// R2[0..k, k]), so Q[:, :r]^T S[:, piv[k]] = R2[0..r-1, k] -- the first r entries of that
// stored column, zero below row k.  No pass over the d-row basis.
__global__ void alpha_from_r_kernel(const double* __restrict__ Rs, int mr, const int* __restrict__ piv, int m,
                                    int steps, int c0, int r, double* __restrict__ alpha) {
  __shared__ int s_k;
  const int c = c0 + blockIdx.x;
  if (threadIdx.x == 0) s_k = m;  // never pivoted (m > mr): every stored row is an R entry
  __syncthreads();
  for (int k = threadIdx.x; k < steps; k += blockDim.x)
    if (piv[k] == c) s_k = k;
  __syncthreads();
  const int k = s_k;
  const double* col = Rs + (size_t)c * mr;
  for (int i = threadIdx.x; i < r; i += blockDim.x) alpha[(size_t)blockIdx.x * r + i] = (i <= k) ? col[i] : 0.0;
}

void launch_alpha_from_r(Ctx& c, const double* Rs, int mr, const int* piv, int m, int c0, int nc, int r,
                         double* alpha) {
  if (r <= 0 || nc <= 0) return;
  alpha_from_r_kernel<<<nc, 256, 0, c.stream>>>(Rs, mr, piv, m, mr < m ? mr : m, c0, r, alpha);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

static int cg_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PW_CG_VARIANT");  // tuning hook (scripts/ubench_gemv.cu)
    v = (e && *e) ? atoi(e) : 0;
  }
  return v;
}

// persistent grid of at most per_sm CTAs per SM, sized so every CTA walks the same number of
// 1024-row tiles (768 tiles at c3 -> 384 CTAs x 2 tiles instead of 444 CTAs x 1.73)
int combine_grid(const Ctx& c, long long d, int per_sm) {
  const long long ntiles = (d + kCgRows - 1) / kCgRows;
  const long long cap = std::max<long long>(1, (long long)per_sm * c.num_sms);
  const long long per_cta = (ntiles + cap - 1) / cap;
  return (int)std::max<long long>(1, (ntiles + per_cta - 1) / per_cta);
}

template <int UNR, int MINB, bool V2>
static int launch_cg(Ctx& c, cudaStream_t st, const double* g, const double* D, int rd,
                      const double* cvec, const double* alpha, const double* Q, int rq, long long d,
                      long long ld, double* y, double* part, int nblk, const double* alpha_sub) {
  auto kern = combine_gemv_kernel<UNR, MINB, V2>;
  if (nblk <= 0) nblk = combine_grid(c, d, MINB);
  size_t smem = sizeof(double) * ((size_t)rd + (size_t)rq * kCgWarps + 1);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    PW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  kern<<<nblk, kCgThreads, smem, st>>>(g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, alpha_sub);
  return nblk;
}

void launch_combine_gemv(Ctx& c, cudaStream_t st, const double* g, const double* D, int rd,
                         const double* cvec, const double* alpha, const double* Q, int rq,
                         long long d, double* y, double* alpha_next, double* part, int nblk,
                         long long ld, const double* alpha_sub) {
  if (ld <= 0) ld = d;
  // 16-byte pairs need every column (and the row block) 16-byte aligned
  const bool v2 = (d % 2 == 0) && (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(D) |
                  reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(y) |
                  reinterpret_cast<uintptr_t>(cvec) | reinterpret_cast<uintptr_t>(g)) % 16 == 0);
  const int var = cg_variant();  // 0: TMA kernel when the layout allows it, 6: LSU kernel
  const size_t tma_extra =
      2 * kTmaStages * sizeof(uint64_t) + sizeof(double) * ((size_t)rd + (size_t)rq * kCgWarps + 2);
  const int tma_nst = (int)std::min<size_t>(kTmaStages, (227u * 1024 - tma_extra) / kTmaStageBytes);
  if ((var == 0 || var == 5) && v2 && d >= kTmaRows && tma_extra < 227u * 1024 && tma_nst >= 2) {
    const long long ntiles = (d + kTmaRows - 1) / kTmaRows;
    if (nblk <= 0) {
      const long long per = (ntiles + c.num_sms - 1) / c.num_sms;
      nblk = (int)((ntiles + per - 1) / per);
    }
    const size_t smem = tma_nst * kTmaStageBytes + 2 * tma_nst * sizeof(uint64_t) +
                        sizeof(double) * ((size_t)rd + (size_t)rq * kCgWarps + 2);
    kernel_setup(c.device, reinterpret_cast<const void*>(combine_tma_kernel), kTmaThreads, 227 * 1024);
    if (!c.tma_done) {
      PW_CUDA(cudaMalloc(&c.tma_done, sizeof(unsigned int)));
      PW_CUDA(cudaMemsetAsync(c.tma_done, 0, sizeof(unsigned int), st));
    }
    combine_tma_kernel<<<nblk, kTmaThreads, smem, st>>>(g, D, rd, cvec, alpha, Q, rq, d, ld, y, part,
                                                        tma_nst, c.tma_done, alpha_next, alpha_sub);
    c.launches += 1;
    PW_LAUNCH_CHECK();
    return;
  }
  switch (var) {
    case 1: nblk = launch_cg<4, 2, false>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub); break;
    case 2: nblk = launch_cg<4, 3, false>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub); break;
    case 3:
      nblk = v2 ? launch_cg<4, 4, true>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub)
                : launch_cg<4, 4, false>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub);
      break;
    case 4:
      nblk = v2 ? launch_cg<8, 3, true>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub)
                : launch_cg<4, 3, false>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub);
      break;
    default:
      nblk = v2 ? launch_cg<4, 3, true>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub)
                : launch_cg<4, 3, false>(c, st, g, D, rd, cvec, alpha, Q, rq, d, ld, y, part, nblk, alpha_sub);
      break;
  }
  c.launches += 1;
  if (rq > 0) {
    reduce_parts_kernel<<<(rq + 31) / 32, 256, 0, st>>>(part, nblk, rq, alpha_next);
    c.launches += 1;
  }
  PW_LAUNCH_CHECK();
}

void launch_project_gemv(Ctx& c, const double* Q, int r, long long d, const double* v,
                         double* alpha, double* part) {
  if (r <= 0) return;
  const int nblk = combine_grid(c, d);
  size_t smem = sizeof(double) * (size_t)r * kCgWarps;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    PW_CUDA(cudaFuncSetAttribute(project_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  project_partial_kernel<<<nblk, kCgThreads, smem, c.stream>>>(Q, r, d, v, part);
  reduce_parts_kernel<<<(r + 31) / 32, 256, 0, c.stream>>>(part, nblk, r, alpha);
  c.launches += 2;
  PW_LAUNCH_CHECK();
}

// one warp per output: fixed summation order (4 interleaved chains per lane, then the
// shuffle tree), so the serial sweep stays deterministic
__global__ void __launch_bounds__(256) implicit_alpha_kernel(const double* __restrict__ C, int ldc,
                                                             const double* __restrict__ xt, int n1,
                                                             const double* __restrict__ g, int n2, int r,
                                                             double* __restrict__ alpha) {
  const int w = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= r) return;
  const double* col = C + (size_t)w * ldc;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  int i = lane;
  for (; i + 96 < n1; i += 128) {
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = fma(col[i + 32 * u], xt[i + 32 * u], s[u]);
  }
  for (; i < n1; i += 32) s[0] = fma(col[i], xt[i], s[0]);
  col += n1;
  i = lane;
  for (; i + 96 < n2; i += 128) {
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = fma(col[i + 32 * u], g[i + 32 * u], s[u]);
  }
  for (; i < n2; i += 32) s[0] = fma(col[i], g[i], s[0]);
  double t = (s[0] + s[1]) + (s[2] + s[3]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) alpha[w] = t;
}

void launch_implicit_alpha(Ctx& c, const double* C, int ldc, const double* xt, int n1, const double* g, int n2,
                           int r, double* alpha) {
  if (r <= 0) return;
  implicit_alpha_kernel<<<(r + 7) / 8, 256, 0, c.stream>>>(C, ldc, xt, n1, g, n2, r, alpha);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

size_t combine_part_doubles(long long d, int r) {
  // >= grid x r for both the 1024-row LSU kernel and the 512-row TMA kernel
  return (size_t)((d + kTmaRows - 1) / kTmaRows) * (size_t)std::max(r, 1);
}

}  // namespace pw
