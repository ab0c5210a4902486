// Fused, batched fine RK3 step for constant advecting velocity (sm_100a, fp64).
//
// Replaces the fine predictor's inner loop: propagate() x rk3_step()
// (integrators.py:79-85, 126-146) x acoustic_rhs (numba_backend.py:119-128)
// for all P slices of a Parareal iteration in one launch per RK3 step.
//
// Arithmetic.  For a constant face velocity every flux order's flux
// divergence telescopes into a fixed 7-point stencil per direction:
//   -(F_{i+1}-F_i)/dx = sum_k c_k q_{i+k},  c_k = -(w_{k+2}-w_{k+3})/dx
// with w the linear face-flux weights of _face_flux (numba_backend.py:13-30).
// Each stage is folded into  s_out = q + beta*f(s_in)  with the stage
// factor beta (h/3, h/2, h) pre-multiplied into every coefficient, so one
// stage costs ~40 DP ops per cell instead of the reference form's ~106.
// Results differ from the reference only by rounding (tests: <=1e-12 rel).
//
// Data movement (the roofline unit: 48 B per cell-update = read + write
// (u,v,p) once).  A CTA owns an x-strip of TX output columns and a y-segment
// of TY output rows.  It streams q rows top-to-bottom through shared-memory
// rings (cp.async, asynchronous one tick ahead) and runs the three stages as
// a row pipeline: stage k trails stage k-1 by RY rows, so all three stages
// are fused per tile with halos only in x (3 cells per stage) and a
// 6*RY-row warm-up per segment; q, s1, s2 never touch HBM.
#include <cuda_pipeline.h>

#include "pw_internal.h"

namespace pw {
namespace {

constexpr int H = 3;  // x radius of one stage (order-6 flux: 3; damping: 2)

__device__ __forceinline__ int wrapi(int k, int n) {
  k %= n;
  return k < 0 ? k + n : k;
}

template <int TX, int TY, int RY, int R, int NT, bool VADV>
struct Cfg {
  static constexpr int WQ = TX + 6 * H;  // q ring row width (cols -3H .. TX+3H)
  static constexpr int W1 = TX + 4 * H;  // s1 ring row width
  static constexpr int W2 = TX + 2 * H;  // s2 ring row width
  static constexpr int NQ = 3 * RY + 2 * R;
  static constexpr int NS = 2 * RY + R;
  static constexpr int NTICK = (TY + 6 * RY) / R;
  static constexpr size_t SMEM = sizeof(double) * 3 * ((size_t)NQ * WQ + (size_t)NS * W1 + (size_t)NS * W2);
  static_assert((TY + 6 * RY) % R == 0, "R must divide TY + 6 RY");
};

// One stage over R rows of the output region of width WO.
//   in ring  : rows of the stage input (width WI = WO + 2H), NI slots
//   q ring   : step-start state (width WQ), column offset (WQ-WO)/2 to the output region
//   rel0     : ring-relative row of the first output row this tick
//   out      : ring (NO slots, width WO) or global (when GLOBAL)
template <int WO, int RY, int R, int NT, bool VADV, bool GLOBAL>
__device__ __forceinline__ void stage(const double* __restrict__ in_ring, int NI,
                                      const double* __restrict__ q_ring, int NQ, int WQ,
                                      int rel0, int rel_lo, int rel_hi, double* __restrict__ out,
                                      int NO, const StageCoef& C, double sx, double sy,
                                      // global-output addressing (stage 3)
                                      double* __restrict__ gout, long long n, int nx, int ny,
                                      int x0, int qs) {
  constexpr int WI = WO + 2 * H;
  const int qoff = (WQ - WO) / 2;
  for (int item = threadIdx.x; item < R * WO; item += NT) {
    const int rr = item / WO;
    const int c = item - rr * WO;
    const int rel = rel0 + rr;
    if (rel < rel_lo || rel >= rel_hi) continue;
    const int ci = c + H;
    // ring row pointers for dy = -RY..RY (field-major inside a slot)
    const double* row[2 * RY + 1];
#pragma unroll
    for (int dy = -RY; dy <= RY; ++dy) row[dy + RY] = in_ring + (size_t)((rel + dy) % NI) * 3 * WI;
    const double* u0 = row[RY];
    const double* v0 = row[RY] + WI;
    const double* p0 = row[RY] + 2 * WI;
#define U(dy, dx) (row[RY + (dy)][ci + (dx)])
#define V(dy, dx) (row[RY + (dy)][WI + ci + (dx)])
#define P(dy, dx) (row[RY + (dy)][2 * WI + ci + (dx)])
    const double* qrow = q_ring + (size_t)(rel % NQ) * 3 * WQ;
    double au = qrow[qoff + c];
    double av = qrow[WQ + qoff + c];
    double ap = qrow[2 * WQ + qoff + c];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      au = fma(C.cx[k], u0[ci + k - 3], au);
      av = fma(C.cx[k], v0[ci + k - 3], av);
      ap = fma(C.cx[k], p0[ci + k - 3], ap);
    }
    if constexpr (VADV) {
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        if (k == 3) continue;
        au = fma(C.cy[k], U(k - 3, 0), au);
        av = fma(C.cy[k], V(k - 3, 0), av);
        ap = fma(C.cy[k], P(k - 3, 0), ap);
      }
      au = fma(C.cy[3], U(0, 0), au);
      av = fma(C.cy[3], V(0, 0), av);
      ap = fma(C.cy[3], P(0, 0), ap);
    }
    // velocity divergence (unscaled by beta): div = sx (u_{i+1}-u_{i-1}) + sy (v_{j+1}-v_{j-1})
    const double d_c = sx * (U(0, 1) - U(0, -1)) + sy * (V(1, 0) - V(-1, 0));
    const double d_e = sx * (U(0, 2) - U(0, 0)) + sy * (V(1, 1) - V(-1, 1));
    const double d_w = sx * (U(0, 0) - U(0, -2)) + sy * (V(1, -1) - V(-1, -1));
    const double d_n = sx * (U(1, 1) - U(1, -1)) + sy * (V(2, 0) - V(0, 0));
    const double d_s = sx * (U(-1, 1) - U(-1, -1)) + sy * (V(0, 0) - V(-2, 0));
    au = fma(C.pgx, P(0, 1) - P(0, -1), au);
    au = fma(C.dmx, d_e - d_w, au);
    av = fma(C.pgy, P(1, 0) - P(-1, 0), av);
    av = fma(C.dmy, d_n - d_s, av);
    ap = fma(C.pdiv, d_c, ap);
#undef U
#undef V
#undef P
    if constexpr (GLOBAL) {
      const int gy = wrapi(qs + rel, ny);
      const long long off = (long long)gy * nx + x0 + c;
      gout[off] = au;
      gout[n + off] = av;
      gout[2 * n + off] = ap;
    } else {
      double* orow = out + (size_t)(rel % NO) * 3 * WO;
      orow[c] = au;
      orow[WO + c] = av;
      orow[2 * WO + c] = ap;
    }
  }
}

template <int TX, int TY, int RY, int R, int NT, bool VADV>
__global__ void __launch_bounds__(NT) rk3_fused_kernel(const double* __restrict__ in,
                                                       double* __restrict__ out, FusedParams P) {
  using K = Cfg<TX, TY, RY, R, NT, VADV>;
  extern __shared__ __align__(16) double smem[];
  double* q_ring = smem;
  double* s1_ring = q_ring + (size_t)K::NQ * 3 * K::WQ;
  double* s2_ring = s1_ring + (size_t)K::NS * 3 * K::W1;

  const int nx = P.nx, ny = P.ny;
  const long long n = (long long)nx * ny;
  const int x0 = blockIdx.x * TX;
  const int y0 = blockIdx.y * TY;
  const double* src = in + (long long)blockIdx.z * P.ld_in;
  double* dst = out + (long long)blockIdx.z * P.ld_out;
  const int qs = y0 - 3 * RY;  // ring-relative row 0

  auto load_rows = [&](int rel_first) {
    // R rows x 3 fields x WQ columns, 8-byte cp.async (LDGSTS), wrapped indices
    constexpr int PER_ROW = 3 * K::WQ;
    for (int e = threadIdx.x; e < R * PER_ROW; e += NT) {
      const int rr = e / PER_ROW;
      const int rem = e - rr * PER_ROW;
      const int f = rem / K::WQ;
      const int col = rem - f * K::WQ;
      const int rel = rel_first + rr;
      const int gy = wrapi(qs + rel, ny);
      const int gx = wrapi(x0 - 3 * H + col, nx);
      double* d = q_ring + (size_t)(rel % K::NQ) * 3 * K::WQ + f * K::WQ + col;
      __pipeline_memcpy_async(d, src + f * n + (long long)gy * nx + gx, sizeof(double));
    }
    __pipeline_commit();
  };

  load_rows(0);
  for (int t = 0; t < K::NTICK; ++t) {
    __pipeline_wait_prior(0);
    __syncthreads();
    if (t + 1 < K::NTICK) load_rows((t + 1) * R);
    // stage 1: s1 = q + (h/3) f(q)    rows rel [tR-RY, tR-RY+R), valid [RY, TY+5RY)
    stage<K::W1, RY, R, NT, VADV, false>(q_ring, K::NQ, q_ring, K::NQ, K::WQ, t * R - RY, RY,
                                         TY + 5 * RY, s1_ring, K::NS, P.st[0], P.sx, P.sy,
                                         nullptr, n, nx, ny, x0, qs);
    __syncthreads();
    // stage 2: s2 = q + (h/2) f(s1)   valid [2RY, TY+4RY)
    stage<K::W2, RY, R, NT, VADV, false>(s1_ring, K::NS, q_ring, K::NQ, K::WQ, t * R - 2 * RY,
                                         2 * RY, TY + 4 * RY, s2_ring, K::NS, P.st[1], P.sx,
                                         P.sy, nullptr, n, nx, ny, x0, qs);
    __syncthreads();
    // stage 3: q+ = q + h f(s2)       valid [3RY, TY+3RY) -> global
    stage<TX, RY, R, NT, VADV, true>(s2_ring, K::NS, q_ring, K::NQ, K::WQ, t * R - 3 * RY,
                                     3 * RY, TY + 3 * RY, nullptr, 0, P.st[2], P.sx, P.sy, dst, n,
                                     nx, ny, x0, qs);
  }
}

template <int TX, int TY, int RY, bool VADV>
void launch_cfg(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch) {
  constexpr int R = 2, NT = 128;
  using K = Cfg<TX, TY, RY, R, NT, VADV>;
  auto kern = rk3_fused_kernel<TX, TY, RY, R, NT, VADV>;
  static bool attr_set = false;
  if (!attr_set) {
    PW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM));
    attr_set = true;
  }
  dim3 grid(fp.nx / TX, fp.ny / TY, batch);
  kern<<<grid, NT, K::SMEM, c.stream>>>(in, out, fp);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

template <int RY, bool VADV>
void launch_ry(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch) {
  const int nx = fp.nx, ny = fp.ny;
  // x strip 64 (or 32/16/8 for small grids); y segment 128 (or the grid height)
  if (nx % 64 == 0) {
    if (ny % 128 == 0) return launch_cfg<64, 128, RY, VADV>(c, fp, in, out, batch);
    if (ny % 64 == 0) return launch_cfg<64, 64, RY, VADV>(c, fp, in, out, batch);
  }
  if (nx % 32 == 0 && ny % 32 == 0) return launch_cfg<32, 32, RY, VADV>(c, fp, in, out, batch);
  if (nx % 16 == 0 && ny % 16 == 0) return launch_cfg<16, 16, RY, VADV>(c, fp, in, out, batch);
  if (nx % 8 == 0 && ny % 8 == 0) return launch_cfg<8, 8, RY, VADV>(c, fp, in, out, batch);
  throw Error{PW_ERR_VALUE, "fused RK3 needs nx, ny multiples of 8"};
}

// linear face-flux weights w[0..5] on the window (q_{f-3}..q_{f+2}) for a
// constant face velocity u (numba_backend._face_flux, numba_backend.py:13-30)
void flux_weights(int order, double u, double w[6]) {
  for (int m = 0; m < 6; ++m) w[m] = 0.0;
  const double a = u < 0 ? -u : u;
  switch (order) {
    case 1:
      if (u >= 0.0) w[2] = u; else w[3] = u;
      break;
    case 2:
      w[2] = w[3] = 0.5 * u;
      break;
    case 3:
    case 4:
      w[1] = -u / 12.0; w[2] = 7.0 * u / 12.0; w[3] = 7.0 * u / 12.0; w[4] = -u / 12.0;
      if (order == 3) { w[1] += -a / 12.0; w[2] += 3.0 * a / 12.0; w[3] += -3.0 * a / 12.0; w[4] += a / 12.0; }
      break;
    case 5:
    case 6:
      w[0] = u / 60.0; w[1] = -8.0 * u / 60.0; w[2] = 37.0 * u / 60.0;
      w[3] = 37.0 * u / 60.0; w[4] = -8.0 * u / 60.0; w[5] = u / 60.0;
      if (order == 5) {
        w[0] += a / 60.0; w[1] += -5.0 * a / 60.0; w[2] += 10.0 * a / 60.0;
        w[3] += -10.0 * a / 60.0; w[4] += 5.0 * a / 60.0; w[5] += -a / 60.0;
      }
      break;
    default:
      throw Error{PW_ERR_VALUE, "flux order must be in 1..6"};
  }
}

}  // namespace

bool fused_supported(int nx, int ny) { return nx % 8 == 0 && ny % 8 == 0; }

void make_fused_params(FusedParams& fp, int nx, int ny, double dx, double dy, double cs,
                       int order, double U, double V, double a1, double a2, double h) {
  fp.nx = nx;
  fp.ny = ny;
  fp.sx = 0.5 / dx;
  fp.sy = 0.5 / dy;
  double wx[6], wy[6], cx[7], cy[7];
  flux_weights(order, U, wx);
  flux_weights(order, V, wy);
  for (int k = -3; k <= 3; ++k) {
    const double a = (k + 2 >= 0 && k + 2 < 6) ? wx[k + 2] : 0.0;
    const double b = (k + 3 >= 0 && k + 3 < 6) ? wx[k + 3] : 0.0;
    cx[k + 3] = -(a - b) / dx;
    const double ay = (k + 2 >= 0 && k + 2 < 6) ? wy[k + 2] : 0.0;
    const double by = (k + 3 >= 0 && k + 3 < 6) ? wy[k + 3] : 0.0;
    cy[k + 3] = -(ay - by) / dy;
  }
  const double betas[3] = {h / 3.0, h / 2.0, h};
  for (int s = 0; s < 3; ++s) {
    const double b = betas[s];
    StageCoef& C = fp.st[s];
    for (int k = 0; k < 7; ++k) {
      C.cx[k] = b * cx[k];
      C.cy[k] = b * cy[k];
    }
    C.pgx = -b * cs * fp.sx;
    C.pgy = -b * cs * fp.sy;
    C.dmx = b * a1 * fp.sx;
    C.dmy = b * a2 * fp.sy;
    C.pdiv = -b * cs;
  }
}

void launch_rk3_fused(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch,
                      bool vadv) {
  if (vadv) launch_ry<3, true>(c, fp, in, out, batch);
  else launch_ry<2, false>(c, fp, in, out, batch);
}

}  // namespace pw
