// Reference-operation-order stencil kernels (compiled with -fmad=false).
//
// Each expression below is evaluated in exactly the order of the reference's
// numba kernels, with every multiply and add separately rounded, so these
// kernels reproduce the reference BITWISE (the oracle test suite checks it):
//   _face_flux            pkg/src/pitwave/kernels/numba_backend.py:13-30
//   flux_x / flux_y       numba_backend.py:33-66  (face f between cells f-1 | f)
//   flux_divergence       numba_backend.py:69-78
//   centered_dx / dy      numba_backend.py:81-105 ((f[i+1]-f[i-1]) * (0.5/dx))
//   acoustic_rhs          numba_backend.py:119-128
//   damping_tendencies    numba_backend.py:108-111
//   rk3_step              integrators.py:79-85   (s = q + f*(h/3), q + f*(h/2), q + f*h)
//   split_fe_fb_step      integrators.py:103-106 + fb_substeps numba_backend.py:131-146
// They accept arbitrary face-velocity arrays (ConstantVelocity or
// SolidBodyRotation, mesh.py:162-199) and every flux order 1..6.
//
// Roles: (1) the coarse propagator G of the Parareal sweep -- one cooperative
// persistent launch per call, all FE-FB substeps separated by grid barriers
// (latency-bound serial work: no per-substep launches); (2) the fine RK3 for
// spatially varying velocity or when the context is in strict mode.
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include <cmath>
#include <utility>

#include "pw_internal.h"

namespace cg = cooperative_groups;

namespace pw {
namespace {

// neighbour index wrap: offsets are at most 3 cells and grids have >= 8 cells
__device__ __forceinline__ int wrapi(int k, int n) { return k < 0 ? k + n : (k >= n ? k - n : k); }

__device__ __forceinline__ double face_flux(int order, double u, double qm2, double qm1,
                                            double q0, double qp1, double qp2, double qp3) {
  if (order == 1) return u >= 0.0 ? u * q0 : u * qp1;
  if (order == 2) return u * 0.5 * (q0 + qp1);
  double f4 = u * (7.0 * (q0 + qp1) - (qm1 + qp2)) / 12.0;
  if (order == 3) return f4 - fabs(u) * (3.0 * (qp1 - q0) - (qp2 - qm1)) / 12.0;
  if (order == 4) return f4;
  double f6 = u * (37.0 * (q0 + qp1) - 8.0 * (qm1 + qp2) + (qm2 + qp3)) / 60.0;
  if (order == 5)
    return f6 - fabs(u) * (10.0 * (qp1 - q0) - 5.0 * (qp2 - qm1) + (qp3 - qm2)) / 60.0;
  return f6;
}

// x-face flux on face f of row j (window cells f-3..f+2)
__device__ __forceinline__ double fx_at(const ExactParams& p, const double* __restrict__ q, int j,
                                        int f, int order) {
  const double* row = q + (size_t)j * p.nx;
  return face_flux(order, p.uf[(size_t)j * p.nx + f], row[wrapi(f - 3, p.nx)],
                   row[wrapi(f - 2, p.nx)], row[wrapi(f - 1, p.nx)], row[f],
                   row[wrapi(f + 1, p.nx)], row[wrapi(f + 2, p.nx)]);
}

__device__ __forceinline__ double gy_at(const ExactParams& p, const double* __restrict__ q, int f,
                                        int i, int order) {
  const int nx = p.nx, ny = p.ny;
  return face_flux(order, p.vf[(size_t)f * nx + i], q[(size_t)wrapi(f - 3, ny) * nx + i],
                   q[(size_t)wrapi(f - 2, ny) * nx + i], q[(size_t)wrapi(f - 1, ny) * nx + i],
                   q[(size_t)f * nx + i], q[(size_t)wrapi(f + 1, ny) * nx + i],
                   q[(size_t)wrapi(f + 2, ny) * nx + i]);
}

// advective_tendency = flux_divergence(flux_x, flux_y) at cell (j, i); ORD > 0 fixes the
// flux order at compile time (the coarse propagator's order-1 flux), 0 reads p.order
template <int ORD = 0>
__device__ __forceinline__ double adv_at(const ExactParams& p, const double* __restrict__ q, int j,
                                         int i) {
  const int order = ORD > 0 ? ORD : p.order;
  const int ip = i + 1 < p.nx ? i + 1 : 0;
  const int jp = j + 1 < p.ny ? j + 1 : 0;
  const double fxi = fx_at(p, q, j, i, order), fxp = fx_at(p, q, j, ip, order);
  const double gyj = gy_at(p, q, j, i, order), gyp = gy_at(p, q, jp, i, order);
  const double tx = -(fxp - fxi), ty = (gyp - gyj);
  return (p.inv_dx != 0.0 ? tx * p.inv_dx : tx / p.dx) - (p.inv_dy != 0.0 ? ty * p.inv_dy : ty / p.dy);
}

__device__ __forceinline__ double cdx(const ExactParams& p, const double* __restrict__ f, int j,
                                      int i, double sx) {
  const double* row = f + (size_t)j * p.nx;
  return (row[wrapi(i + 1, p.nx)] - row[wrapi(i - 1, p.nx)]) * sx;
}

__device__ __forceinline__ double cdy(const ExactParams& p, const double* __restrict__ f, int j,
                                      int i, double sy) {
  return (f[(size_t)wrapi(j + 1, p.ny) * p.nx + i] - f[(size_t)wrapi(j - 1, p.ny) * p.nx + i]) *
         sy;
}

// one RK3 stage: out = q + f(s) * beta   (out may alias q: reads q only at the own cell)
__global__ void rk3_stage_exact(const double* q, const double* __restrict__ s, double* out,
                                int batch, long long ldq, long long lds, long long ldo,
                                ExactParams p, double beta) {
  const int n = p.nx * p.ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy, cs = p.cs;
  const long long b = blockIdx.y;
  (void)batch;
  for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < n; cell += gridDim.x * blockDim.x) {
    const int j = cell / p.nx, i = cell - j * p.nx;
    const double* su = s + b * lds;
    const double* sv = su + n;
    const double* sp = sv + n;
    double du = adv_at(p, su, j, i) - cs * cdx(p, sp, j, i, sx);
    double dv = adv_at(p, sv, j, i) - cs * cdy(p, sp, j, i, sy);
    double dp = adv_at(p, sp, j, i) - cs * (cdx(p, su, j, i, sx) + cdy(p, sv, j, i, sy));
    if (p.a1 != 0.0 || p.a2 != 0.0) {
      const int im = wrapi(i - 1, p.nx), ipp = wrapi(i + 1, p.nx);
      const int jm = wrapi(j - 1, p.ny), jpp = wrapi(j + 1, p.ny);
      const double div_ip = cdx(p, su, j, ipp, sx) + cdy(p, sv, j, ipp, sy);
      const double div_im = cdx(p, su, j, im, sx) + cdy(p, sv, j, im, sy);
      const double div_jp = cdx(p, su, jpp, i, sx) + cdy(p, sv, jpp, i, sy);
      const double div_jm = cdx(p, su, jm, i, sx) + cdy(p, sv, jm, i, sy);
      du = du + p.a1 * ((div_ip - div_im) * sx);
      dv = dv + p.a2 * ((div_jp - div_jm) * sy);
    }
    const double* qb = q + b * ldq;
    double* ob = out + b * ldo;
    const double qu = qb[cell], qv = qb[n + cell], qp = qb[2 * n + cell];
    ob[cell] = qu + du * beta;
    ob[n + cell] = qv + dv * beta;
    ob[2 * n + cell] = qp + dp * beta;
  }
}

// scalar advection RK3 stage (physics.advection_rhs, physics.py:77-80): out = q + adv(s) * beta
__global__ void rk3_stage_exact_scalar(const double* q, const double* __restrict__ s, double* out,
                                       long long ldq, long long lds, long long ldo, ExactParams p,
                                       double beta) {
  const int n = p.nx * p.ny;
  const long long b = blockIdx.y;
  for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < n; cell += gridDim.x * blockDim.x) {
    const int j = cell / p.nx, i = cell - j * p.nx;
    const double f = adv_at(p, s + b * lds, j, i);
    out[b * ldo + cell] = q[b * ldq + cell] + f * beta;
  }
}

// advective tendencies of the 3 acoustic fields of `cur` (physics.advective_tendencies,
// physics.py:67-74) into work planes 0..2 of each state (split RK3-FB stages)
__global__ void adv3_exact(const double* __restrict__ cur, long long ld, double* __restrict__ work,
                           ExactParams p) {
  const int n = p.nx * p.ny;
  const long long b = blockIdx.y;
  const double* q = cur + b * ld;
  double* w = work + b * 6 * (long long)n;
  for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < n; cell += gridDim.x * blockDim.x) {
    const int j = cell / p.nx, i = cell - j * p.nx;
    w[cell] = adv_at(p, q, j, i);
    w[n + cell] = adv_at(p, q + n, j, i);
    w[2 * n + cell] = adv_at(p, q + 2 * n, j, i);
  }
}

// Split FE-FB (integrators.py:103-106 / fb_substeps numba_backend.py:131-146),
// nsteps coarse steps in ONE cooperative launch.  One grid barrier per acoustic
// substep: the pressure update needs the new velocities of its 4 neighbours,
// which each thread recomputes from the old state with the same expression
// (bitwise identical to storing them), reading a ping-pong copy of (u, v, p).
// work per state: [au, av, ap, u', v', p'] (6 planes).
// 7x7 neighbourhood of a cell, wrapped once: rows j-3..j+3, cols i-3..i+3
struct Nbr {
  int ro[7];
  int co[7];
  __device__ __forceinline__ double at(const double* f, int dy, int dx) const {
    return f[ro[dy + 3] + co[dx + 3]];
  }
};
__device__ __forceinline__ void make_nbr(Nbr& N, int j, int i, int nx, int ny) {
#pragma unroll
  for (int k = -3; k <= 3; ++k) {
    int jj = j + k;
    jj = jj < 0 ? jj + ny : (jj >= ny ? jj - ny : jj);
    int ii = i + k;
    ii = ii < 0 ? ii + nx : (ii >= nx ? ii - nx : ii);
    N.ro[k + 3] = jj * nx;
    N.co[k + 3] = ii;
  }
}
// Field access for the FB substep: global memory through a wrapped 7x7 neighbourhood ...
struct GAcc {
  Nbr N;
  const double* __restrict__ cu;
  const double* __restrict__ cv;
  const double* __restrict__ cp;
  const double* __restrict__ au;
  const double* __restrict__ av;
  __device__ __forceinline__ double u(int dy, int dx) const { return N.at(cu, dy, dx); }
  __device__ __forceinline__ double v(int dy, int dx) const { return N.at(cv, dy, dx); }
  __device__ __forceinline__ double p(int dy, int dx) const { return N.at(cp, dy, dx); }
  __device__ __forceinline__ double a_u(int dy, int dx) const { return N.at(au, dy, dx); }
  __device__ __forceinline__ double a_v(int dy, int dx) const { return N.at(av, dy, dx); }
};
// ... or a shared-memory tile (pointers at the cell, row pitch W; a-tiles pitch WA)
struct SAcc {
  const double* su;
  const double* sv;
  const double* sp;
  int W;
  const double* sau;
  const double* sav;
  int WA;
  __device__ __forceinline__ double u(int dy, int dx) const { return su[dy * W + dx]; }
  __device__ __forceinline__ double v(int dy, int dx) const { return sv[dy * W + dx]; }
  __device__ __forceinline__ double p(int dy, int dx) const { return sp[dy * W + dx]; }
  __device__ __forceinline__ double a_u(int dy, int dx) const { return sau[dy * WA + dx]; }
  __device__ __forceinline__ double a_v(int dy, int dx) const { return sav[dy * WA + dx]; }
};

// ... or a shared-memory tile with the cell's own frozen tendencies in registers (only the
// <0, 0> velocity updates, which read a_u / a_v at the cell itself)
struct SAccV {
  const double* su;
  const double* sv;
  const double* sp;
  int W;
  double au, av;
  __device__ __forceinline__ double u(int dy, int dx) const { return su[dy * W + dx]; }
  __device__ __forceinline__ double v(int dy, int dx) const { return sv[dy * W + dx]; }
  __device__ __forceinline__ double p(int dy, int dx) const { return sp[dy * W + dx]; }
  __device__ __forceinline__ double a_u(int, int) const { return au; }
  __device__ __forceinline__ double a_v(int, int) const { return av; }
};

// u' and v' of one FB substep at (j+DY, i+DX), reference operation order (fb_substeps,
// numba_backend.py:137-143): du = au - cs dx(p) [+ a1 dx(div)], u' = u + tau du
template <int DY, int DX, class A>
__device__ __forceinline__ double un_at(const A& a, const ExactParams& p, double sx, double sy,
                                        double tau, bool damp) {
  double du = a.a_u(DY, DX) - p.cs * ((a.p(DY, DX + 1) - a.p(DY, DX - 1)) * sx);
  if (damp) {
    const double div_ip = (a.u(DY, DX + 2) - a.u(DY, DX)) * sx +
                          (a.v(DY + 1, DX + 1) - a.v(DY - 1, DX + 1)) * sy;
    const double div_im = (a.u(DY, DX) - a.u(DY, DX - 2)) * sx +
                          (a.v(DY + 1, DX - 1) - a.v(DY - 1, DX - 1)) * sy;
    du = du + p.a1 * ((div_ip - div_im) * sx);
  }
  return a.u(DY, DX) + tau * du;
}
template <int DY, int DX, class A>
__device__ __forceinline__ double vn_at(const A& a, const ExactParams& p, double sx, double sy,
                                        double tau, bool damp) {
  double dv = a.a_v(DY, DX) - p.cs * ((a.p(DY + 1, DX) - a.p(DY - 1, DX)) * sy);
  if (damp) {
    const double div_jp = (a.u(DY + 1, DX + 1) - a.u(DY + 1, DX - 1)) * sx +
                          (a.v(DY + 2, DX) - a.v(DY, DX)) * sy;
    const double div_jm = (a.u(DY - 1, DX + 1) - a.u(DY - 1, DX - 1)) * sx +
                          (a.v(DY, DX) - a.v(DY - 2, DX)) * sy;
    dv = dv + p.a2 * ((div_jp - div_jm) * sy);
  }
  return a.v(DY, DX) + tau * dv;
}

// one cell's substep: new (u, v, p), p from the recomputed neighbour velocities
template <class A>
__device__ __forceinline__ void fb_cell(const A& a, const ExactParams& p, double sx, double sy,
                                        double tau, bool damp, double ap_c, double p_c,
                                        double& un, double& vn, double& pn) {
  un = un_at<0, 0>(a, p, sx, sy, tau, damp);
  vn = vn_at<0, 0>(a, p, sx, sy, tau, damp);
  const double u_e = un_at<0, 1>(a, p, sx, sy, tau, damp);
  const double u_w = un_at<0, -1>(a, p, sx, sy, tau, damp);
  const double v_n = vn_at<1, 0>(a, p, sx, sy, tau, damp);
  const double v_s = vn_at<-1, 0>(a, p, sx, sy, tau, damp);
  const double divn = (u_e - u_w) * sx + (v_n - v_s) * sy;
  pn = p_c + tau * (ap_c - p.cs * divn);
}

__global__ void __launch_bounds__(128) fefb_coop(double* st, int batch, long long ld, ExactParams p,
                                                 int nsteps, double tau, int nsub, double* work,
                                                 int adv_given) {
  cg::grid_group grid = cg::this_grid();
  const int n = p.nx * p.ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy, cs = p.cs;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  const int stride = gridDim.x * blockDim.x;
  const int first = blockIdx.x * blockDim.x + threadIdx.x;
  for (int step = 0; step < nsteps; ++step) {
    // frozen slow tendency A(q) (physics.advective_tendencies, physics.py:67-74); split
    // RK3-FB stages pass it precomputed from another state (adv_given)
    if (!adv_given)
    for (long long b = 0; b < batch; ++b)
    for (int cell = first; cell < n; cell += stride) {
      const int j = cell / p.nx, i = cell - j * p.nx;
      const double* q = st + b * ld;
      double* w = work + b * 6 * n;
      w[cell] = adv_at(p, q, j, i);
      w[n + cell] = adv_at(p, q + n, j, i);
      w[2 * n + cell] = adv_at(p, q + 2 * n, j, i);
    }
    grid.sync();
    for (int sub = 0; sub < nsub; ++sub) {
      const bool from_state = (sub % 2 == 0);
      for (long long b = 0; b < batch; ++b)
      for (int cell = first; cell < n; cell += stride) {
        const int j = cell / p.nx, i = cell - j * p.nx;
        double* w = work + b * 6 * n;
        double* sb = st + b * ld;
        const double* __restrict__ cu = from_state ? sb : w + 3 * n;
        const double* __restrict__ cv = cu + n;
        const double* __restrict__ cp = cu + 2 * n;
        double* __restrict__ nu = from_state ? w + 3 * n : sb;
        GAcc acc;
        make_nbr(acc.N, j, i, p.nx, p.ny);
        acc.cu = cu;
        acc.cv = cv;
        acc.cp = cp;
        acc.au = w;
        acc.av = w + n;
        double un, vn, pn;
        fb_cell(acc, p, sx, sy, tau, damp, w[2 * n + cell], cp[cell], un, vn, pn);
        nu[cell] = un;
        nu[n + cell] = vn;
        nu[2 * n + cell] = pn;
      }
      grid.sync();
    }
    if (nsub % 2 == 1) {
      for (long long b = 0; b < batch; ++b)
      for (int cell = first; cell < n; cell += stride) {
        double* w = work + b * 6 * n;
        double* sb = st + b * ld;
        sb[cell] = w[3 * n + cell];
        sb[n + cell] = w[4 * n + cell];
        sb[2 * n + cell] = w[5 * n + cell];
      }
      grid.sync();
    }
  }
}

// Tiled variant for grids divisible by T: per substep every CTA stages its
// T x T tile of (u, v, p) with a 3-cell halo and (au, av) with a 1-cell halo in
// shared memory, then computes T*T/256 cells per thread from the tile with
// compile-time offsets (same expressions as the global variant: bitwise equal).
template <int T>
__global__ void __launch_bounds__(256, 2) fefb_tiled_coop(double* st, int batch, long long ld,
                                                       ExactParams p, int nsteps, double tau,
                                                       int nsub, double* work) {
  cg::grid_group grid = cg::this_grid();
  constexpr int W = T + 6, WA = T + 2;
  extern __shared__ double sm[];
  double* su = sm;
  double* sv = su + W * W;
  double* sp = sv + W * W;
  double* sau = sp + W * W;
  double* sav = sau + WA * WA;
  const int nx = p.nx, ny = p.ny;
  const int n = nx * ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  const int tiles_x = nx / T, tiles = tiles_x * (ny / T);
  const long long work_items = (long long)tiles * batch;
  const int stride = gridDim.x * blockDim.x;
  const int first = blockIdx.x * blockDim.x + threadIdx.x;
  for (int step = 0; step < nsteps; ++step) {
    for (long long b = 0; b < batch; ++b)
      for (int cell = first; cell < n; cell += stride) {
        const int j = cell / nx, i = cell - j * nx;
        const double* q = st + b * ld;
        double* w = work + b * 6 * n;
        w[cell] = adv_at(p, q, j, i);
        w[n + cell] = adv_at(p, q + n, j, i);
        w[2 * n + cell] = adv_at(p, q + 2 * n, j, i);
      }
    grid.sync();
    for (int sub = 0; sub < nsub; ++sub) {
      const bool from_state = (sub % 2 == 0);
      for (long long it = blockIdx.x; it < work_items; it += gridDim.x) {
        const long long b = it / tiles;
        const int t = (int)(it - b * tiles);
        const int ty0 = (t / tiles_x) * T, tx0 = (t % tiles_x) * T;
        double* w = work + b * 6 * n;
        double* sb = st + b * ld;
        const double* __restrict__ cu = from_state ? sb : w + 3 * n;
        double* __restrict__ nu = from_state ? w + 3 * n : sb;
        // stage (u, v, p) with halo 3 and (au, av) with halo 1: warp w stages rows
        // w, w+8, ...; lanes cover x and x+32 (column wraps computed once per tile)
        {
          const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
          auto wrapx = [&](int x) { return x < 0 ? x + nx : (x >= nx ? x - nx : x); };
          auto wrapy = [&](int y) { return y < 0 ? y + ny : (y >= ny ? y - ny : y); };
          const int gx0 = wrapx(lane < W ? tx0 - 3 + lane : 0);
          const int gx1 = wrapx(tx0 - 3 + lane + 32 < nx + 3 ? tx0 - 3 + lane + 32 : 0);
          for (int y = warp; y < W; y += 8) {
            const double* row = cu + wrapy(ty0 - 3 + y) * nx;
#pragma unroll
            for (int f = 0; f < 3; ++f) {
              if (lane < W) __pipeline_memcpy_async(&sm[f * W * W + y * W + lane], row + f * n + gx0, 8);
              if (lane + 32 < W)
                __pipeline_memcpy_async(&sm[f * W * W + y * W + lane + 32], row + f * n + gx1, 8);
            }
          }
          const int ga0 = wrapx(lane < WA ? tx0 - 1 + lane : 0);
          const int ga1 = wrapx(tx0 - 1 + lane + 32 < nx + 1 ? tx0 - 1 + lane + 32 : 0);
          for (int y = warp; y < WA; y += 8) {
            const double* row = w + wrapy(ty0 - 1 + y) * nx;
#pragma unroll
            for (int f = 0; f < 2; ++f) {
              if (lane < WA) __pipeline_memcpy_async(&sau[f * WA * WA + y * WA + lane], row + f * n + ga0, 8);
              if (lane + 32 < WA)
                __pipeline_memcpy_async(&sau[f * WA * WA + y * WA + lane + 32], row + f * n + ga1, 8);
            }
          }
          __pipeline_commit();
          __pipeline_wait_prior(0);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < T * T / 256; ++k) {
          const int c = threadIdx.x + k * 256;
          const int ly = c / T, lx = c - ly * T;
          const int off = (ly + 3) * W + (lx + 3);
          const int offa = (ly + 1) * WA + (lx + 1);
          SAcc acc{su + off, sv + off, sp + off, W, sau + offa, sav + offa, WA};
          const int cell = (ty0 + ly) * nx + tx0 + lx;
          double un, vn, pn;
          fb_cell(acc, p, sx, sy, tau, damp, w[2 * n + cell], sp[off], un, vn, pn);
          nu[cell] = un;
          nu[n + cell] = vn;
          nu[2 * n + cell] = pn;
        }
        __syncthreads();
      }
      grid.sync();
    }
    if (nsub % 2 == 1) {
      for (long long b = 0; b < batch; ++b)
        for (int cell = first; cell < n; cell += stride) {
          double* w = work + b * 6 * n;
          double* sb = st + b * ld;
          sb[cell] = w[3 * n + cell];
          sb[n + cell] = w[4 * n + cell];
          sb[2 * n + cell] = w[5 * n + cell];
        }
      grid.sync();
    }
  }
}

// Temporal-blocked variant: K substeps per grid barrier.  Each CTA stages its T x T
// tile of (u, v, p) with a 3K-cell halo, then runs the K substeps on shrinking regions
// in shared memory: u', v' of the whole region first (stored), one CTA barrier, then
// p' from the stored neighbour velocities (no recomputation), p updated in place and
// the (u, v) / (u', v') planes swapped.  Region margins per substep (M = 3K at entry):
// u', v' on M - 2, p' on M - 3, next M = M - 3, so the last p' lands on the tile.
// Same expressions as fb_cell (bitwise equal to the per-cell variants).
struct TbPlanes {
  double* u;
  double* v;
  double* p;
  double* un;
  double* vn;
};

template <int TMX, int TMY, int K, bool FIXX, bool FIXY>
__device__ __forceinline__ void tb_block(double* sm, const double* __restrict__ cu,
                                         double* __restrict__ nu, const double* __restrict__ w,
                                         int tx0, int ty0, int twx_, int twy_, const ExactParams& p,
                                         double sx, double sy, double tau, bool damp) {
  // TMX x TMY: largest tile (fixes the shared-memory planes); this tile is twx x twy
  // (FIXX / FIXY: every tile has the full extent -- compile-time loop bounds)
  const int twx = FIXX ? TMX : twx_, twy = FIXY ? TMY : twy_;
  constexpr int H = 3 * K, W = TMX + 2 * H, WW = W * (TMY + 2 * H);
  const int nx = p.nx, ny = p.ny, n = nx * ny;
  double* planes = sm;  // u, v, p, un, vn : W x W each
  // ---- stage (u, v, p) with halo H
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    constexpr int CX = (W + 31) / 32;
    int gx[CX];
#pragma unroll
    for (int k = 0; k < CX; ++k) {
      int x = tx0 - H + lane + 32 * k;
      x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
      gx[k] = x;
    }
    for (int y = warp; y < twy + 2 * H; y += nwarp) {
      int gy = ty0 - H + y;
      gy = gy < 0 ? gy + ny : (gy >= ny ? gy - ny : gy);
      const double* row = cu + (size_t)gy * nx;
#pragma unroll
      for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int k = 0; k < CX; ++k)
          if (lane + 32 * k < twx + 2 * H)
            __pipeline_memcpy_async(&planes[f * WW + y * W + lane + 32 * k], row + (size_t)f * n + gx[k], 8);
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
  }
  __syncthreads();
  double* su = planes;
  double* sv = planes + WW;
  double* sp = planes + 2 * WW;
  double* sun = planes + 3 * WW;
  double* svn = planes + 4 * WW;
  const double* au = w;
  const double* av = w + n;
  const double* ap = w + 2 * n;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int M = H - 3 * s;
    // u', v' on margin M - 2 (frozen tendencies read from global memory / L2)
    {
      const int m = M - 2, Rx = twx + 2 * m, Ry = twy + 2 * m, o = H - m;
      for (int c = threadIdx.x; c < Rx * Ry; c += blockDim.x) {
        const int ly = c / Rx, lx = c - ly * Rx;
        const int off = (ly + o) * W + (lx + o);
        int gy = ty0 - m + ly, gxx = tx0 - m + lx;
        gy = gy < 0 ? gy + ny : (gy >= ny ? gy - ny : gy);
        gxx = gxx < 0 ? gxx + nx : (gxx >= nx ? gxx - nx : gxx);
        const int cell = gy * nx + gxx;
        const SAccV acc{su + off, sv + off, sp + off, W, au[cell], av[cell]};
        sun[off] = un_at<0, 0>(acc, p, sx, sy, tau, damp);
        svn[off] = vn_at<0, 0>(acc, p, sx, sy, tau, damp);
      }
    }
    __syncthreads();
    // p' on margin M - 3 (in place: every thread reads and writes only its own p cells)
    {
      const int m = M - 3, Rx = twx + 2 * m, Ry = twy + 2 * m, o = H - m;
      for (int c = threadIdx.x; c < Rx * Ry; c += blockDim.x) {
        const int ly = c / Rx, lx = c - ly * Rx;
        const int off = (ly + o) * W + (lx + o);
        int gy = ty0 - m + ly, gxx = tx0 - m + lx;
        gy = gy < 0 ? gy + ny : (gy >= ny ? gy - ny : gy);
        gxx = gxx < 0 ? gxx + nx : (gxx >= nx ? gxx - nx : gxx);
        const int cell = gy * nx + gxx;
        const double divn = (sun[off + 1] - sun[off - 1]) * sx + (svn[off + W] - svn[off - W]) * sy;
        sp[off] = sp[off] + tau * (ap[cell] - p.cs * divn);
      }
    }
    __syncthreads();
    double* t = su; su = sun; sun = t;
    t = sv; sv = svn; svn = t;
  }
  // ---- the tile's new (u, v, p)
  for (int c = threadIdx.x; c < twx * twy; c += blockDim.x) {
    const int ly = c / twx, lx = c - ly * twx;
    const int off = (ly + H) * W + (lx + H);
    const int cell = (ty0 + ly) * nx + tx0 + lx;
    nu[cell] = su[off];
    nu[n + cell] = sv[off];
    nu[2 * n + cell] = sp[off];
  }
  __syncthreads();
}

template <int TMX, int TMY, int K, int NT, int MINB, bool FIXX, bool FIXY, int ORD>
__global__ void __launch_bounds__(NT, MINB) fefb_tb_coop(double* st, int batch, long long ld,
                                                   ExactParams p, int nsteps, double tau, int nsub,
                                                   double* work, int tiles_x, int tiles_y) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  const int nx = p.nx, ny = p.ny;
  const int n = nx * ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  // tiles_x x tiles_y near-equal tiles of at most TMX x TMY (edges floor(k n / tiles))
  const int tiles = tiles_x * tiles_y;
  const long long work_items = (long long)tiles * batch;
  const int stride = gridDim.x * blockDim.x;
  const int first = blockIdx.x * blockDim.x + threadIdx.x;
  const int nblk = nsub / K, ntail = nsub - nblk * K;
  for (int step = 0; step < nsteps; ++step) {
    for (long long b = 0; b < batch; ++b)
      for (int cell = first; cell < n; cell += stride) {
        const int j = cell / nx, i = cell - j * nx;
        const double* q = st + b * ld;
        double* w = work + b * 6 * n;
        w[cell] = adv_at<ORD>(p, q, j, i);
        w[n + cell] = adv_at<ORD>(p, q + n, j, i);
        w[2 * n + cell] = adv_at<ORD>(p, q + 2 * n, j, i);
      }
    grid.sync();
    int blk = 0;
    for (; blk < nblk + ntail; ++blk) {
      const bool from_state = (blk % 2 == 0);
      for (long long it = blockIdx.x; it < work_items; it += gridDim.x) {
        const long long b = it / tiles;
        const int t = (int)(it - b * tiles);
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int ty0 = (int)((long long)iy * ny / tiles_y), tx0 = (int)((long long)ix * nx / tiles_x);
        const int twy = (int)((long long)(iy + 1) * ny / tiles_y) - ty0;
        const int twx = (int)((long long)(ix + 1) * nx / tiles_x) - tx0;
        double* w = work + b * 6 * n;
        double* sb = st + b * ld;
        const double* cu = from_state ? sb : w + 3 * n;
        double* nu = from_state ? w + 3 * n : sb;
        if (blk < nblk)
          tb_block<TMX, TMY, K, FIXX, FIXY>(sm, cu, nu, w, tx0, ty0, twx, twy, p, sx, sy, tau, damp);
        else
          tb_block<TMX, TMY, 1, FIXX, FIXY>(sm, cu, nu, w, tx0, ty0, twx, twy, p, sx, sy, tau, damp);
      }
      grid.sync();
    }
    if (blk % 2 == 1) {
      for (long long b = 0; b < batch; ++b)
        for (int cell = first; cell < n; cell += stride) {
          double* w = work + b * 6 * n;
          double* sb = st + b * ld;
          sb[cell] = w[3 * n + cell];
          sb[n + cell] = w[4 * n + cell];
          sb[2 * n + cell] = w[5 * n + cell];
        }
      grid.sync();
    }
  }
}

// ---------------------------------------------------------------- neighbour-flag G
// One FE-FB propagation (split_fe_fb_step x nsteps, integrators.py:103-106 with
// fb_substeps, numba_backend.py:131-146) of ONE state as a persistent cooperative launch
// without grid barriers.  The state is cut into 32 x TY tiles; per step a tile runs phase A
// (its cells' frozen advective tendencies) and ceil(nsub / K) substep blocks, each block K
// substeps on its tile plus a 3K-cell halo in shared memory (temporal blocking).  Before a
// phase a tile waits only until its 8 neighbour tiles have finished the previous phase
// (per-tile phase counters, release / acquire): that orders both the halo it reads (RAW)
// and the buffer it overwrites, which those neighbours read in the previous phase (WAR).
// A CTA walks its tiles phase by phase, so every wait points at a lower phase: no deadlock.
//
// Same expressions as fb_cell (bitwise equal to the reference; -fmad=false), restructured:
// the divergence D = dx(u) + dy(v) that both damping terms difference is computed once per
// cell and substep (the reference's own damping_tendencies form), each thread owns one
// column of cells of the region (compile-time strip), its cells' tendencies stay in
// registers for the whole block, and staging loads bypass L1 (ld.global.cg).
template <int TMY, int K, int NT>
struct NfCfg {
  // x halo rounded up to even (HX): staged rows start 16-byte aligned (cp.async of pairs)
  static constexpr int TX = 32, H = 3 * K, HX = (H + 1) / 2 * 2, RX = TX + 2 * HX, RYM = TMY + 2 * H;
  static constexpr int NSTR = NT / RX;                // column strips of the region
  static constexpr int S = (RYM + NSTR - 1) / NSTR;   // cells per thread (one column)
  // plane: NSTR * S rows (>= RYM) plus a padding row above and below (branch-free passes)
  static constexpr int PL = RX * (NSTR * S + 2);
  static constexpr size_t SMEM = sizeof(double) * 6 * PL;
  static_assert(NSTR >= 1, "the region must be at most NT columns wide");
};

// Global storage of the neighbour-flag G.  Three plane families of (u, v, p): the state (0),
// the ping-pong state (1) and the frozen tendencies (2).  FlatAcc: one state and one work
// buffer (the production layout).  ShardAcc: the grid's rows split into row shards
// [s R, (s+1) R), each shard with its own state, work and flag buffers -- the storage of a
// row-sharded G, where a tile reads its halo rows from the neighbouring
// shard's buffers and waits on that shard's flags.
constexpr int kMaxRowShards = 8;
struct NfShards {
  double* st[kMaxRowShards];    // rows [s R, (s+1) R) of u, v, p (field stride R nx)
  double* work[kMaxRowShards];  // au, av, ap, then the ping-pong u, v, p (field stride R nx)
  int* flags[kMaxRowShards];    // phase counters of the shard's tiles
  int rows;                     // R
  int tiles;                    // tiles per shard (tile rows per shard x tiles_x)
};
struct FlatAcc {
  double* st;
  double* work;
  int* fl;
  long long n;
  int nx;
  __device__ __forceinline__ double* pl(int fam, int f, int gy) const {
    double* b = fam == 0 ? st : work + (fam == 1 ? 3 : 0) * n;
    return b + f * n + (long long)gy * nx;
  }
  __device__ __forceinline__ int* flag(int t) const { return fl + t; }
};
struct ShardAcc {
  NfShards sh;
  int nx;
  __device__ __forceinline__ double* pl(int fam, int f, int gy) const {
    const int s = gy / sh.rows;
    const long long fs = (long long)sh.rows * nx;
    double* b = fam == 0 ? sh.st[s] : sh.work[s] + (fam == 1 ? 3 : 0) * fs;
    return b + f * fs + (long long)(gy - s * sh.rows) * nx;
  }
  __device__ __forceinline__ int* flag(int t) const {
    const int s = t / sh.tiles;
    return sh.flags[s] + (t - s * sh.tiles);
  }
};

// adv_at with the field's rows through an accessor (same expressions, same order)
template <int ORD, class R>
__device__ __forceinline__ double adv_at_rows(const ExactParams& p, const R& row, int j, int i) {
  const int order = ORD > 0 ? ORD : p.order;
  const int nx = p.nx, ny = p.ny;
  const int ip = i + 1 < nx ? i + 1 : 0;
  const int jp = j + 1 < ny ? j + 1 : 0;
  auto fx = [&](int jj, int f) {
    const double* r = row(jj);
    return face_flux(order, p.uf[(size_t)jj * nx + f], r[wrapi(f - 3, nx)], r[wrapi(f - 2, nx)],
                     r[wrapi(f - 1, nx)], r[f], r[wrapi(f + 1, nx)], r[wrapi(f + 2, nx)]);
  };
  auto gyf = [&](int f, int ii) {
    return face_flux(order, p.vf[(size_t)f * nx + ii], row(wrapi(f - 3, ny))[ii], row(wrapi(f - 2, ny))[ii],
                     row(wrapi(f - 1, ny))[ii], row(f)[ii], row(wrapi(f + 1, ny))[ii], row(wrapi(f + 2, ny))[ii]);
  };
  const double fxi = fx(j, i), fxp = fx(j, ip);
  const double gyj = gyf(j, i), gyp = gyf(jp, i);
  const double tx = -(fxp - fxi), ty = (gyp - gyj);
  return (p.inv_dx != 0.0 ? tx * p.inv_dx : tx / p.dx) - (p.inv_dy != 0.0 ? ty * p.inv_dy : ty / p.dy);
}

__device__ __forceinline__ int nf_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void nf_st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef NF_SLEEP
#define NF_SLEEP 1
#endif
#ifndef NF_FENCE
#define NF_FENCE 1
#endif
// wait until the 8 neighbours of tile (ix, iy) have completed phase `ph`
template <class A>
__device__ __forceinline__ void nf_wait(const A& acc, int ix, int iy, int tiles_x, int tiles_y, int ph) {
  if (ph > 0 && threadIdx.x < 9 && threadIdx.x != 4) {
    int jx = ix + (int)threadIdx.x % 3 - 1, jy = iy + (int)threadIdx.x / 3 - 1;
    jx += jx < 0 ? tiles_x : 0;
    jx -= jx >= tiles_x ? tiles_x : 0;
    jy += jy < 0 ? tiles_y : 0;
    jy -= jy >= tiles_y ? tiles_y : 0;
    const int* f = acc.flag(jy * tiles_x + jx);
    long long spins = 0;
    while (nf_ld_acquire(f) < ph) {
      if (NF_SLEEP) __nanosleep(32);
      if (++spins > (1LL << 28)) __trap();  // a broken dependency fails, never hangs
    }
  }
  __syncthreads();
}
// the CTA barrier orders every thread's stores before thread 0's fence (cumulative) and
// release, as cooperative groups' grid barrier does
template <class A>
__device__ __forceinline__ void nf_signal(const A& acc, int tile, int ph) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (NF_FENCE) __threadfence();
    nf_st_release(acc.flag(tile), ph);
  }
}

template <int TMY, int K, int NT, int ORD, class ACC>
__device__ __forceinline__ void fefb_nf_body(const ACC& acc, ExactParams p, int nsteps, double tau, int nsub,
                                             int tiles_x, int tiles_y, int tile_lo, int tile_hi) {
  using C = NfCfg<TMY, K, NT>;
  constexpr int TX = C::TX, H = C::H, HX = C::HX, RX = C::RX, PL = C::PL, S = C::S;
  extern __shared__ double sm[];
  const int nx = p.nx, ny = p.ny;
  const long long n = (long long)nx * ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy, cs = p.cs, a1 = p.a1, a2 = p.a2;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  (void)n;
  const int tid = threadIdx.x;
  const int cx = tid % RX, strip = tid / RX;  // this thread's column and strip of the region
  const bool comp = strip < C::NSTR;
  const int y0s = strip * S;
  const int nblk = (nsub + K - 1) / K;
  int ph = 0;
  for (int step = 0; step < nsteps; ++step) {
    // ---- phase A: frozen advective tendency of the tile's cells (physics.py:67-74)
    for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
      const int iy = t / tiles_x, ix = t - iy * tiles_x;
      const int ty0 = (int)((long long)iy * ny / tiles_y), ty1 = (int)((long long)(iy + 1) * ny / tiles_y);
      nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
      for (int c = tid; c < TX * (ty1 - ty0); c += NT) {
        const int j = ty0 + c / TX, i = ix * TX + c % TX;
#pragma unroll
        for (int f = 0; f < 3; ++f)
          acc.pl(2, f, j)[i] = adv_at_rows<ORD>(p, [&](int r) -> const double* { return acc.pl(0, f, r); }, j, i);
      }
      nf_signal(acc, t, ph + 1);
    }
    ++ph;
    // ---- substep blocks
    for (int blk = 0; blk < nblk; ++blk) {
      const int ks = min(K, nsub - blk * K);
      const int fsrc = (blk % 2 == 0) ? 0 : 1, fdst = 1 - fsrc;  // state <-> ping-pong planes
      for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int tx0 = ix * TX;
        const int ty0 = (int)((long long)iy * ny / tiles_y);
        const int TY = (int)((long long)(iy + 1) * ny / tiles_y) - ty0;
        const int RY = TY + 2 * H;
        nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
        double* su = sm + RX;  // row 0 of the region (one padding row above)
        double* sv = su + PL;
        double* sp = sv + PL;
        double* sd = sp + PL;
        double* sun = sd + PL;
        double* svn = sun + PL;
        // stage (u, v, p) of the region [tx0 - HX, tx0 + TX + HX) x [ty0 - H, ty0 + TY + H):
        // 16-byte cp.async.cg (L2 only) of column pairs, all in flight before one wait
        for (int c = tid; c < (RX / 2) * RY; c += NT) {
          const int y = c / (RX / 2), x = 2 * (c - y * (RX / 2));
          int gx = tx0 - HX + x, gy = ty0 - H + y;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          gy += gy < 0 ? ny : 0;
          gy -= gy >= ny ? ny : 0;
          const int o = y * RX + x;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(su + f * PL + o);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(acc.pl(fsrc, f, gy) + gx)
                         : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // this thread's cells' tendencies (registers for the whole block)
        double tu[S], tv[S], tp[S];
        if (comp) {
          int gx = tx0 - HX + cx;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          int gy = ty0 - H + y0s;
          gy += gy < 0 ? ny : 0;
          gy -= gy >= ny ? ny : 0;
#pragma unroll
          for (int r = 0; r < S; ++r) {
            tu[r] = __ldcg(acc.pl(2, 0, gy) + gx);
            tv[r] = __ldcg(acc.pl(2, 1, gy) + gx);
            tp[r] = __ldcg(acc.pl(2, 2, gy) + gx);
            // next row, wrapping at the bottom edge (rows past the region: any valid row)
            if (++gy >= ny) gy = 0;
          }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        // Each pass computes all S cells of the thread's column branch-free (independent
        // rows: full ILP), then stores the rows inside the pass's margin.  Rows outside it
        // carry garbage that no valid cell ever reads (the margins shrink by the stencil
        // radius); planes have a padding row above and below, so no access leaves them.
        for (int ss = 0; ss < ks; ++ss) {
          const int M = H - 3 * ss;  // (u, v, p) valid on margin M of the tile
          // D = dx(u) + dy(v) on margin M - 1 (damping_tendencies' div, numba_backend.py:108-111)
          if (damp && comp && cx >= HX - (M - 1) && cx < HX + TX + (M - 1) &&
              y0s + S > H - (M - 1) && y0s < H + TY + (M - 1)) {
            double dd[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = (y0s + r) * RX + cx;
              dd[r] = (su[o + 1] - su[o - 1]) * sx + (sv[o + RX] - sv[o - RX]) * sy;
            }
            const int lo = H - (M - 1) - y0s, hi = H + TY + (M - 1) - y0s;
#pragma unroll
            for (int r = 0; r < S; ++r)
              if (r >= lo && r < hi) sd[(y0s + r) * RX + cx] = dd[r];
          }
          __syncthreads();
          // u', v' on margin M - 2 (fb_substeps, numba_backend.py:137-143)
          if (comp && cx >= HX - (M - 2) && cx < HX + TX + (M - 2) &&
              y0s + S > H - (M - 2) && y0s < H + TY + (M - 2)) {
            double nu_[S], nv_[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = (y0s + r) * RX + cx;
              double du = tu[r] - cs * ((sp[o + 1] - sp[o - 1]) * sx);
              double dv = tv[r] - cs * ((sp[o + RX] - sp[o - RX]) * sy);
              if (damp) {
                du = du + a1 * ((sd[o + 1] - sd[o - 1]) * sx);
                dv = dv + a2 * ((sd[o + RX] - sd[o - RX]) * sy);
              }
              nu_[r] = su[o] + tau * du;
              nv_[r] = sv[o] + tau * dv;
            }
            const int lo = H - (M - 2) - y0s, hi = H + TY + (M - 2) - y0s;
#pragma unroll
            for (int r = 0; r < S; ++r)
              if (r >= lo && r < hi) {
                sun[(y0s + r) * RX + cx] = nu_[r];
                svn[(y0s + r) * RX + cx] = nv_[r];
              }
          }
          __syncthreads();
          // p' on margin M - 3 from the new velocities (numba_backend.py:144-145)
          if (comp && cx >= HX - (M - 3) && cx < HX + TX + (M - 3) &&
              y0s + S > H - (M - 3) && y0s < H + TY + (M - 3)) {
            double np_[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = (y0s + r) * RX + cx;
              const double divn = (sun[o + 1] - sun[o - 1]) * sx + (svn[o + RX] - svn[o - RX]) * sy;
              np_[r] = sp[o] + tau * (tp[r] - cs * divn);
            }
            const int lo = H - (M - 3) - y0s, hi = H + TY + (M - 3) - y0s;
#pragma unroll
            for (int r = 0; r < S; ++r)
              if (r >= lo && r < hi) sp[(y0s + r) * RX + cx] = np_[r];
          }
          __syncthreads();
          double* tt = su;
          su = sun;
          sun = tt;
          tt = sv;
          sv = svn;
          svn = tt;
        }
        // the tile's new (u, v, p)
        for (int c = tid; c < TX * TY; c += NT) {
          const int ly = c / TX, lx = c - ly * TX;
          const int o = (ly + H) * RX + lx + HX;
          const int gy = ty0 + ly, gx = tx0 + lx;
          acc.pl(fdst, 0, gy)[gx] = su[o];
          acc.pl(fdst, 1, gy)[gx] = sv[o];
          acc.pl(fdst, 2, gy)[gx] = sp[o];
        }
        nf_signal(acc, t, ph + 1);
      }
      ++ph;
    }
    if (nblk % 2 == 1) {  // the last block wrote ws: copy the tiles back (WAR on st: a phase)
      for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int ty0 = (int)((long long)iy * ny / tiles_y), ty1 = (int)((long long)(iy + 1) * ny / tiles_y);
        nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
        for (int c = tid; c < TX * (ty1 - ty0); c += NT) {
          const int gy = ty0 + c / TX, gx = ix * TX + c % TX;
#pragma unroll
          for (int f = 0; f < 3; ++f) acc.pl(0, f, gy)[gx] = acc.pl(1, f, gy)[gx];
        }
        nf_signal(acc, t, ph + 1);
      }
      ++ph;
    }
  }
}

// ---- the same G with phase A folded into the first substep block of each step.
// The first block stages the region with E more cells of margin (the flux stencil's reach:
// 1 for the order-1 coarse flux, 3 otherwise) and computes the frozen advective tendencies
// of every region cell within the 3K margin from shared memory (adv_at's expressions and
// order, bitwise), so no phase of its own is needed and no tendency halo is exchanged.
// When each CTA owns one tile the tendencies stay in registers for the whole step;
// otherwise the tile's own cells are written to the tendency planes and later blocks read
// them (neighbours' halo included) back, as the phase-A form does.
template <int TMY, int K, int NT, int E>
struct NfmCfg {
  static constexpr int TX = 32, H = 3 * K, HE = H + E, HX = (HE + 1) / 2 * 2, RX = TX + 2 * HX, RYM = TMY + 2 * HE;
  static constexpr int NSTR = NT / RX;
  static constexpr int S = (RYM + NSTR - 1) / NSTR;
  static constexpr int PL = RX * (NSTR * S + 2);
  static constexpr size_t SMEM = sizeof(double) * 6 * PL;
  static_assert(NSTR >= 1, "the region must be at most NT columns wide");
};
template <int ORD>
__host__ __device__ constexpr int nfm_reach() { return ORD == 1 ? 1 : 3; }

// adv_at (flux_divergence of flux_x / flux_y) of region cell (x, y) from a staged plane;
// gx, gy: the cell's global column and row
template <int ORD, int RX>
__device__ __forceinline__ double adv_smem(const ExactParams& p, const double* pl, int x, int y, int gx, int gy) {
  const int order = ORD > 0 ? ORD : p.order;
  const int nx = p.nx, ny = p.ny;
  const int gxp = gx + 1 < nx ? gx + 1 : 0;
  const int gyp = gy + 1 < ny ? gy + 1 : 0;
  const double* r = pl + y * RX;
  auto fx = [&](int f, int gf) {  // face between region cells f-1 | f of row y
    const double uface = p.cvel ? p.uc : __ldg(p.uf + (size_t)gy * nx + gf);
    return face_flux(order, uface, r[f - 3], r[f - 2], r[f - 1], r[f], r[f + 1], r[f + 2]);
  };
  auto gyf = [&](int f, int gf) {  // face between region rows f-1 | f of column x
    const double* c = pl + x;
    const double vface = p.cvel ? p.vc : __ldg(p.vf + (size_t)gf * nx + gx);
    return face_flux(order, vface, c[(f - 3) * RX], c[(f - 2) * RX], c[(f - 1) * RX],
                     c[f * RX], c[(f + 1) * RX], c[(f + 2) * RX]);
  };
  const double fxi = fx(x, gx), fxp = fx(x + 1, gxp);
  const double gyj = gyf(y, gy), gyq = gyf(y + 1, gyp);
  const double tx = -(fxp - fxi), ty = (gyq - gyj);
  return (p.inv_dx != 0.0 ? tx * p.inv_dx : tx / p.dx) - (p.inv_dy != 0.0 ? ty * p.inv_dy : ty / p.dy);
}

template <int TMY, int K, int NT, int ORD, class ACC>
__device__ __forceinline__ void fefb_nfm_body(const ACC& acc, ExactParams p, int nsteps, double tau, int nsub,
                                              int tiles_x, int tiles_y, int tile_lo, int tile_hi) {
  using C = NfmCfg<TMY, K, NT, nfm_reach<ORD>()>;
  constexpr int TX = C::TX, H = C::H, HE = C::HE, HX = C::HX, RX = C::RX, PL = C::PL, S = C::S;
  extern __shared__ double sm[];
  const int nx = p.nx, ny = p.ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy, cs = p.cs, a1 = p.a1, a2 = p.a2;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  const int tid = threadIdx.x;
  const int cx = tid % RX, strip = tid / RX;  // this thread's column and strip of the region
  const bool comp = strip < C::NSTR;
  const int y0s = strip * S;
  const int nblk = (nsub + K - 1) / K;
  const bool resident = tile_hi - tile_lo <= (int)gridDim.x;  // one tile per CTA: tendencies stay in registers
  double tu[S], tv[S], tp[S];
  int ph = 0;
  for (int step = 0; step < nsteps; ++step) {
    for (int blk = 0; blk < nblk; ++blk) {
      const int ks = min(K, nsub - blk * K);
      const int fsrc = (blk % 2 == 0) ? 0 : 1, fdst = 1 - fsrc;  // state <-> ping-pong planes
      for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int tx0 = ix * TX;
        const int ty0 = (int)((long long)iy * ny / tiles_y);
        const int TY = (int)((long long)(iy + 1) * ny / tiles_y) - ty0;
        const int RY = TY + 2 * HE;
        nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
        double* su = sm + RX;  // row 0 of the region (one padding row above)
        double* sv = su + PL;
        double* sp = sv + PL;
        double* sd = sp + PL;
        double* sun = sd + PL;
        double* svn = sun + PL;
        for (int c = tid; c < (RX / 2) * RY; c += NT) {
          const int y = c / (RX / 2), x = 2 * (c - y * (RX / 2));
          int gx = tx0 - HX + x, gy = ty0 - HE + y;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          gy += gy < 0 ? ny : 0;
          gy -= gy >= ny ? ny : 0;
          const int o = y * RX + x;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(su + f * PL + o);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(acc.pl(fsrc, f, gy) + gx)
                         : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (blk > 0 && !resident && comp) {  // tendencies of this tile's region (own + neighbours')
          int gx = tx0 - HX + cx;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          int gy = ty0 - HE + y0s;
          gy += gy < 0 ? ny : 0;
          gy -= gy >= ny ? ny : 0;
#pragma unroll
          for (int r = 0; r < S; ++r) {
            tu[r] = __ldcg(acc.pl(2, 0, gy) + gx);
            tv[r] = __ldcg(acc.pl(2, 1, gy) + gx);
            tp[r] = __ldcg(acc.pl(2, 2, gy) + gx);
            if (++gy >= ny) gy = 0;
          }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (blk == 0 && comp) {  // frozen advective tendencies (physics.py:67-74) on margin H
          int gx = tx0 - HX + cx;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          const bool colin = cx >= HX - H && cx < HX + TX + H;
          const bool own_x = cx >= HX && cx < HX + TX;
#pragma unroll
          for (int r = 0; r < S; ++r) {
            const int y = y0s + r;
            if (colin && y >= HE - H && y < HE + TY + H) {
              int gy = ty0 - HE + y;
              gy += gy < 0 ? ny : 0;
              gy -= gy >= ny ? ny : 0;
              tu[r] = adv_smem<ORD, RX>(p, su, cx, y, gx, gy);
              tv[r] = adv_smem<ORD, RX>(p, sv, cx, y, gx, gy);
              tp[r] = adv_smem<ORD, RX>(p, sp, cx, y, gx, gy);
              if (!resident && own_x && y >= HE && y < HE + TY) {
                acc.pl(2, 0, gy)[gx] = tu[r];
                acc.pl(2, 1, gy)[gx] = tv[r];
                acc.pl(2, 2, gy)[gx] = tp[r];
              }
            } else {
              tu[r] = tv[r] = tp[r] = 0.0;
            }
          }
        }
        for (int ss = 0; ss < ks; ++ss) {
          const int M = H - 3 * ss;  // (u, v, p) valid on margin M of the tile
          // D = dx(u) + dy(v) on margin M - 1 (damping_tendencies' div, numba_backend.py:108-111)
          if (damp && comp && cx >= HX - (M - 1) && cx < HX + TX + (M - 1) &&
              y0s + S > HE - (M - 1) && y0s < HE + TY + (M - 1)) {
            double dd[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = (y0s + r) * RX + cx;
              dd[r] = (su[o + 1] - su[o - 1]) * sx + (sv[o + RX] - sv[o - RX]) * sy;
            }
            const int lo = HE - (M - 1) - y0s, hi = HE + TY + (M - 1) - y0s;
#pragma unroll
            for (int r = 0; r < S; ++r)
              if (r >= lo && r < hi) sd[(y0s + r) * RX + cx] = dd[r];
          }
          __syncthreads();
          // u', v' on margin M - 2 (fb_substeps, numba_backend.py:137-143)
          if (comp && cx >= HX - (M - 2) && cx < HX + TX + (M - 2) &&
              y0s + S > HE - (M - 2) && y0s < HE + TY + (M - 2)) {
            double nu_[S], nv_[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = (y0s + r) * RX + cx;
              double du = tu[r] - cs * ((sp[o + 1] - sp[o - 1]) * sx);
              double dv = tv[r] - cs * ((sp[o + RX] - sp[o - RX]) * sy);
              if (damp) {
                du = du + a1 * ((sd[o + 1] - sd[o - 1]) * sx);
                dv = dv + a2 * ((sd[o + RX] - sd[o - RX]) * sy);
              }
              nu_[r] = su[o] + tau * du;
              nv_[r] = sv[o] + tau * dv;
            }
            const int lo = HE - (M - 2) - y0s, hi = HE + TY + (M - 2) - y0s;
#pragma unroll
            for (int r = 0; r < S; ++r)
              if (r >= lo && r < hi) {
                sun[(y0s + r) * RX + cx] = nu_[r];
                svn[(y0s + r) * RX + cx] = nv_[r];
              }
          }
          __syncthreads();
          // p' on margin M - 3 from the new velocities (numba_backend.py:144-145)
          if (comp && cx >= HX - (M - 3) && cx < HX + TX + (M - 3) &&
              y0s + S > HE - (M - 3) && y0s < HE + TY + (M - 3)) {
            double np_[S];
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = (y0s + r) * RX + cx;
              const double divn = (sun[o + 1] - sun[o - 1]) * sx + (svn[o + RX] - svn[o - RX]) * sy;
              np_[r] = sp[o] + tau * (tp[r] - cs * divn);
            }
            const int lo = HE - (M - 3) - y0s, hi = HE + TY + (M - 3) - y0s;
#pragma unroll
            for (int r = 0; r < S; ++r)
              if (r >= lo && r < hi) sp[(y0s + r) * RX + cx] = np_[r];
          }
          __syncthreads();
          double* tt = su;
          su = sun;
          sun = tt;
          tt = sv;
          sv = svn;
          svn = tt;
        }
        for (int c = tid; c < TX * TY; c += NT) {
          const int ly = c / TX, lx = c - ly * TX;
          const int o = (ly + HE) * RX + lx + HX;
          const int gy = ty0 + ly, gx = tx0 + lx;
          acc.pl(fdst, 0, gy)[gx] = su[o];
          acc.pl(fdst, 1, gy)[gx] = sv[o];
          acc.pl(fdst, 2, gy)[gx] = sp[o];
        }
        nf_signal(acc, t, ph + 1);
      }
      ++ph;
    }
    if (nblk % 2 == 1) {  // the last block wrote ws: copy the tiles back (WAR on st: a phase)
      for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int ty0 = (int)((long long)iy * ny / tiles_y), ty1 = (int)((long long)(iy + 1) * ny / tiles_y);
        nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
        for (int c = tid; c < TX * (ty1 - ty0); c += NT) {
          const int gy = ty0 + c / TX, gx = ix * TX + c % TX;
#pragma unroll
          for (int f = 0; f < 3; ++f) acc.pl(0, f, gy)[gx] = acc.pl(1, f, gy)[gx];
        }
        nf_signal(acc, t, ph + 1);
      }
      ++ph;
    }
  }
}

template <int TMY, int K, int NT, int ORD, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) fefb_nfm_kernel(double* st, ExactParams p, int nsteps, double tau,
                                                         int nsub, double* work, int tiles_x, int tiles_y,
                                                         int* flags) {
  const FlatAcc acc{st, work, flags, (long long)p.nx * p.ny, p.nx};
  fefb_nfm_body<TMY, K, NT, ORD>(acc, p, nsteps, tau, nsub, tiles_x, tiles_y, 0, tiles_x * tiles_y);
}

// ---- the folded G with register-resident columns.  Each thread keeps its column strip's
// v, p, D (= div(u, v)) and frozen p-tendency in registers, so the y-neighbours of a
// stencil are registers (only a strip's two end rows read the next strip's values from
// shared memory) and only x-neighbours, u and the frozen u/v tendencies come from shared
// memory: ~9 shared loads per cell and substep instead of 19.  The damping divergence of
// substep k+1, dx(u) + dy(v) of the new velocities, is the same expression (same operands,
// same order) as the divergence in substep k's pressure update, so it is taken from there:
// two passes per substep (u'/v', then p' and D) plus one D pass per block.  Passes run
// branch-free over every cell of the strip; cells outside a pass's valid margin hold values
// no valid cell ever reads (the margins shrink by the stencil radius), as in fefb_nf_body.
template <int TMY, int K, int NT, int ORD, class ACC>
__device__ __forceinline__ void fefb_nfr_body(const ACC& acc, ExactParams p, int nsteps, double tau, int nsub,
                                              int tiles_x, int tiles_y, int tile_lo, int tile_hi) {
  using C = NfmCfg<TMY, K, NT, nfm_reach<ORD>()>;
  constexpr int TX = C::TX, H = C::H, HE = C::HE, HX = C::HX, RX = C::RX, PL = C::PL, S = C::S;
  extern __shared__ double sm[];
  const int nx = p.nx, ny = p.ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy, cs = p.cs, a1 = p.a1, a2 = p.a2;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  const int tid = threadIdx.x;
  const int cx = tid % RX, strip = tid / RX;
  const bool comp = strip < C::NSTR;
  const int y0s = strip * S;
  const int nblk = (nsub + K - 1) / K;
  const bool resident = tile_hi - tile_lo <= (int)gridDim.x;
  // one tile per CTA and an even block count per step: the tile's own cells stay in shared
  // memory from block to block (and step to step).  A block then stages only the halo ring
  // and stores only the band its neighbours' regions reach (HX columns / HE rows from the
  // tile's edges); the whole tile goes out after the call's last block.
  const bool keep = resident && nblk % 2 == 0;
  double* const U = sm + RX;  // row 0 of the region (one padding row above each plane)
  double* const V = U + PL;
  double* const P = V + PL;
  double* const Dp = P + PL;
  double* const TU = Dp + PL;
  double* const TV = TU + PL;
  const int oc = y0s * RX + cx;  // this thread's first cell
  // does this thread's strip touch margin m of the tile (the cells a pass must produce)?
  auto inm = [&](int m, int TY) {
    return comp && cx >= HX - m && cx < HX + TX + m && y0s + S > HE - m && y0s < HE + TY + m;
  };
  double v[S], pr[S], dv_[S], tp[S];
  int ph = 0;
#ifdef PW_NF_PROF
  long long pt[7] = {0, 0, 0, 0, 0, 0, 0}, t0 = 0, t1 = 0;
#define NFP(k) do { t1 = clock64(); pt[k] += t1 - t0; t0 = t1; } while (0)
#else
#define NFP(k) do {} while (0)
#endif
  for (int step = 0; step < nsteps; ++step) {
    for (int blk = 0; blk < nblk; ++blk) {
      const int ks = min(K, nsub - blk * K);
      const int fsrc = (blk % 2 == 0) ? 0 : 1, fdst = 1 - fsrc;
      for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int tx0 = ix * TX;
        const int ty0 = (int)((long long)iy * ny / tiles_y);
        const int TY = (int)((long long)(iy + 1) * ny / tiles_y) - ty0;
        const int RY = TY + 2 * HE;
#ifdef PW_NF_PROF
        t0 = clock64();
#endif
        nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
        NFP(0);
        const bool ld_tend = blk > 0 && !resident;
        const bool ring_only = keep && (step > 0 || blk > 0);
        const bool last = step == nsteps - 1 && blk == nblk - 1;
        for (int c = tid; c < (RX / 2) * RY; c += NT) {
          const int y = c / (RX / 2), x = 2 * (c - y * (RX / 2));
          if (ring_only && x >= HX && x < HX + TX && y >= HE && y < HE + TY) continue;  // own cells: on chip
          int gx = tx0 - HX + x, gy = ty0 - HE + y;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          gy += gy < 0 ? ny : 0;
          gy -= gy >= ny ? ny : 0;
          const int o = y * RX + x;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(U + f * PL + o);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(acc.pl(fsrc, f, gy) + gx)
                         : "memory");
          }
          if (ld_tend) {
#pragma unroll
            for (int f = 0; f < 2; ++f) {
              const unsigned sa = (unsigned)__cvta_generic_to_shared(TU + f * PL + o);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(acc.pl(2, f, gy) + gx)
                           : "memory");
            }
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (ld_tend && comp) {
          int gx = tx0 - HX + cx;
          gx += gx < 0 ? nx : 0;
          gx -= gx >= nx ? nx : 0;
          int gy = ty0 - HE + y0s;
          gy += gy < 0 ? ny : 0;
          gy -= gy >= ny ? ny : 0;
#pragma unroll
          for (int r = 0; r < S; ++r) {
            tp[r] = __ldcg(acc.pl(2, 2, gy) + gx);
            if (++gy >= ny) gy = 0;
          }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        NFP(1);
        if (comp) {
          if (blk == 0) {  // frozen advective tendencies (physics.py:67-74) on margin H
            int gx = tx0 - HX + cx;
            gx += gx < 0 ? nx : 0;
            gx -= gx >= nx ? nx : 0;
            const bool colin = cx >= HX - H && cx < HX + TX + H;
            const bool own_x = cx >= HX && cx < HX + TX;
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int y = y0s + r;
              double au = 0.0, av = 0.0, ap = 0.0;
              if (colin && y >= HE - H && y < HE + TY + H) {
                int gy = ty0 - HE + y;
                gy += gy < 0 ? ny : 0;
                gy -= gy >= ny ? ny : 0;
                au = adv_smem<ORD, RX>(p, U, cx, y, gx, gy);
                av = adv_smem<ORD, RX>(p, V, cx, y, gx, gy);
                ap = adv_smem<ORD, RX>(p, P, cx, y, gx, gy);
                if (!resident && own_x && y >= HE && y < HE + TY) {
                  acc.pl(2, 0, gy)[gx] = au;
                  acc.pl(2, 1, gy)[gx] = av;
                  acc.pl(2, 2, gy)[gx] = ap;
                }
              }
              TU[oc + r * RX] = au;
              TV[oc + r * RX] = av;
              tp[r] = ap;
            }
          }
#pragma unroll
          for (int r = 0; r < S; ++r) {
            v[r] = V[oc + r * RX];
            pr[r] = P[oc + r * RX];
          }
          if (damp && inm(H - 1, TY)) {  // D = dx(u) + dy(v) (damping_tendencies' div, numba_backend.py:108-111)
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = oc + r * RX;
              const double vm = r > 0 ? v[r - 1] : V[o - RX];
              const double vp = r < S - 1 ? v[r + 1] : V[o + RX];
              dv_[r] = (U[o + 1] - U[o - 1]) * sx + (vp - vm) * sy;
              Dp[o] = dv_[r];
            }
          }
        }
        __syncthreads();
        NFP(2);
        for (int ss = 0; ss < ks; ++ss) {
          const int M = H - 3 * ss;  // (u, v, p) valid on margin M of the tile
          // u', v' on margin M - 2 (fb_substeps, numba_backend.py:137-143)
          if (inm(M - 2, TY)) {
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = oc + r * RX;
              const double pm = r > 0 ? pr[r - 1] : P[o - RX];
              const double pp = r < S - 1 ? pr[r + 1] : P[o + RX];
              double du = TU[o] - cs * ((P[o + 1] - P[o - 1]) * sx);
              double dv = TV[o] - cs * ((pp - pm) * sy);
              if (damp) {
                const double dm = r > 0 ? dv_[r - 1] : Dp[o - RX];
                const double dq = r < S - 1 ? dv_[r + 1] : Dp[o + RX];
                du = du + a1 * ((Dp[o + 1] - Dp[o - 1]) * sx);
                dv = dv + a2 * ((dq - dm) * sy);
              }
              U[o] = U[o] + tau * du;
              v[r] = v[r] + tau * dv;
            }
            V[oc] = v[0];
            V[oc + (S - 1) * RX] = v[S - 1];
          }
          __syncthreads();
          // p' on margin M - 3 from the new velocities (numba_backend.py:144-145); its
          // divergence is the next substep's D (needed on margin M - 4)
          if (inm(M - 3, TY)) {
#pragma unroll
            for (int r = 0; r < S; ++r) {
              const int o = oc + r * RX;
              const double vm = r > 0 ? v[r - 1] : V[o - RX];
              const double vp = r < S - 1 ? v[r + 1] : V[o + RX];
              const double divn = (U[o + 1] - U[o - 1]) * sx + (vp - vm) * sy;
              pr[r] = pr[r] + tau * (tp[r] - cs * divn);
              dv_[r] = divn;
            }
#pragma unroll
            for (int r = 0; r < S; ++r) {
              P[oc + r * RX] = pr[r];
              if (damp) Dp[oc + r * RX] = dv_[r];
            }
          }
          __syncthreads();
        }
        NFP(3);
        if (comp) {
#pragma unroll
          for (int r = 0; r < S; ++r) V[oc + r * RX] = v[r];
        }
        __syncthreads();
        NFP(4);
        for (int c = tid; c < TX * TY; c += NT) {
          const int ly = c / TX, lx = c - ly * TX;
          if (keep && !last && lx >= HX && lx < TX - HX && ly >= HE && ly < TY - HE) continue;  // no neighbour reads it
          const int o = (ly + HE) * RX + lx + HX;
          const int gy = ty0 + ly, gx = tx0 + lx;
          acc.pl(fdst, 0, gy)[gx] = U[o];
          acc.pl(fdst, 1, gy)[gx] = V[o];
          acc.pl(fdst, 2, gy)[gx] = P[o];
        }
        NFP(5);
        nf_signal(acc, t, ph + 1);
        NFP(6);
      }
      ++ph;
    }
    if (nblk % 2 == 1) {
      for (int t = tile_lo + blockIdx.x; t < tile_hi; t += gridDim.x) {
        const int iy = t / tiles_x, ix = t - iy * tiles_x;
        const int ty0 = (int)((long long)iy * ny / tiles_y), ty1 = (int)((long long)(iy + 1) * ny / tiles_y);
        nf_wait(acc, ix, iy, tiles_x, tiles_y, ph);
        for (int c = tid; c < TX * (ty1 - ty0); c += NT) {
          const int gy = ty0 + c / TX, gx = ix * TX + c % TX;
#pragma unroll
          for (int f = 0; f < 3; ++f) acc.pl(0, f, gy)[gx] = acc.pl(1, f, gy)[gx];
        }
        nf_signal(acc, t, ph + 1);
      }
      ++ph;
    }
  }
#ifdef PW_NF_PROF
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 70))
    printf("nfr cta %d: wait %lld stage %lld adv+D %lld passes %lld vsync %lld store %lld signal %lld cycles\n",
           blockIdx.x, pt[0], pt[1], pt[2], pt[3], pt[4], pt[5], pt[6]);
#endif
}

template <int TMY, int K, int NT, int ORD>
__global__ void __launch_bounds__(NT, 1) fefb_nfr_shard_kernel(NfShards sh, ExactParams p, int nsteps, double tau,
                                                               int nsub, int tiles_x, int tiles_y, int tile_lo,
                                                               int tile_hi) {
  const ShardAcc acc{sh, p.nx};
  fefb_nfr_body<TMY, K, NT, ORD>(acc, p, nsteps, tau, nsub, tiles_x, tiles_y, tile_lo, tile_hi);
}

template <int TMY, int K, int NT, int ORD, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) fefb_nfr_kernel(double* st, ExactParams p, int nsteps, double tau,
                                                         int nsub, double* work, int tiles_x, int tiles_y,
                                                         int* flags) {
  const FlatAcc acc{st, work, flags, (long long)p.nx * p.ny, p.nx};
  fefb_nfr_body<TMY, K, NT, ORD>(acc, p, nsteps, tau, nsub, tiles_x, tiles_y, 0, tiles_x * tiles_y);
}


template <int TMY, int K, int NT, int ORD, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) fefb_nf_kernel(double* st, ExactParams p, int nsteps, double tau,
                                                       int nsub, double* work, int tiles_x, int tiles_y,
                                                       int* flags) {
  const FlatAcc acc{st, work, flags, (long long)p.nx * p.ny, p.nx};
  fefb_nf_body<TMY, K, NT, ORD>(acc, p, nsteps, tau, nsub, tiles_x, tiles_y, 0, tiles_x * tiles_y);
}


template <int TMX, int TMY, int K>
constexpr size_t tb_smem() {
  return sizeof(double) * 5 * (TMX + 6 * K) * (TMY + 6 * K);
}

template <int T>
constexpr size_t tiled_smem() {
  return sizeof(double) * (3 * (T + 6) * (T + 6) + 2 * (T + 2) * (T + 2));
}

constexpr int kThreads = 256;
constexpr int kCoopThreads = 128;

}  // namespace

size_t rk3_exact_work_doubles(const ExactParams& p, int batch) {
  return (size_t)2 * 3 * p.nx * p.ny * (size_t)batch;
}

size_t fefb_exact_work_doubles(const ExactParams& p, int batch) {
  // + the neighbour-flag kernel's per-tile phase counters (<= nx/32 x ny/8 ints)
  return (size_t)6 * p.nx * p.ny * (size_t)batch + (size_t)p.nx * p.ny / 512 + 64;
}

void launch_rk3_exact(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                      int nsteps, double h, double* work) {
  const long long n3 = 3LL * p.nx * p.ny;
  const long long total = (long long)p.nx * p.ny * batch;
  const long long ncell = (long long)p.nx * p.ny;
  int bx = (int)std::min<long long>((ncell + kThreads - 1) / kThreads, (long long)c.num_sms * 16);
  if (bx < 1) bx = 1;
  PW_CHECK(batch <= 65535, PW_ERR_VALUE, "batch too large for one launch");
  const dim3 blocks(bx, batch);
  double* s1 = work;
  double* s2 = work + n3 * batch;
  const double h3 = h / 3.0, h2 = h / 2.0;
  for (int s = 0; s < nsteps; ++s) {
    rk3_stage_exact<<<blocks, kThreads, 0, c.stream>>>(states, states, s1, batch, ld, ld, n3, p, h3);
    rk3_stage_exact<<<blocks, kThreads, 0, c.stream>>>(states, s1, s2, batch, ld, n3, n3, p, h2);
    rk3_stage_exact<<<blocks, kThreads, 0, c.stream>>>(states, s2, states, batch, ld, n3, ld, p, h);
    c.launches += 3;
  }
  PW_LAUNCH_CHECK();
}

template <int T>
static void launch_tiled(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                         int nsteps, double h, int nsub, double* work) {
  constexpr size_t smem = tiled_smem<T>();
  const int per_sm = kernel_setup(c, fefb_tiled_coop<T>, 256, smem);
  const long long items = (long long)(p.nx / T) * (p.ny / T) * batch;
  const int cap_sm = c.coop_blocks_per_sm > 0 ? std::min(per_sm, c.coop_blocks_per_sm) : per_sm;
  int blocks = (int)std::max<long long>(1, std::min<long long>(items, (long long)c.num_sms * cap_sm));
  double tau = h / nsub;
  ExactParams pp = p;
  void* args[] = {&states, &batch, &ld, &pp, &nsteps, &tau, &nsub, &work};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)fefb_tiled_coop<T>, dim3(blocks), dim3(256), args, smem,
                                      c.stream));
  c.launches += 1;
}

// tiles_y <= 0: ceil(ny / TMY) (tall tiles: at least one tile row per ~SM budget)
template <int TMX, int TMY, int K, int NT, int MINB, bool FIXX, bool FIXY, int ORD = 0>
static void launch_tb(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                      int nsteps, double h, int nsub, double* work, bool fill_sms = false) {
  auto kern = fefb_tb_coop<TMX, TMY, K, NT, MINB, FIXX, FIXY, ORD>;
  constexpr size_t smem = tb_smem<TMX, TMY, K>();
  const int per_sm = kernel_setup(c, kern, NT, smem);
  int tiles_x = (p.nx + TMX - 1) / TMX, tiles_y = (p.ny + TMY - 1) / TMY;
  if (fill_sms) {  // as many tile rows as keep every SM busy with one tile (batch 1)
    const int want = (c.num_sms * per_sm) / std::max(1, tiles_x * batch);
    tiles_y = std::min(p.ny, std::max(tiles_y, want));
  }
  const long long items = (long long)tiles_x * tiles_y * batch;
  const int cap_sm = c.coop_blocks_per_sm > 0 ? std::min(per_sm, c.coop_blocks_per_sm) : per_sm;
  int blocks = (int)std::max<long long>(1, std::min<long long>(items, (long long)c.num_sms * cap_sm));
  double tau = h / nsub;
  ExactParams pp = p;
  void* args[] = {&states, &batch, &ld, &pp, &nsteps, &tau, &nsub, &work, &tiles_x, &tiles_y};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(blocks), dim3(NT), args, smem, c.stream));
  c.launches += 1;
}

static int coarse_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PW_COARSE_VARIANT");  // tuning hook (scripts/microbench.py coarse)
    v = (e && *e) ? atoi(e) : 0;
  }
  return v;
}

// Neighbour-flag G for one state (serial sweep): tiles of 32 x <= TMY rows, as many tile
// rows as fill the resident CTA slots (near-equal heights); the flags follow the 6 n work
// doubles (fefb_exact_work_doubles reserves them).  Returns false when the grid does not fit.
template <int TMY, int K, int NT, int ORD, int MINB = 1>
static bool launch_nf(Ctx& c, const ExactParams& p, double* states, int nsteps, double h, int nsub, double* work) {
  using C = NfCfg<TMY, K, NT>;
  auto kern = fefb_nf_kernel<TMY, K, NT, ORD, MINB>;
  const int per_sm = kernel_setup(c, kern, NT, C::SMEM);
  const int tiles_x = p.nx / 32;
  const int slots = c.num_sms * per_sm;
  int tiles_y = (p.ny + TMY - 1) / TMY;                        // smallest count with TY <= TMY
  const int fill = std::max(1, slots / std::max(1, tiles_x));  // one tile per CTA when it fits
  if (tiles_x * tiles_y < slots) tiles_y = std::max(tiles_y, std::min(p.ny / (3 * K), fill));
  if (p.ny / tiles_y < 3 * K || tiles_x * 32 != p.nx) return false;  // halo must stay in the 8 neighbours
  if (((uintptr_t)states | (uintptr_t)work) & 15) return false;      // 16-byte staging copies
  const int tiles = tiles_x * tiles_y;
  const int grid = std::min(tiles, slots);
  int* flags = reinterpret_cast<int*>(work + 6 * (size_t)p.nx * p.ny);
  PW_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)tiles, c.stream));
  double tau = h / nsub;
  ExactParams pp = p;
  int tx = tiles_x, ty = tiles_y;
  void* args[] = {&states, &pp, &nsteps, &tau, &nsub, &work, &tx, &ty, &flags};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(NT), args, C::SMEM, c.stream));
  c.launches += 1;
  return true;
}

// The folded form of launch_nf (fefb_nfm_kernel): same tiling rule, E more margin.
template <int TMY_, int K, int NT, int ORD, int MINB = 1, bool REG = false>
static bool launch_nfm(Ctx& c, const ExactParams& p, double* states, int nsteps, double h, int nsub, double* work) {
  constexpr int TMY = ORD == 1 ? TMY_ : TMY_ - 8;  // reach 3: shorter tiles keep the planes in shared memory
  using C = NfmCfg<TMY, K, NT, nfm_reach<ORD>()>;
  auto kern = REG ? fefb_nfr_kernel<TMY, K, NT, ORD, MINB> : fefb_nfm_kernel<TMY, K, NT, ORD, MINB>;
  const int per_sm = kernel_setup(c, kern, NT, C::SMEM);
  const int tiles_x = p.nx / 32;
  const int slots = c.num_sms * per_sm;
  int tiles_y = (p.ny + TMY - 1) / TMY;
  const int fill = std::max(1, slots / std::max(1, tiles_x));
  if (tiles_x * tiles_y < slots) tiles_y = std::max(tiles_y, std::min(p.ny / C::HE, fill));
  if (p.ny / tiles_y < C::HE || tiles_x * 32 != p.nx) return false;  // halo must stay in the 8 neighbours
  if (((uintptr_t)states | (uintptr_t)work) & 15) return false;
  const int tiles = tiles_x * tiles_y;
  const int grid = std::min(tiles, slots);
  int* flags = reinterpret_cast<int*>(work + 6 * (size_t)p.nx * p.ny);
  PW_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)tiles, c.stream));
  double tau = h / nsub;
  ExactParams pp = p;
  int tx = tiles_x, ty = tiles_y;
  void* args[] = {&states, &pp, &nsteps, &tau, &nsub, &work, &tx, &ty, &flags};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(NT), args, C::SMEM, c.stream));
  c.launches += 1;
  return true;
}

static int nf_variant() {
  // 0: the grid-barrier kernels; 2 / 3 / 4: substeps per phase (phase-A form); 6 / 10: phase A
  // folded into the first block (K = 3 / 2); 11 / 12: folded + register-resident columns
  // (K = 3 / 2; 12 is the default: 512^2 2-step call 160 us, 1024^2 623 us, from 200 / 698)
  // -1 (default): 11 where one 60-row tile per SM covers the grid (512^2: 151 us per 2-step call
  // against 155 with K = 2, both with resident tiles), else K = 2 with 64-row (12) or 58-row (17)
  // tiles, whichever needs fewer CTA rounds x tile rows (1024^2: 576 tiles of 57 rows are four
  // 97 %-full rounds of 148 CTAs, 584 us against 606 with 512 tiles of 64 rows)
  const char* e = getenv("PW_COARSE_NF");
  return (e && *e) ? atoi(e) : -1;
}

// Row-sharded G: one state whose rows live in nsh row shards, shard s holding
// rows [s R, (s+1) R) in its own state / work / flag buffers.  All shards' tiles run in this one
// launch; tile rows are aligned to the shard boundaries (tiles_y a multiple of nsh).  The
// default G's body (fefb_nfr_body, K = 2) through the shard accessor -- bitwise equal to the
// replicated G.
constexpr int kRsK = 2;
static int rs_tmy(const ExactParams& p) { return p.order == 1 ? 64 : 56; }
static int rs_tiles_y(const ExactParams& p, int nsh) { return ((p.ny + rs_tmy(p) - 1) / rs_tmy(p) + nsh - 1) / nsh * nsh; }
size_t rowshard_work_doubles(const ExactParams& p, int nsh) { return (size_t)6 * p.nx * (p.ny / nsh); }
int rowshard_flag_ints(const ExactParams& p, int nsh) { return (p.nx / 32) * rs_tiles_y(p, nsh) / nsh; }
void launch_fefb_rowshard(Ctx& c, const ExactParams& p, int nsh, double* const* st, double* const* work,
                          int* const* flags, int nsteps, double h, int nsub) {
  PW_CHECK(nsh >= 1 && nsh <= kMaxRowShards, PW_ERR_VALUE, "row shards: 1..8");
  PW_CHECK(p.nx % 32 == 0 && p.ny % nsh == 0, PW_ERR_VALUE, "row shards need nx % 32 == 0 and ny % nshard == 0");
  constexpr int NT = 512;
  const bool o1 = p.order == 1;
  using C1 = NfmCfg<64, kRsK, NT, 1>;
  using C0 = NfmCfg<56, kRsK, NT, 3>;
  auto kern = o1 ? fefb_nfr_shard_kernel<64, kRsK, NT, 1> : fefb_nfr_shard_kernel<56, kRsK, NT, 0>;
  const size_t smem = o1 ? C1::SMEM : C0::SMEM;
  const int he = o1 ? C1::HE : C0::HE;
  const int per_sm = kernel_setup(c, kern, NT, smem);
  const int tiles_x = p.nx / 32;
  const int tiles_y = rs_tiles_y(p, nsh);  // shard-aligned tile rows
  PW_CHECK(p.ny / tiles_y >= he, PW_ERR_VALUE, "row shards: tiles too short for the halo");
  NfShards sh{};
  sh.rows = p.ny / nsh;
  sh.tiles = tiles_x * tiles_y / nsh;
  for (int s = 0; s < nsh; ++s) {
    sh.st[s] = st[s];
    sh.work[s] = work[s];
    sh.flags[s] = flags[s];
    PW_CUDA(cudaMemsetAsync(flags[s], 0, sizeof(int) * (size_t)sh.tiles, c.stream));
  }
  const int tiles = tiles_x * tiles_y;
  const int grid = std::min(tiles, c.num_sms * per_sm);
  double tau = h / nsub;
  ExactParams pp = p;
  int tx = tiles_x, ty = tiles_y, lo = 0, hi = tiles;
  void* args[] = {&sh, &pp, &nsteps, &tau, &nsub, &tx, &ty, &lo, &hi};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(NT), args, smem, c.stream));
  c.launches += 1;
}

void launch_fefb_exact(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                       int nsteps, double h, int nsub, double* work) {
  if (nsteps <= 0 || batch <= 0) return;
  PW_CHECK((long long)p.nx * p.ny < (1LL << 31), PW_ERR_VALUE, "grid too large");
  if (!c.strict && batch == 1 && ld >= 3LL * p.nx * p.ny && p.nx % 32 == 0 && p.ny >= 64 &&
      (long long)p.nx * p.ny >= 16384 && nf_variant() != 0) {
    const bool o1 = p.order == 1;
    bool ok = false;
    int variant = nf_variant();
    if (variant < 0) {
      const int t60 = (p.nx / 32) * ((p.ny + 59) / 60);
      const int sms = c.num_sms > 0 ? c.num_sms : 148;
      // tiles outnumber the SMs: rounds of CTAs x rows per tile, for 64- and 58-row tiles
      auto cost = [&](int tmy) {
        const int ty = (p.ny + tmy - 1) / tmy, tiles = (p.nx / 32) * ty;
        return (long long)((tiles + sms - 1) / sms) * ((p.ny + ty - 1) / ty);
      };
      variant = (t60 <= sms && 2 * t60 >= sms) ? 11 : (cost(58) < cost(64) ? 17 : 12);
    }
    switch (variant) {
      case 2: ok = o1 ? launch_nf<64, 2, 512, 1>(c, p, states, nsteps, h, nsub, work)
                      : launch_nf<64, 2, 512, 0>(c, p, states, nsteps, h, nsub, work); break;
      case 4: ok = o1 ? launch_nf<56, 4, 512, 1>(c, p, states, nsteps, h, nsub, work)
                      : launch_nf<56, 4, 512, 0>(c, p, states, nsteps, h, nsub, work); break;
      case 5:  // smaller tiles, 2 CTAs (2 tiles in flight) per SM: measured 207 vs 195 us at 512^2
        ok = o1 ? launch_nf<32, 2, 256, 1, 2>(c, p, states, nsteps, h, nsub, work)
                : launch_nf<32, 2, 256, 0, 2>(c, p, states, nsteps, h, nsub, work); break;
      case 6: ok = o1 ? launch_nfm<60, 3, 512, 1>(c, p, states, nsteps, h, nsub, work)
                      : launch_nfm<60, 3, 512, 0>(c, p, states, nsteps, h, nsub, work); break;
      case 7: ok = o1 ? launch_nf<32, 2, 512, 1, 2>(c, p, states, nsteps, h, nsub, work)
                      : launch_nf<32, 2, 512, 0, 2>(c, p, states, nsteps, h, nsub, work); break;
      case 8: ok = o1 ? launch_nfm<26, 2, 512, 1, 2>(c, p, states, nsteps, h, nsub, work)
                      : launch_nfm<26, 2, 512, 0, 2>(c, p, states, nsteps, h, nsub, work); break;
      case 9: ok = o1 ? launch_nfm<46, 4, 512, 1>(c, p, states, nsteps, h, nsub, work)
                      : launch_nfm<46, 4, 512, 0>(c, p, states, nsteps, h, nsub, work); break;
      case 10: ok = o1 ? launch_nfm<64, 2, 512, 1>(c, p, states, nsteps, h, nsub, work)
                       : launch_nfm<64, 2, 512, 0>(c, p, states, nsteps, h, nsub, work); break;
      case 11: ok = o1 ? launch_nfm<60, 3, 512, 1, 1, true>(c, p, states, nsteps, h, nsub, work)
                       : launch_nfm<60, 3, 512, 0, 1, true>(c, p, states, nsteps, h, nsub, work); break;
      case 12: ok = o1 ? launch_nfm<64, 2, 512, 1, 1, true>(c, p, states, nsteps, h, nsub, work)
                       : launch_nfm<64, 2, 512, 0, 1, true>(c, p, states, nsteps, h, nsub, work); break;
      case 17:  // K = 2 with 58-row tiles: 1024^2 in 576 tiles of 57 rows (4 rounds of 148 CTAs, 97 % full)
        ok = o1 ? launch_nfm<58, 2, 512, 1, 1, true>(c, p, states, nsteps, h, nsub, work)
                : launch_nfm<58, 2, 512, 0, 1, true>(c, p, states, nsteps, h, nsub, work); break;
      case 13: ok = o1 ? launch_nfm<30, 2, 256, 1, 2, true>(c, p, states, nsteps, h, nsub, work)
                       : launch_nfm<30, 2, 256, 0, 2, true>(c, p, states, nsteps, h, nsub, work); break;
      default: ok = o1 ? launch_nf<60, 3, 512, 1>(c, p, states, nsteps, h, nsub, work)
                       : launch_nf<60, 3, 512, 0>(c, p, states, nsteps, h, nsub, work); break;
    }
    if (ok) return;
  }
  if (!c.strict && p.nx % 32 == 0 && p.ny % 32 == 0 && (long long)p.nx * p.ny >= 65536) {
    const bool o1 = p.order == 1;
    switch (coarse_variant()) {
      case 1: return launch_tiled<32>(c, p, states, batch, ld, nsteps, h, nsub, work);
      case 2: return launch_tb<32, 32, 1, 256, 2, true, true>(c, p, states, batch, ld, nsteps, h, nsub, work);
      case 3:  // tall near-equal tiles, one 512-thread CTA per SM
        if (o1) return launch_tb<32, 60, 2, 512, 1, true, false, 1>(c, p, states, batch, ld, nsteps, h, nsub, work, true);
        return launch_tb<32, 60, 2, 512, 1, true, false>(c, p, states, batch, ld, nsteps, h, nsub, work, true);
      case 5:  // tall tiles, 3 substeps per barrier
        if (o1) return launch_tb<32, 60, 3, 512, 1, true, false, 1>(c, p, states, batch, ld, nsteps, h, nsub, work, true);
        return launch_tb<32, 60, 3, 512, 1, true, false>(c, p, states, batch, ld, nsteps, h, nsub, work, true);
      case 4:
        if (o1) return launch_tb<32, 32, 2, 256, 2, true, true, 1>(c, p, states, batch, ld, nsteps, h, nsub, work);
        return launch_tb<32, 32, 2, 256, 2, true, true>(c, p, states, batch, ld, nsteps, h, nsub, work);
      default:
        // one state (the serial sweep): tall tiles, one per SM (balanced barrier phases),
        // 3 substeps per grid barrier; batches: 32 x 32 tiles, 2 CTAs per SM, 2 substeps
        if (batch == 1 && o1)
          return launch_tb<32, 60, 3, 512, 1, true, false, 1>(c, p, states, batch, ld, nsteps, h, nsub, work, true);
        if (o1) return launch_tb<32, 32, 2, 256, 2, true, true, 1>(c, p, states, batch, ld, nsteps, h, nsub, work);
        return launch_tb<32, 32, 2, 256, 2, true, true>(c, p, states, batch, ld, nsteps, h, nsub, work);
    }
  }
  if (!c.strict && p.nx % 16 == 0 && p.ny % 16 == 0)
    return launch_tiled<16>(c, p, states, batch, ld, nsteps, h, nsub, work);
  launch_fefb_coop(c, p, states, batch, ld, nsteps, h / nsub, nsub, work, 0);
}

// per-cell cooperative FE-FB: nsteps x (A phase unless adv_given, nsub substeps of tau)
void launch_fefb_coop(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                      int nsteps, double tau, int nsub, double* work, int adv_given) {
  const int max_per_sm = kernel_setup(c, fefb_coop, kCoopThreads, 0);
  const long long total = (long long)p.nx * p.ny * batch;
  long long want = (total + kCoopThreads - 1) / kCoopThreads;
  long long cap = (long long)c.num_sms * max_per_sm;
  int blocks = (int)std::max<long long>(1, std::min(want, cap));
  ExactParams pp = p;
  void* args[] = {&states, &batch, &ld, &pp, &nsteps, &tau, &nsub, &work, &adv_given};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)fefb_coop, dim3(blocks), dim3(kCoopThreads), args, 0,
                                      c.stream));
  c.launches += 1;
}

size_t scalar_rk3_work_doubles(const ExactParams& p, int batch) {
  return (size_t)2 * p.nx * p.ny * (size_t)batch;
}

void launch_rk3_exact_scalar(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                             int nsteps, double h, double* work) {
  const long long n = (long long)p.nx * p.ny;
  int bx = (int)std::min<long long>((n + kThreads - 1) / kThreads, (long long)c.num_sms * 16);
  if (bx < 1) bx = 1;
  PW_CHECK(batch <= 65535, PW_ERR_VALUE, "batch too large for one launch");
  const dim3 blocks(bx, batch);
  double* s1 = work;
  double* s2 = work + n * batch;
  const double h3 = h / 3.0, h2 = h / 2.0;
  for (int s = 0; s < nsteps; ++s) {
    rk3_stage_exact_scalar<<<blocks, kThreads, 0, c.stream>>>(states, states, s1, ld, ld, n, p, h3);
    rk3_stage_exact_scalar<<<blocks, kThreads, 0, c.stream>>>(states, s1, s2, ld, n, n, p, h2);
    rk3_stage_exact_scalar<<<blocks, kThreads, 0, c.stream>>>(states, s2, states, ld, n, ld, p, h);
    c.launches += 3;
  }
  PW_LAUNCH_CHECK();
}

size_t split_rk3_fb_work_doubles(const ExactParams& p, int batch) {
  return (size_t)(6 + 3 + 3) * p.nx * p.ny * (size_t)batch;  // FB work, stage start copy, cur
}

// split_rk3_fb_step (integrators.py:109-120): three stages; stage k takes the advective
// tendency of the latest stage result and restarts the FB integration from the step-start
// state over frac*dt with ceil(n_sound*frac) substeps; damping from the stage's tau.
void launch_split_rk3_fb(Ctx& c, const ExactParams& p, double nu, double* states, int batch,
                         long long ld, int nsteps, double dt, int n_sound, double* work) {
  const long long n = (long long)p.nx * p.ny, n3 = 3 * n;
  double* fbw = work;                      // 6 planes per state (A + ping-pong)
  double* start = work + 6 * n * batch;    // stage integration buffer (d x batch, ld n3)
  double* cur = start + n3 * batch;        // latest stage result (ld n3)
  int bx = (int)std::min<long long>((n + kThreads - 1) / kThreads, (long long)c.num_sms * 16);
  if (bx < 1) bx = 1;
  PW_CHECK(batch <= 65535, PW_ERR_VALUE, "batch too large for one launch");
  const double fracs[3] = {1.0 / 3.0, 0.5, 1.0};
  for (int s = 0; s < nsteps; ++s) {
    for (int st = 0; st < 3; ++st) {
      const double frac = fracs[st];
      const int nsub = std::max(1, (int)std::ceil(n_sound * frac));
      const double tau = frac * dt / nsub;
      ExactParams q = p;
      if (nu > 0.0) {
        q.a1 = nu * p.dx * p.dx / tau;
        q.a2 = nu * p.dy * p.dy / tau;
      } else {
        q.a1 = q.a2 = 0.0;
      }
      // A(latest stage) -> fbw planes 0..2
      adv3_exact<<<dim3(bx, batch), kThreads, 0, c.stream>>>(st == 0 ? states : cur, st == 0 ? ld : n3, fbw, q);
      c.launches += 1;
      // integrate from the step-start state
      PW_CUDA(cudaMemcpy2DAsync(start, n3 * sizeof(double), states, ld * sizeof(double), n3 * sizeof(double),
                                batch, cudaMemcpyDeviceToDevice, c.stream));
      launch_fefb_coop(c, q, start, batch, n3, 1, tau, nsub, fbw, 1);
      std::swap(start, cur);
    }
    PW_CUDA(cudaMemcpy2DAsync(states, ld * sizeof(double), cur, n3 * sizeof(double), n3 * sizeof(double),
                              batch, cudaMemcpyDeviceToDevice, c.stream));
  }
  PW_LAUNCH_CHECK();
}

}  // namespace pw
