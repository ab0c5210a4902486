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
                                        int f) {
  const double* row = q + (size_t)j * p.nx;
  return face_flux(p.order, p.uf[(size_t)j * p.nx + f], row[wrapi(f - 3, p.nx)],
                   row[wrapi(f - 2, p.nx)], row[wrapi(f - 1, p.nx)], row[f],
                   row[wrapi(f + 1, p.nx)], row[wrapi(f + 2, p.nx)]);
}

__device__ __forceinline__ double gy_at(const ExactParams& p, const double* __restrict__ q, int f,
                                        int i) {
  const int nx = p.nx, ny = p.ny;
  return face_flux(p.order, p.vf[(size_t)f * nx + i], q[(size_t)wrapi(f - 3, ny) * nx + i],
                   q[(size_t)wrapi(f - 2, ny) * nx + i], q[(size_t)wrapi(f - 1, ny) * nx + i],
                   q[(size_t)f * nx + i], q[(size_t)wrapi(f + 1, ny) * nx + i],
                   q[(size_t)wrapi(f + 2, ny) * nx + i]);
}

// advective_tendency = flux_divergence(flux_x, flux_y) at cell (j, i)
__device__ __forceinline__ double adv_at(const ExactParams& p, const double* __restrict__ q, int j,
                                         int i) {
  const int ip = i + 1 < p.nx ? i + 1 : 0;
  const int jp = j + 1 < p.ny ? j + 1 : 0;
  const double fxi = fx_at(p, q, j, i), fxp = fx_at(p, q, j, ip);
  const double gyj = gy_at(p, q, j, i), gyp = gy_at(p, q, jp, i);
  return -(fxp - fxi) / p.dx - (gyp - gyj) / p.dy;
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

// Split FE-FB (integrators.py:103-106 / fb_substeps numba_backend.py:131-146),
// nsteps coarse steps in ONE cooperative launch.  One grid barrier per acoustic
// substep: the pressure update needs the new velocities of its 4 neighbours,
// which each thread recomputes from the old state with the same expression
// (bitwise identical to storing them), reading a ping-pong copy of (u, v, p).
// work per state: [au, av, ap, u', v', p'] (6 planes).
__device__ __forceinline__ double u_new(const ExactParams& p, const double* cu, const double* cv,
                                        const double* pp, const double* au, int j, int i,
                                        double sx, double sy, double tau, bool damp) {
  const size_t c = (size_t)j * p.nx + i;
  double du = au[c] - p.cs * cdx(p, pp, j, i, sx);
  if (damp) {
    const int im = wrapi(i - 1, p.nx), ipp = wrapi(i + 1, p.nx);
    const double div_ip = cdx(p, cu, j, ipp, sx) + cdy(p, cv, j, ipp, sy);
    const double div_im = cdx(p, cu, j, im, sx) + cdy(p, cv, j, im, sy);
    du = du + p.a1 * ((div_ip - div_im) * sx);
  }
  return cu[c] + tau * du;
}

__device__ __forceinline__ double v_new(const ExactParams& p, const double* cu, const double* cv,
                                        const double* pp, const double* av, int j, int i,
                                        double sx, double sy, double tau, bool damp) {
  const size_t c = (size_t)j * p.nx + i;
  double dv = av[c] - p.cs * cdy(p, pp, j, i, sy);
  if (damp) {
    const int jm = wrapi(j - 1, p.ny), jpp = wrapi(j + 1, p.ny);
    const double div_jp = cdx(p, cu, jpp, i, sx) + cdy(p, cv, jpp, i, sy);
    const double div_jm = cdx(p, cu, jm, i, sx) + cdy(p, cv, jm, i, sy);
    dv = dv + p.a2 * ((div_jp - div_jm) * sy);
  }
  return cv[c] + tau * dv;
}

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
// u' and v' of one FB substep at (j+DY, i+DX), reference operation order (fb_substeps)
template <int DY, int DX>
__device__ __forceinline__ double un_at(const Nbr& N, const ExactParams& p, const double* cu,
                                        const double* cv, const double* cp, const double* au,
                                        double sx, double sy, double tau, bool damp) {
  double du = N.at(au, DY, DX) - p.cs * ((N.at(cp, DY, DX + 1) - N.at(cp, DY, DX - 1)) * sx);
  if (damp) {
    const double div_ip = (N.at(cu, DY, DX + 2) - N.at(cu, DY, DX)) * sx +
                          (N.at(cv, DY + 1, DX + 1) - N.at(cv, DY - 1, DX + 1)) * sy;
    const double div_im = (N.at(cu, DY, DX) - N.at(cu, DY, DX - 2)) * sx +
                          (N.at(cv, DY + 1, DX - 1) - N.at(cv, DY - 1, DX - 1)) * sy;
    du = du + p.a1 * ((div_ip - div_im) * sx);
  }
  return N.at(cu, DY, DX) + tau * du;
}
template <int DY, int DX>
__device__ __forceinline__ double vn_at(const Nbr& N, const ExactParams& p, const double* cu,
                                        const double* cv, const double* cp, const double* av,
                                        double sx, double sy, double tau, bool damp) {
  double dv = N.at(av, DY, DX) - p.cs * ((N.at(cp, DY + 1, DX) - N.at(cp, DY - 1, DX)) * sy);
  if (damp) {
    const double div_jp = (N.at(cu, DY + 1, DX + 1) - N.at(cu, DY + 1, DX - 1)) * sx +
                          (N.at(cv, DY + 2, DX) - N.at(cv, DY, DX)) * sy;
    const double div_jm = (N.at(cu, DY - 1, DX + 1) - N.at(cu, DY - 1, DX - 1)) * sx +
                          (N.at(cv, DY, DX) - N.at(cv, DY - 2, DX)) * sy;
    dv = dv + p.a2 * ((div_jp - div_jm) * sy);
  }
  return N.at(cv, DY, DX) + tau * dv;
}

__global__ void __launch_bounds__(128) fefb_coop(double* st, int batch, long long ld, ExactParams p,
                                                 int nsteps, double tau, int nsub, double* work) {
  cg::grid_group grid = cg::this_grid();
  const int n = p.nx * p.ny;
  const double sx = 0.5 / p.dx, sy = 0.5 / p.dy, cs = p.cs;
  const bool damp = (p.a1 != 0.0 || p.a2 != 0.0);
  const int stride = gridDim.x * blockDim.x;
  const int first = blockIdx.x * blockDim.x + threadIdx.x;
  for (int step = 0; step < nsteps; ++step) {
    // frozen slow tendency A(q) (physics.advective_tendencies, physics.py:67-74)
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
        const double* cu = from_state ? sb : w + 3 * n;
        const double* cv = cu + n;
        const double* cp = cu + 2 * n;
        double* nu = from_state ? w + 3 * n : sb;
        Nbr N;
        make_nbr(N, j, i, p.nx, p.ny);
        // momentum: current p gradient + current-velocity damping
        const double un = un_at<0, 0>(N, p, cu, cv, cp, w, sx, sy, tau, damp);
        const double vn = vn_at<0, 0>(N, p, cu, cv, cp, w + n, sx, sy, tau, damp);
        // pressure from the freshly updated velocity divergence (neighbour velocities recomputed)
        const double u_e = un_at<0, 1>(N, p, cu, cv, cp, w, sx, sy, tau, damp);
        const double u_w = un_at<0, -1>(N, p, cu, cv, cp, w, sx, sy, tau, damp);
        const double v_n = vn_at<1, 0>(N, p, cu, cv, cp, w + n, sx, sy, tau, damp);
        const double v_s = vn_at<-1, 0>(N, p, cu, cv, cp, w + n, sx, sy, tau, damp);
        const double divn = (u_e - u_w) * sx + (v_n - v_s) * sy;
        nu[cell] = un;
        nu[n + cell] = vn;
        nu[2 * n + cell] = cp[cell] + tau * (w[2 * n + cell] - cs * divn);
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

constexpr int kThreads = 256;
constexpr int kCoopThreads = 128;

}  // namespace

size_t rk3_exact_work_doubles(const ExactParams& p, int batch) {
  return (size_t)2 * 3 * p.nx * p.ny * (size_t)batch;
}

size_t fefb_exact_work_doubles(const ExactParams& p, int batch) {
  return (size_t)6 * p.nx * p.ny * (size_t)batch;
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

void launch_fefb_exact(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                       int nsteps, double h, int nsub, double* work) {
  if (nsteps <= 0 || batch <= 0) return;
  static int max_per_sm = -1;
  if (max_per_sm < 0) {
    PW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_per_sm, fefb_coop, kCoopThreads, 0));
    if (max_per_sm < 1) max_per_sm = 1;
  }
  const long long total = (long long)p.nx * p.ny * batch;
  long long want = (total + kCoopThreads - 1) / kCoopThreads;
  PW_CHECK((long long)p.nx * p.ny < (1LL << 31), PW_ERR_VALUE, "grid too large");
  long long cap = (long long)c.num_sms * max_per_sm;
  int blocks = (int)std::max<long long>(1, std::min(want, cap));
  double tau = h / nsub;
  ExactParams pp = p;
  void* args[] = {&states, &batch, &ld, &pp, &nsteps, &tau, &nsub, &work};
  PW_CUDA(cudaLaunchCooperativeKernel((void*)fefb_coop, dim3(blocks), dim3(kCoopThreads), args, 0,
                                      c.stream));
  c.launches += 1;
}

}  // namespace pw
