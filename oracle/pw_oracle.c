#define _GNU_SOURCE
/*
 * pw_oracle.c -- CPU restatement of the reference's grid arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 kernels and the CPU baseline timed by bench.py (--impl reference /
 * cpu_baseline).  Nothing in the product path (paper_1510_02237_b200/)
 * links or calls it.
 *
 * It restates, operation for operation, the reference's numba kernels so
 * that -ffp-contract=off builds reproduce the reference bitwise:
 *   _face_flux          pkg/src/pitwave/kernels/numba_backend.py:13-30
 *   flux_x / flux_y     numba_backend.py:33-66
 *   flux_divergence     numba_backend.py:69-78
 *   centered_dx / dy    numba_backend.py:81-105
 *   damping_tendencies  numba_backend.py:108-111
 *   acoustic_rhs        numba_backend.py:119-128
 *   fb_substeps         numba_backend.py:131-146
 *   rk3_step            pkg/src/pitwave/integrators.py:79-85
 *   split_fe_fb_step    integrators.py:103-106 (+ _fb_integrate 88-100,
 *                       physics.advective_tendencies physics.py:67-74)
 *   propagate           integrators.py:126-146 (fixed step loop)
 * The face-velocity arrays (mesh.face_normal_velocities, mesh.py:232-247)
 * are passed in, so constant and solid-body velocities are both covered.
 *
 * State layout: (nvar=3, ny, nx) fp64, x fastest (mesh.State, mesh.py:74-138);
 * a batch is B such states back to back.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define IDX(j, i) ((size_t)(j) * (size_t)nx + (size_t)(i))

static inline double face_flux(int order, double u, double qm2, double qm1, double q0,
                               double qp1, double qp2, double qp3) {
    /* numba_backend.py:13-30 -- interface between formula cells q0 and qp1 */
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

static inline int wrap(int k, int n) { k %= n; return k < 0 ? k + n : k; }

static void flux_x(const double *q, const double *uf, int order, int nx, int ny, double *out) {
    /* numba_backend.py:33-48: out[j,f] on the face x=f*dx (cells f-1 | f) */
    for (int j = 0; j < ny; ++j)
        for (int f = 0; f < nx; ++f)
            out[IDX(j, f)] = face_flux(order, uf[IDX(j, f)],
                                       q[IDX(j, wrap(f - 3, nx))], q[IDX(j, wrap(f - 2, nx))],
                                       q[IDX(j, wrap(f - 1, nx))], q[IDX(j, f)],
                                       q[IDX(j, wrap(f + 1, nx))], q[IDX(j, wrap(f + 2, nx))]);
}

static void flux_y(const double *q, const double *vf, int order, int nx, int ny, double *out) {
    /* numba_backend.py:51-66 */
    for (int f = 0; f < ny; ++f)
        for (int i = 0; i < nx; ++i)
            out[IDX(f, i)] = face_flux(order, vf[IDX(f, i)],
                                       q[IDX(wrap(f - 3, ny), i)], q[IDX(wrap(f - 2, ny), i)],
                                       q[IDX(wrap(f - 1, ny), i)], q[IDX(f, i)],
                                       q[IDX(wrap(f + 1, ny), i)], q[IDX(wrap(f + 2, ny), i)]);
}

static void flux_divergence(const double *fx, const double *gy, int nx, int ny, double dx,
                            double dy, double *out) {
    /* numba_backend.py:69-78 */
    for (int j = 0; j < ny; ++j) {
        int jp = j + 1 < ny ? j + 1 : 0;
        for (int i = 0; i < nx; ++i) {
            int ip = i + 1 < nx ? i + 1 : 0;
            out[IDX(j, i)] = -(fx[IDX(j, ip)] - fx[IDX(j, i)]) / dx - (gy[IDX(jp, i)] - gy[IDX(j, i)]) / dy;
        }
    }
}

static void centered_dx(const double *f, int nx, int ny, double dx, double *out) {
    /* numba_backend.py:81-91 */
    double s = 0.5 / dx;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            out[IDX(j, i)] = (f[IDX(j, wrap(i + 1, nx))] - f[IDX(j, wrap(i - 1, nx))]) * s;
}

static void centered_dy(const double *f, int nx, int ny, double dy, double *out) {
    /* numba_backend.py:94-105 */
    double s = 0.5 / dy;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            out[IDX(j, i)] = (f[IDX(wrap(j + 1, ny), i)] - f[IDX(wrap(j - 1, ny), i)]) * s;
}

typedef struct {
    int nx, ny, order;
    double dx, dy, cs, a1, a2;
    const double *uf, *vf;
} pwo_grid;

/* scratch: 8 planes of nx*ny doubles */
static void advective_tendency(const pwo_grid *g, const double *q, double *out, double *scr) {
    /* numba_backend.py:114-116 */
    int nx = g->nx, ny = g->ny;
    double *fx = scr, *gy = scr + (size_t)nx * ny;
    flux_x(q, g->uf, g->order, nx, ny, fx);
    flux_y(q, g->vf, g->order, nx, ny, gy);
    flux_divergence(fx, gy, nx, ny, g->dx, g->dy, out);
}

static void acoustic_rhs(const pwo_grid *g, const double *s, double *ds, double *scr) {
    /* numba_backend.py:119-128; s and ds are (3, ny, nx) */
    int nx = g->nx, ny = g->ny;
    size_t n = (size_t)nx * ny;
    const double *u = s, *v = s + n, *p = s + 2 * n;
    double *du = ds, *dv = ds + n, *dp = ds + 2 * n;
    double *t1 = scr + 2 * n, *t2 = scr + 3 * n, *t3 = scr + 4 * n, *t4 = scr + 5 * n;
    double cs = g->cs;

    advective_tendency(g, u, t1, scr);
    centered_dx(p, nx, ny, g->dx, t2);
    for (size_t k = 0; k < n; ++k) du[k] = t1[k] - cs * t2[k];

    advective_tendency(g, v, t1, scr);
    centered_dy(p, nx, ny, g->dy, t2);
    for (size_t k = 0; k < n; ++k) dv[k] = t1[k] - cs * t2[k];

    advective_tendency(g, p, t1, scr);
    centered_dx(u, nx, ny, g->dx, t2);
    centered_dy(v, nx, ny, g->dy, t3);
    for (size_t k = 0; k < n; ++k) dp[k] = t1[k] - cs * (t2[k] + t3[k]);

    if (g->a1 != 0.0 || g->a2 != 0.0) {
        /* damping_tendencies, numba_backend.py:108-111: div = dx(u) + dy(v) */
        for (size_t k = 0; k < n; ++k) t4[k] = t2[k] + t3[k];
        centered_dx(t4, nx, ny, g->dx, t1);
        centered_dy(t4, nx, ny, g->dy, t2);
        for (size_t k = 0; k < n; ++k) {
            du[k] = du[k] + g->a1 * t1[k];
            dv[k] = dv[k] + g->a2 * t2[k];
        }
    }
}

/* scratch for one rk3 step: 3 states (9 planes) + 8 planes */
static void rk3_step(const pwo_grid *g, double *q, double h, double *work) {
    /* integrators.py:79-85: s1 = q + (h/3) f(q); s2 = q + (h/2) f(s1); q+ = q + h f(s2) */
    size_t n3 = 3 * (size_t)g->nx * g->ny;
    double *f = work, *s = work + n3, *scr = work + 2 * n3;
    double h3 = h / 3.0, h2 = h / 2.0;
    acoustic_rhs(g, q, f, scr);
    for (size_t k = 0; k < n3; ++k) s[k] = q[k] + f[k] * h3;
    acoustic_rhs(g, s, f, scr);
    for (size_t k = 0; k < n3; ++k) s[k] = q[k] + f[k] * h2;
    acoustic_rhs(g, s, f, scr);
    for (size_t k = 0; k < n3; ++k) q[k] = q[k] + f[k] * h;
}

static void fefb_step(const pwo_grid *g, double *q, double dt, int nsub, double a1, double a2,
                      double *work) {
    /* integrators.py:103-106 + 88-100 and numba fb_substeps 131-146 */
    int nx = g->nx, ny = g->ny;
    size_t n = (size_t)nx * ny;
    double *adv = work, *scr = work + 3 * n;  /* adv: 3 planes; scr: 8 planes */
    double *du = scr + 2 * n, *dv = scr + 3 * n, *t1 = scr + 4 * n, *t2 = scr + 5 * n,
           *t3 = scr + 6 * n, *t4 = scr + 7 * n;
    double *u = q, *v = q + n, *p = q + 2 * n;
    double cs = g->cs, tau = dt / nsub;
    for (int k = 0; k < 3; ++k) advective_tendency(g, q + k * n, adv + k * n, scr);
    const double *au = adv, *av = adv + n, *ap = adv + 2 * n;
    for (int it = 0; it < nsub; ++it) {
        centered_dx(p, nx, ny, g->dx, t1);
        centered_dy(p, nx, ny, g->dy, t2);
        for (size_t k = 0; k < n; ++k) { du[k] = au[k] - cs * t1[k]; dv[k] = av[k] - cs * t2[k]; }
        if (a1 != 0.0 || a2 != 0.0) {
            centered_dx(u, nx, ny, g->dx, t1);
            centered_dy(v, nx, ny, g->dy, t2);
            for (size_t k = 0; k < n; ++k) t4[k] = t1[k] + t2[k];
            centered_dx(t4, nx, ny, g->dx, t1);
            centered_dy(t4, nx, ny, g->dy, t2);
            for (size_t k = 0; k < n; ++k) {
                t3[k] = a1 * t1[k];
                du[k] = du[k] + t3[k];
                t3[k] = a2 * t2[k];
                dv[k] = dv[k] + t3[k];
            }
        }
        for (size_t k = 0; k < n; ++k) { u[k] += tau * du[k]; v[k] += tau * dv[k]; }
        centered_dx(u, nx, ny, g->dx, t1);
        centered_dy(v, nx, ny, g->dy, t2);
        for (size_t k = 0; k < n; ++k) p[k] += tau * (ap[k] - cs * (t1[k] + t2[k]));
    }
}

/*
 * Batched fixed-step propagation, in place on `states` (B x 3 x ny x nx).
 * scheme 0 = rk3 (a1/a2 of the fine model), 1 = split_fe_fb (a1/a2 of one
 * substep, tau = h/n_sound).  Slices are independent (the reference's
 * _fine_all thread pool, parareal.py:62-65); nthreads<=0 uses all cores.
 */
typedef struct {
    int scheme, batch, nsteps, n_sound;
    double *states, h, a1, a2;
    const pwo_grid *g;
    int next;              /* shared work counter (dynamic schedule, one slice per grab) */
    pthread_mutex_t mu;
    int err;
} pwo_job;

static void *pwo_worker(void *arg) {
    pwo_job *job = (pwo_job *)arg;
    size_t n = (size_t)job->g->nx * job->g->ny;
    double *work = (double *)malloc(sizeof(double) * 17 * n);
    if (!work) { pthread_mutex_lock(&job->mu); job->err = -3; pthread_mutex_unlock(&job->mu); return 0; }
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int b = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (b >= job->batch) break;
        double *q = job->states + (size_t)b * 3 * n;
        for (int s = 0; s < job->nsteps; ++s) {
            if (job->scheme == 0) rk3_step(job->g, q, job->h, work);
            else fefb_step(job->g, q, job->h, job->n_sound, job->a1, job->a2, work);
        }
    }
    free(work);
    return 0;
}

/*
 * Batched fixed-step propagation, in place on `states` (B x 3 x ny x nx).
 * scheme 0 = rk3 (a1/a2 of the fine model), 1 = split_fe_fb (a1/a2 of one
 * substep, tau = h/n_sound).  Slices are independent and are spread over
 * `nthreads` POSIX threads, one slice per grab -- the reference's _fine_all
 * thread pool (parareal.py:62-65).  nthreads<=0 uses every online core.
 */
int pwo_propagate(int scheme, double *states, int batch, int nsteps, int nx, int ny, double dx,
                  double dy, double cs, int order, double a1, double a2, double h, int n_sound,
                  const double *uf, const double *vf, int nthreads) {
    if (nx < 8 || ny < 8 || batch < 0 || nsteps < 0 || order < 1 || order > 6) return -1;
    if (scheme != 0 && scheme != 1) return -2;
    if (scheme == 1 && n_sound < 1) return -2;
    pwo_grid g = {nx, ny, order, dx, dy, cs, a1, a2, uf, vf};
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads > batch) nthreads = batch;
    if (nthreads < 1) nthreads = 1;
    pwo_job job;
    job.scheme = scheme; job.batch = batch; job.nsteps = nsteps; job.n_sound = n_sound;
    job.states = states; job.h = h; job.a1 = a1; job.a2 = a2; job.g = &g;
    job.next = 0; job.err = 0;
    pthread_mutex_init(&job.mu, 0);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, pwo_worker, &job);
    pwo_worker(&job);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
    free(th);
    pthread_mutex_destroy(&job.mu);
    return job.err;
}

/* One acoustic RHS evaluation (for stencil-level parity tests). */
int pwo_acoustic_rhs(const double *state, double *out, int nx, int ny, double dx, double dy,
                     double cs, int order, double a1, double a2, const double *uf,
                     const double *vf) {
    size_t n = (size_t)nx * ny;
    double *scr = (double *)malloc(sizeof(double) * 8 * n);
    if (!scr) return -3;
    pwo_grid g = {nx, ny, order, dx, dy, cs, a1, a2, uf, vf};
    acoustic_rhs(&g, state, out, scr);
    free(scr);
    return 0;
}

int pwo_num_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
