// Internal declarations of the sm_100a KSE-Parareal library (libpitwave_b200.so).
// The public C ABI lives in include/pitwave_b200.h; nothing here crosses it.
#pragma once

#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/pitwave_b200.h"

namespace pw {

// NVTX range for profilers (nsys / ncu --nvtx): named after the reference's phases
// (parareal.py:31-47: coarse / fine / qr).  nvtx3 is header-only; without a tool attached
// a push / pop costs a few ns.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};

#define PW_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      throw pw::Error{PW_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) +    \
                                       " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
    }                                                                                       \
  } while (0)

#define PW_CHECK(cond, code, msg)                 \
  do {                                            \
    if (!(cond)) throw pw::Error{(code), (msg)};  \
  } while (0)

#define PW_LAUNCH_CHECK() PW_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- grid description
// State layout (reference mesh.State, mesh.py:74-138): (3, ny, nx) fp64,
// x fastest; a batch is B states at stride `ld` doubles.
struct GridDesc {
  int nx, ny;
  double dx, dy;
};

// Exact-order (reference operation order, no FMA contraction) stencil
// parameters: face-velocity arrays live on the device (mesh.face_normal_velocities).
struct ExactParams {
  int nx, ny, order;
  double dx, dy, cs, a1, a2;
  const double* uf;  // (ny, nx) x-face normal velocity
  const double* vf;  // (ny, nx) y-face normal velocity
  // 1/dx, 1/dy when dx, dy are powers of two: x/dx == x*(1/dx) exactly then,
  // so the divisions of flux_divergence become multiplies without changing a bit
  double inv_dx = 0.0, inv_dy = 0.0;
  // the face velocities when every face carries the same value (cvel = 1): the shared-memory
  // tendency pass of the coarse G takes them from here instead of two global loads per face
  int cvel = 0;
  double uc = 0.0, vc = 0.0;
};

// Folded constant-velocity RK3 coefficients for one stage with factor beta
// (s_out = q + beta * f(s_in)); see fine_fused.cu.
// Divergence damping is expanded and folded (a1 dx(div) = a1 sx^2 dxx(u) +
// a1 sx sy dx dy(v), a2 dy(div) likewise), so per cell only x stencils, a
// few y differences and two mixed differences remain.
struct StageCoef {
  double cxu[7];  // beta * (x advection + a1 sx^2 [1,0,-2,0,1]) on u, offsets -3..3
  double cxv[7];  // beta * x advection on v, centre - 2 beta a2 sy^2
  double cxp[7];  // beta * x advection on p
  double cy[7];   // beta * y advection stencil (used only when V != 0)
  double pgx;     // -beta cs sx     du += pgx (p_{i+1} - p_{i-1})
  double pgy;     // -beta cs sy     dv += pgy (p_{j+1} - p_{j-1})
  double cuv;     // beta a1 sx sy   du += cuv (a_{i+1} - a_{i-1}),  a = v_{j+1} - v_{j-1}
  double cvu;     // beta a2 sx sy   dv += cvu (b_{i+1} - b_{i-1}),  b = u_{j+1} - u_{j-1}
  double dv2;     // beta a2 sy^2    dv += dv2 (v_{j+2} + v_{j-2})
  double pu;      // -beta cs sx     dp += pu (u_{i+1} - u_{i-1})
  double pv;      // -beta cs sy     dp += pv a_i
};
constexpr int kMaxPeers = 7;  // peers of one rank in an 8-GPU NVSwitch node
struct FusedParams {
  int nx, ny;
  int zmask = 0;  // always 0: (tick & zmask) keeps per-tick coefficient loads in the loop
  // fused slice all-gather (pw_prop_apply_to_peers): the row-marching kernel also stores
  // each output row at out + peer_delta[i] bytes, i < npeer (peer-mapped buffers)
  int npeer = 0;
  long long peer_delta[kMaxPeers] = {};
  long long ld_in, ld_out;
  double sx, sy;  // 0.5/dx, 0.5/dy
  StageCoef st[3];
};

// ---------------------------------------------------------------- context
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  void* cublas = nullptr;    // cublasHandle_t
  void* cusolver = nullptr;  // cusolverDnHandle_t
  void* cusolver_params = nullptr;  // cusolverDnParams_t (64-bit X API)
  void* blas_ws = nullptr;   // fixed cuBLAS workspace
  // scratch for grid barriers / reductions
  double* red = nullptr;     // reduction scratch (doubles)
  unsigned int* tma_done = nullptr;  // last-CTA counter of the TMA serial-step kernel
  size_t red_cap = 0;
  int launches = 0;          // kernels launched by this library (bench gpu_launches)
  bool strict = false;       // force reference-order kernels everywhere
  int coop_blocks_per_sm = 0;        // cap for cooperative G launches (0 = occupancy max)
  cudaStream_t side = nullptr;       // second stream: subspace QR beside the fine sweep
  cudaStream_t outer = nullptr;      // while work runs on `side`: the context's own stream
  bool qr_overlap = true;            // PW_QR_OVERLAP=0: QR after the fine sweep, one stream
  bool tsqr = false;                 // row-sharded (TSQR) subspace factorisation in sharded sweeps
  // row-sharded serial correction: across ranks through the comm hooks (pw_ctx_set_comm),
  // or vshards > 1 row shards in one process (tests, PW_ROW_SHARDS)
  int comm_rank = 0, comm_world = 1, vshards = 1;
  pw_allreduce_hook allreduce_hook = nullptr;
  pw_allgather_hook allgather_hook = nullptr;
  void* comm_user = nullptr;
  void* nccl = nullptr;              // ncclComm_t owned by the library (pw_ctx_set_nccl), or null
  double* comm_scratch = nullptr;    // world x block doubles for the padded NCCL all-gather
  size_t comm_scratch_n = 0;
  pw_fine_hook fine_hook = nullptr;  // slice-sharded fine predictor (multi-GPU), see header
  pw_fine_rows_hook fine_rows_hook = nullptr;  // ... delivering this rank's rows (row-local sweeps)
  void* fine_rows_user = nullptr;
  void* fine_hook_user = nullptr;
};

// One-time per-(device, kernel) launch setup: raises the dynamic shared-memory limit to
// `smem` (when above the 48 KB default) and returns the resident CTAs per SM for
// `threads` x `smem`.  The attribute is a per-device property, so a process that drives
// several GPUs sets it once on each (cached under a mutex; api.cu).
int kernel_setup(int device, const void* kern, int threads, size_t smem);
template <class F>
inline int kernel_setup(const Ctx& c, F* kern, int threads, size_t smem) {
  return kernel_setup(c.device, reinterpret_cast<const void*>(kern), threads, smem);
}

// ---------------------------------------------------------------- collectives (comm.cu)
// The row-sharded sweep's collectives on the context stream: NCCL when the context owns a
// communicator (pw_ctx_set_nccl), else the pw_ctx_set_comm hooks.
void nccl_unique_id(unsigned char* out128);
void nccl_init(Ctx& c, const unsigned char* id128, int rank, int world);
void nccl_destroy(Ctx& c);
void comm_allreduce(Ctx& c, double* data, long long count);
void comm_allgather(Ctx& c, double* data, long long block, long long total);

// ---------------------------------------------------------------- kernels (launchers)
// exact.cu  (compiled with -fmad=false: reference operation order, bitwise)
void launch_rk3_exact(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                      int nsteps, double h, double* work);
void launch_fefb_exact(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                       int nsteps, double h, int nsub, double* work);
size_t rk3_exact_work_doubles(const ExactParams& p, int batch);
// per-cell cooperative FE-FB (adv_given: A already in the work planes 0..2)
void launch_fefb_coop(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                      int nsteps, double tau, int nsub, double* work, int adv_given);
// scalar advection RK3 (one field per state), reference order
size_t scalar_rk3_work_doubles(const ExactParams& p, int batch);
void launch_rk3_exact_scalar(Ctx& c, const ExactParams& p, double* states, int batch, long long ld,
                             int nsteps, double h, double* work);
// split RK3-FB, reference order; damping per stage from nu
size_t split_rk3_fb_work_doubles(const ExactParams& p, int batch);
void launch_split_rk3_fb(Ctx& c, const ExactParams& p, double nu, double* states, int batch,
                         long long ld, int nsteps, double dt, int n_sound, double* work);
size_t fefb_exact_work_doubles(const ExactParams& p, int batch);
// row-sharded G (one state in nsh row shards, every shard's tiles in one launch)
size_t rowshard_work_doubles(const ExactParams& p, int nsh);
int rowshard_flag_ints(const ExactParams& p, int nsh);
void launch_fefb_rowshard(Ctx& c, const ExactParams& p, int nsh, double* const* st, double* const* work,
                          int* const* flags, int nsteps, double h, int nsub);

// fine_fused.cu
void make_fused_params(FusedParams& fp, int nx, int ny, double dx, double dy, double cs,
                       int order, double U, double V, double a1, double a2, double h);
void launch_rk3_fused(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch,
                      bool vadv);
bool fused_supported(int nx, int ny);
// fine_march.cu: row-marching variant for V = 0 and whole-row CTAs
bool march_supported(int nx, int ny, long long ld_in, long long ld_out, const void* in,
                     const void* out);
void launch_rk3_march(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch);
bool march_peer_capable(int nx);  // launch_rk3_march handles fp.npeer > 0 for this nx
// persistent march over all steps of one propagation (PW_MARCH_PERSIST=1): one launch,
// work items (step, state, segment) with per-segment step counters in sync
bool march_persist_enabled(int nx);
size_t march_persist_sync_ints(int ny, int batch);
void launch_rk3_march_persist(Ctx& c, const FusedParams& fp, const double* in, double* out, double* tmp,
                              int batch, int nsteps, long long d, int* sync);

// march_tma.cu: the TMA-fed persistent row march (K1; default, PW_MARCH_V2=0 turns it off)
bool mtma_enabled();
bool mtma_supported(int nx, int ny, long long ld_in, long long ld_out, const void* in, const void* out,
                    const void* tmp);
void launch_rk3_mtma(Ctx& c, const FusedParams& fp, const double* in, double* out, double* tmp, int batch,
                     int nsteps, long long d, int* sync);

// linalg.cu
void launch_axpby_cols(Ctx& c, double* y, const double* a, const double* b, double alpha,
                       double beta, size_t n);
void launch_extract_upper(Ctx& c, const double* W, long long ldw, int mr, int m, double* R);
void launch_zero_strict_lower_block(Ctx& c, double* A, long long ld, int rows, int cols);
// k Householder vectors stored from column A (rows off.. of their block) -> explicit
// unit-lower trapezoidal form: zero above the diagonal entry off + j, 1 on it
void launch_make_unit_lower(Ctx& c, double* A, long long ld, int off, int k);
// dlarft recurrence for reflector columns col0..col0+p-1 of T (ld ldt), G = V^T V_new (m x p)
void launch_larft_cols(Ctx& c, double* T, int ldt, const double* G, const double* tau, int col0, int p);
void launch_set_diag_block(Ctx& c, double* A, long long ld, int k, double v);
size_t residual_scratch_doubles(int ncols, long long nrows);
// fp64 DMMA GEMM (dgemm.cu): C = alpha op(A) B + beta C, column-major, 64-bit sizes;
// acol gathers op(A)'s columns (op N), b_upper skips the zero lower part of an upper-
// triangular B
void dgemm(Ctx& c, bool ta, long long m, long long n, long long k, double alpha, const double* A, long long lda,
           const double* B, long long ldb, double beta, double* C, long long ldc, const int* acol = nullptr,
           bool b_upper = false);

// Xc (r x r) = rows piv[0..r) of X (m x r): R11^-1 back from its scattered form
void launch_gather_rows(Ctx& c, const double* X, int m, const int* piv, int r, double* Xc);
// alpha (r x nc, ld r) = Q^T S[:, c0 .. c0 + nc) from the pivoted factor stored in Rs (mr x m)
void launch_alpha_from_r(Ctx& c, const double* Rs, int mr, const int* piv, int m, int c0, int nc, int r,
                         double* alpha);

// tall-skinny Householder QR (tsqr.cu): LAPACK geqrf's output format for rows x p
void tsqr_geqrf(Ctx& c, long long rows, int p, double* A, long long lda, double* tau);

// K7: out[0] = max|q| (NaN wins), out[1] = cell_area * sum q^2, out[2] = #non-finite,
// out[3 + k] = q[probes[k]]
size_t window_diag_scratch_doubles(const Ctx& c);
void launch_window_diag(Ctx& c, const double* q, long long n, double cell_area, const long long* probes_dev,
                        int nprobe, double* scratch, double* out_dev);
void launch_residual(Ctx& c, const double* a, long long lda, const double* b, long long ldb,
                     int ncols, long long nrows, double* scratch, double* out_dev);
// fp64 pipe peak probe (probe.cu): best-of-3 DFMA throughput in TFLOP/s
double probe_fp64_tflops(Ctx& c, int iters);

// balanced persistent grid for the combine/projection kernels: <= per_sm CTAs per SM
int combine_grid(const Ctx& c, long long d, int per_sm = 2);
size_t combine_part_doubles(long long d, int r);
// R: mr x m (lda mr), mr = min(d, m); returns rank, fills piv (m), tau/diag (min(mr, m))
int pivoted_qr_small(Ctx& c, double* R, int mr, int m, double rank_tol, int* piv_dev,
                     double* tau_dev, double* diag_dev, int* rank_host);
void form_q2(Ctx& c, const double* R, int mr, const int* piv, const double* tau, int r,
             double* Q2);
void tri_inverse_scatter(Ctx& c, const double* R, int mr, int m, const int* piv, int r,
                         double* X);
// y = [g +] c + D (alpha [- alpha_sub]) (rd cols) and alpha_next = Q^T y (rq cols); nblk <= 0: default grid
// d rows from the given pointers; D / Q columns ld apart (ld <= 0: ld = d)
void launch_combine_gemv(Ctx& c, cudaStream_t st, const double* g, const double* D, int rd,
                         const double* cvec, const double* alpha, const double* Q, int rq,
                         long long d, double* y, double* alpha_next, double* part, int nblk = 0,
                         long long ld = 0, const double* alpha_sub = nullptr);
// alpha[j] = C[0:n1, j] . xt + C[n1:n1+n2, j] . g for j < r (C column-major, ld ldc): the
// small step that turns the reflector products V^T x into Q^T x when Q is kept implicit
void launch_implicit_alpha(Ctx& c, const double* C, int ldc, const double* xt, int n1, const double* g, int n2,
                           int r, double* alpha);
void launch_project_gemv(Ctx& c, const double* Q, int r, long long d, const double* v,
                         double* alpha, double* part);

}  // namespace pw
