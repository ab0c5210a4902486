// C ABI of the B200 KSE-Parareal hot path (include/pitwave_b200.h).
//
// Objects: a context (device, stream, cuBLAS/cuSOLVER handles), propagators
// (PDE over a slice, or a dense test matrix), the device-resident Krylov
// basis, and the sweep driver.  Every sweep step is enqueued on the context
// stream from this host loop; the only host round-trips are the rank read
// after each subspace refactorisation and (optionally) the residual for a
// tol early exit -- the reference's own per-iteration decisions.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>

#include "pw_internal.h"

using pw::Ctx;
using pw::Error;

namespace pw {
int kernel_setup(int device, const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({device, kern});
  if (it != cache.end()) return it->second;
  // always explicit: with static shared memory as well, the default dynamic limit is
  // 48 KB minus the static part
  if (smem > 0) PW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  per_sm = std::max(per_sm, 1);
  cache[{device, kern}] = per_sm;
  return per_sm;
}
}  // namespace pw

struct pw_ctx {
  Ctx c;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PW_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return PW_ERR_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PW_ERR_STATE;
  }
}

#define PW_BLAS(call)                                                                     \
  do {                                                                                    \
    cublasStatus_t s_ = (call);                                                           \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                      \
      throw Error{PW_ERR_LIBRARY, std::string(#call) + " -> cublas status " + std::to_string((int)s_)}; \
  } while (0)
#define PW_SOLVER(call)                                                                   \
  do {                                                                                    \
    cusolverStatus_t s_ = (call);                                                         \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                    \
      throw Error{PW_ERR_LIBRARY, std::string(#call) + " -> cusolver status " + std::to_string((int)s_)}; \
  } while (0)

inline cublasHandle_t blas(Ctx& c) { return static_cast<cublasHandle_t>(c.cublas); }
inline cusolverDnHandle_t solver(Ctx& c) { return static_cast<cusolverDnHandle_t>(c.cusolver); }

// Stream-ordered device buffer.
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  double* ensure(Ctx& c, size_t count) {
    if (count <= n && p) return p;
    release();
    s = c.stream;
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(double), s);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      throw Error{PW_ERR_MEMORY, "device allocation of " + std::to_string(count * 8) +
                                     " bytes failed: " + cudaGetErrorString(e)};
    }
    n = count;
    return p;
  }
};

struct IBuf {
  int* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  ~IBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  int* ensure(Ctx& c, size_t count) {
    if (count <= n && p) return p;
    if (p) cudaFreeAsync(p, s);
    s = c.stream;
    PW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(int), s));
    n = count;
    return p;
  }
};

void copy_cols(Ctx& c, double* dst, long long ldd, const double* src, long long lds,
               long long rows, long long cols) {
  if (rows <= 0 || cols <= 0 || dst == src) return;
  if (ldd == rows && lds == rows) {
    PW_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, c.stream));
  } else {
    PW_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double),
                              rows * sizeof(double), cols, cudaMemcpyDeviceToDevice, c.stream));
  }
}

// C(m x n) = alpha * op(A) * op(B) + beta * C, column-major
bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && *e == '1';
}

void gemm(Ctx& c, bool ta, bool tb, long long m, long long n, long long k, double alpha,
          const double* A, long long lda, const double* B, long long ldb, double beta, double* C,
          long long ldc) {
  if (m <= 0 || n <= 0) return;
  if (k <= 0) {
    PW_CHECK(beta == 1.0 || beta == 0.0, PW_ERR_STATE, "gemm with k=0 and beta not in {0,1}");
    if (beta == 0.0)
      PW_CUDA(cudaMemset2DAsync(C, ldc * sizeof(double), 0, m * sizeof(double), n, c.stream));
    return;
  }
  PW_CHECK(!tb, PW_ERR_STATE, "gemm: op(B) = B^T is not used by the library");
  if (getenv_flag("PW_CUBLAS")) {  // A/B comparison against the vendor GEMM (tests, profiling)
    PW_BLAS(cublasDgemm_64(blas(c), ta ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &alpha, A, lda, B,
                           ldb, &beta, C, ldc));
    return;
  }
  pw::dgemm(c, ta, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // namespace

// ============================================================ propagators
struct pw_prop {
  pw_ctx* ctx = nullptr;
  int kind = 0;  // 0 = PDE, 1 = dense
  long long dim = 0;
  pw_pde_desc desc{};
  pw::ExactParams ex{};
  DBuf uf, vf;
  bool const_vel = false;
  pw::FusedParams fp{};
  bool vadv = false;
  DBuf A;  // dense
  DBuf t1, t2, work;
  DBuf sync;  // persistent march: work counter + per-segment step counters (ints)
};

namespace {

bool use_fused(const pw_prop* P) {
  return P->kind == 0 && P->desc.scheme == PW_SCHEME_RK3 && P->const_vel && !P->ctx->c.strict &&
         pw::fused_supported(P->desc.nx, P->desc.ny);
}

// Returns true when the last fused step already stored the result into the npeer
// peer buffers (row-marching epilogue); otherwise prop_apply copies it there.
bool prop_apply_impl(pw_prop* P, const double* in, double* out, int batch, long long ld, int npeer,
                     double* const* peers) {
  Ctx& c = P->ctx->c;
  const long long d = P->dim;
  PW_CHECK(batch >= 0, PW_ERR_VALUE, "batch must be non-negative");
  PW_CHECK(ld >= d, PW_ERR_VALUE, "ld must be >= state dimension");
  if (batch == 0) return true;
  if (P->kind == 1) {
    const double* src = in;
    if (in == out) {
      double* t = P->t1.ensure(c, (size_t)d * batch);
      copy_cols(c, t, d, in, ld, d, batch);
      src = t;
    }
    gemm(c, false, false, d, batch, d, 1.0, P->A.p, d, src, src == in ? ld : d, 0.0, out, ld);
    return false;
  }
  const pw_pde_desc& D = P->desc;
  const int nsteps = D.nsteps;
  if (nsteps == 0) {
    copy_cols(c, out, ld, in, ld, d, batch);
    return false;
  }
  if (use_fused(P)) {
    // ping-pong so that the last step lands in `out`; in != dst always
    const double* src = in;
    long long ld_src = ld;
    if (in == out) {
      double* t = P->t1.ensure(c, (size_t)d * batch);
      copy_cols(c, t, d, in, ld, d, batch);
      src = t;
      ld_src = d;
    }
    double* tmp = P->t2.ensure(c, (size_t)d * batch);
    bool peers_ok = true;  // the epilogue's 16-byte peer stores need 16-byte buffers
    for (int i = 0; i < npeer; ++i) peers_ok &= ((uintptr_t)peers[i] & 15) == 0;
    if (peers_ok && !P->vadv && pw::mtma_enabled() &&
        pw::mtma_supported(P->fp.nx, P->fp.ny, ld_src, ld, src, out, tmp)) {
      // K1: TMA-fed persistent row march over all nsteps (march_tma.cu); with peers, the
      // last step's rows also go straight into every peer's buffer (fused all-gather)
      int* sync = reinterpret_cast<int*>(
          P->sync.ensure(c, (pw::march_persist_sync_ints(P->fp.ny, batch) + 1) / 2));
      pw::FusedParams fp = P->fp;
      fp.ld_in = ld_src;
      fp.ld_out = ld;
      fp.npeer = npeer;
      for (int i = 0; i < npeer; ++i) fp.peer_delta[i] = (long long)((uintptr_t)peers[i] - (uintptr_t)out);
      pw::launch_rk3_mtma(c, fp, src, out, tmp, batch, nsteps, d, sync);
      return npeer > 0;
    }
    if (npeer == 0 && nsteps >= 2 && !P->vadv && pw::march_persist_enabled(P->fp.nx) &&
        pw::march_supported(P->fp.nx, P->fp.ny, ld_src, ld, src, out) &&
        pw::march_supported(P->fp.nx, P->fp.ny, d, d, tmp, tmp)) {
      int* sync = reinterpret_cast<int*>(
          P->sync.ensure(c, (pw::march_persist_sync_ints(P->fp.ny, batch) + 1) / 2));
      pw::FusedParams fp = P->fp;
      fp.ld_in = ld_src;
      fp.ld_out = ld;
      pw::launch_rk3_march_persist(c, fp, src, out, tmp, batch, nsteps, d, sync);
      return false;
    }
    bool peers_done = false;
    for (int s = 0; s < nsteps; ++s) {
      const bool to_out = ((nsteps - 1 - s) % 2) == 0;
      double* dst = to_out ? out : tmp;
      const long long ld_dst = to_out ? ld : d;
      pw::FusedParams fp = P->fp;
      fp.ld_in = ld_src;
      fp.ld_out = ld_dst;
      bool peers_aligned = true;  // the epilogue's 16-byte peer stores need 16-byte buffers
      for (int i = 0; i < npeer; ++i) peers_aligned &= ((uintptr_t)peers[i] & 15) == 0;
      if (s == nsteps - 1 && npeer > 0 && peers_aligned && !P->vadv && pw::march_peer_capable(fp.nx) &&
          pw::march_supported(fp.nx, fp.ny, ld_src, ld_dst, src, dst)) {
        fp.npeer = npeer;
        for (int i = 0; i < npeer; ++i)
          fp.peer_delta[i] = (long long)((uintptr_t)peers[i] - (uintptr_t)out);
        peers_done = true;
      }
      pw::launch_rk3_fused(c, fp, src, dst, batch, P->vadv);
      src = dst;
      ld_src = ld_dst;
    }
    return peers_done;
  }
  // reference-order kernels, in place on `out`
  copy_cols(c, out, ld, in, ld, d, batch);
  if (D.scheme == PW_SCHEME_RK3_SCALAR) {
    double* w = P->work.ensure(c, pw::scalar_rk3_work_doubles(P->ex, batch));
    pw::launch_rk3_exact_scalar(c, P->ex, out, batch, ld, nsteps, D.h, w);
  } else if (D.scheme == PW_SCHEME_SPLIT_RK3_FB) {
    double* w = P->work.ensure(c, pw::split_rk3_fb_work_doubles(P->ex, batch));
    pw::launch_split_rk3_fb(c, P->ex, D.nu_damp, out, batch, ld, nsteps, D.h, D.n_sound, w);
  } else if (D.scheme == PW_SCHEME_RK3) {
    double* w = P->work.ensure(c, pw::rk3_exact_work_doubles(P->ex, batch));
    pw::launch_rk3_exact(c, P->ex, out, batch, ld, nsteps, D.h, w);
  } else {
    double* w = P->work.ensure(c, pw::fefb_exact_work_doubles(P->ex, batch));
    pw::launch_fefb_exact(c, P->ex, out, batch, ld, nsteps, D.h, D.n_sound, w);
  }
  return false;
}

void prop_apply(pw_prop* P, const double* in, double* out, int batch, long long ld, int npeer = 0,
                double* const* peers = nullptr) {
  PW_CHECK(npeer >= 0 && npeer <= pw::kMaxPeers, PW_ERR_VALUE, "npeer must be in [0, 7]");
  for (int i = 0; i < npeer; ++i) PW_CHECK(peers && peers[i], PW_ERR_VALUE, "NULL peer buffer");
  if (prop_apply_impl(P, in, out, batch, ld, npeer, peers) || batch == 0) return;
  Ctx& c = P->ctx->c;
  for (int i = 0; i < npeer; ++i)  // not fused: copy-engine stores into each peer (P2P)
    PW_CUDA(cudaMemcpy2DAsync(peers[i], (size_t)ld * 8, out, (size_t)ld * 8, (size_t)P->dim * 8, batch,
                              cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace

// ============================================================ Krylov basis
struct pw_basis {
  pw_ctx* ctx = nullptr;
  long long dim = 0;
  double rank_tol = 1e-10;
  int cap = 0;
  int m = 0;
  int r = 0;
  bool diff_mode = false;  // M holds F(S)-G(S) (sweep) instead of F(S) (Subspace API)
  pw_prop* coarse = nullptr;
  DBuf S, M, W, Q, Y;      // d x cap (S, M, W); d x r (Q, Y)
  DBuf Rs, tau1, tau2, diag, Q2, X, cs_work, lazy_fq, lazy_img, tmp, alpha;
  DBuf R1;                 // unpivoted R of all snapshots (cap x cap)
  DBuf Xc;                 // compact R11^-1 (r x r) for the gathered image product
  // row-sharded (TSQR) factorisation: per-shard tau, the stacked shard R factors and
  // their own QR, the small Z = Q_RR [Q2; 0], and per-shard T scratch
  DBuf tauS, RR, RG, tauRR, Trr, Zq, Tg;
  bool sweep_tsqr = false;  // set by pw_sweep: factor by TSQR when the context is sharded
  // row-local storage (multi-rank TSQR sweeps): the basis holds only this rank's rows
  // [row_lo, row_lo + dim) of the global_dim-row snapshots, images, Q and Y
  bool local_rows = false;
  long long row_lo = 0, global_dim = 0;
  int tsqr_g0 = 0, tsqr_g1 = 0, tsqr_nsh = 1;
  long long tsqr_blk = 0;
  DBuf T, wy1, wy2;        // compact-WY T of all reflectors (cap x cap) and two cap x cap temps
  std::vector<char> cs_host;  // cuSOLVER host workspace (X API)
  int v_cols = 0;          // reflectors held in W (explicit unit-lower V); incremental path
  bool lean = false;       // sweep under memory pressure: no separate snapshot copy S
  IBuf piv, info;
  std::vector<double> diag_h;
  std::vector<int> piv_h;
  bool fq_valid = false, img_valid = false;
  // Q kept implicit (sweeps on one unsharded GPU): Q = [Q2; 0] - V X2 is never formed; the
  // serial step takes Q^T x = Cq^T [x[0:mr]; V^T x] with Cq = [Q2; -X2] ((mr + k) x r).  The
  // explicit Q (d x r, 2 d k r flops) is formed on first use by basis_q().
  bool implicit_q = false, q_valid = false;
  int implicit_steps = 0;  // serial steps per update (the pass over V reads m columns, Q has r)
  DBuf Cq;
  int cq_n1 = 0, cq_n2 = 0;
};

namespace {

// PW_QR_TIMING=1 prints the refactorisation phase times (CUDA events) to stderr
struct PhaseClock {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  explicit PhaseClock(cudaStream_t st) : s(st) {
    const char* e = getenv("PW_QR_TIMING");
    on = e && *e == '1';
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
  }
  ~PhaseClock() {
    if (!on || ev.size() < 2) return;
    cudaEventSynchronize(ev.back().second);
    fprintf(stderr, "[pw qr]");
    for (size_t k = 1; k < ev.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[k - 1].second, ev[k].second);
      fprintf(stderr, " %s=%.3fms", ev[k].first, ms);
    }
    fprintf(stderr, "\n");
    for (auto& x : ev) cudaEventDestroy(x.second);
  }
};

// Unpivoted Householder QR  S = Q1 R1  of all m snapshots, kept in compact WY form:
//   Q1 = I - V T V^T,  V (d x k, W's columns, explicit unit-lower trapezoidal),
//   T (k x k upper triangular, ld cap),  k = min(d, m)
// and R1 copied to a cap x cap buffer.  When the sweep appends p columns N, only they
// are processed: N <- Q1^T N = N - V T^T V^T N (three GEMMs), a 64-bit geqrf of the
// trailing (d - m_old) x p block, then T grows by the new panel's larft block and the
// coupling block -T_old (V_old^T V_new) T_new.  That is exactly a blocked Householder
// QR of the whole d x m block (no orthogonality loss on the near-duplicate snapshots
// Parareal produces), without ever forming Q1: the basis Q = Q1 [Q2; 0] is one more
// GEMM pass over V.  The pivoted QR of R1 below then picks dgeqp3's pivots on S
// (SURVEY.md 8(c)).  All solver calls are the 64-bit X API and every GEMM is
// cublasDgemm_64, so d x m may exceed 2^31 (c4: 3.1M x 1024).
static PhaseClock* g_clk = nullptr;  // optional fine-grained marks (PW_QR_TIMING=1)
static void mark(const char* n) { if (g_clk) g_clk->mark(n); }

static cusolverDnParams_t solver_params(Ctx& c) {
  if (!c.cusolver_params) {
    cusolverDnParams_t prm;
    PW_SOLVER(cusolverDnCreateParams(&prm));
    c.cusolver_params = prm;
  }
  return static_cast<cusolverDnParams_t>(c.cusolver_params);
}

// cuSOLVER workspace, sized once for the largest call this basis can make (geqrf / larft
// at k = capacity): growing it update by update re-allocated (and re-mapped) pool memory
// inside the refactorisation and stalled the stream for up to ~0.2 s.
static void presize_solver_ws(pw_basis* B) {
  if (B->cs_work.p) return;
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const long long cap = std::min<long long>(B->cap, B->dim);
  double* any = B->W.p;  // size queries only: the pointers are not dereferenced
  size_t dev = 8, host = 0, dv = 0, hv = 0;
  PW_SOLVER(cusolverDnXgeqrf_bufferSize(solver(c), solver_params(c), d, cap, CUDA_R_64F, any, d,
                                        CUDA_R_64F, any, CUDA_R_64F, &dv, &hv));
  dev = std::max(dev, dv);
  host = std::max(host, hv);
  PW_SOLVER(cusolverDnXlarft_bufferSize(solver(c), solver_params(c), CUBLAS_DIRECT_FORWARD,
                                        CUBLAS_STOREV_COLUMNWISE, d, cap, CUDA_R_64F, any, d, CUDA_R_64F,
                                        any, CUDA_R_64F, any, B->cap, CUDA_R_64F, &dv, &hv));
  dev = std::max(dev, dv);
  host = std::max(host, hv);
  B->cs_work.ensure(c, dev / sizeof(double) + 1);
  B->cs_host.resize(std::max<size_t>(host, 1));
}

// Contexts alive in this process.  With more than one (several host threads driving the
// same GPU, as the thread-rank tests do), concurrent cusolverDnXgeqrf calls on different
// handles intermittently returned CUSOLVER_STATUS_INTERNAL_ERROR, so they are serialised
// (call and completion) across contexts.  One context per process (the production layout,
// one process per GPU) takes the plain path.
static std::atomic<int> g_live_ctx{0};
static std::mutex g_geqrf_mu;

static void xgeqrf(pw_basis* B, long long rows, long long cols, double* A, long long lda, double* tau) {
  Ctx& c = B->ctx->c;
  if (!getenv_flag("PW_CUSOLVER")) {  // default: the library's TSQR panel (tsqr.cu)
    pw::tsqr_geqrf(c, rows, (int)cols, A, lda, tau);
    return;
  }
  int* info = B->info.ensure(c, 1);
  auto call = [&] {
    PW_SOLVER(cusolverDnXgeqrf(solver(c), solver_params(c), rows, cols, CUDA_R_64F, A, lda, CUDA_R_64F, tau,
                               CUDA_R_64F, B->cs_work.p, B->cs_work.n * sizeof(double), B->cs_host.data(),
                               B->cs_host.size(), info));
  };
  if (g_live_ctx.load() > 1) {
    std::lock_guard<std::mutex> lock(g_geqrf_mu);
    call();
    PW_CUDA(cudaStreamSynchronize(c.stream));
  } else {
    call();
  }
}

// Householder QR of the panel W[row0:, col0:col0+p] (ld d) into tau1[col0..], its larft
// block into T[col0.., col0..], then explicit unit-lower V for the panel (rows above the
// panel's diagonal zeroed: R1 already holds them).  Returns the reflector count.
static int factor_panel(pw_basis* B, int col0, int p) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const long long rows = d - col0;
  const int k = (int)std::min<long long>(rows, p);
  if (k <= 0) return 0;
  double* P = B->W.p + (size_t)col0 * d + col0;
  double* tau = B->tau1.p + col0;
  presize_solver_ws(B);
  xgeqrf(B, rows, p, P, d, tau);
  mark("geqrf");
  return k;
}

static void panel_to_wy(pw_basis* B, int col0, int k) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const size_t capc = (size_t)B->cap;
  pw::launch_make_unit_lower(c, B->W.p + (size_t)col0 * d, d, col0, k);
  // G = V[col0:, 0:m]^T V_new[col0:, :]  (V_new is zero above row col0), then T's new columns
  const int m = col0 + k;
  double* G = B->wy1.ensure(c, capc * capc);
  gemm(c, true, false, m, k, d - col0, 1.0, B->W.p + col0, d, B->W.p + (size_t)col0 * d + col0, d, 0.0,
       G, m);
  pw::launch_larft_cols(c, B->T.p, B->cap, G, B->tau1.p, col0, k);
  if (col0 > 0) {  // T[0:col0, new] = -T_old (G[0:col0, :] T_new)
    double* X2 = B->wy2.ensure(c, capc * capc);
    double* Tn = B->T.p + (size_t)col0 * capc + col0;
    gemm(c, false, false, col0, k, k, 1.0, G, m, Tn, B->cap, 0.0, X2, col0);
    gemm(c, false, false, col0, k, col0, -1.0, B->T.p, B->cap, X2, col0, 0.0, B->T.p + (size_t)col0 * capc,
         B->cap);
  }
  mark("larft");
}

static void alloc_factor(pw_basis* B) {
  Ctx& c = B->ctx->c;
  const size_t capc = (size_t)B->cap;
  B->W.ensure(c, (size_t)B->dim * capc);
  B->tau1.ensure(c, capc);
  if (B->T.p == nullptr) {  // T's strict lower part is never written
    B->T.ensure(c, capc * capc);
    PW_CUDA(cudaMemsetAsync(B->T.p, 0, capc * capc * sizeof(double), c.stream));
  }
  presize_solver_ws(B);
}

static void factor_full(pw_basis* B, int mr) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const int m = B->m;
  const size_t capc = (size_t)B->cap;
  alloc_factor(B);
  PW_CUDA(cudaMemsetAsync(B->T.p, 0, capc * capc * sizeof(double), c.stream));
  mark("full.alloc");
  if (!B->lean) copy_cols(c, B->W.p, d, B->S.p, d, d, m);
  const int k = factor_panel(B, 0, m);
  double* R1 = B->R1.ensure(c, capc * capc);
  double* tmp = B->Rs.ensure(c, capc * capc);
  pw::launch_extract_upper(c, B->W.p, d, mr, m, tmp);  // mr x m, ld mr
  PW_CUDA(cudaMemcpy2DAsync(R1, capc * sizeof(double), tmp, mr * sizeof(double), mr * sizeof(double),
                            m, cudaMemcpyDeviceToDevice, c.stream));
  panel_to_wy(B, 0, k);
  B->v_cols = k;
}

static void factor_append(pw_basis* B, int m_old) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const int m = B->m, p = m - m_old;
  const size_t capc = (size_t)B->cap;
  alloc_factor(B);
  double* W = B->W.p;
  double* Wn = W + (size_t)m_old * d;
  if (!B->lean) copy_cols(c, Wn, d, B->S.p + (size_t)m_old * d, d, d, p);
  mark("a.copy");
  // N <- Q1^T N = N - V T^T (V^T N)   (V = the m_old explicit reflectors)
  double* X1 = B->wy1.ensure(c, capc * capc);
  double* X2 = B->wy2.ensure(c, capc * capc);
  gemm(c, true, false, m_old, p, d, 1.0, W, d, Wn, d, 0.0, X1, m_old);
  gemm(c, true, false, m_old, p, m_old, 1.0, B->T.p, B->cap, X1, m_old, 0.0, X2, m_old);
  gemm(c, false, false, d, p, m_old, -1.0, W, d, X2, m_old, 1.0, Wn, d);
  mark("a.applyQ1T");
  // Householder QR of the trailing rows m_old..d-1 of the new block
  const int k = factor_panel(B, m_old, p);
  // R1[:, m_old:m] = [ (Q1^T N)[0:m_old] ; upper(R_N) ]
  double* R1 = B->R1.p;
  double* tmp = B->Rs.ensure(c, capc * capc);
  PW_CUDA(cudaMemcpy2DAsync(tmp, m * sizeof(double), Wn, d * sizeof(double), m * sizeof(double), p,
                            cudaMemcpyDeviceToDevice, c.stream));
  pw::launch_zero_strict_lower_block(c, tmp + m_old, m, p, p);
  PW_CUDA(cudaMemcpy2DAsync(R1 + (size_t)m_old * capc, capc * sizeof(double), tmp, m * sizeof(double),
                            m * sizeof(double), p, cudaMemcpyDeviceToDevice, c.stream));
  mark("a.R1");
  panel_to_wy(B, m_old, k);
  B->v_cols = m_old + k;
}


// ---- row-sharded subspace factorisation (distributed TSQR) --------------
// Shard g owns rows [g blk, (g+1) blk) of S (the serial correction's row blocks).  Each
// shard factors its row block of S by Householder QR (reflectors left in W's rows), the
// shards' m x m R factors are stacked (all-gathered across ranks) and factored once more:
// that R is the R1 of the whole S (unique up to row signs, which the pivoted QR of R1
// absorbs).  Q = diag(Q_g) Q_RR [Q2; 0] is then formed shard by shard.  Across ranks each
// rank factors and forms only its own rows; the collectives are one all-gather of m x m
// doubles per update.  Returns false (caller uses the replicated QR) when the sweep is not
// sharded, the basis is lean, or a shard has fewer rows than there are snapshots.
static bool tsqr_applicable(pw_basis* B) {
  Ctx& c = B->ctx->c;
  if (!B->sweep_tsqr || !c.tsqr || B->lean) return false;
  const bool comm = c.comm_world > 1;
  const int nsh = comm ? c.comm_world : c.vshards;
  if (nsh <= 1) return false;
  const long long d = B->local_rows ? B->global_dim : B->dim;
  const long long blk = ((d + nsh - 1) / nsh + 1) / 2 * 2;
  if (d - (long long)(nsh - 1) * blk < B->m) {
    // the same test on every rank: a row-local basis has no replicated fallback
    PW_CHECK(!B->local_rows, PW_ERR_STATE,
             "row-sharded subspace: the smallest row block has fewer rows than the " +
                 std::to_string(B->m) + " snapshots");
    return false;
  }
  B->tsqr_nsh = nsh;
  B->tsqr_blk = blk;
  B->tsqr_g0 = comm ? c.comm_rank : 0;
  B->tsqr_g1 = comm ? c.comm_rank + 1 : nsh;
  return true;
}

// storage rows of shard g: its block of the replicated arrays, or all rows of a row-local basis
static void tsqr_rows(const pw_basis* B, int g, long long& lo, long long& rows) {
  if (B->local_rows) {
    lo = 0;
    rows = B->dim;
    return;
  }
  lo = g * B->tsqr_blk;
  rows = std::min<long long>(B->dim, lo + B->tsqr_blk) - lo;
}

static void factor_tsqr(pw_basis* B) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const int m = B->m, nsh = B->tsqr_nsh;
  const size_t capc = (size_t)B->cap;
  const long long nm = (long long)nsh * m;  // rows of the stacked R
  alloc_factor(B);
  copy_cols(c, B->W.p, d, B->S.p, d, d, m);
  double* tauS = B->tauS.ensure(c, (size_t)nsh * capc);
  double* RR = B->RR.ensure(c, (size_t)nsh * capc * capc);
  double* RG = B->RG.ensure(c, (size_t)nsh * capc * capc);
  int* info = B->info.ensure(c, 1);
  for (int g = B->tsqr_g0; g < B->tsqr_g1; ++g) {
    long long lo, rows;
    tsqr_rows(B, g, lo, rows);
    xgeqrf(B, rows, m, B->W.p + lo, d, tauS + (size_t)g * capc);
    pw::launch_extract_upper(c, B->W.p + lo, d, m, m, RG + (size_t)g * m * m);  // m x m, ld m
  }
  mark("tsqr.local");
  if (c.comm_world > 1) {
    // the hooks work on the context's main stream; this may run on the side stream (beside
    // the fine sweep): hand the R factors over and take the gathered ones back with syncs of
    // the two streams (once per update)
    PW_CUDA(cudaStreamSynchronize(c.stream));
    pw::comm_allgather(c, RG, (long long)m * m, (long long)nsh * m * m);  // TSQR R factors
    if (c.outer) PW_CUDA(cudaStreamSynchronize(c.outer));
  }
  for (int g = 0; g < nsh; ++g)  // stack: RR[g m : (g+1) m, :] = R_g
    PW_CUDA(cudaMemcpy2DAsync(RR + (size_t)g * m, nm * sizeof(double), RG + (size_t)g * m * m,
                              m * sizeof(double), m * sizeof(double), m, cudaMemcpyDeviceToDevice, c.stream));
  double* tauRR = B->tauRR.ensure(c, capc);
  xgeqrf(B, nm, m, RR, nm, tauRR);
  double* tmp = B->Rs.ensure(c, capc * capc);
  pw::launch_extract_upper(c, RR, nm, m, m, tmp);
  PW_CUDA(cudaMemcpy2DAsync(B->R1.p, capc * sizeof(double), tmp, m * sizeof(double), m * sizeof(double), m,
                            cudaMemcpyDeviceToDevice, c.stream));
  B->v_cols = -1;  // W holds per-shard reflectors: the next update refactors in full
  mark("tsqr.stack");
}

// T of the k explicit unit-lower reflectors V (rows x k, ld ldv): T = larft(V^T V, tau)
static void wy_t(pw_basis* B, const double* V, long long ldv, long long rows, int k, const double* tau,
                 double* T, int ldt) {
  Ctx& c = B->ctx->c;
  double* G = B->wy1.ensure(c, (size_t)B->cap * B->cap);
  gemm(c, true, false, k, k, rows, 1.0, V, ldv, V, ldv, 0.0, G, k);
  PW_CUDA(cudaMemsetAsync(T, 0, sizeof(double) * (size_t)ldt * k, c.stream));
  pw::launch_larft_cols(c, T, ldt, G, tau, 0, k);
}

// Q rows of the own shards: Q[lo:hi] = Q_g [Z_g; 0] with Z = Q_RR [Q2; 0]
static void form_q_tsqr(pw_basis* B, const double* Q2, int r, double* Q) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const int m = B->m, nsh = B->tsqr_nsh;
  const size_t capc = (size_t)B->cap;
  const long long nm = (long long)nsh * m;
  double* X1 = B->wy2.ensure(c, capc * capc);
  double* X2 = B->tmp.ensure(c, capc * capc);
  // Z = [Q2; 0] - V_RR (T_RR (V_RR[0:m]^T Q2))
  double* RR = B->RR.p;
  pw::launch_make_unit_lower(c, RR, nm, 0, m);
  double* Trr = B->Trr.ensure(c, capc * capc);
  wy_t(B, RR, nm, nm, m, B->tauRR.p, Trr, m);
  double* Z = B->Zq.ensure(c, (size_t)nm * capc);
  gemm(c, true, false, m, r, m, 1.0, RR, nm, Q2, m, 0.0, X1, m);
  gemm(c, false, false, m, r, m, 1.0, Trr, m, X1, m, 0.0, X2, m);
  PW_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * (size_t)nm * r, c.stream));
  copy_cols(c, Z, nm, Q2, m, m, r);
  gemm(c, false, false, nm, r, m, -1.0, RR, nm, X2, m, 1.0, Z, nm);
  mark("tsqr.Z");
  PW_CUDA(cudaMemsetAsync(Q, 0, sizeof(double) * (size_t)d * r, c.stream));
  double* Tg = B->Tg.ensure(c, capc * capc);
  for (int g = B->tsqr_g0; g < B->tsqr_g1; ++g) {
    long long lo, rows;
    tsqr_rows(B, g, lo, rows);
    double* V = B->W.p + lo;
    pw::launch_make_unit_lower(c, V, d, 0, m);
    wy_t(B, V, d, rows, m, B->tauS.p + (size_t)g * capc, Tg, m);
    const double* Zg = Z + (size_t)g * m;
    gemm(c, true, false, m, r, m, 1.0, V, d, Zg, nm, 0.0, X1, m);
    gemm(c, false, false, m, r, m, 1.0, Tg, m, X1, m, 0.0, X2, m);
    copy_cols(c, Q + lo, d, Zg, nm, m, r);
    gemm(c, false, false, rows, r, m, -1.0, V, d, X2, m, 1.0, Q + lo, d);
  }
  mark("tsqr.Q");
}

// The explicit orthonormal basis Q (d x r), formed on first use: Q = [Q2; 0] + V Cq[mr:, :]
static const double* basis_q(pw_basis* B) {
  if (B->q_valid || B->r == 0) return B->Q.p;
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  const int r = B->r, mr = B->cq_n1, k = B->cq_n2, lc = mr + k;
  PW_CHECK(mr > 0 && B->Cq.p, PW_ERR_STATE, "subspace basis is not factored");
  double* Q = B->Q.ensure(c, (size_t)d * std::min<size_t>((size_t)B->cap, (size_t)d));
  PW_CUDA(cudaMemsetAsync(Q, 0, sizeof(double) * (size_t)d * r, c.stream));
  copy_cols(c, Q, d, B->Cq.p, lc, mr, r);
  gemm(c, false, false, d, r, k, 1.0, B->W.p, d, B->Cq.p + mr, lc, 1.0, Q, d);
  B->q_valid = true;
  return Q;
}

// Everything of the refactorisation that depends on the snapshots only: the QR of S, the
// pivoted QR of R1 and the rank, Q, and the scattered R11^-1 (X).  The sweep runs it on the
// side stream while the fine propagator runs (the images are not needed until Y).
void basis_factor(pw_basis* B, int m_old) {
  Ctx& c = B->ctx->c;
  PhaseClock clk(c.stream);
  clk.mark("start");
  const long long d = B->dim;
  const int m = B->m;
  B->fq_valid = B->img_valid = false;
  B->r = 0;
  if (m == 0) return;
  const int mr = (int)std::min<long long>(d, m);  // rows of R1
  const size_t capc = (size_t)B->cap;
  if (B->R1.p == nullptr) {  // R1 starts zero: its strict lower part is never written
    B->R1.ensure(c, capc * capc);
    PW_CUDA(cudaMemsetAsync(B->R1.p, 0, capc * capc * sizeof(double), c.stream));
  }
  const bool tsqr = tsqr_applicable(B);
  const bool incremental = !tsqr && m <= d && m_old > 0 && B->v_cols == m_old;
  PW_CHECK(!B->lean || incremental || m_old == 0, PW_ERR_STATE,
           "lean subspace cannot be refactored from scratch (snapshots not retained)");
  g_clk = clk.on ? &clk : nullptr;
  if (tsqr) factor_tsqr(B);
  else if (incremental) factor_append(B, m_old);
  else factor_full(B, mr);
  clk.mark(tsqr ? "tsqr(total)" : incremental ? "append(total)" : "full(total)");
  // column-pivoted QR of the mr x m factor R1 (same pivots as dgeqp3 on S)
  double* Rs = B->Rs.ensure(c, capc * capc);
  PW_CUDA(cudaMemcpy2DAsync(Rs, mr * sizeof(double), B->R1.p, capc * sizeof(double), mr * sizeof(double),
                            m, cudaMemcpyDeviceToDevice, c.stream));
  int* piv = B->piv.ensure(c, capc);
  double* tau2 = B->tau2.ensure(c, capc);
  double* diag = B->diag.ensure(c, capc);
  int r = 0;
  pw::pivoted_qr_small(c, Rs, mr, m, B->rank_tol, piv, tau2, diag, &r);
  clk.mark("pivqr+rank");
  B->diag_h.assign(mr, 0.0);
  B->piv_h.assign(m, 0);
  PW_CUDA(cudaMemcpyAsync(B->diag_h.data(), diag, sizeof(double) * mr, cudaMemcpyDeviceToHost, c.stream));
  PW_CUDA(cudaMemcpyAsync(B->piv_h.data(), piv, sizeof(int) * m, cudaMemcpyDeviceToHost, c.stream));
  B->r = r;
  if (r == 0) return;
  // Q = Q1 [Q2[:, :r]; 0] = [Q2; 0] - V (T (V[0:mr]^T Q2))
  double* Q2 = B->Q2.ensure(c, capc * capc);
  pw::form_q2(c, Rs, mr, piv, tau2, r, Q2);
  B->q_valid = false;
  B->cq_n1 = B->cq_n2 = 0;
  if (tsqr) {
    double* Q = B->Q.ensure(c, (size_t)d * std::min<size_t>(capc, (size_t)d));
    form_q_tsqr(B, Q2, r, Q);
    B->q_valid = true;
  } else {
    // Cq = [Q2; -X2], X2 = T (V[0:mr]^T Q2): the small factors of Q = [Q2; 0] - V X2
    const int k = B->v_cols;  // == mr
    const int lc = mr + k;
    double* X1 = B->wy1.ensure(c, capc * capc);
    double* Cq = B->Cq.ensure(c, 2 * capc * capc);
    gemm(c, true, false, k, r, mr, 1.0, B->W.p, d, Q2, mr, 0.0, X1, k);
    copy_cols(c, Cq, lc, Q2, mr, mr, r);
    gemm(c, false, false, k, r, k, -1.0, B->T.p, B->cap, X1, k, 0.0, Cq + mr, lc);
    B->cq_n1 = mr;
    B->cq_n2 = k;
    // worth it while the m - r extra columns the serial passes read (V has m columns, Q r)
    // cost less than the 2 d k r flops of forming Q: HBM at ~6.5 TB/s against ~25 TFLOP/s
    const double extra_s = (double)(k - r) * B->implicit_steps * 8.0 / 6.5e12;
    const double form_s = 2.0 * (double)k * r / 25e12;
    if (!B->implicit_q || extra_s >= form_s) basis_q(B);
  }
  clk.mark("Q=Q1Q2");
  double* X = B->X.ensure(c, capc * capc);
  pw::tri_inverse_scatter(c, Rs, mr, m, piv, r, X);
  B->Y.ensure(c, (size_t)d * std::min<size_t>(capc, (size_t)d));
  clk.mark("Rinv");
}

// Y = M scatter(R11^-1)   (FQ, or D = (F-G)(S) R^-1 in the sweep) -- the only part of the
// refactorisation that needs the images.  Gathering the r pivot columns and an in-place
// cublasDtrmm_64 (d r^2 flops) measured slower than this GEMM (186 vs 111 ms, c4).
void basis_images_gemm(pw_basis* B) {
  Ctx& c = B->ctx->c;
  if (B->r == 0) return;
  const long long d = B->dim;
  if (getenv_flag("PW_CUBLAS")) {
    gemm(c, false, false, d, B->r, B->m, 1.0, B->M.p, d, B->X.p, B->m, 0.0, B->Y.p, d);
    return;
  }
  // X = scatter(R11^-1) has only the r pivot rows: Y = M[:, piv[0:r]] R11^-1, the column
  // gather and the triangle both in the DMMA GEMM (d r^2 flops instead of 2 d m r)
  const int r = B->r;
  double* Xc = B->Xc.ensure(c, (size_t)r * r);
  pw::launch_gather_rows(c, B->X.p, B->m, B->piv.p, r, Xc);
  pw::dgemm(c, false, d, r, r, 1.0, B->M.p, d, Xc, r, 0.0, B->Y.p, d, B->piv.p, true);
}

void basis_refactor(pw_basis* B, int m_old) {
  basis_factor(B, m_old);
  basis_images_gemm(B);
  PW_CUDA(cudaStreamSynchronize(B->ctx->c.stream));
}

// snapshot columns (lean sweeps keep them only as W's not-yet-factored columns)
void basis_append_snapshots(pw_basis* B, const double* states, long long lds, int p) {
  Ctx& c = B->ctx->c;
  PW_CHECK(p >= 0, PW_ERR_VALUE, "negative column count");
  PW_CHECK(B->m + p <= B->cap, PW_ERR_VALUE,
           "subspace capacity exceeded (" + std::to_string(B->m + p) + " > " + std::to_string(B->cap) + ")");
  const long long d = B->dim;
  double* S = B->lean ? B->W.ensure(c, (size_t)d * B->cap) : B->S.ensure(c, (size_t)d * B->cap);
  copy_cols(c, S + (size_t)B->m * d, d, states, lds, d, p);
  B->m += p;
}

// the matching image columns at column offset col0
void basis_append_images(pw_basis* B, int col0, const double* m_cols, long long ldm, int p) {
  Ctx& c = B->ctx->c;
  const long long d = B->dim;
  double* M = B->M.ensure(c, (size_t)d * B->cap);
  copy_cols(c, M + (size_t)col0 * d, d, m_cols, ldm, d, p);
}

void basis_append(pw_basis* B, const double* states, long long lds, const double* m_cols,
                  long long ldm, int p) {
  const int m_old = B->m;
  basis_append_snapshots(B, states, lds, p);
  basis_append_images(B, m_old, m_cols, ldm, p);
}

// alpha (r x batch) = Q^T v
double* basis_coeffs(pw_basis* B, const double* v, int batch, long long ld) {
  Ctx& c = B->ctx->c;
  double* a = B->alpha.ensure(c, (size_t)std::max(B->r, 1) * batch);
  gemm(c, true, false, B->r, batch, B->dim, 1.0, basis_q(B), B->dim, v, ld, 0.0, a, std::max(B->r, 1));
  return a;
}

const double* basis_fq(pw_basis* B) {
  if (!B->diff_mode) return B->Y.p;
  Ctx& c = B->ctx->c;
  if (!B->fq_valid && B->r > 0) {
    // FQ = D + G(Q)   (G linear: D = (F - G)(S) R^-1 and Q = S R^-1)
    double* fq = B->lazy_fq.ensure(c, (size_t)B->dim * B->r);
    prop_apply(B->coarse, basis_q(B), fq, B->r, B->dim);
    pw::launch_axpby_cols(c, fq, fq, B->Y.p, 1.0, 1.0, (size_t)B->dim * B->r);
    B->fq_valid = true;
  }
  return B->lazy_fq.p;
}

const double* basis_images(pw_basis* B) {
  if (!B->diff_mode) return B->M.p;
  Ctx& c = B->ctx->c;
  if (!B->img_valid && B->m > 0) {
    double* im = B->lazy_img.ensure(c, (size_t)B->dim * B->m);
    prop_apply(B->coarse, B->S.p, im, B->m, B->dim);
    pw::launch_axpby_cols(c, im, im, B->M.p, 1.0, 1.0, (size_t)B->dim * B->m);
    B->img_valid = true;
  }
  return B->lazy_img.p;
}

pw_basis* basis_new(pw_ctx* ctx, long long dim, double rank_tol, int capacity) {
  PW_CHECK(dim >= 1, PW_ERR_VALUE, "dimension must be positive");
  PW_CHECK(capacity >= 1, PW_ERR_VALUE, "capacity must be positive");
  auto* B = new pw_basis();
  B->ctx = ctx;
  B->dim = dim;
  B->rank_tol = rank_tol;
  B->cap = capacity;
  return B;
}

}  // namespace

// ============================================================ C ABI
extern "C" {

const char* pw_last_error(void) { return g_last_error.c_str(); }
int pw_version(void) { return 100; }

int pw_ctx_create(int device, void* stream, pw_ctx** out) {
  return guarded([&] {
    PW_CHECK(out != nullptr, PW_ERR_VALUE, "out is NULL");
    int ndev = 0;
    PW_CUDA(cudaGetDeviceCount(&ndev));
    PW_CHECK(device >= 0 && device < ndev, PW_ERR_VALUE, "no such CUDA device");
    PW_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    PW_CUDA(cudaGetDeviceProperties(&prop, device));
    PW_CHECK(prop.major == 10, PW_ERR_CUDA,
             std::string("this library is built for sm_100a (B200); device is ") + prop.name);
    // keep freed device memory in the stream-ordered pool: sweeps re-allocate their
    // (multi-GB) basis buffers every window, and re-mapping them costs ~100 ms
    cudaMemPool_t pool;
    PW_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    PW_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    auto ctx = std::make_unique<pw_ctx>();
    ctx->c.device = device;
    ctx->c.stream = static_cast<cudaStream_t>(stream);
    ctx->c.num_sms = prop.multiProcessorCount;
    cublasHandle_t h;
    PW_BLAS(cublasCreate(&h));
    PW_BLAS(cublasSetStream(h, ctx->c.stream));
    PW_BLAS(cublasSetMathMode(h, CUBLAS_DEFAULT_MATH));
    {
      const size_t ws = 64u << 20;  // fixed cuBLAS workspace: no allocations inside GEMM calls
      void* wp = nullptr;
      PW_CUDA(cudaMalloc(&wp, ws));
      ctx->c.blas_ws = wp;
      PW_BLAS(cublasSetWorkspace(h, wp, ws));
    }
    ctx->c.cublas = h;
    cusolverDnHandle_t sh;
    PW_SOLVER(cusolverDnCreate(&sh));
    PW_SOLVER(cusolverDnSetStream(sh, ctx->c.stream));
    ctx->c.cusolver = sh;
    if (const char* e = std::getenv("PW_ROW_SHARDS")) ctx->c.vshards = std::atoi(e);
    PW_CUDA(cudaStreamCreateWithFlags(&ctx->c.side, cudaStreamNonBlocking));
    if (const char* e = std::getenv("PW_QR_OVERLAP")) ctx->c.qr_overlap = std::atoi(e) != 0;
    if (const char* e = std::getenv("PW_TSQR")) ctx->c.tsqr = std::atoi(e) != 0;
    *out = ctx.release();
    g_live_ctx.fetch_add(1);
  });
}

int pw_ctx_destroy(pw_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    g_live_ctx.fetch_sub(1);
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.red) cudaFree(ctx->c.red);
    if (ctx->c.tma_done) cudaFree(ctx->c.tma_done);
    if (ctx->c.side) {
      cudaStreamSynchronize(ctx->c.side);
      cudaStreamDestroy(ctx->c.side);
    }
    pw::nccl_destroy(ctx->c);
    if (ctx->c.comm_scratch) cudaFree(ctx->c.comm_scratch);
    if (ctx->c.blas_ws) cudaFree(ctx->c.blas_ws);
    if (ctx->c.cublas) cublasDestroy(blas(ctx->c));
    if (ctx->c.cusolver_params) cusolverDnDestroyParams(static_cast<cusolverDnParams_t>(ctx->c.cusolver_params));
    if (ctx->c.cusolver) cusolverDnDestroy(solver(ctx->c));
    delete ctx;
  });
}

int pw_ctx_set_comm(pw_ctx* ctx, int rank, int world, pw_allreduce_hook allreduce,
                    pw_allgather_hook allgather, void* user) {
  return guarded([&] {
    PW_CHECK(ctx, PW_ERR_VALUE, "ctx is NULL");
    PW_CHECK(world >= 1 && rank >= 0 && rank < world, PW_ERR_VALUE, "bad rank / world");
    PW_CHECK(world == 1 || (allreduce && allgather), PW_ERR_VALUE, "world > 1 needs both hooks");
    ctx->c.comm_rank = rank;
    ctx->c.comm_world = world;
    ctx->c.allreduce_hook = allreduce;
    ctx->c.allgather_hook = allgather;
    ctx->c.comm_user = user;
  });
}

int pw_prop_apply_rowshard(pw_prop* prop, int nshard, double* const* state_rows, double* const* work_rows,
                           int* const* flags) {
  return guarded([&] {
    PW_CHECK(prop && state_rows && work_rows && flags, PW_ERR_VALUE, "bad argument");
    PW_CHECK(prop->kind == 0 && prop->desc.scheme == PW_SCHEME_SPLIT_FE_FB, PW_ERR_VALUE,
             "row-sharded apply is the split FE-FB coarse propagator's");
    for (int s = 0; s < nshard; ++s)
      PW_CHECK(state_rows[s] && work_rows[s] && flags[s] && (((uintptr_t)state_rows[s] | (uintptr_t)work_rows[s]) & 15) == 0,
               PW_ERR_VALUE, "row shard buffers must be non-NULL and 16-byte aligned");
    const pw_pde_desc& D = prop->desc;
    pw::launch_fefb_rowshard(prop->ctx->c, prop->ex, nshard, state_rows, work_rows, flags, D.nsteps, D.h,
                             D.n_sound);
  });
}

long long pw_rowshard_sizes(pw_prop* prop, int nshard, long long* work_doubles) {
  if (!prop || nshard < 1) return -1;
  if (work_doubles) *work_doubles = (long long)pw::rowshard_work_doubles(prop->ex, nshard);
  return pw::rowshard_flag_ints(prop->ex, nshard);
}

int pw_nccl_unique_id(unsigned char* id128) {
  return guarded([&] {
    PW_CHECK(id128 != nullptr, PW_ERR_VALUE, "id buffer is NULL");
    pw::nccl_unique_id(id128);
  });
}

int pw_ctx_set_nccl(pw_ctx* ctx, const unsigned char* id128, int rank, int world) {
  return guarded([&] {
    PW_CHECK(ctx && id128, PW_ERR_VALUE, "bad argument");
    PW_CHECK(world >= 1 && rank >= 0 && rank < world, PW_ERR_VALUE, "bad rank / world");
    pw::nccl_init(ctx->c, id128, rank, world);
  });
}

int pw_comm_allreduce(pw_ctx* ctx, double* data, long long count) {
  return guarded([&] {
    PW_CHECK(ctx && data && count >= 0, PW_ERR_VALUE, "bad argument");
    if (ctx->c.comm_world > 1 || ctx->c.nccl) pw::comm_allreduce(ctx->c, data, count);
  });
}

int pw_comm_allgather(pw_ctx* ctx, double* data, long long block, long long total) {
  return guarded([&] {
    PW_CHECK(ctx && data && block >= 1 && total >= 0, PW_ERR_VALUE, "bad argument");
    if (ctx->c.comm_world > 1 || ctx->c.nccl) pw::comm_allgather(ctx->c, data, block, total);
  });
}

int pw_ctx_set_row_shards(pw_ctx* ctx, int nshards) {
  return guarded([&] {
    PW_CHECK(ctx && nshards >= 1, PW_ERR_VALUE, "bad argument");
    ctx->c.vshards = nshards;
  });
}

int pw_ctx_set_fine_rows_hook(pw_ctx* ctx, pw_fine_rows_hook hook, void* user) {
  return guarded([&] {
    PW_CHECK(ctx != nullptr, PW_ERR_VALUE, "bad argument");
    ctx->c.fine_rows_hook = hook;
    ctx->c.fine_rows_user = user;
  });
}

int pw_ctx_set_tsqr(pw_ctx* ctx, int on) {
  return guarded([&] {
    PW_CHECK(ctx != nullptr, PW_ERR_VALUE, "bad argument");
    ctx->c.tsqr = on != 0;
  });
}

int pw_serial_step(pw_ctx* ctx, const double* g, const double* D, int rd, const double* cv,
                   const double* alpha, const double* Q, int rq, long long d, long long ld,
                   double* y, double* alpha_next) {
  return guarded([&] {
    PW_CHECK(ctx && cv && y && d >= 1 && ld >= d && rd >= 0 && rq >= 0, PW_ERR_VALUE, "bad argument");
    PW_CHECK(rd == 0 || (D && alpha), PW_ERR_VALUE, "rd > 0 needs D and alpha");
    PW_CHECK(rq == 0 || (Q && alpha_next), PW_ERR_VALUE, "rq > 0 needs Q and alpha_next");
    Ctx& c = ctx->c;
    DBuf part;
    double* pp = part.ensure(c, pw::combine_part_doubles(d, std::max(rq, 1)));
    pw::launch_combine_gemv(c, c.stream, g, D, rd, cv, alpha, Q, rq, d, y, alpha_next, pp, 0, ld);
    PW_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int pw_probe_fp64_peak(pw_ctx* ctx, int iters, double* tflops) {
  return guarded([&] {
    PW_CHECK(ctx && tflops && iters > 0, PW_ERR_VALUE, "bad argument");
    *tflops = pw::probe_fp64_tflops(ctx->c, iters);
  });
}

int pw_mem_stats(pw_ctx* ctx, int reset, long long* pool_used_high, long long* pool_reserved_high,
                 long long* device_used_now) {
  return guarded([&] {
    PW_CHECK(ctx, PW_ERR_VALUE, "ctx is NULL");
    PW_CUDA(cudaSetDevice(ctx->c.device));
    cudaMemPool_t pool;
    PW_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->c.device));
    uint64_t used = 0, reserved = 0;
    PW_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &used));
    PW_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &reserved));
    size_t free_b = 0, total_b = 0;
    PW_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (pool_used_high) *pool_used_high = (long long)used;
    if (pool_reserved_high) *pool_reserved_high = (long long)reserved;
    if (device_used_now) *device_used_now = (long long)(total_b - free_b);
    if (reset) {
      uint64_t zero = 0;
      PW_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero));
      PW_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &zero));
    }
  });
}

int pw_ctx_set_stream(pw_ctx* ctx, void* stream) {
  return guarded([&] {
    PW_CHECK(ctx, PW_ERR_VALUE, "ctx is NULL");
    ctx->c.stream = static_cast<cudaStream_t>(stream);
    PW_BLAS(cublasSetStream(blas(ctx->c), ctx->c.stream));
    PW_SOLVER(cusolverDnSetStream(solver(ctx->c), ctx->c.stream));
  });
}

int pw_ctx_synchronize(pw_ctx* ctx) {
  return guarded([&] { PW_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

int pw_ctx_set_fine_hook(pw_ctx* ctx, pw_fine_hook hook, void* user) {
  return guarded([&] {
    PW_CHECK(ctx, PW_ERR_VALUE, "ctx is NULL");
    ctx->c.fine_hook = hook;
    ctx->c.fine_hook_user = user;
  });
}

int pw_ctx_set_strict(pw_ctx* ctx, int strict) {
  return guarded([&] { ctx->c.strict = strict != 0; });
}

long long pw_ctx_launch_count(pw_ctx* ctx) { return ctx ? ctx->c.launches : -1; }

int pw_prop_create_pde(pw_ctx* ctx, const pw_pde_desc* desc, pw_prop** out) {
  return guarded([&] {
    PW_CHECK(ctx && desc && out, PW_ERR_VALUE, "NULL argument");
    const pw_pde_desc& D = *desc;
    PW_CHECK(D.scheme == PW_SCHEME_RK3 || D.scheme == PW_SCHEME_SPLIT_FE_FB ||
                 D.scheme == PW_SCHEME_RK3_SCALAR || D.scheme == PW_SCHEME_SPLIT_RK3_FB,
             PW_ERR_VALUE, "scheme must be rk3, split_fe_fb, rk3_scalar or split_rk3_fb");
    const bool scalar = D.scheme == PW_SCHEME_RK3_SCALAR;
    PW_CHECK(D.nx >= 8 && D.ny >= 8, PW_ERR_VALUE, "grid too small (need at least 8 cells per direction)");
    PW_CHECK(D.order >= 1 && D.order <= 6, PW_ERR_VALUE, "flux order must be in 1..6");
    PW_CHECK(D.nsteps >= 0, PW_ERR_VALUE, "nsteps must be non-negative");
    PW_CHECK(D.scheme == PW_SCHEME_RK3 || D.n_sound >= 1, PW_ERR_VALUE, "n_sound must be at least 1");
    PW_CHECK(D.h > 0 && D.dx > 0 && D.dy > 0 && (scalar || D.cs > 0), PW_ERR_VALUE,
             "non-positive step/spacing/sound speed");
    PW_CHECK(D.scheme != PW_SCHEME_SPLIT_RK3_FB || D.nu_damp >= 0, PW_ERR_VALUE, "negative nu_damp");
    Ctx& c = ctx->c;
    auto P = std::make_unique<pw_prop>();
    P->ctx = ctx;
    P->kind = 0;
    P->desc = D;
    P->desc.uf = P->desc.vf = nullptr;
    P->dim = (scalar ? 1LL : 3LL) * D.nx * D.ny;
    const size_t n = (size_t)D.nx * D.ny;
    std::vector<double> hu(n), hv(n);
    if (D.const_velocity) {
      std::fill(hu.begin(), hu.end(), D.vel_u);
      std::fill(hv.begin(), hv.end(), D.vel_v);
    } else {
      PW_CHECK(D.uf && D.vf, PW_ERR_VALUE, "face velocity arrays required");
      std::memcpy(hu.data(), D.uf, n * sizeof(double));
      std::memcpy(hv.data(), D.vf, n * sizeof(double));
    }
    // a velocity field that is constant on every face is handled by the folded kernel
    bool cst = true;
    for (size_t k = 1; k < n && cst; ++k) cst = (hu[k] == hu[0] && hv[k] == hv[0]);
    P->const_vel = cst;
    double* du = P->uf.ensure(c, n);
    double* dv = P->vf.ensure(c, n);
    PW_CUDA(cudaMemcpyAsync(du, hu.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    PW_CUDA(cudaMemcpyAsync(dv, hv.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    PW_CUDA(cudaStreamSynchronize(c.stream));
    P->ex = pw::ExactParams{D.nx, D.ny, D.order, D.dx, D.dy, D.cs, D.a1, D.a2, du, dv};
    auto pow2_inv = [](double x) {  // 1/x if x is an exact power of two, else 0
      int e = 0;
      const double m = std::frexp(x, &e);
      return (m == 0.5) ? std::ldexp(1.0, 1 - e) : 0.0;
    };
    P->ex.inv_dx = pow2_inv(D.dx);
    P->ex.inv_dy = pow2_inv(D.dy);
    P->ex.cvel = cst ? 1 : 0;
    P->ex.uc = hu[0];
    P->ex.vc = hv[0];
    if (D.scheme == PW_SCHEME_RK3 && cst) {
      pw::make_fused_params(P->fp, D.nx, D.ny, D.dx, D.dy, D.cs, D.order, hu[0], hv[0], D.a1,
                            D.a2, D.h);
      P->vadv = hv[0] != 0.0;
    }
    *out = P.release();
  });
}

int pw_prop_create_dense(pw_ctx* ctx, const double* a, int d, pw_prop** out) {
  return guarded([&] {
    PW_CHECK(ctx && a && out, PW_ERR_VALUE, "NULL argument");
    PW_CHECK(d >= 1, PW_ERR_VALUE, "dimension must be positive");
    auto P = std::make_unique<pw_prop>();
    P->ctx = ctx;
    P->kind = 1;
    P->dim = d;
    double* A = P->A.ensure(ctx->c, (size_t)d * d);
    PW_CUDA(cudaMemcpyAsync(A, a, sizeof(double) * d * d, cudaMemcpyDeviceToDevice, ctx->c.stream));
    *out = P.release();
  });
}

int pw_prop_destroy(pw_prop* prop) {
  return guarded([&] {
    if (!prop) return;
    cudaStreamSynchronize(prop->ctx->c.stream);
    delete prop;
  });
}

long long pw_prop_dim(const pw_prop* prop) { return prop ? prop->dim : -1; }

int pw_prop_apply(pw_prop* prop, const double* in, double* out, int batch, long long ld) {
  return guarded([&] {
    PW_CHECK(prop && in && out, PW_ERR_VALUE, "NULL argument");
    prop_apply(prop, in, out, batch, ld);
  });
}

int pw_prop_apply_to_peers(pw_prop* prop, const double* in, double* out, int batch, long long ld, int npeer,
                           double* const* peer_out) {
  return guarded([&] {
    PW_CHECK(prop && in && out, PW_ERR_VALUE, "NULL argument");
    prop_apply(prop, in, out, batch, ld, npeer, peer_out);
  });
}

int pw_ipc_alloc(pw_ctx* ctx, long long bytes, void** ptr, unsigned char handle[64]) {
  return guarded([&] {
    PW_CHECK(ctx && ptr && handle && bytes > 0, PW_ERR_VALUE, "bad argument");
    PW_CUDA(cudaSetDevice(ctx->c.device));
    void* p = nullptr;
    PW_CUDA(cudaMalloc(&p, (size_t)bytes));  // own allocation: IPC handles name its base
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      PW_CUDA(e);
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &h, 64);
    *ptr = p;
  });
}

int pw_ipc_free(pw_ctx* ctx, void* ptr) {
  return guarded([&] {
    PW_CHECK(ctx, PW_ERR_VALUE, "NULL context");
    if (!ptr) return;
    PW_CUDA(cudaSetDevice(ctx->c.device));
    PW_CUDA(cudaStreamSynchronize(ctx->c.stream));
    PW_CUDA(cudaFree(ptr));
  });
}

int pw_ipc_open(pw_ctx* ctx, const unsigned char handle[64], void** ptr) {
  return guarded([&] {
    PW_CHECK(ctx && handle && ptr, PW_ERR_VALUE, "NULL argument");
    PW_CUDA(cudaSetDevice(ctx->c.device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    PW_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int pw_ipc_close(pw_ctx* ctx, void* ptr) {
  return guarded([&] {
    PW_CHECK(ctx, PW_ERR_VALUE, "NULL context");
    if (!ptr) return;
    PW_CUDA(cudaSetDevice(ctx->c.device));
    PW_CUDA(cudaStreamSynchronize(ctx->c.stream));
    PW_CUDA(cudaIpcCloseMemHandle(ptr));
  });
}

int pw_basis_create(pw_ctx* ctx, long long dim, double rank_tol, int capacity, pw_basis** out) {
  return guarded([&] {
    PW_CHECK(ctx && out, PW_ERR_VALUE, "NULL argument");
    *out = basis_new(ctx, dim, rank_tol, capacity);
  });
}

int pw_basis_destroy(pw_basis* basis) {
  return guarded([&] {
    if (!basis) return;
    cudaStreamSynchronize(basis->ctx->c.stream);
    delete basis;
  });
}

int pw_basis_update(pw_basis* basis, const double* states, const double* images, int p) {
  return guarded([&] {
    PW_CHECK(basis, PW_ERR_VALUE, "NULL basis");
    PW_CHECK(!basis->diff_mode, PW_ERR_STATE, "sweep-internal subspace cannot be updated with images");
    PW_CHECK(p == 0 || (states && images), PW_ERR_VALUE, "NULL snapshot/image pointer");
    const int m_old = basis->m;
    basis_append(basis, states, basis->dim, images, basis->dim, p);
    basis_refactor(basis, m_old);
  });
}

int pw_basis_rank(const pw_basis* basis) { return basis ? basis->r : -1; }
int pw_basis_ncols(const pw_basis* basis) { return basis ? basis->m : -1; }

int pw_basis_views(const pw_basis* basis, const double** q, const double** fq,
                   const double** snapshots, const double** images) {
  return guarded([&] {
    PW_CHECK(basis, PW_ERR_VALUE, "NULL basis");
    pw_basis* B = const_cast<pw_basis*>(basis);
    if (q) *q = basis_q(B);
    if (fq) *fq = B->r > 0 ? basis_fq(B) : nullptr;
    if (snapshots) *snapshots = B->lean ? nullptr : B->S.p;
    if (images) *images = (B->m > 0 && !B->lean) ? basis_images(B) : nullptr;
    PW_CUDA(cudaStreamSynchronize(B->ctx->c.stream));
  });
}

int pw_basis_diag(const pw_basis* basis, double* ratios_host, int* piv_host) {
  return guarded([&] {
    PW_CHECK(basis, PW_ERR_VALUE, "NULL basis");
    const int nd = (int)basis->diag_h.size();
    for (int k = 0; k < nd && ratios_host; ++k)
      ratios_host[k] = basis->diag_h[0] != 0.0 ? basis->diag_h[k] / basis->diag_h[0] : 0.0;
    for (int k = 0; k < (int)basis->piv_h.size() && piv_host; ++k) piv_host[k] = basis->piv_h[k];
  });
}

int pw_basis_project(pw_basis* basis, const double* v, double* out, int batch, long long ld) {
  return guarded([&] {
    PW_CHECK(basis && v && out, PW_ERR_VALUE, "NULL argument");
    Ctx& c = basis->ctx->c;
    if (basis->r == 0) {
      PW_CUDA(cudaMemset2DAsync(out, ld * sizeof(double), 0, basis->dim * sizeof(double), batch, c.stream));
      return;
    }
    double* a = basis_coeffs(basis, v, batch, ld);
    gemm(c, false, false, basis->dim, batch, basis->r, 1.0, basis_q(basis), basis->dim, a, basis->r,
         0.0, out, ld);
  });
}

int pw_basis_fine_on_projection(pw_basis* basis, const double* v, double* out, int batch,
                                long long ld) {
  return guarded([&] {
    PW_CHECK(basis && v && out, PW_ERR_VALUE, "NULL argument");
    Ctx& c = basis->ctx->c;
    if (basis->r == 0) {
      PW_CUDA(cudaMemset2DAsync(out, ld * sizeof(double), 0, basis->dim * sizeof(double), batch, c.stream));
      return;
    }
    const double* fq = basis_fq(basis);
    double* a = basis_coeffs(basis, v, batch, ld);
    gemm(c, false, false, basis->dim, batch, basis->r, 1.0, fq, basis->dim, a, basis->r, 0.0, out, ld);
  });
}

int pw_kse_coarse(pw_basis* basis, pw_prop* coarse, const double* v, double* out, int batch,
                  long long ld) {
  return guarded([&] {
    PW_CHECK(basis && coarse && v && out, PW_ERR_VALUE, "NULL argument");
    PW_CHECK(coarse->dim == basis->dim, PW_ERR_VALUE, "coarse propagator dimension mismatch");
    Ctx& c = basis->ctx->c;
    const long long d = basis->dim;
    if (basis->r == 0) {
      prop_apply(coarse, v, out, batch, ld);
      return;
    }
    // K(q) = G(q - Q Q^T q) + FQ Q^T q    (subspace.py:105-111)
    const double* fq = basis_fq(basis);
    double* a = basis_coeffs(basis, v, batch, ld);
    double* w = basis->tmp.ensure(c, (size_t)d * batch);
    copy_cols(c, w, d, v, ld, d, batch);
    gemm(c, false, false, d, batch, basis->r, -1.0, basis_q(basis), d, a, basis->r, 1.0, w, d);
    prop_apply(coarse, w, out, batch, ld);
    // out is (d x batch) with stride ld; add FQ a
    gemm(c, false, false, d, batch, basis->r, 1.0, fq, d, a, basis->r, 1.0, out, ld);
  });
}

int pw_copy(pw_ctx* ctx, void* dst, const void* src, long long nbytes) {
  return guarded([&] {
    PW_CHECK(ctx && dst && src && nbytes >= 0, PW_ERR_VALUE, "bad pw_copy arguments");
    if (nbytes == 0) return;
    PW_CUDA(cudaMemcpyAsync(dst, src, (size_t)nbytes, cudaMemcpyDefault, ctx->c.stream));
    PW_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int pw_residual(pw_ctx* ctx, const double* a, const double* b, int n, long long dim,
                double* out_host) {
  return guarded([&] {
    PW_CHECK(ctx && out_host, PW_ERR_VALUE, "NULL argument");
    Ctx& c = ctx->c;
    DBuf scr;
    double* s = scr.ensure(c, pw::residual_scratch_doubles(n, dim) + 1);
    pw::launch_residual(c, a, dim, b, dim, n, dim, s + 1, s);
    PW_CUDA(cudaMemcpyAsync(out_host, s, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    PW_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int pw_dgemm(pw_ctx* ctx, int trans_a, long long m, long long n, long long k, double alpha, const double* a,
             long long lda, const double* b, long long ldb, double beta, double* c, long long ldc) {
  return guarded([&] {
    PW_CHECK(ctx && (m <= 0 || n <= 0 || (c && (k <= 0 || (a && b)))), PW_ERR_VALUE, "NULL argument");
    PW_CHECK(m >= 0 && n >= 0 && k >= 0, PW_ERR_VALUE, "negative dimension");
    PW_CHECK(ldc >= std::max<long long>(1, m) && ldb >= std::max<long long>(1, k) &&
                 lda >= std::max<long long>(1, trans_a ? k : m),
             PW_ERR_VALUE, "leading dimension too small");
    gemm(ctx->c, trans_a != 0, false, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
  });
}

int pw_geqrf(pw_ctx* ctx, long long rows, int cols, double* a, long long lda, double* tau) {
  return guarded([&] {
    PW_CHECK(ctx && a && tau, PW_ERR_VALUE, "NULL argument");
    PW_CHECK(rows >= 0 && cols >= 0 && lda >= std::max<long long>(1, rows), PW_ERR_VALUE, "bad geqrf shape");
    pw::tsqr_geqrf(ctx->c, rows, cols, a, lda, tau);
  });
}

int pw_window_diag(pw_ctx* ctx, const double* q, long long dim, double cell_area, const long long* probes,
                   int nprobe, double* out_host) {
  return guarded([&] {
    PW_CHECK(ctx && q && out_host && dim >= 1, PW_ERR_VALUE, "bad pw_window_diag arguments");
    PW_CHECK(nprobe >= 0 && nprobe <= 4 && (nprobe == 0 || probes), PW_ERR_VALUE, "0..4 probe indices");
    for (int k = 0; k < nprobe; ++k)
      PW_CHECK(probes[k] >= 0 && probes[k] < dim, PW_ERR_VALUE, "probe index outside the state");
    Ctx& c = ctx->c;
    DBuf scr;
    const size_t ns = pw::window_diag_scratch_doubles(c);
    double* s = scr.ensure(c, ns + 8 + 4);
    long long* pr = reinterpret_cast<long long*>(s + ns + 8);
    if (nprobe > 0)
      PW_CUDA(cudaMemcpyAsync(pr, probes, sizeof(long long) * nprobe, cudaMemcpyHostToDevice, c.stream));
    pw::launch_window_diag(c, q, dim, cell_area, pr, nprobe, s, s + ns);
    PW_CUDA(cudaMemcpyAsync(out_host, s + ns, sizeof(double) * (3 + nprobe), cudaMemcpyDeviceToHost, c.stream));
    PW_CUDA(cudaStreamSynchronize(c.stream));
  });
}

// ------------------------------------------------------------ the sweep
namespace {
// Run a scope's launches (our kernels, cuBLAS, cuSOLVER) on another stream.
struct StreamScope {
  Ctx& c;
  cudaStream_t saved;
  StreamScope(Ctx& ctx, cudaStream_t s) : c(ctx), saved(ctx.stream) {
    c.outer = saved;  // the stream the comm hooks work on (torch's current stream)
    set(s);
  }
  ~StreamScope() {
    set(saved);
    c.outer = nullptr;
  }
  void set(cudaStream_t s) {
    c.stream = s;
    cublasSetStream(blas(c), s);
    cusolverDnSetStream(solver(c), s);
  }
};
struct SyncEvents {
  cudaEvent_t snap = nullptr, fact = nullptr, pass = nullptr, coef = nullptr;
  SyncEvents() {
    PW_CUDA(cudaEventCreateWithFlags(&snap, cudaEventDisableTiming));
    PW_CUDA(cudaEventCreateWithFlags(&fact, cudaEventDisableTiming));
    PW_CUDA(cudaEventCreateWithFlags(&pass, cudaEventDisableTiming));
    PW_CUDA(cudaEventCreateWithFlags(&coef, cudaEventDisableTiming));
  }
  ~SyncEvents() {
    cudaEventDestroy(snap);
    cudaEventDestroy(fact);
    cudaEventDestroy(pass);
    cudaEventDestroy(coef);
  }
};
}  // namespace

int pw_sweep(pw_ctx* ctx, int mode, pw_prop* fine, pw_prop* coarse, const double* q0, int n_c,
             int n_it, double tol, double rank_tol, double* out_states, double* residuals,
             int* n_done, double* timings, int* ranks, pw_basis** out_basis) {
  return guarded([&] {
    PW_CHECK(ctx && fine && coarse && q0 && out_states && residuals && n_done, PW_ERR_VALUE,
             "NULL argument");
    PW_CHECK(mode == PW_MODE_ORIGINAL || mode == PW_MODE_KSE, PW_ERR_VALUE, "unknown mode");
    PW_CHECK(n_c >= 1 && n_it >= 1, PW_ERR_VALUE, "n_c and n_it must be at least 1");
    PW_CHECK(fine->dim == coarse->dim, PW_ERR_VALUE, "fine and coarse propagators must share the grid");
    Ctx& c = ctx->c;
    const long long d = fine->dim;
    const bool kse = mode == PW_MODE_KSE;
    // buffers (column-major, ld = d)
    // Row-local sweep (multi-rank KSE with TSQR): the basis, the fine images (PRED) and the
    // coarse images (GK, GN) hold only this rank's rows [lo, lo + ldr); the iterates QK,
    // QN stay whole (G and the fine sweep need whole states).  Otherwise ldr = d, roff = 0.
    const bool local = kse && c.comm_world > 1 && c.tsqr;
    // one unsharded GPU: the serial step works on the reflectors, Q is never formed
    // (PW_IMPLICIT_Q=0 keeps the explicit Q = Q1 Q2 product of every update)
    const char* iq_env = std::getenv("PW_IMPLICIT_Q");
    const bool implicit_q = kse && c.comm_world <= 1 && c.vshards <= 1 && !(iq_env && *iq_env == '0');
    // Folded correction (single unsharded GPU; PW_FOLD_CORRECTION=0 restores the GEMM form):
    // c_i keeps only F(qk_i) - G(qk_i) and the serial pass applies D (alpha(qn_i) - alpha(qk_i)) in
    // one go, instead of subtracting D alpha(qk_i) from c_i by a d x P x r GEMM and adding
    // D alpha(qn_i) in the pass: K(qn_i) - K(qk_i) with the two projections differenced before D.
    // Same deviations from the reference runs (c3 3.7e-7, c4 2.0e-6), and a converged first slice
    // still reproduces its iterate exactly (alpha(qn_0) and alpha(qk_0) are the same vector).
    const char* fc_env = getenv("PW_FOLD_CORRECTION");
    const bool fold_corr = kse && c.comm_world <= 1 && c.vshards <= 1 && !(fc_env && *fc_env == '0');
    // Q^T qk_i read off the pivoted factor instead of a GEMM over the d rows (PW_ALPHA_FROM_R=0
    // restores the GEMM): the qk_i are this update's snapshots, so Q^T S = R2[:r, :] Pi^T holds their
    // projections already.  Same c3 / c4 deviations from the reference runs.  (With the folded
    // correction the first slice's projection cancels exactly whatever its bits, so a converged
    // first slice still repeats bit for bit.)  The row-sharded paths keep the GEMM.
    const char* ar_env = getenv("PW_ALPHA_FROM_R");
    const bool alpha_from_r = kse && c.comm_world <= 1 && c.vshards <= 1 && !(ar_env && *ar_env == '0');
    long long roff = 0, ldr = d;
    if (local) {
      const long long blk = ((d + c.comm_world - 1) / c.comm_world + 1) / 2 * 2;
      roff = std::min<long long>(d, (long long)c.comm_rank * blk);
      ldr = std::min<long long>(d, roff + blk) - roff;
      PW_CHECK(ldr >= 1, PW_ERR_VALUE, "row-sharded sweep: this rank has no rows");
    }
    DBuf bQK, bQN, bPred, bGK, bGN, bGF, bRes, bScr, bAlpha, bPart, bAlphaPart, bGv;
    double* QK = bQK.ensure(c, (size_t)d * (n_c + 1));
    double* QN = bQN.ensure(c, (size_t)d * (n_c + 1));
    double* PRED = bPred.ensure(c, (size_t)ldr * n_c);
    double* GK = bGK.ensure(c, (size_t)ldr * n_c);
    double* GN = bGN.ensure(c, (size_t)ldr * n_c);
    double* GF = local ? bGF.ensure(c, (size_t)d) : nullptr;  // one whole G(qn_i) (row-local)
    double* res_dev = bRes.ensure(c, n_it);
    double* scr = bScr.ensure(c, pw::residual_scratch_doubles(n_c, d));
    std::unique_ptr<pw_basis> B;
    if (kse) {
      // multi-rank TSQR sweeps keep only this rank's rows of the basis (memory / world)
      const long long lo = roff, nrow = ldr;
      B.reset(basis_new(ctx, nrow, rank_tol, n_c * n_it));
      B->diff_mode = true;
      B->coarse = coarse;
      B->sweep_tsqr = true;
      B->local_rows = local;
      B->row_lo = lo;
      B->global_dim = d;
      // lean mode when the d x cap matrices (S, M, W, Q, Y) plus propagator temporaries
      // would not fit next to the sweep buffers (c4 on one GPU: 5 x 25.8 GB)
      size_t free_b = 0, total_b = 0;
      PW_CUDA(cudaMemGetInfo(&free_b, &total_b));
      {  // memory the stream-ordered pool holds but does not use is free for our allocations
        cudaMemPool_t pool;
        uint64_t reserved = 0, used = 0;
        PW_CUDA(cudaDeviceGetDefaultMemPool(&pool, c.device));
        PW_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
        PW_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
        if (reserved > used) free_b += (size_t)(reserved - used);
      }
      const double col = 8.0 * (double)d, bcol = 8.0 * (double)B->dim;
      // (the sweep buffers are allocated already: col * n_c * 3 is headroom for propagator
      // temporaries, calibrated on c4)
      const double need = bcol * std::min<long long>(B->cap, B->dim) * 5.0 + col * n_c * 3.0 +
                          std::max(4.0 * (1ull << 30), 0.06 * (double)total_b);
      const char* e = getenv("PW_SWEEP_LEAN");
      B->lean = !B->local_rows && ((e && *e == '1') || need > (double)free_b);
      // even lean (4 d x cap matrices) must fit, or fail now instead of after the first fine
      // sweep (c5 on one GPU: 4 x 96 GiB; it needs the row-sharded basis of SURVEY 8(e))
      const double need_lean = need - (B->local_rows ? 0.0 : bcol * std::min<long long>(B->cap, B->dim));
      PW_CHECK(need_lean <= (double)free_b, PW_ERR_MEMORY,
               "KSE sweep needs ~" + std::to_string((long long)(need_lean / (1 << 30))) +
                   " GiB for its d x " + std::to_string(B->cap) + " basis even without a snapshot copy; " +
                   std::to_string((long long)(free_b >> 30)) + " GiB free on this device");
    }
    struct Events {  // destroyed on every exit path, errors included
      cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
      ~Events() {
        for (auto& x : e)
          if (x) cudaEventDestroy(x);
      }
    } evs;
    cudaEvent_t* ev = evs.e;
    const bool timed = timings != nullptr;
    double t_coarse = 0, t_fine = 0, t_qr = 0;
    if (timed) for (int i = 0; i < 4; ++i) PW_CUDA(cudaEventCreate(&ev[i]));
    auto elapsed = [&](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0;
      PW_CUDA(cudaEventSynchronize(b));
      PW_CUDA(cudaEventElapsedTime(&ms, a, b));
      return ms * 1e-3;
    };

    pw::NvtxRange nv_sweep(kse ? "pitwave.kse_sweep" : "pitwave.parareal_sweep");
    // serial coarse initialisation qk[i+1] = G(qk[i])  (parareal.py:112-116)
    if (timed) PW_CUDA(cudaEventRecord(ev[0], c.stream));
    std::unique_ptr<pw::NvtxRange> nv_phase(new pw::NvtxRange("coarse.init"));
    copy_cols(c, QK, d, q0, d, d, 1);
    for (int i = 0; i < n_c; ++i) prop_apply(coarse, QK + (size_t)i * d, QK + (size_t)(i + 1) * d, 1, d);
    copy_cols(c, GK, ldr, QK + d + roff, d, ldr, n_c);  // G(qk[i]) for the first correction
    if (timed) {
      PW_CUDA(cudaEventRecord(ev[1], c.stream));
      t_coarse += elapsed(ev[0], ev[1]);
    }
    SyncEvents sync;
    int k_done = 0;
    nv_phase.reset();
    for (int k = 0; k < n_it; ++k) {
      pw::NvtxRange nv_it("iteration");
      nv_phase.reset(new pw::NvtxRange("fine"));
      if (timed) PW_CUDA(cudaEventRecord(ev[0], c.stream));
      // the snapshots qk[0..P-1] are final here: their QR runs on the side stream while
      // the fine propagator runs on the main one (only Y needs the fine images)
      if (kse) PW_CUDA(cudaEventRecord(sync.snap, c.stream));
      // fine predictor over all slices at once (_fine_all, parareal.py:62-65)
      if (local && c.fine_rows_hook) {  // this rank's rows of all fine images (all-to-all)
        const int rc = c.fine_rows_hook(c.fine_rows_user, QK, PRED, n_c, d, roff, ldr);
        PW_CHECK(rc == 0, PW_ERR_STATE, "fine rows hook failed (rc=" + std::to_string(rc) + ")");
      } else if (local) {  // propagate every slice here, keep this rank's rows
        const int chunk = (int)std::max<long long>(1, std::min<long long>(n_c, (1ll << 27) / d));
        double* tmp = bGF.ensure(c, (size_t)d * chunk);
        GF = tmp;
        for (int i0 = 0; i0 < n_c; i0 += chunk) {
          const int nb = std::min(chunk, n_c - i0);
          prop_apply(fine, QK + (size_t)i0 * d, tmp, nb, d);
          copy_cols(c, PRED + (size_t)i0 * ldr, ldr, tmp + roff, d, ldr, nb);
        }
      } else if (c.fine_hook) {
        const int rc = c.fine_hook(c.fine_hook_user, QK, PRED, n_c, d);
        PW_CHECK(rc == 0, PW_ERR_STATE, "fine hook failed (rc=" + std::to_string(rc) + ")");
      } else {
        prop_apply(fine, QK, PRED, n_c, d);
      }
      if (timed) PW_CUDA(cudaEventRecord(ev[1], c.stream));
      const int m_old = kse ? B->m : 0;
      nv_phase.reset(new pw::NvtxRange("qr"));
      if (kse) {
        StreamScope side(c, c.qr_overlap ? c.side : c.stream);
        PW_CUDA(cudaStreamWaitEvent(c.stream, sync.snap, 0));
        B->implicit_q = implicit_q;
        B->implicit_steps = n_c;
        basis_append_snapshots(B.get(), QK + B->row_lo, d, n_c);
        basis_factor(B.get(), m_old);  // blocks the host at the rank read; the fine sweep runs on
        PW_CUDA(cudaEventRecord(sync.fact, c.stream));
      }
      // c_i = F(qk[i]) - G(qk[i])  [- D Q^T qk[i] in KSE mode]
      pw::launch_axpby_cols(c, PRED, PRED, GK, 1.0, -1.0, (size_t)ldr * n_c);
      int r = 0;
      double* alpha = nullptr;
      double* alpha_next = nullptr;
      if (kse) {
        basis_append_images(B.get(), m_old, PRED, ldr, n_c);  // rows roff.. (all rows: ldr = d)
        PW_CUDA(cudaStreamWaitEvent(c.stream, sync.fact, 0));
        basis_images_gemm(B.get());
        r = B->r;
        if (ranks) ranks[k] = r;
        if (r > 0) {
          double* ab = bAlpha.ensure(c, (size_t)std::min<long long>(B->cap, d) * (n_c + 2));
          if (B->local_rows) {
            // row-local (TSQR) basis: Q and Y hold this rank's rows; alpha is the sum over
            // ranks of Q_g^T qk_g, and only this rank's rows of c_i are corrected (the serial
            // correction reads no others)
            const long long lo = B->row_lo, nr = B->dim;
            gemm(c, true, false, r, n_c, nr, 1.0, basis_q(B.get()), nr, QK + lo, d, 0.0, ab, r);
            pw::comm_allreduce(c, ab, (long long)r * n_c);  // TSQR projection partials
            gemm(c, false, false, nr, n_c, r, -1.0, B->Y.p, nr, ab, r, 1.0, PRED, ldr);
          } else if (B->cq_n1 > 0 && !B->q_valid) {
            // implicit Q: Q^T QK = Q2^T QK[0:mr] - X2^T (V^T QK)
            const int mr = B->cq_n1, kv = B->cq_n2, lc = mr + kv;
            double* gv = bGv.ensure(c, (size_t)kv * (n_c + 1));
            if (alpha_from_r && !tsqr_applicable(B.get())) {
              // the qk are this update's snapshots: Q^T qk_i is a column of the pivoted factor
              pw::launch_alpha_from_r(c, B->Rs.p, (int)std::min<long long>(d, B->m), B->piv.p, B->m, m_old, n_c, r, ab);
            } else {
              gemm(c, true, false, kv, n_c, d, 1.0, B->W.p, d, QK, d, 0.0, gv, kv);
              gemm(c, true, false, r, n_c, mr, 1.0, B->Cq.p, lc, QK, d, 0.0, ab, r);
              gemm(c, true, false, r, n_c, kv, 1.0, B->Cq.p + mr, lc, gv, kv, 1.0, ab, r);
            }
            if (!fold_corr) gemm(c, false, false, d, n_c, r, -1.0, B->Y.p, d, ab, r, 1.0, PRED, d);
          } else {
            if (alpha_from_r && !tsqr_applicable(B.get()))
              pw::launch_alpha_from_r(c, B->Rs.p, (int)std::min<long long>(d, B->m), B->piv.p, B->m, m_old, n_c, r, ab);
            else
              gemm(c, true, false, r, n_c, d, 1.0, basis_q(B.get()), d, QK, d, 0.0, ab, r);
            if (!fold_corr) gemm(c, false, false, d, n_c, r, -1.0, B->Y.p, d, ab, r, 1.0, PRED, d);
          }
          alpha = ab;                             // column 0 = Q^T q0
          alpha_next = ab + (size_t)r * n_c;      // scratch pair after the block
        }
      }
      if (timed) PW_CUDA(cudaEventRecord(ev[2], c.stream));
      nv_phase.reset(new pw::NvtxRange("coarse.correction"));
      // serial correction sweep (parareal.py:128-132)
      copy_cols(c, QN, d, q0, d, d, 1);
      double* part = bPart.ensure(c, pw::combine_part_doubles(d, kse ? (int)std::min<long long>(B->cap, d) : 1));
      double* a_cur = alpha;
      double* a_buf[2] = {alpha_next, alpha_next ? alpha_next + r : nullptr};
      const bool comm = c.comm_world > 1;
      const int nsh = local ? c.comm_world : (r > 0) ? (comm ? c.comm_world : std::max(1, c.vshards)) : 1;
      if (nsh > 1) {
        // Row-sharded serial correction: shard s owns rows [s blk, (s+1) blk)
        // of D and Q.  Per step: G(qn_i) (replicated), the combine pass over the shard's rows
        // -> partial alpha_{i+1}, a sum of the partials over the shards, and the shards' rows
        // of qn_{i+1} gathered back into every replica.  Across ranks (comm hooks) the sum is
        // an allreduce of r doubles and the gather an all-gather of d doubles; a single
        // process with vshards > 1 runs every shard itself and sums in shard order (tests).
        const long long blk = ((d + nsh - 1) / nsh + 1) / 2 * 2;  // even: 16-byte row blocks
        double* a_part = bAlphaPart.ensure(c, (size_t)std::max(r, 1) * nsh);
        if (comm) {  // every replica must have found the same rank
          double* rr = a_part;
          const double rv = (double)r;
          PW_CUDA(cudaMemcpyAsync(rr, &rv, sizeof(double), cudaMemcpyHostToDevice, c.stream));
          pw::comm_allreduce(c, rr, 1);
          double tot = 0.0;
          PW_CUDA(cudaMemcpyAsync(&tot, rr, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
          PW_CUDA(cudaStreamSynchronize(c.stream));
          PW_CHECK(tot == rv * c.comm_world, PW_ERR_STATE,
                   "replicas disagree on the subspace rank (" + std::to_string(r) + " here)");
        }
        for (int i = 0; i < n_c; ++i) {
          // G(qn_i): whole, into GN's column (or GF, whose rows GN keeps, row-local)
          double* gi = local ? GF : GN + (size_t)i * d;
          prop_apply(coarse, QN + (size_t)i * d, gi, 1, d);
          double* a_nxt = a_buf[i % 2];
          const int s0 = comm ? c.comm_rank : 0, s1 = comm ? c.comm_rank + 1 : nsh;
          for (int sh = s0; sh < s1; ++sh) {
            const long long lo = std::min<long long>(d, sh * blk), hi = std::min<long long>(d, lo + blk);
            double* dst = comm ? a_nxt : a_part + (size_t)sh * r;
            if (hi <= lo) {
              PW_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * r, c.stream));
              continue;
            }
            // row-local basis: this rank's rows start at row 0 of Y and Q (ld = their rows)
            const long long boff = B->local_rows ? 0 : lo, bld = B->local_rows ? B->dim : d;
            const double* ci = local ? PRED + (size_t)i * ldr : PRED + (size_t)i * d + lo;
            pw::launch_combine_gemv(c, c.stream, gi + lo, r > 0 ? B->Y.p + boff : nullptr, r, ci, a_cur,
                                    r > 0 ? basis_q(B.get()) + boff : nullptr, r, hi - lo,
                                    QN + (size_t)(i + 1) * d + lo, dst, part, 0, bld);
            if (local)
              PW_CUDA(cudaMemcpyAsync(GN + (size_t)i * ldr, gi + lo, sizeof(double) * (size_t)ldr,
                                      cudaMemcpyDeviceToDevice, c.stream));
          }
          if (comm) {
            pw::comm_allreduce(c, a_nxt, r);
            pw::comm_allgather(c, QN + (size_t)(i + 1) * d, blk, d);
          } else {
            pw::launch_axpby_cols(c, a_nxt, a_part, a_part + r, 1.0, 1.0, (size_t)r);
            for (int sh = 2; sh < nsh; ++sh)
              pw::launch_axpby_cols(c, a_nxt, a_nxt, a_part + (size_t)sh * r, 1.0, 1.0, (size_t)r);
          }
          a_cur = a_nxt;
        }
      } else {
        const char* co_env = getenv("PW_COEF_OVERLAP");
        const bool coef_overlap = !(co_env && *co_env == '0');
        bool coef_pending = false;
        for (int i = 0; i < n_c; ++i) {
          prop_apply(coarse, QN + (size_t)i * d, GN + (size_t)i * d, 1, d);
          double* a_nxt = (r > 0) ? a_buf[i % 2] : nullptr;
          if (r > 0 && B->cq_n1 > 0 && !B->q_valid) {
            // implicit Q: the pass reduces against the reflectors V (d x kv), then
            // alpha_{i+1} = Cq^T [qn_{i+1}[0:mr]; V^T qn_{i+1}]
            const int mr = B->cq_n1, kv = B->cq_n2;
            double* gv = bGv.p + (size_t)kv * n_c;
            // the small step alpha_{i+1} = Cq^T [qn_{i+1}[0:mr]; gv] runs on the side stream beside the
            // next G (whose persistent CTAs leave a few SMs free): the pass of step i+1 waits for it
            if (coef_pending) {
              PW_CUDA(cudaStreamWaitEvent(c.stream, sync.coef, 0));
              coef_pending = false;
            }
            pw::launch_combine_gemv(c, c.stream, GN + (size_t)i * d, B->Y.p, r, PRED + (size_t)i * d, a_cur,
                                    B->W.p, kv, d, QN + (size_t)(i + 1) * d, gv, part, 0, 0,
                                    fold_corr ? alpha + (size_t)i * r : nullptr);
            if (coef_overlap && c.side) {
              PW_CUDA(cudaEventRecord(sync.pass, c.stream));
              PW_CUDA(cudaStreamWaitEvent(c.side, sync.pass, 0));
              {
                StreamScope side(c, c.side);
                pw::launch_implicit_alpha(c, B->Cq.p, mr + kv, QN + (size_t)(i + 1) * d, mr, gv, kv, r, a_nxt);
              }
              PW_CUDA(cudaEventRecord(sync.coef, c.side));
              coef_pending = true;
            } else {
              pw::launch_implicit_alpha(c, B->Cq.p, mr + kv, QN + (size_t)(i + 1) * d, mr, gv, kv, r, a_nxt);
            }
          } else {
            pw::launch_combine_gemv(c, c.stream, GN + (size_t)i * d, B ? B->Y.p : nullptr, r,
                                    PRED + (size_t)i * d, a_cur, (B && r > 0) ? basis_q(B.get()) : nullptr, r, d,
                                    QN + (size_t)(i + 1) * d, a_nxt, part, 0, 0,
                                    (fold_corr && r > 0) ? alpha + (size_t)i * r : nullptr);
          }
          a_cur = a_nxt;
        }
        if (coef_pending) PW_CUDA(cudaStreamWaitEvent(c.stream, sync.coef, 0));  // join the side stream
      }
      pw::launch_residual(c, QK + d, d, QN + d, d, n_c, d, scr, res_dev + k);
      nv_phase.reset();
      if (timed) {
        PW_CUDA(cudaEventRecord(ev[3], c.stream));
        t_fine += elapsed(ev[0], ev[1]);
        t_qr += elapsed(ev[1], ev[2]);
        t_coarse += elapsed(ev[2], ev[3]);
      }
      std::swap(bQK.p, bQN.p);
      std::swap(bQK.n, bQN.n);
      std::swap(bGK.p, bGN.p);
      std::swap(bGK.n, bGN.n);
      QK = bQK.p;
      QN = bQN.p;
      GK = bGK.p;
      GN = bGN.p;
      k_done = k + 1;
      if (tol >= 0.0) {
        double rk = 0;
        PW_CUDA(cudaMemcpyAsync(&rk, res_dev + k, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        PW_CUDA(cudaStreamSynchronize(c.stream));
        if (rk <= tol) break;
      }
    }
    copy_cols(c, out_states, d, QK + d, d, d, n_c);
    PW_CUDA(cudaMemcpyAsync(residuals, res_dev, sizeof(double) * k_done, cudaMemcpyDeviceToHost, c.stream));
    PW_CUDA(cudaStreamSynchronize(c.stream));
    *n_done = k_done;
    if (timed) {
      timings[0] = t_coarse;
      timings[1] = t_fine;
      timings[2] = t_qr;
    }
    if (out_basis) *out_basis = B.release();
  });
}

}  // extern "C"
