/*
 * pitwave_b200.h -- C ABI of the B200 (sm_100a) KSE-Parareal hot path.
 *
 * Drop-in boundary for the reference package `pitwave` (arXiv 1510.02237).
 * The reference is pure Python; its FFI-free seam for this path is the set
 * of propagator callables, the Subspace object and the sweep cores.  Every
 * entry point below replaces one of them (reference file:line cited) and is
 * bound from Python with ctypes (paper_1510_02237_b200/_lib.py; see
 * INTEGRATION.md for the binding a pitwave maintainer would add).
 *
 * Conventions
 *  - plain pointers and sizes, no torch or C++ types;
 *  - `double*` arguments documented "device" are CUDA device pointers on
 *    the context's device, "host" are host pointers;
 *  - a state is (3, ny, nx) fp64, x fastest (mesh.State, mesh.py:74-138);
 *    batches are `batch` states at a stride of `ld` doubles;
 *  - every call returns PW_OK (0) or a negative status; the message of the
 *    last failure on the calling thread is in pw_last_error().  Structural
 *    errors map to the reference's ValueError, numerical blow-up is NOT an
 *    error (the reference silences overflow, integrators.py:141-145).
 *  - all work is enqueued on the context stream; calls return without
 *    synchronising unless they return a host value (documented).
 */
#ifndef PITWAVE_B200_H
#define PITWAVE_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define PW_OK 0
#define PW_ERR_VALUE (-1)     /* reference ValueError (bad shape, ratio, order ...) */
#define PW_ERR_CUDA (-2)      /* CUDA / driver failure                             */
#define PW_ERR_LIBRARY (-3)   /* cuBLAS / cuSOLVER failure                          */
#define PW_ERR_MEMORY (-4)    /* device allocation failed                           */
#define PW_ERR_STATE (-5)     /* object used in the wrong state                     */

#define PW_SCHEME_RK3 0          /* integrators.rk3_step, integrators.py:79-85         */
#define PW_SCHEME_SPLIT_FE_FB 1  /* integrators.split_fe_fb_step, integrators.py:103-106 */
#define PW_SCHEME_RK3_SCALAR 2   /* rk3_step on the scalar advection model (physics.py:77-80);
                                    states are one (ny, nx) field                            */
#define PW_SCHEME_SPLIT_RK3_FB 3 /* integrators.split_rk3_fb_step, integrators.py:109-120:
                                    damping per stage from nu_damp (a1/a2 unused)           */

#define PW_MODE_ORIGINAL 0       /* parareal.parareal_sweep, parareal.py:68-97 */
#define PW_MODE_KSE 1            /* parareal.kse_sweep,      parareal.py:100-138 */

typedef struct pw_ctx pw_ctx;
typedef struct pw_prop pw_prop;
typedef struct pw_basis pw_basis;

/* Propagator description: integrators.PropagatorSpec (integrators.py:26-61)
 * + make_propagator (64-76) + the step count of one propagate() call
 * (126-146).  h = PropagatorSpec.dt; a1/a2 = damping_coefficients
 * (physics.py:54-58) of the step (RK3) or of one acoustic substep (FE-FB).
 * uf/vf: host (ny*nx) face-velocity arrays (mesh.face_normal_velocities,
 * mesh.py:232-247), copied to the device; if const_velocity != 0 they may be
 * NULL and (vel_u, vel_v) is used (mesh.ConstantVelocity, mesh.py:162-176). */
typedef struct pw_pde_desc {
  int scheme;
  int nx, ny;
  double dx, dy;
  double cs;
  int order;        /* advective flux order 1..6 (stencils.VALID_ORDERS) */
  double a1, a2;
  double h;
  int n_sound;
  int nsteps;       /* fixed steps per apply */
  int const_velocity;
  double vel_u, vel_v;
  const double* uf; /* host */
  const double* vf; /* host */
  double nu_damp;   /* PW_SCHEME_SPLIT_RK3_FB: alpha = nu_damp (dx^2, dy^2) / tau per stage */
} pw_pde_desc;

/* ---- library / context ------------------------------------------------ */
const char* pw_last_error(void);
int pw_version(void);
/* stream: a cudaStream_t (NULL = legacy default stream). */
int pw_ctx_create(int device, void* stream, pw_ctx** out);
int pw_ctx_destroy(pw_ctx* ctx);
int pw_ctx_set_stream(pw_ctx* ctx, void* stream);
int pw_ctx_synchronize(pw_ctx* ctx);
/* strict != 0: run the reference-operation-order kernels everywhere (bitwise
 * parity mode); default uses the folded fused RK3 kernel for constant velocity. */
int pw_ctx_set_strict(pw_ctx* ctx, int strict);
/* number of kernels this library has launched on the context (host value). */
long long pw_ctx_launch_count(pw_ctx* ctx);

/* ---- propagators: the reference's fine/coarse callables -----------------
 * replaces PitConfig.vector_propagators closures (parareal.py:182-194) and
 * propagate() (integrators.py:126-146), batched over slices (_fine_all,
 * parareal.py:62-65). */
int pw_prop_create_pde(pw_ctx* ctx, const pw_pde_desc* desc, pw_prop** out);
/* dense linear propagator q -> A q (the reference tests' matrix seam,
 * tests/test_parareal.py:14-15); a: device, d x d, column-major. */
int pw_prop_create_dense(pw_ctx* ctx, const double* a, int d, pw_prop** out);
int pw_prop_destroy(pw_prop* prop);
long long pw_prop_dim(const pw_prop* prop);
/* out[b] = P(in[b]) for b < batch; in/out device, stride ld (>= dim); in == out allowed. */
int pw_prop_apply(pw_prop* prop, const double* in, double* out, int batch, long long ld);
/* pw_prop_apply that also stores the result into npeer (<= 7) more buffers laid out
 * like out (same ld): the slice-sharded fine sweep's all-gather of end states
 * (replaces the gather of _fine_all's results, parareal.py:62-65, across
 * ranks). peer_out[i] are device pointers usable from this context: other ranks'
 * buffers mapped by pw_ipc_open (NVLink peer memory) or local buffers. For the
 * row-marching RK3 grids (nx 128/256/384/512) the last step's kernel stores every
 * output row to all of them as it is produced; otherwise the result is copied
 * afterwards (cudaMemcpy2DAsync, peer to peer). Enqueued on the context stream: the
 * caller synchronises and runs a cross-rank barrier before the peers read. */
int pw_prop_apply_to_peers(pw_prop* prop, const double* in, double* out, int batch, long long ld,
                           int npeer, double* const* peer_out);

/* ---- Krylov subspace: subspace.Subspace (subspace.py:31-98) ----------- */
/* capacity: max snapshot columns kept (the reference keeps all). */
int pw_basis_create(pw_ctx* ctx, long long dim, double rank_tol, int capacity, pw_basis** out);
int pw_basis_destroy(pw_basis* basis);
/* Subspace.update (subspace.py:46-80): append p snapshot/image pairs (device,
 * column-major d x p, ld = dim) and refactor all columns (pivoted QR,
 * rank_tol truncation, FQ = images * scatter(R^-1)).  Synchronises (rank). */
int pw_basis_update(pw_basis* basis, const double* states, const double* images, int p);
int pw_basis_rank(const pw_basis* basis);
int pw_basis_ncols(const pw_basis* basis);
/* device pointers (column-major, ld = dim) valid until the next update */
int pw_basis_views(const pw_basis* basis, const double** q, const double** fq,
                   const double** snapshots, const double** images);
/* host copy of |R_jj| / |R_11| for j < ncols (rank diagnostics) and pivots */
int pw_basis_diag(const pw_basis* basis, double* ratios_host, int* piv_host);
/* Subspace.project (82-89): out = Q (Q^T v); v/out device (batch vectors, stride ld) */
int pw_basis_project(pw_basis* basis, const double* v, double* out, int batch, long long ld);
/* Subspace.fine_on_projection (91-98): out = FQ (Q^T v) */
int pw_basis_fine_on_projection(pw_basis* basis, const double* v, double* out, int batch,
                                long long ld);
/* kse_coarse (subspace.py:105-111): out = G(v - Pv) + FQ (Q^T v) */
int pw_kse_coarse(pw_basis* basis, pw_prop* coarse, const double* v, double* out, int batch,
                  long long ld);

/* ---- sweeps: parareal_sweep / kse_sweep (parareal.py:68-138) ------------
 * q0: device (dim).  out_states: device, n_c x dim (endpoints q_1..q_{n_c}).
 * residuals: host, n_it entries; *n_done = iterations run (tol early exit).
 * tol < 0 disables the early exit (reference tol=None).
 * timings: host [coarse, fine, qr] seconds (reference Timings, parareal.py:31-47), may be NULL.
 * out_basis (KSE only, may be NULL): receives the final subspace (caller destroys).
 * Synchronises once per iteration only when tol >= 0 or timings != NULL. */
int pw_sweep(pw_ctx* ctx, int mode, pw_prop* fine, pw_prop* coarse, const double* q0, int n_c,
             int n_it, double tol, double rank_tol, double* out_states, double* residuals,
             int* n_done, double* timings, int* ranks, pw_basis** out_basis);

/* ---- slice-sharded fine predictor (multi-GPU) ----------------------------
 * If set, pw_sweep calls hook(user, qk, pred, n_c, dim) instead of applying
 * the fine propagator itself: qk = the n_c predictor inputs, pred = where the
 * n_c fine images must land (both device, column-major, ld = dim).  The hook
 * runs on the calling thread and must leave its work ordered on the context
 * stream; it returns 0 on success.  Used to shard the P independent fine
 * propagations over GPUs (each rank propagates P/N slices, then an NCCL
 * all-gather over NVLink): the reference's _fine_all pool (parareal.py:62-65)
 * spread over devices.  hook = NULL restores the local fine propagator. */
typedef int (*pw_fine_hook)(void* user, const double* qk, double* pred, int n_c, long long dim);
int pw_ctx_set_fine_hook(pw_ctx* ctx, pw_fine_hook hook, void* user);

/* Row-local variant for multi-rank TSQR sweeps (pw_ctx_set_tsqr with world > 1), where
 * the fine and coarse images are kept as this rank's rows only: the hook fills
 * pred_rows (rows x n_c, ld = rows) with rows [row_lo, row_lo + rows) of the n_c fine
 * images of qk (ld = dim).  Across ranks that is the all-to-all of SURVEY 8(e): each rank
 * propagates its slices and sends every other rank that rank's rows.  Without it such a
 * sweep propagates all slices itself and keeps its rows. */
typedef int (*pw_fine_rows_hook)(void* user, const double* qk, double* pred_rows, int n_c, long long dim,
                                 long long row_lo, long long rows);
int pw_ctx_set_fine_rows_hook(pw_ctx* ctx, pw_fine_rows_hook hook, void* user);

/* ---- row-sharded serial correction --------------------------
 * With world > 1 every rank keeps the whole subspace (replicated, deterministic
 * refactorisation) but streams only its row block [rank*blk, (rank+1)*blk) of D
 * and Q in each serial step (blk = ceil(dim/world) rounded up to even).  Per step
 * the sweep calls, on the context stream:
 *   allreduce(user, data, count)        in-place sum over ranks of count doubles
 *                                       (the partial alpha_{i+1} = Q_g^T y_g)
 *   allgather(user, data, block, total) data[rank*block .. +block) is valid on this
 *                                       rank; fill the other ranks' blocks (the
 *                                       last block may be shorter than `block`)
 * Both return 0 on success.  world = 1 (default) keeps the single-device loop.
 * pw_ctx_set_row_shards(ctx, n) runs n row shards inside one process, summing
 * the partials in shard order (the same arithmetic as n ranks; for tests). */
typedef int (*pw_allreduce_hook)(void* user, double* data, long long count);
typedef int (*pw_allgather_hook)(void* user, double* data, long long block, long long total);
int pw_ctx_set_comm(pw_ctx* ctx, int rank, int world, pw_allreduce_hook allreduce,
                    pw_allgather_hook allgather, void* user);
int pw_ctx_set_row_shards(pw_ctx* ctx, int nshards);
/* Native NCCL transport for the same collectives (replaces the hooks above; the serial
 * step's allreduce and all-gather are then enqueued from the library on the context
 * stream, no host round-trip per step -- reference serial loop parareal.py:128-132):
 *   pw_nccl_unique_id(id)   rank 0: 128-byte ncclUniqueId to broadcast to the others
 *   pw_ctx_set_nccl(ctx, id, rank, world)   every rank: ncclCommInitRank on the
 *                           context's device; sets rank / world like pw_ctx_set_comm.
 * NCCL is resolved at run time (libnccl.so.2 already in the process, e.g. torch's).
 * pw_comm_allreduce / pw_comm_allgather expose the transport (hooks or NCCL) directly:
 * allreduce = in-place sum of count doubles; allgather = as the hook above. */
/* Row-sharded coarse propagator: ONE state whose grid rows live in
 * nshard row shards, shard s holding rows [s R, (s+1) R) (R = ny / nshard) as u, v, p planes
 * of R x nx in state_rows[s], with work_rows[s] (pw_rowshard_sizes: work doubles) and
 * flags[s] (its return value: ints) of its own.  Applies the split FE-FB propagator (its
 * nsteps) to the sharded state in place: every tile waits only on its 8 neighbours'
 * phase counters, and tiles on a shard edge read their halo rows from the neighbouring
 * shard's buffers -- the halo exchange of a row-sharded G, here with every shard's tiles in
 * one launch on one device.  Bitwise equal to pw_prop_apply (integrators.py:103-106).
 * nx % 32 == 0, ny % nshard == 0, nshard <= 8. */
int pw_prop_apply_rowshard(pw_prop* prop, int nshard, double* const* state_rows, double* const* work_rows,
                           int* const* flags);
long long pw_rowshard_sizes(pw_prop* prop, int nshard, long long* work_doubles);
int pw_nccl_unique_id(unsigned char* id128);
int pw_ctx_set_nccl(pw_ctx* ctx, const unsigned char* id128, int rank, int world);
int pw_comm_allreduce(pw_ctx* ctx, double* data, long long count);
int pw_comm_allgather(pw_ctx* ctx, double* data, long long block, long long total);
/* Row-sharded subspace factorisation (distributed TSQR) for sharded sweeps
 * (world > 1 or row shards > 1): each shard Householder-factors its row block of the
 * snapshots, the m x m R factors are all-gathered (allgather hook, block m*m) and factored
 * once more, and each shard forms its own rows of Q.  Across ranks the projection
 * alpha = Q^T qk becomes a per-rank partial plus an allreduce of r x n_c doubles.
 * Replaces src/subspace.py:60-74 (the scipy qr of all snapshots) in that setting.
 * on = 0 (default; env PW_TSQR) keeps the replicated factorisation. */
int pw_ctx_set_tsqr(pw_ctx* ctx, int on);

/* ---- peer memory (CUDA IPC) for pw_prop_apply_to_peers -------------------
 * pw_ipc_alloc: bytes of device memory of its own (cudaMalloc) and its 64-byte
 * IPC handle, to send to the other ranks; pw_ipc_free releases it.
 * pw_ipc_open maps another process's handle on this context's device (NVLink peer
 * access enabled lazily); pw_ipc_close unmaps it. Same-process buffers need no
 * mapping: pass their pointers directly. */
int pw_ipc_alloc(pw_ctx* ctx, long long bytes, void** ptr, unsigned char handle[64]);
int pw_ipc_free(pw_ctx* ctx, void* ptr);
int pw_ipc_open(pw_ctx* ctx, const unsigned char handle[64], void** ptr);
int pw_ipc_close(pw_ctx* ctx, void* ptr);

/* ---- memory helper ------------------------------------------------------
 * stream-ordered copy of nbytes between any host/device pointers (UVA,
 * cudaMemcpyDefault), synchronising the context stream afterwards. */
int pw_copy(pw_ctx* ctx, void* dst, const void* src, long long nbytes);

/* ---- diagnostics --------------------------------------------------------
 * iteration_residual (parareal.py:50-59): max_i ||a_i - b_i||_2 (host result). */
int pw_residual(pw_ctx* ctx, const double* a, const double* b, int n, long long dim,
                double* out_host);

/* The library's fp64 tensor-core GEMM (DMMA, csrc/dgemm.cu) on caller device buffers:
 * C (m x n) = alpha op(A) B + beta C, column-major, op(A) = A (trans_a = 0) or A^T.
 * Every dense product of the subspace (Subspace.update / project / fine_on_projection,
 * subspace.py:66-98, and the sweep's batched K(qk)) runs on it; exported for tests and
 * benchmarks.  beta == 0 does not read C. */
int pw_dgemm(pw_ctx* ctx, int trans_a, long long m, long long n, long long k, double alpha, const double* a,
             long long lda, const double* b, long long ldb, double beta, double* c, long long ldc);

/* The library's tall-skinny Householder QR (csrc/tsqr.cu: TSQR + Householder
 * reconstruction, 32-column sub-panels) on a caller device buffer, in LAPACK dgeqrf's
 * output format: R on and above the diagonal of a (rows x cols, ld lda), the unit-lower
 * reflectors below it, tau[min(rows, cols)].  The subspace update factors every appended
 * snapshot block with it (reference subspace.py:66-68: scipy qr, LAPACK); exported for
 * tests and benchmarks. */
int pw_geqrf(pw_ctx* ctx, long long rows, int cols, double* a, long long lda, double* tau);

/* Window diagnostics of one device state q (dim doubles) in one pass -- the per-window
 * record of run_windowed (parareal.py:253-263, 316-318): out_host[0] = max|q| (max_norm,
 * diagnostics.py:34-36; NaN propagates), out_host[1] = cell_area * sum q^2 (total_energy,
 * diagnostics.py:20-23), out_host[2] = number of non-finite entries (State.all_finite,
 * mesh.py:140-141), out_host[3 + k] = q[probes[k]] for nprobe <= 4 flat indices (ProbeSeries,
 * diagnostics.py:39-66).  out_host holds 3 + nprobe doubles. */
int pw_window_diag(pw_ctx* ctx, const double* q, long long dim, double cell_area, const long long* probes,
                   int nprobe, double* out_host);

/* The sweep's fused serial-step pass on caller buffers (device pointers; test and
 * diagnostic entry):  y = [g +] c + D alpha  (rd columns of D) and
 * alpha_next = Q^T y (rq columns of Q); D and Q are column-major with leading
 * dimension ld >= d; g may be NULL; rd or rq may be 0. */
int pw_serial_step(pw_ctx* ctx, const double* g, const double* D, int rd, const double* c,
                   const double* alpha, const double* Q, int rq, long long d, long long ld,
                   double* y, double* alpha_next);

/* fp64 pipe peak (TFLOP/s) from a DFMA-throughput probe kernel: the fp64
 * half of the roofline; no reference counterpart. */
int pw_probe_fp64_peak(pw_ctx* ctx, int iters, double* tflops);

/* Device memory high-water marks of the context's device (bench reporting; no
 * reference counterpart): the stream-ordered pool every library buffer comes from
 * (used and reserved bytes since the last reset) and cudaMemGetInfo's in-use bytes
 * now (all allocators of the process, torch's caching allocator included).
 * reset != 0 restarts the pool's high-water marks after reading them. */
int pw_mem_stats(pw_ctx* ctx, int reset, long long* pool_used_high, long long* pool_reserved_high,
                 long long* device_used_now);

#ifdef __cplusplus
}
#endif
#endif /* PITWAVE_B200_H */
