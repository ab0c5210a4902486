// Row-marching fused RK3 step for constant x-advection (V = 0), sm_100a, fp64.
//
// Same operator as rk3_fused_kernel (fine_fused.cu: the folded constant-
// velocity RK3 of integrators.py:126-146 with acoustic_rhs,
// numba_backend.py:119-128), with a data movement built around the fact that
// the y coupling of the operator is narrow (radius 1, radius 2 only for the
// v damping) while the x stencils are 7 wide:
//
// * A CTA owns whole grid rows (TX = nx, periodic in x: 4 ghost columns on
//   each side of every ring row, so there is no x halo recompute) and a
//   y-segment of TY rows of one state.  It marches down the segment one row
//   per tick.
// * Three warp groups, one per RK stage.  In tick t stage 1 consumes q row
//   t-6, stage 2 s1 row t-9, stage 3 s2 row t-12: each group reads rows the
//   previous group finished in an earlier tick, so one barrier per tick.
// * y coupling in registers ("scatter"): a thread consuming input row k adds
//   its x-stencil terms to row k and its y-difference terms to the
//   accumulators of rows k-2..k+2, which it keeps in registers (u, p: 3 rows,
//   v: 5 rows).  Rows k-1 (u, p) and k-2 (v) are then complete and stored
//   (stage 1/2: shared ring; stage 3: global).  Only the input row's x
//   windows come from shared memory: 3 fields x (BX+8) doubles per BX cells.
// * q rows arrive by 16-byte cp.async two ticks ahead into an 8-row ring;
//   stages 2/3 take their q base from it when a row's accumulator is born.
// * The tick loop is unrolled 3x: u/p accumulators of row r live in slot
//   r mod 3 (compile time), only v's five rows shift.  The stage index comes
//   through __shfl_sync, so the compiler knows it is warp-uniform and keeps each
//   stage's 28 coefficients in uniform registers (DFMA operands).  6-warp CTAs
//   (nx <= 256) branch on the stage inside one loop; 12-warp CTAs (nx = 512)
//   give each stage group its own loop.
// * Segments: each state is cut into y-segments; the count minimises waves x
//   (TY + 14) over the resident CTA slots.  (MC::NS > 1 would put NS states
//   side by side in one CTA; measured slower, not dispatched.)
//
// Shared-memory rows are chunk-swizzled (chunk c at c ^ ((c >> 3) & (BX/2-1)))
// so the BX/2-chunk thread stride of the window loads is conflict free.
#include <cooperative_groups.h>
#include <type_traits>

#include "pw_internal.h"

#include <algorithm>

namespace cg = cooperative_groups;

namespace pw {
namespace {

template <int NX_, int BX_, int NS_ = 1, int CL_ = 1, int PR_ = 0>
struct MC {
  static constexpr int NX = NX_, BX = BX_, NS = NS_;  // NS states side by side per CTA
  // PR_: stage 3 also stores every output row into the peers' buffers (FusedParams
  // npeer / peer_delta): the slice all-gather fused into the last RK3 step's epilogue
  static constexpr bool PEERS = PR_ == 1;
  // PR_ == 2: persistent kernel; the item's src / dst live in shared memory (seg_shared)
  // and are re-read where used, so they take no registers across the tick loop
  static constexpr bool PERSIST = PR_ == 2;
  // CL CTAs of one thread-block cluster share each grid row (NX columns each; ghost
  // columns exchanged through distributed shared memory): rows of NXT = CL * NX cells
  static constexpr int CL = CL_, NXT = CL * NX;
  static constexpr int GS = NX / BX;   // threads per state row
  static constexpr int G = NS * GS;    // threads per stage group
  static constexpr int NT = 3 * G;
  static constexpr int RW = NX + 8;    // doubles per ring field row: cols [-4, NX+4)
  static constexpr int CHR = RW / 2;   // 16-byte chunks per field row
  static constexpr int SROW = 3 * RW;  // one state's row (u, v, p)
  static constexpr int SLOT = NS * SROW;  // doubles per ring slot
  static constexpr int NQ = 8, N1 = 3, N2 = 3;
  static constexpr size_t SMEM = sizeof(double) * SLOT * (NQ + N1 + N2);
  static constexpr int SWZ = BX / 2 - 1;
  static constexpr int WN = BX + 8;    // window: cols [x-4, x+BX+4)
  static constexpr int WC = WN / 2;    // window chunks
  static constexpr int NCH = NS * 3 * CHR;  // chunks per ring slot
  static constexpr int NLD = (NCH + NT - 1) / NT;
  // element offset of a copied chunk from the group's first state (32-bit for one state)
  using GOff = typename std::conditional<(NS > 1), long long, int>::type;
  static constexpr int MINB = (int)((227 * 1024) / (SMEM + 1024)) < 1 ? 1 : (int)((227 * 1024) / (SMEM + 1024));
  static_assert(G % 32 == 0, "stage groups must be whole warps");
  static_assert(BX == 4 || BX == 8, "BX is 4 or 8");
  static_assert(NCH >= NT, "copy entries past the row wrap once");
  static_assert(CHR % 4 == 0, "row chunks must be a multiple of the swizzle block");
};

// lags: stage S consumes row t - LAG[S] in tick t; it is active for rows [LO, HI + TY]
__host__ __device__ constexpr int lag_of(int S) { return S == 0 ? 6 : S == 1 ? 9 : 12; }
__host__ __device__ constexpr int lo_of(int S) { return S == 0 ? -6 : S == 1 ? -4 : -2; }
__host__ __device__ constexpr int hi_of(int S) { return S == 0 ? 5 : S == 1 ? 3 : 1; }

__device__ __forceinline__ int swz(int c, int m) { return c ^ ((c >> 3) & m); }

__device__ __forceinline__ void bar_sync() { asm volatile("bar.sync 0;" ::: "memory"); }
// the tick barrier: the CTA, or the whole cluster when ghost columns come from other CTAs
template <class K>
__device__ __forceinline__ void tick_sync() {
  if constexpr (K::CL > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    bar_sync();
  }
}

struct SegShared {
  const double* src;
  double* dst;
};
template <class K>
__device__ __forceinline__ SegShared& seg_shared() {
  __shared__ SegShared sh;
  return sh;
}
template <class K>
__device__ __forceinline__ const double* seg_src(const double* reg) {
  if constexpr (K::PERSIST) return *reinterpret_cast<const double* const volatile*>(&seg_shared<K>().src);
  else return reg;
}
template <class K>
__device__ __forceinline__ double* seg_dst(double* reg) {
  if constexpr (K::PERSIST) return *reinterpret_cast<double* const volatile*>(&seg_shared<K>().dst);
  else return reg;
}
// this CTA's rank in its cluster (0 without clusters: blockIdx.x is then free)
template <class K>
__device__ __forceinline__ int crank() {
  if constexpr (K::CL > 1) return (int)blockIdx.x;
  else return 0;
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void ld_chunks(double (&w)[2 * N], const double* row, const int* off) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double2 t = *reinterpret_cast<const double2*>(row + off[j]);
    w[2 * j] = t.x;
    w[2 * j + 1] = t.y;
  }
}

template <int N>
__device__ __forceinline__ void st_chunks(double* row, const int* off, const double (&v)[2 * N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) *reinterpret_cast<double2*>(row + off[j]) = make_double2(v[2 * j], v[2 * j + 1]);
}

// One stage thread's state: accumulators of rows k-1..k+1 (u, p) and k-2..k+2 (v)
// relative to the row k it consumes next.
template <class K>
struct Acc {
  double u[3][K::BX], p[3][K::BX], v[5][K::BX];
};

// Consume input row `in` (3 field rows, RW apart).  base_up / base_v: q rows k+1 and
// k+2 (S > 0; the births of rows k+1 (u, p) and k+2 (v) start from q there).
template <class K, int S, int PH>
__device__ __forceinline__ void consume(Acc<K>& A, const double* in, const double* base_up,
                                        const double* base_v, const int* woff, const StageCoef& C) {
  constexpr int BX = K::BX;
  // u, p of rows k-1, k, k+1 in slots (PH+2)%3, PH, (PH+1)%3 (PH = k mod 3, compile time);
  // v of rows k-2 .. k+2 in v[0..4] (shifted after every row)
  constexpr int U0 = (PH + 2) % 3, U1 = PH, U2 = (PH + 1) % 3;
  double w[K::WN];
  // ---- v: x stencil of row k; v_x (mixed damping of u) and v itself (p's v_y, v_yy)
  //      go to rows k+-1 / k+-2; births of rows k+1 (u, p) and k+2 (v)
  ld_chunks<K::WC>(w, in + K::RW, woff);
#pragma unroll
  for (int m = 0; m < 7; ++m)
#pragma unroll
    for (int c = 0; c < BX; ++c)  // cxv equals cxp off the centre (fewer coefficient loads)
      A.v[2][c] = fma(m == 3 ? C.cxv[3] : C.cxp[m], w[c + 1 + m], A.v[2][c]);
  {
    double b[BX];
    if constexpr (S > 0) ld_chunks<BX / 2>(b, base_up, woff + 2);
#pragma unroll
    for (int c = 0; c < BX; ++c) {
      const double t1 = C.cuv * (w[c + 5] - w[c + 3]);
      A.u[U0][c] += t1;
      A.u[U2][c] = (S > 0) ? b[c] - t1 : -t1;
    }
  }
  {
    double b[BX];
    if constexpr (S > 0) ld_chunks<BX / 2>(b, base_up + 2 * K::RW, woff + 2);
#pragma unroll
    for (int c = 0; c < BX; ++c) {
      A.p[U0][c] = fma(C.pv, w[c + 4], A.p[U0][c]);
      A.p[U2][c] = (S > 0) ? fma(-C.pv, w[c + 4], b[c]) : -C.pv * w[c + 4];
    }
  }
  {
    double b[BX];
    if constexpr (S > 0) ld_chunks<BX / 2>(b, base_v + K::RW, woff + 2);
#pragma unroll
    for (int c = 0; c < BX; ++c) {
      A.v[0][c] = fma(C.dv2, w[c + 4], A.v[0][c]);
      A.v[4][c] = (S > 0) ? fma(C.dv2, w[c + 4], b[c]) : C.dv2 * w[c + 4];
    }
  }
  // ---- u: x stencil of row k, u_x for p(k) and the mixed damping of v(k+-1)
  double t2[BX];
  ld_chunks<K::WC>(w, in, woff);
#pragma unroll
  for (int m = 0; m < 7; ++m)
#pragma unroll
    for (int c = 0; c < BX; ++c)  // cxu equals cxp at the odd offsets -3, -1, 1, 3
      A.u[U1][c] = fma((m & 1) ? C.cxu[m] : C.cxp[m], w[c + 1 + m], A.u[U1][c]);
#pragma unroll
  for (int c = 0; c < BX; ++c) {
    const double bx = w[c + 5] - w[c + 3];
    A.p[U1][c] = fma(C.pu, bx, A.p[U1][c]);
    t2[c] = C.cvu * bx;
  }
  // ---- p: x stencil of row k, p_x for u(k), p_y for v(k+-1)
  ld_chunks<K::WC>(w, in + 2 * K::RW, woff);
#pragma unroll
  for (int m = 0; m < 7; ++m)
#pragma unroll
    for (int c = 0; c < BX; ++c) A.p[U1][c] = fma(C.cxp[m], w[c + 1 + m], A.p[U1][c]);
#pragma unroll
  for (int c = 0; c < BX; ++c) {
    A.u[U1][c] = fma(C.pu, w[c + 5] - w[c + 3], A.u[U1][c]);  // pgx == pu
    t2[c] = fma(C.pv, w[c + 4], t2[c]);  // pgy == pv
    A.v[1][c] += t2[c];
    A.v[3][c] -= t2[c];
  }
}

template <class K>
__device__ __forceinline__ void rotate_v(Acc<K>& A) {
#pragma unroll
  for (int c = 0; c < K::BX; ++c) {
    A.v[0][c] = A.v[1][c];
    A.v[1][c] = A.v[2][c];
    A.v[2][c] = A.v[3][c];
    A.v[3][c] = A.v[4][c];
  }
}

struct Seg {
  const double* src;  // first state of the CTA's group (loads add each chunk's state offset)
  double* dst;        // this thread's state (stage 3 stores)
  long long n;        // nx * ny
  int ny, y0, TY;
  bool st_ok;         // this thread's state exists (the last group may be short)
};

// Consume row k and store the completed rows (k-1: u, p; k-2: v) of stage S.
template <class K, int S, int PH>
__device__ __forceinline__ void stage_tick(Acc<K>& A, double* sm, const Seg& sg, const FusedParams& P,
                                           int g, int k, int z, const int* woff, int goff0, int goff1,
                                           bool ghost) {
  constexpr int k3 = PH, U0 = (PH + 2) % 3;  // ring slot of row k (k mod 3), u/p slot of row k-1
  constexpr int BX = K::BX;
  double* qring = sm;
  double* r1 = qring + K::NQ * K::SLOT;
  double* r2 = r1 + K::N1 * K::SLOT;
  const double* in;
  if constexpr (S == 0) in = qring + (size_t)(k & 7) * K::SLOT;
  else if constexpr (S == 1) in = r1 + (size_t)k3 * K::SLOT;
  else in = r2 + (size_t)k3 * K::SLOT;
  const double* bup = qring + (size_t)((k + 1) & 7) * K::SLOT;
  const double* bv = qring + (size_t)((k + 2) & 7) * K::SLOT;
  // z is 0; the per-stage loops pass it opaque (t & zmask) so the stage's coefficients
  // load inside the tick instead of being hoisted out of the loop
  consume<K, S, PH>(A, in, bup, bv, woff, P.st[S + z]);
  if constexpr (S < 2) {
    double* out = (S == 0 ? r1 : r2);
    // k3 = k mod 3: rows k-1 and k-2 sit in slots (k3 + 2) mod 3 and (k3 + 1) mod 3
    double* o1 = out + (size_t)(k3 == 0 ? 2 : k3 - 1) * K::SLOT;
    double* o2 = out + (size_t)(k3 == 2 ? 0 : k3 + 1) * K::SLOT;
    st_chunks<BX / 2>(o1, woff + 2, A.u[U0]);
    st_chunks<BX / 2>(o1 + 2 * K::RW, woff + 2, A.p[U0]);
    st_chunks<BX / 2>(o2 + K::RW, woff + 2, A.v[0]);
    if (ghost) {
      // mirrored columns: the first 4 of thread 0's block, the last 4 of the last thread's --
      // into this CTA's ghost columns, or (cluster) the neighbouring CTA's on the same rows
      if constexpr (K::CL > 1) {
        const unsigned me = blockIdx.x;
        const unsigned tgt = (g == 0) ? (me + K::CL - 1) % K::CL : (me + 1) % K::CL;
        cg::cluster_group cl = cg::this_cluster();
        o1 = cl.map_shared_rank(o1, tgt);
        o2 = cl.map_shared_rank(o2, tgt);
      }
      const bool first = (g == 0);
      double gu[4], gp[4], gv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        gu[j] = first ? A.u[U0][j] : A.u[U0][BX - 4 + j];
        gp[j] = first ? A.p[U0][j] : A.p[U0][BX - 4 + j];
        gv[j] = first ? A.v[0][j] : A.v[0][BX - 4 + j];
      }
      *reinterpret_cast<double2*>(o1 + goff0) = make_double2(gu[0], gu[1]);
      *reinterpret_cast<double2*>(o1 + goff1) = make_double2(gu[2], gu[3]);
      *reinterpret_cast<double2*>(o1 + 2 * K::RW + goff0) = make_double2(gp[0], gp[1]);
      *reinterpret_cast<double2*>(o1 + 2 * K::RW + goff1) = make_double2(gp[2], gp[3]);
      *reinterpret_cast<double2*>(o2 + K::RW + goff0) = make_double2(gv[0], gv[1]);
      *reinterpret_cast<double2*>(o2 + K::RW + goff1) = make_double2(gv[2], gv[3]);
    }
  } else {
    const int x = crank<K>() * K::NX + g * BX;
    if (sg.st_ok && k - 1 >= 0 && k - 1 < sg.TY) {
      double* o = seg_dst<K>(sg.dst) + (long long)(sg.y0 + k - 1) * K::NXT + x;
#pragma unroll
      for (int c = 0; c < BX; c += 2) {
        *reinterpret_cast<double2*>(o + c) = make_double2(A.u[U0][c], A.u[U0][c + 1]);
        *reinterpret_cast<double2*>(o + 2 * sg.n + c) = make_double2(A.p[U0][c], A.p[U0][c + 1]);
      }
      if constexpr (K::PEERS) {
        for (int i = 0; i < P.npeer; ++i) {  // NVLink stores into the peers' copies
          double* q = reinterpret_cast<double*>(reinterpret_cast<char*>(o) + P.peer_delta[i]);
#pragma unroll
          for (int c = 0; c < BX; c += 2) {
            __stcg(reinterpret_cast<double2*>(q + c), make_double2(A.u[U0][c], A.u[U0][c + 1]));
            __stcg(reinterpret_cast<double2*>(q + 2 * sg.n + c), make_double2(A.p[U0][c], A.p[U0][c + 1]));
          }
        }
      }
    }
    if (sg.st_ok && k - 2 >= 0 && k - 2 < sg.TY) {
      double* o = seg_dst<K>(sg.dst) + sg.n + (long long)(sg.y0 + k - 2) * K::NXT + x;
#pragma unroll
      for (int c = 0; c < BX; c += 2) *reinterpret_cast<double2*>(o + c) = make_double2(A.v[0][c], A.v[0][c + 1]);
      if constexpr (K::PEERS) {
        for (int i = 0; i < P.npeer; ++i) {
          double* q = reinterpret_cast<double*>(reinterpret_cast<char*>(o) + P.peer_delta[i]);
#pragma unroll
          for (int c = 0; c < BX; c += 2) __stcg(reinterpret_cast<double2*>(q + c), make_double2(A.v[0][c], A.v[0][c + 1]));
        }
      }
    }
  }
}

// One tick of stage S: the CTA barrier, the q-row load two ticks ahead, then row
// k = t - lag.  I = t mod 3 = k mod 3 (the lags are multiples of 3) is a compile-time
// constant, so the u/p accumulator slots and the s-ring slots are too.
template <class K, int S, int I>
__device__ __forceinline__ void tick(Acc<K>& A, double* sm, double* smj, const Seg& sg, const FusedParams& P, int g,
                                     int t, const int* ld_soff, const typename K::GOff* ld_goff, int* woff,
                                     int goff0, int goff1, bool ghost) {
  const int TY = sg.TY;
  cp_wait1();
  tick_sync<K>();
  {
    const int rr = t - 4;  // q row needed by stage 1 in tick t+2, into slot rr & 7
    if (rr <= TY + 5) {
      int gy = sg.y0 + rr;
      gy += (gy < 0) ? sg.ny : 0;
      gy -= (gy >= sg.ny) ? sg.ny : 0;
      double* slot = sm + (size_t)(rr & 7) * K::SLOT;
      const double* rowp = seg_src<K>(sg.src) + (long long)gy * K::NXT;
#pragma unroll
      for (int j = 0; j < K::NLD; ++j) cp16(slot + ld_soff[j], rowp + ld_goff[j]);
    }
    cp_commit();
  }
  const int k = t - lag_of(S);
  if (k < lo_of(S) || k > TY + hi_of(S)) return;
  // z = t & zmask = 0, opaque: the stage's coefficients load inside the tick (uniform
  // registers) instead of 28 doubles being hoisted out of the loop
  stage_tick<K, S, I>(A, smj, sg, P, g, k, t & P.zmask, woff, goff0, goff1, ghost);
  rotate_v(A);
}

// Single loop over ticks for all stages (the stage branch inside), unrolled 3x so the
// u/p accumulator slots are compile-time (I = t mod 3 = k mod 3).
template <class K, int I>
__device__ __forceinline__ void tick_all(Acc<K>& A, double* sm, double* smj, const Seg& sg,
                                         const FusedParams& P, int S, int g, int t,
                                         const int* ld_soff, const typename K::GOff* ld_goff,
                                         int* woff, int goff0, int goff1, bool ghost) {
  const int TY = sg.TY;
  cp_wait1();
  tick_sync<K>();
  {
    const int rr = t - 4;  // q row needed by stage 1 in tick t+2, into slot rr & 7
    if (rr <= TY + 5) {
      int gy = sg.y0 + rr;
      gy += (gy < 0) ? sg.ny : 0;
      gy -= (gy >= sg.ny) ? sg.ny : 0;
      double* slot = sm + (size_t)(rr & 7) * K::SLOT;
      const double* rowp = seg_src<K>(sg.src) + (long long)gy * K::NXT;
#pragma unroll
      for (int j = 0; j < K::NLD; ++j) cp16(slot + ld_soff[j], rowp + ld_goff[j]);
    }
    cp_commit();
  }
  const int lag = S == 0 ? lag_of(0) : S == 1 ? lag_of(1) : lag_of(2);
  const int lo = S == 0 ? lo_of(0) : S == 1 ? lo_of(1) : lo_of(2);
  const int hi = TY + (S == 0 ? hi_of(0) : S == 1 ? hi_of(1) : hi_of(2));
  const int k = t - lag;
  if (k < lo || k > hi) return;
#pragma unroll
  for (int j = 0; j < K::WC; ++j) asm volatile("" : "+r"(woff[j]));
  if (S == 0) stage_tick<K, 0, I>(A, smj, sg, P, g, k, 0, woff, goff0, goff1, ghost);
  else if (S == 1) stage_tick<K, 1, I>(A, smj, sg, P, g, k, 0, woff, goff0, goff1, ghost);
  else stage_tick<K, 2, I>(A, smj, sg, P, g, k, 0, woff, goff0, goff1, ghost);
  rotate_v(A);
}

template <class K, int S>
__device__ __forceinline__ void stage_loop(double* sm, double* smj, const Seg& sg, const FusedParams& P, int g,
                                           const int* ld_soff, const typename K::GOff* ld_goff, int* woff,
                                           int goff0, int goff1, bool ghost) {
  Acc<K> A;
#pragma unroll
  for (int c = 0; c < K::BX; ++c) {
#pragma unroll
    for (int r = 0; r < 3; ++r) A.u[r][c] = A.p[r][c] = 0.0;
#pragma unroll
    for (int r = 0; r < 5; ++r) A.v[r][c] = 0.0;
  }
  // tick count rounded up to the unroll (the same for every warp: equal barrier counts)
  const int nt = (sg.TY + 14 + 2) / 3 * 3;
  for (int t = 0; t < nt; t += 3) {
    tick<K, S, 0>(A, sm, smj, sg, P, g, t, ld_soff, ld_goff, woff, goff0, goff1, ghost);
    tick<K, S, 1>(A, sm, smj, sg, P, g, t + 1, ld_soff, ld_goff, woff, goff0, goff1, ghost);
    tick<K, S, 2>(A, sm, smj, sg, P, g, t + 2, ld_soff, ld_goff, woff, goff0, goff1, ghost);
  }
}

// One CTA's march: segment segi of state group grpz (blockIdx.y / .z of the plain
// launch; a work item of the persistent one).  ld_in / ld_out override P's (per step).
template <class K>
__device__ __forceinline__ void march_body(double* sm, const double* __restrict__ in, double* __restrict__ out,
                                           const FusedParams& P, long long ld_in, long long ld_out, int nseg,
                                           int batch, int segi, int grpz) {
  const int ny = P.ny;
  Seg sg;
  sg.n = (long long)K::NXT * ny;
  sg.ny = ny;
  sg.y0 = (int)((long long)segi * ny / nseg);
  sg.TY = (int)((long long)(segi + 1) * ny / nseg) - sg.y0;
  const int grp0 = grpz * K::NS;  // first state of this CTA
  sg.src = in + (long long)grp0 * ld_in;
  const int tid = threadIdx.x;
  // q-row copy assignment: chunk e = tid + j*NT of the 3 x CHR chunks of a row
  int ld_soff[K::NLD];
  typename K::GOff ld_goff[K::NLD];
  // entries past the row (e >= NCH) repeat an earlier chunk: the same bytes to the same
  // place, so every thread issues NLD copies and the tick loop has no divergent branch
#pragma unroll
  for (int j = 0; j < K::NLD; ++j) {
    int e = tid + j * K::NT;
    e -= (e >= K::NCH) ? K::NCH : 0;
    const int js = e / (3 * K::CHR);
    const int r = e - js * 3 * K::CHR;
    const int f = r / K::CHR, c = r - f * K::CHR;
    int col = crank<K>() * K::NX + 2 * c - 4;  // this cluster rank's columns
    col += (col < 0) ? K::NXT : 0;
    col -= (col >= K::NXT) ? K::NXT : 0;
    // a missing state of a short last group copies the group's first state (never stored)
    const int jsrc = (grp0 + js < batch) ? js : 0;
    ld_soff[j] = js * K::SROW + f * K::RW + 2 * swz(c, K::SWZ);
    ld_goff[j] = (typename K::GOff)((long long)jsrc * ld_in + f * sg.n + col);
  }
  // prologue: q rows -6 and -5 (ticks 0 and 1 of stage 1)
  for (int rr = -6; rr <= -5; ++rr) {
    int gy = sg.y0 + rr;
    gy += (gy < 0) ? ny : 0;
    double* slot = sm + (size_t)(rr & 7) * K::SLOT;
    const double* rowp = sg.src + (long long)gy * K::NXT;
#pragma unroll
    for (int j = 0; j < K::NLD; ++j)
      cp16(slot + ld_soff[j], rowp + ld_goff[j]);
    cp_commit();
  }
  // warp uniform, and read through a shuffle so the compiler knows it: the stage
  // coefficients then load into uniform registers (DFMA takes them as operands)
  const int S = __shfl_sync(0xffffffffu, tid / K::G, 0);
  // this thread's state within the group and its column group within the state row (one
  // state: compile-time 0, so dst and the ring base stay CTA-uniform)
  const int jst = K::NS > 1 ? (tid - S * K::G) / K::GS : 0;
  const int g = tid - S * K::G - jst * K::GS;
  sg.dst = out + (long long)(grp0 + jst) * ld_out;
  if constexpr (K::PERSIST) {  // read back after the first tick's barrier
    static_assert(K::NS == 1, "one state per CTA");
    if (threadIdx.x == 0) {
      seg_shared<K>().src = sg.src;
      seg_shared<K>().dst = sg.dst;
    }
  }
  sg.st_ok = K::NS > 1 ? grp0 + jst < batch : true;
  double* smj = sm + jst * K::SROW;  // ring rows of this thread's state
  constexpr int BX = K::BX;
  // this thread's window chunk offsets inside a field row (fixed for the whole march)
  int woff[K::WC];
#pragma unroll
  for (int j = 0; j < K::WC; ++j) woff[j] = 2 * swz(g * (BX / 2) + j, K::SWZ);
  // ghost chunk offsets: thread 0 mirrors cols [0,4) to [NX, NX+4), the last thread
  // cols [NX-4, NX) to [-4, 0)
  int goff0 = 0, goff1 = 0;
  if (g == 0) {
    goff0 = 2 * swz(K::NX / 2 + 2, K::SWZ);
    goff1 = 2 * swz(K::NX / 2 + 3, K::SWZ);
  } else if (g == K::GS - 1) {
    goff0 = 2 * swz(0, K::SWZ);
    goff1 = 2 * swz(1, K::SWZ);
  }
  const bool ghost = (g == 0) || (g == K::GS - 1);
  if constexpr (K::G >= 128) {  // four warps per stage group: per-stage loops, unrolled 3x
    if (S == 0) stage_loop<K, 0>(sm, smj, sg, P, g, ld_soff, ld_goff, woff, goff0, goff1, ghost);
    else if (S == 1) stage_loop<K, 1>(sm, smj, sg, P, g, ld_soff, ld_goff, woff, goff0, goff1, ghost);
    else stage_loop<K, 2>(sm, smj, sg, P, g, ld_soff, ld_goff, woff, goff0, goff1, ghost);
  } else {  // two CTAs of 6 warps per SM: one loop with the stage branch inside, unrolled 3x
    // (per-stage loops measured 44 G/s here, the rotating single loop 53.7, this 54.8)
    Acc<K> A;
#pragma unroll
    for (int c = 0; c < BX; ++c) {
#pragma unroll
      for (int r = 0; r < 3; ++r) A.u[r][c] = A.p[r][c] = 0.0;
#pragma unroll
      for (int r = 0; r < 5; ++r) A.v[r][c] = 0.0;
    }
    const int nt = (sg.TY + 14 + 2) / 3 * 3;
    for (int t = 0; t < nt; t += 3) {
      tick_all<K, 0>(A, sm, smj, sg, P, S, g, t, ld_soff, ld_goff, woff, goff0, goff1, ghost);
      tick_all<K, 1>(A, sm, smj, sg, P, S, g, t + 1, ld_soff, ld_goff, woff, goff0, goff1, ghost);
      tick_all<K, 2>(A, sm, smj, sg, P, S, g, t + 2, ld_soff, ld_goff, woff, goff0, goff1, ghost);
    }
  }
  // no CTA of a cluster leaves while a neighbour may still store its last ghost columns
  if constexpr (K::CL > 1) tick_sync<K>();
}

template <class K>
__global__ void __launch_bounds__(K::NT, K::MINB) rk3_march_kernel(const double* __restrict__ in,
                                                                  double* __restrict__ out,
                                                                  FusedParams P, int nseg, int batch) {
  extern __shared__ __align__(16) double sm[];
  march_body<K>(sm, in, out, P, P.ld_in, P.ld_out, nseg, batch, blockIdx.y, blockIdx.z);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Persistent march over all nsteps RK3 steps (PW_MARCH_PERSIST): one launch, CTAs take
// work items (step, state, segment) in order from an atomic counter.  Item (s, b, j)
// reads step s-1's rows of segments j-1..j+1 of state b (the 6-row y halo) and
// overwrites the buffer step s-2 wrote, which those same three items read: so it waits
// until done[b][j-1..j+1] >= s.  Items are taken in order, so every item waited on was
// taken by a running CTA: no deadlock, and no wave quantisation between steps.
// sync[0]: the counter; sync[1 + b * nseg + j]: steps finished by segment j of state b.
template <class K>
__global__ void __launch_bounds__(K::NT, K::MINB) rk3_march_persist_kernel(
    const double* __restrict__ in, double* out, double* tmp, FusedParams P, int nseg, int batch, int nsteps,
    long long d, int* sync) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_item;
  const int per_step = nseg * batch;
  const long long total = (long long)per_step * nsteps;
  int* done = sync + 1;
  for (;;) {
    __syncthreads();  // s_item of the previous item is no longer read
    if (threadIdx.x == 0) s_item = atomicAdd(sync, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= total) break;
    const int s = item / per_step;
    const int r = item - s * per_step;
    const int b = r / nseg, j = r - b * nseg;
    if (s > 0 && threadIdx.x < 3) {  // three neighbours, one thread each
      int jj = j + (int)threadIdx.x - 1;
      jj += (jj < 0) ? nseg : 0;
      jj -= (jj >= nseg) ? nseg : 0;
      const int* f = done + b * nseg + jj;
      long long spins = 0;
      while (ld_acquire(f) < s) {
        __nanosleep(100);
        if (++spins > (1LL << 26)) __trap();  // a broken dependency fails, never hangs
      }
    }
    __syncthreads();
    // ping-pong so that the last step lands in out (as prop_apply)
    const bool to_out = ((nsteps - 1 - s) % 2) == 0;
    double* dst = to_out ? out : tmp;
    const long long ld_dst = to_out ? P.ld_out : d;
    const double* src = s == 0 ? in : (to_out ? tmp : out);
    const long long ld_src = s == 0 ? P.ld_in : (to_out ? d : P.ld_out);
    march_body<K>(sm, src, dst, P, ld_src, ld_dst, nseg, batch, j, b);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(done + b * nseg + j, s + 1);
  }
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

template <class K>
void launch_march_cfg(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch) {
  auto kern = rk3_march_kernel<K>;
  const int per_sm = kernel_setup(c, kern, K::NT, K::SMEM);  // per device (api.cu)
  // segments per state: minimise waves x ticks per CTA (TY + 14), waves = CTAs over
  // the resident CTA slots (c2: 4 segments, one wave; c3: 2 segments, one wave)
  int nseg = env_int("PW_MARCH_NSEG", 0);
  if (nseg <= 0) {
    const long long slots = (long long)(c.num_sms > 0 ? c.num_sms : 148) * per_sm;
    double best = 1e300;
    for (int s = 1; s <= fp.ny / 16; ++s) {
      const long long ngrp = (batch + K::NS - 1) / K::NS;
      const long long waves = (ngrp * s * K::CL + slots - 1) / slots;
      const double cost = (double)waves * ((double)fp.ny / s + 14.0);
      if (cost < best - 1e-9) {
        best = cost;
        nseg = s;
      }
    }
    if (nseg <= 0) nseg = 1;
  }
  dim3 grid(K::CL, nseg, (batch + K::NS - 1) / K::NS);
  if constexpr (K::CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(K::NT);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PW_CUDA(cudaLaunchKernelEx(&cfg, kern, in, out, fp, nseg, batch));
  } else {
    kern<<<grid, K::NT, K::SMEM, c.stream>>>(in, out, fp, nseg, batch);
  }
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

template <class K>
void launch_march_persist_cfg(Ctx& c, const FusedParams& fp, const double* in, double* out, double* tmp,
                              int batch, int nsteps, long long d, int* sync) {
  auto kern = rk3_march_persist_kernel<K>;
  const int per_sm = kernel_setup(c, kern, K::NT, K::SMEM);  // per device (api.cu)
  const long long slots = (long long)(c.num_sms > 0 ? c.num_sms : 148) * per_sm;
  // segments per state: no waves here, so minimise ticks per item x max(1, items / slots)
  // (the second factor: fewer items than CTA slots leave slots idle)
  int nseg = env_int("PW_MARCH_NSEG", 0);
  if (nseg <= 0) {
    double best = 1e300;
    for (int s = 1; s <= fp.ny / 16; ++s) {
      const double items = (double)batch * s;
      const double cost = ((double)fp.ny / s + 14.0) * std::max(1.0, items / (double)slots);
      if (cost < best - 1e-9) {
        best = cost;
        nseg = s;
      }
    }
    if (nseg <= 0) nseg = 1;
  }
  // the sync buffer holds ny / 16 + 1 counters per state, and a segment needs >= 16 rows
  // (the 6-row halo of the neighbour dependency): clamp the override too
  nseg = std::max(1, std::min(nseg, fp.ny / 16));
  const long long items = (long long)batch * nseg * nsteps;
  const int grid = (int)std::min<long long>(slots, items);
  PW_CUDA(cudaMemsetAsync(sync, 0, sizeof(int) * (1 + (size_t)batch * nseg), c.stream));
  kern<<<grid, K::NT, K::SMEM, c.stream>>>(in, out, tmp, fp, nseg, batch, nsteps, d, sync);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

}  // namespace

// default: on for the two-CTA-per-SM grids (nx 128 / 256), where it removes the idle
// CTA slots of the per-step launches (c2: 58.4 vs 55.3 G/s over 200 steps); 512 measured
// slower (57.0 vs 58.3 G/s, 4 steps).  PW_MARCH_PERSIST=1 forces it on, 0 off.
bool march_persist_enabled(int nx) {
  const int e = env_int("PW_MARCH_PERSIST", -1);
  if (e == 0) return false;
  if (e > 0) return nx == 128 || nx == 256 || nx == 384 || nx == 512;
  return nx == 128 || nx == 256;
}

size_t march_persist_sync_ints(int ny, int batch) { return 1 + (size_t)batch * (size_t)(ny / 16 + 1); }

void launch_rk3_march_persist(Ctx& c, const FusedParams& fp, const double* in, double* out, double* tmp,
                              int batch, int nsteps, long long d, int* sync) {
  switch (fp.nx) {
    case 128: return launch_march_persist_cfg<MC<128, 4, 1, 1, 2>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 256: return launch_march_persist_cfg<MC<256, 4, 1, 1, 2>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 384: return launch_march_persist_cfg<MC<384, 4, 1, 1, 2>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 512: return launch_march_persist_cfg<MC<512, 4, 1, 1, 2>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    default: throw Error{PW_ERR_VALUE, "persistent march needs nx in {128, 256, 384, 512}"};
  }
}

bool march_supported(int nx, int ny, long long ld_in, long long ld_out, const void* in,
                     const void* out) {
  if (env_int("PW_MARCH", 1) == 0) return false;
  // 1024 / 2048: clusters sharing each row work (tests) but the per-tick cluster barrier
  // made them slower than the tile kernel (35.5 vs 42.5 G/s at 1024^2 x 16): opt-in only
  const bool cluster = (nx == 1024 || nx == 2048) && env_int("PW_MARCH_CLUSTER", 0) != 0;
  if (!(nx == 128 || nx == 256 || nx == 384 || nx == 512 || cluster)) return false;
  if (ny < 32) return false;
  if ((ld_in & 1) || (ld_out & 1)) return false;
  if (((uintptr_t)in & 15) || ((uintptr_t)out & 15)) return false;
  return true;
}

bool march_peer_capable(int nx) { return nx == 128 || nx == 256 || nx == 384 || nx == 512; }

void launch_rk3_march(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch) {
  if (fp.npeer > 0) {
    switch (fp.nx) {
      case 128: return launch_march_cfg<MC<128, 4, 1, 1, 1>>(c, fp, in, out, batch);
      case 256: return launch_march_cfg<MC<256, 4, 1, 1, 1>>(c, fp, in, out, batch);
      case 384: return launch_march_cfg<MC<384, 4, 1, 1, 1>>(c, fp, in, out, batch);
      case 512: return launch_march_cfg<MC<512, 4, 1, 1, 1>>(c, fp, in, out, batch);
      default: throw Error{PW_ERR_VALUE, "peer stores need nx in {128, 256, 384, 512}"};
    }
  }
  switch (fp.nx) {
    case 128: return launch_march_cfg<MC<128, 4>>(c, fp, in, out, batch);
    // MC<256, 4, 2> (two states per 12-warp CTA) passes the parity tests but spills and
    // measured 42.7 G/s against 53.7 for two 6-warp CTAs per SM
    case 256: return launch_march_cfg<MC<256, 4>>(c, fp, in, out, batch);
    case 384: return launch_march_cfg<MC<384, 4>>(c, fp, in, out, batch);
    case 512: return launch_march_cfg<MC<512, 4>>(c, fp, in, out, batch);
    // wider rows: clusters of 512-column CTAs, ghost columns through distributed smem
    case 1024: return launch_march_cfg<MC<512, 4, 1, 2>>(c, fp, in, out, batch);
    case 2048: return launch_march_cfg<MC<512, 4, 1, 4>>(c, fp, in, out, batch);
    default:
      throw Error{PW_ERR_VALUE, "row-marching RK3 needs nx in {128, 256, 384, 512}"};
  }
}

}  // namespace pw
