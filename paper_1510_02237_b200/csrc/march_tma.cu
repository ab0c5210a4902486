// K1: TMA-fed, row-marching, persistent RK3 propagation for constant x-advection (V = 0),
// sm_100a, fp64.  The production fine kernel for rows of 128 / 256 / 384 / 512 cells.
//
// Operator: the folded constant-velocity WS-RK3 step of fine_fused.cu (integrators.py:126-146
// rk3_step with acoustic_rhs, numba_backend.py:119-128): stage S computes
// s_out = q + beta_S L(s_in) as 7-point x stencils plus narrow y differences (radius 1 for u
// and p, radius 2 for the v damping).  Results equal the reference up to rounding (tests:
// <= 1e-12 relative against the oracle).
//
// Data movement, designed from the previous kernel's ncu profile (fine_march.cu: issue-bound,
// ~110 of ~290 instructions per thread and tick were cp.async address generation, spill
// reloads and the v register rotation):
//
// * A CTA owns whole grid rows of one state and a y-segment of TY rows.  Three warp groups,
//   one per RK stage, march down the segment one row per tick: in tick t stage 1 consumes
//   q row t-6, stage 2 s1 row t-9, stage 3 s2 row t-12, all reading rows finished in an
//   earlier tick, so one CTA barrier per tick.
// * q rows arrive by ONE 5-D TMA copy per row (u, v, p together: box {4, NX/4, 1, 3, 1} of
//   the view {4, NX/4, ny, 3, batch}) issued by one thread two ticks ahead into an 8-slot
//   ring, completion on a per-slot mbarrier.  The copy lands with the 32-byte swizzle, which
//   is exactly the chunk XOR the window loads need (16-byte chunk c at c ^ ((c >> 3) & 1)):
//   the 32-byte per-thread stride of the window loads is bank-conflict free.
// * No ghost columns: the periodic x wrap lives in each thread's window offset table (the
//   first thread's left chunks point at the row's end, the last thread's right chunks at
//   its start), so ring rows are exactly NX doubles and nothing is copied twice.
// * y coupling in registers: a thread consuming row k adds its x-stencil terms to row k and
//   its y-difference terms to rows k-1 and k+1; u and p keep rows k-1..k+1 in 3 fixed slots
//   (row mod 3, the tick loop is unrolled 3x).  v's radius-2 damping keeps only 3 rows plus
//   h = dv2 v(k-1), added when row k+1 is born: no register rotation at all.
// * Persistent: one launch runs every RK3 step of the propagation.  CTAs take work items
//   (step, state, segment) in order from an atomic counter; an item waits on the step
//   counters of its three neighbouring segments (the y halo it reads and the buffer it
//   overwrites), so items never deadlock and there is no wave quantisation between steps.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "pw_internal.h"

namespace pw {
namespace {

// NX columns per CTA; CL CTAs of a thread-block cluster share each grid row (rows of
// NXT = CL NX cells: 1024 and 2048 as 2 and 4 CTAs of 512).  With CL > 1 a ring field row
// carries a 32-double pad: its right halo (the right neighbour's first 4 columns) at
// [NX, NX + 4), its left halo at [NX + 16, NX + 20) -- TMA-loaded for q, stored over DSMEM by
// the neighbour's edge threads for s1 / s2.
// BX columns per thread: 4 (32-byte swizzle, 6-chunk windows) or 8 (64-byte swizzle, 8-chunk
// windows: a third less shared-memory traffic per cell, half the threads; CL = 1 only).
// UNI: the three stage groups run ONE copy of the row code with the stage as a warp-uniform
// run-time value (coefficients in uniform registers), a third of the instruction footprint:
// with BX = 8 the stage-specialised code (72 KB) left the warps waiting on instruction fetch.
template <int NX_, int CL_ = 1, int BX_ = 4, bool UNI_ = (BX_ == 8)>
struct TK {
  static constexpr int NX = NX_, BX = BX_, CL = CL_, NXT = CL * NX;
  static constexpr bool UNI = UNI_;
  static constexpr int NCH = BX / 2 + 4;  // 16-byte chunks of a thread's x window (BX + 8 cells)
  static constexpr int GS = NX / BX;   // threads per stage group
  static constexpr int NT = 3 * GS;
  static constexpr int CH = NX / 2;    // 16-byte chunks per field row
  static constexpr int FS = CL > 1 ? NX + 32 : NX;  // doubles per ring field row
  static constexpr int HR = NX, HL = NX + 16;       // halo offsets in a ring field row (CL > 1)
  static constexpr int SLOT = 3 * FS;  // doubles per ring slot: u, v, p rows
  static constexpr int NQ = 8, N1 = 3, N2 = 3;
  static constexpr size_t RING = sizeof(double) * SLOT * (NQ + N1 + N2);
  static constexpr size_t SMEM = RING + 1024 + 8 * NQ;  // + alignment slack + mbarriers
  // bytes one q row brings: the CTA's 3 x NX cells (+ 3 x 2 halos of 4 cells with CL > 1)
  static constexpr uint32_t ROW_BYTES = (3 * NX + (CL > 1 ? 24 : 0)) * sizeof(double);
  static constexpr int MB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int MB_REGS = 65536 / (NT * (BX == 4 ? 168 : 255));
  static constexpr int MINB = (MB_SMEM < MB_REGS ? MB_SMEM : MB_REGS) < 1 ? 1 : (MB_SMEM < MB_REGS ? MB_SMEM : MB_REGS);
  static_assert(GS % 32 == 0, "stage groups must be whole warps");
  static_assert(BX == 4 || (BX == 8 && CL == 1), "8 columns per thread: one CTA per row only");
  static_assert((FS * 8) % 256 == 0, "ring field rows keep the 256-byte alignment of the 32-byte swizzle");
};

// 16-byte chunk c of a ring field row lands at swz(c): TMA's 32-byte swizzle (address bit 4 ^=
// bit 7) for BX = 4, its 64-byte swizzle (bits 4-5 ^= bits 7-8) for BX = 8.  With 64 bytes per
// lane the bank group of chunk 4 m + r is (m & 1, r ^ ((m >> 1) & 3)): 8 consecutive lanes hit 8
// distinct groups for EVERY window chunk r (the 128-byte swizzle conflicts 2-way on the halo
// chunks: measured, 28 % of the wavefronts).
template <int BX>
__device__ __forceinline__ int swz(int c) {
  return BX == 4 ? c ^ ((c >> 3) & 1) : c ^ ((c >> 3) & 3);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(const uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// one q row (u, v, p of state b, grid row gy) into a ring slot
__device__ __forceinline__ void tma_row(const CUtensorMap* map, double* slot, uint64_t* bar, int gy, int b,
                                        uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(slot)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(0), "r"(gy), "r"(0), "r"(b), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bar_sync() { asm volatile("bar.sync 0;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the same shared-memory location in CTA `rank` of the cluster (generic address)
template <class T>
__device__ __forceinline__ T* peer_smem(T* p, unsigned rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<T*>(out);
}
// one 4-cell tile (16-byte chunks) of the TMA view at (col4, gy, field, b) -> smem
__device__ __forceinline__ void tma_box(const CUtensorMap* map, void* dst, uint64_t* bar, int col4, int gy, int f,
                                        int b) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(col4), "r"(gy), "r"(f), "r"(b), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// A thread's x window (BX + 8 cells, w[1] .. w[BX + 6] are read) as 128-bit chunk loads (the
// compiler narrows the two half-used edge chunks to 64-bit loads, which conflict 2-way at 32
// bytes per lane whatever the swizzle: 14 % of the kernel's shared-memory wavefronts).
// -DPW_K1_SHFL=1 takes the two edge cells from the neighbouring lanes' registers instead (they
// are those lanes' w[BX + 1] and w[6]; 4 SHFL.32 = 4 passes of the pipe against 8; lanes 0 and 31
// load theirs): same values, parity-tested, but measured SLOWER at c2 (59.4 vs 72.8 G/s: the
// shuffles sit between the loads and the first taps, 168 registers and 20 bytes of spills).
#ifndef PW_K1_SHFL
#define PW_K1_SHFL 0
#endif
template <int BX>
__device__ __forceinline__ void ld_window(double (&w)[BX + 8], const double* row, const int* off) {
  constexpr int NCH = BX / 2 + 4;
#if PW_K1_SHFL
#pragma unroll
  for (int j = 1; j < NCH - 1; ++j) {
    const double2 t = *reinterpret_cast<const double2*>(row + off[j]);
    w[2 * j] = t.x;
    w[2 * j + 1] = t.y;
  }
  const int lane = threadIdx.x & 31;
  double lo = __shfl_up_sync(0xffffffffu, w[BX + 1], 1);
  double hi = __shfl_down_sync(0xffffffffu, w[6], 1);
  if (lane == 0) lo = row[off[0] + 1];
  if (lane == 31) hi = row[off[NCH - 1]];
  w[0] = 0.0;
  w[1] = lo;
  w[BX + 6] = hi;
  w[BX + 7] = 0.0;
#else
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const double2 t = *reinterpret_cast<const double2*>(row + off[j]);
    w[2 * j] = t.x;
    w[2 * j + 1] = t.y;
  }
#endif
}
template <int BX>
__device__ __forceinline__ void st4(double* row, const int* off, const double (&v)[BX]) {
#pragma unroll
  for (int j = 0; j < BX / 2; ++j) *reinterpret_cast<double2*>(row + off[j]) = make_double2(v[2 * j], v[2 * j + 1]);
}
template <int BX>
__device__ __forceinline__ void stg4(double* p, const double (&v)[BX]) {
#pragma unroll
  for (int j = 0; j < BX / 2; ++j) *reinterpret_cast<double2*>(p + 2 * j) = make_double2(v[2 * j], v[2 * j + 1]);
}

// One stage thread's registers: u, p rows k-1..k+1 and v rows k-2..k (slot = row mod 3),
// h = dv2 v(k-1) for the birth of v row k+1.
template <int BX>
struct Acc {
  double u[3][BX], p[3][BX], v[3][BX], h[BX];
};

// Where the completed rows go: the next stage's ring (S < 2) or the state in HBM (S = 2).
struct Sink {
  double* ring;     // S < 2: the output ring's slot 0
  unsigned left, right;  // CL > 1: cluster ranks of the CTAs holding the columns left / right
  double* g;        // S = 2: this thread's columns of the segment's first row (u field)
  long long n;      // nx * ny (field stride)
  int TY;
  int npeer;        // last RK3 step of a fused all-gather: also store into npeer peer buffers
  const long long* peer_delta;  // (bytes from out, FusedParams::peer_delta), else npeer = 0
};

// stage 3's 4 cells of one output row: HBM, and (PEERS: fused slice all-gather,
// pw_prop_apply_to_peers) the same bytes into each peer's buffer over NVLink, from the
// registers that hold them.  A separate instantiation: the peer loop in the plain kernel
// cost 11 % (64.6 vs 72.4 G/s at c2).
template <bool PEERS, int BX>
__device__ __forceinline__ void st_out(const Sink& o, double* p, const double (&v)[BX]) {
  stg4<BX>(p, v);
  if constexpr (PEERS)
  for (int i = 0; i < o.npeer; ++i) {
    double* q = reinterpret_cast<double*>(reinterpret_cast<char*>(p) + o.peer_delta[i]);
#pragma unroll
    for (int j = 0; j < BX / 2; ++j)
      __stcg(reinterpret_cast<double2*>(q + 2 * j), make_double2(v[2 * j], v[2 * j + 1]));
  }
}

__device__ __forceinline__ double2 lds2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}
// this thread's 4 cells of a ring row (two 16-byte chunks, always 128-bit loads)
template <int BX>
__device__ __forceinline__ void ld_own(double (&b)[BX], const double* row, const int* off) {
#pragma unroll
  for (int j = 0; j < BX / 2; ++j) {
    const double2 x = lds2(row + off[j]);
    b[2 * j] = x.x;
    b[2 * j + 1] = x.y;
  }
}

// x stencil of one field row into acc (7 taps, cen / e2m / e2p: the centre and -2 / +2
// coefficients, which carry the field's own centre and x-damping terms); d1 = w_1 - w_{-1},
// the centred difference the other fields need (pressure gradient, divergence, mixed damping).
// (Pairing the antisymmetric advection taps, c_j (w_j - w_{-j}), saves 3 of 38 DP ops per cell
// and stage but measured slower: 71.1 vs 72.7 G cell-updates/s at c2, more live registers.)
template <int BX>
__device__ __forceinline__ void xstencil(double (&acc)[BX], double (&d1)[BX], const double (&w)[BX + 8], double cen,
                                         double e2m, double e2p, const StageCoef& C) {
#pragma unroll
  for (int c = 0; c < BX; ++c) {
    d1[c] = w[c + 5] - w[c + 3];
    acc[c] = fma(C.cxp[0], w[c + 1], acc[c]);
    acc[c] = fma(e2m, w[c + 2], acc[c]);
    acc[c] = fma(C.cxp[2], w[c + 3], acc[c]);
    acc[c] = fma(cen, w[c + 4], acc[c]);
    acc[c] = fma(C.cxp[4], w[c + 5], acc[c]);
    acc[c] = fma(e2p, w[c + 6], acc[c]);
    acc[c] = fma(C.cxp[6], w[c + 7], acc[c]);
  }
}

// Consume input row k (ring slot `in`; q row k+1 at `qb` for the births when S > 0), store
// the completed rows: u, p of row k-1 and v of row k-2.  PH = k mod 3 (compile time).
// CL > 1, S < 2: the edge threads also store their outer 4 cells into the neighbouring CTAs'
// halos of the same ring row (DSMEM): g = 0's first cells are the left neighbour's right
// halo, the last thread's last cells the right neighbour's left halo
template <int NX, int FS, int CL, int BX>
__device__ __forceinline__ void st_ring(double* row, const int* woff2, const double (&v)[BX], int g, const Sink& o) {
  st4<BX>(row, woff2, v);
  if constexpr (CL > 1) {
    if (g == 0) {
      double2* h = reinterpret_cast<double2*>(peer_smem(row + NX, o.left));
      h[0] = make_double2(v[0], v[1]);
      h[1] = make_double2(v[2], v[3]);
    } else if (g == NX / 4 - 1) {
      double2* h = reinterpret_cast<double2*>(peer_smem(row + NX + 16, o.right));
      h[0] = make_double2(v[0], v[1]);
      h[1] = make_double2(v[2], v[3]);
    }
  }
}

// S_ >= 0: the stage at compile time; S_ < 0: the stage is the warp-uniform run-time `srt`
// (one copy of the code for the three stage groups; stage 1's missing q base is a zero row in
// registers, so only the sign of a zero can differ from the specialised code)
template <int NX, int S_, int PH, bool PEERS, int FS = NX, int CL = 1, int BX = 4>
__device__ __forceinline__ void row_step(Acc<BX>& A, const double* in, const double* qb, const int* woff,
                                         const StageCoef& C, const Sink& o, int k, int g = 0, int srt = 0) {
  constexpr int NXT = NX * CL;
  constexpr bool RT = S_ < 0;
  const int S = RT ? srt : S_;
  constexpr int NCH = BX / 2 + 4;
  constexpr int U0 = (PH + 2) % 3, U1 = PH, U2 = (PH + 1) % 3;  // u, p: rows k-1, k, k+1
  constexpr int V0 = (PH + 1) % 3, V1 = (PH + 2) % 3, V2 = PH;  // v: rows k-2 (-> k+1), k-1, k
  double w[BX + 8], d1[BX];
  // ---- v row k: x stencil of row k; completes v(k-2); births v(k+1); u_y-mixed / p_y terms
  ld_window<BX>(w, in + FS, woff);
  // v: cxv equals cxp off the centre; the +-2 taps are plain advection
  xstencil<BX>(A.v[V2], d1, w, C.cxv[3], C.cxp[1], C.cxp[5], C);
#pragma unroll
  for (int c = 0; c < BX; ++c) A.v[V0][c] = fma(C.dv2, w[c + 4], A.v[V0][c]);
  if (S < 2) {
    st_ring<NX, FS, CL, BX>(o.ring + ((PH + 1) % 3) * (3 * FS) + FS, woff + 2, A.v[V0], g, o);
  } else {
    if (k - 2 >= 0 && k - 2 < o.TY) st_out<PEERS, BX>(o, o.g + o.n + (long long)(k - 2) * NXT, A.v[V0]);
  }
  {
    double b[BX];
    if (S > 0) ld_own<BX>(b, qb + FS, woff + 2);
    else if constexpr (RT) {
#pragma unroll
      for (int c = 0; c < BX; ++c) b[c] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < BX; ++c) {
      A.v[V0][c] = (RT || S > 0) ? b[c] + A.h[c] : A.h[c];  // v(k+1) = q + dv2 v(k-1)
      A.h[c] = C.dv2 * w[c + 4];
    }
  }
  {
    double bu[BX], bp[BX];
    if (S > 0) {
      ld_own<BX>(bu, qb, woff + 2);
      ld_own<BX>(bp, qb + 2 * FS, woff + 2);
    } else if constexpr (RT) {
#pragma unroll
      for (int c = 0; c < BX; ++c) bu[c] = bp[c] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < BX; ++c) {
      // mixed damping of u (cuv v_x) into rows k-1 (+) and k+1 (-); p_y of p into p(k-1), p(k+1)
      A.u[U0][c] = fma(C.cuv, d1[c], A.u[U0][c]);
      A.u[U2][c] = (RT || S > 0) ? fma(-C.cuv, d1[c], bu[c]) : -C.cuv * d1[c];
      A.p[U0][c] = fma(C.pv, w[c + 4], A.p[U0][c]);
      A.p[U2][c] = (RT || S > 0) ? fma(-C.pv, w[c + 4], bp[c]) : -C.pv * w[c + 4];
    }
  }
  if (S < 2) {
    double* r = o.ring + ((PH + 2) % 3) * (3 * FS);
    st_ring<NX, FS, CL, BX>(r, woff + 2, A.u[U0], g, o);
    st_ring<NX, FS, CL, BX>(r + 2 * FS, woff + 2, A.p[U0], g, o);
  } else {
    if (k - 1 >= 0 && k - 1 < o.TY) {
      double* gp = o.g + (long long)(k - 1) * NXT;
      st_out<PEERS, BX>(o, gp, A.u[U0]);
      st_out<PEERS, BX>(o, gp + 2 * o.n, A.p[U0]);
    }
  }
  // ---- u row k: x stencil (advection + the symmetric x damping at +-2 and the centre);
  //      u_x for p(k) and the mixed damping of v(k-1), v(k+1)
  double t2[BX];
  ld_window<BX>(w, in, woff);
  xstencil<BX>(A.u[U1], d1, w, C.cxu[3], C.cxu[1], C.cxu[5], C);
#pragma unroll
  for (int c = 0; c < BX; ++c) {
    A.p[U1][c] = fma(C.pu, d1[c], A.p[U1][c]);
    t2[c] = C.cvu * d1[c];
  }
  // ---- p row k: x stencil; p_x for u(k), p_y for v(k-1), v(k+1)
  ld_window<BX>(w, in + 2 * FS, woff);
  xstencil<BX>(A.p[U1], d1, w, C.cxp[3], C.cxp[1], C.cxp[5], C);
#pragma unroll
  for (int c = 0; c < BX; ++c) {
    A.u[U1][c] = fma(C.pu, d1[c], A.u[U1][c]);  // pgx == pu
    t2[c] = fma(C.pv, w[c + 4], t2[c]);         // pgy == pv
    A.v[V1][c] += t2[c];
    A.v[V0][c] -= t2[c];
  }
}

struct Item {
  int y0, TY, b;
  int col4;      // CL > 1: this CTA's first column / 4 in the cluster's row
  uint32_t seq;  // q rows this CTA issued before the item (ring slot / mbarrier phase base)
  const CUtensorMap* map;
  const CUtensorMap* hmap;  // CL > 1: the 4-cell halo view of the same buffer
};

// q ring slot and mbarrier parity of segment row r (r >= -6)
__device__ __forceinline__ uint32_t qslot(uint32_t seq, int r) { return (seq + (uint32_t)(r + 6)) & 7u; }
__device__ __forceinline__ uint32_t qpar(uint32_t seq, int r) { return ((seq + (uint32_t)(r + 6)) >> 3) & 1u; }

template <class K>
__device__ __forceinline__ void issue(double* ring, uint64_t* full, const Item& it, int ny, int r) {
  int gy = it.y0 + r;
  gy += (gy < 0) ? ny : 0;
  gy -= (gy >= ny) ? ny : 0;
  const uint32_t s = qslot(it.seq, r);
  if constexpr (K::CL == 1) {
    tma_row(it.map, ring + (size_t)s * K::SLOT, full + s, gy, it.b, K::ROW_BYTES);
  } else {  // per field: the CTA's NX cells, and the 4-cell halos on either side (periodic)
    double* slot = ring + (size_t)s * K::SLOT;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)),
                 "r"(K::ROW_BYTES)
                 : "memory");
    constexpr int C4 = K::NXT / 4;  // 4-cell columns of the whole row
    const int lc = it.col4 == 0 ? C4 - 1 : it.col4 - 1;
    const int rc = it.col4 + K::NX / 4 == C4 ? 0 : it.col4 + K::NX / 4;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double* row = slot + f * K::FS;
      tma_box(it.map, row, full + s, it.col4, gy, f, it.b);
      tma_box(it.hmap, row + K::HR, full + s, rc, gy, f, it.b);
      tma_box(it.hmap, row + K::HL, full + s, lc, gy, f, it.b);
    }
  }
}

// One tick: the CTA barrier, the q row two ticks ahead, then stage S's row k = t - lag.
template <class K, int I, bool PEERS>
__device__ __forceinline__ void tick(Acc<K::BX>& A, double* ring, uint64_t* full, const Item& it, const FusedParams& P,
                                     int S, int t, const int* woff, const Sink& o, bool producer, int g) {
  constexpr int NX = K::NX;
  if constexpr (K::CL > 1) cluster_sync();  // the neighbours' halo stores of the last tick
  else bar_sync();
  if (producer && t - 4 <= it.TY + 5) issue<K>(ring, full, it, P.ny, t - 4);
  double* q = ring;
  double* r1 = ring + K::NQ * K::SLOT;
  double* r2 = r1 + K::N1 * K::SLOT;
  // k = t - lag with lag in {6, 9, 12}: k mod 3 = t mod 3 = I
  if constexpr (K::UNI) {  // one copy of the row code, the stage a warp-uniform value
    const int k = t - 6 - 3 * S;
    if (k < 2 * S - 6 || k > it.TY + 5 - 2 * S) return;
    const double* in;
    const double* qb = nullptr;
    if (S == 0) {
      const uint32_t s = qslot(it.seq, k);
      mbar_wait(full + s, qpar(it.seq, k));
      in = q + (size_t)s * K::SLOT;
    } else {
      in = (S == 1 ? r1 : r2) + (I * K::SLOT);
      qb = q + (size_t)qslot(it.seq, k + 1) * K::SLOT;
    }
    row_step<NX, -1, I, PEERS, K::FS, K::CL, K::BX>(A, in, qb, woff, P.st[S], o, k, g, S);
  } else if (S == 0) {
    const int k = t - 6;
    if (k > it.TY + 5) return;
    const uint32_t s = qslot(it.seq, k);
    mbar_wait(full + s, qpar(it.seq, k));
    row_step<NX, 0, I, PEERS, K::FS, K::CL, K::BX>(A, q + (size_t)s * K::SLOT, nullptr, woff, P.st[0], o, k, g);
  } else if (S == 1) {
    const int k = t - 9;
    if (k < -4 || k > it.TY + 3) return;
    const double* qb = q + (size_t)qslot(it.seq, k + 1) * K::SLOT;
    row_step<NX, 1, I, PEERS, K::FS, K::CL, K::BX>(A, r1 + (I * K::SLOT), qb, woff, P.st[1], o, k, g);
  } else {
    const int k = t - 12;
    if (k < -2 || k > it.TY + 1) return;
    const double* qb = q + (size_t)qslot(it.seq, k + 1) * K::SLOT;
    row_step<NX, 2, I, PEERS, K::FS, K::CL, K::BX>(A, r2 + (I * K::SLOT), qb, woff, P.st[2], o, k, g);
  }
}

template <class K, bool PEERS>
__global__ void __launch_bounds__(K::NT, K::MINB) rk3_mtma_kernel(
    const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_out,
    const __grid_constant__ CUtensorMap map_tmp, const __grid_constant__ CUtensorMap hmap_in,
    const __grid_constant__ CUtensorMap hmap_out, const __grid_constant__ CUtensorMap hmap_tmp, double* out,
    double* tmp, long long ld_out, long long ld_tmp, const __grid_constant__ FusedParams P, int nseg, int batch,
    int nsteps, int* sync) {
  constexpr int NX = K::NX, CL = K::CL;
  // CL > 1: a cluster of CL CTAs marches each row, this CTA owns columns [crank NX, +NX)
  const unsigned crank = CL > 1 ? cluster_rank() : 0u;
  extern __shared__ unsigned char smraw[];
  // 1024-byte aligned ring (offset arithmetic on smraw keeps the shared address space visible)
  double* ring = reinterpret_cast<double*>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)K::SLOT * (K::NQ + K::N1 + K::N2));
  __shared__ int s_item;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < K::NQ; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // warp-uniform stage index (through a shuffle, so the compiler knows it)
  const int S = __shfl_sync(0xffffffffu, tid / K::GS, 0);
  const int g = tid - S * K::GS;
  // window chunk offsets: cols [4g - 4, 4g + 8) as 6 chunks; one CTA per row: wrapped
  // periodically; CL > 1: the outer chunks of the edge threads are the row's halos
  int woff[K::NCH];
#pragma unroll
  for (int j = 0; j < K::NCH; ++j) {
    int c = (K::BX / 2) * g - 2 + j;
    if constexpr (CL == 1) {
      c += (c < 0) ? K::CH : 0;
      c -= (c >= K::CH) ? K::CH : 0;
      woff[j] = 2 * swz<K::BX>(c);
    } else {
      woff[j] = c < 0 ? K::HL + 2 * (c + 2) : (c >= K::CH ? K::HR + 2 * (c - K::CH) : 2 * swz<K::BX>(c));
    }
  }
  const bool producer = (tid == 0);
  const int ny = P.ny;
  const long long n = (long long)K::NXT * ny;
  const int per_step = nseg * batch;
  const long long total = (long long)per_step * nsteps;
  int* done = sync + 1;
  uint32_t seq = 0;
  double* ring_out = S == 0 ? ring + K::NQ * K::SLOT : ring + (K::NQ + K::N1) * K::SLOT;
  for (;;) {
    if constexpr (CL == 1) {
      __syncthreads();  // s_item of the previous item is no longer read; rings are free
      if (tid == 0) s_item = atomicAdd(sync, 1);
      __syncthreads();
    } else {  // the cluster takes an item together: rank 0 draws it, every CTA gets a copy
      cluster_sync();
      if (tid == 0 && crank == 0) {
        const int v = atomicAdd(sync, 1);
        for (int r = 0; r < CL; ++r) *peer_smem(&s_item, (unsigned)r) = v;
      }
      cluster_sync();
    }
    const int item = s_item;
    if (item >= total) break;
    const int s = item / per_step;
    const int rem = item - s * per_step;
    const int b = rem / nseg, j = rem - b * nseg;
    if (s > 0 && tid < 3 && crank == 0) {  // the three neighbouring segments finished step s-1
      int jj = j + tid - 1;
      jj += (jj < 0) ? nseg : 0;
      jj -= (jj >= nseg) ? nseg : 0;
      const int* f = done + b * nseg + jj;
      long long spins = 0;
      while (ld_acquire(f) < s) {
        __nanosleep(64);
        if (++spins > (1LL << 26)) __trap();  // a broken dependency fails, never hangs
      }
    }
    if constexpr (CL == 1) __syncthreads();
    else cluster_sync();
    // the neighbours' generic-proxy stores (seen through the acquire) before this CTA's TMA reads
    if (producer) asm volatile("fence.proxy.async.global;" ::: "memory");
    // ping-pong so that the last step lands in out
    const bool to_out = ((nsteps - 1 - s) % 2) == 0;
    Item it;
    it.y0 = (int)((long long)j * ny / nseg);
    it.TY = (int)((long long)(j + 1) * ny / nseg) - it.y0;
    it.b = b;
    it.seq = seq;
    it.map = s == 0 ? &map_in : (to_out ? &map_tmp : &map_out);
    it.hmap = s == 0 ? &hmap_in : (to_out ? &hmap_tmp : &hmap_out);
    it.col4 = (int)crank * (NX / 4);
    Sink o;
    o.left = (crank + CL - 1) % CL;
    o.right = (crank + 1) % CL;
    o.ring = ring_out;
    o.n = n;
    o.TY = it.TY;
    if constexpr (PEERS) {
      o.npeer = (s == nsteps - 1) ? P.npeer : 0;  // peers get the final state only
      o.peer_delta = P.peer_delta;
    }
    o.g = (to_out ? out + (long long)b * ld_out : tmp + (long long)b * ld_tmp) + (long long)it.y0 * K::NXT +
          (long long)crank * NX + K::BX * g;
    if (producer) {  // prologue: q rows -6 and -5 (stage 1's ticks 0 and 1)
      issue<K>(ring, full, it, ny, -6);
      issue<K>(ring, full, it, ny, -5);
    }
    Acc<K::BX> A;
#pragma unroll
    for (int c = 0; c < K::BX; ++c) {
#pragma unroll
      for (int r = 0; r < 3; ++r) A.u[r][c] = A.p[r][c] = A.v[r][c] = 0.0;
      A.h[c] = 0.0;
    }
    // tick count rounded up to the unroll (equal barrier counts for every warp)
    const int nt = (it.TY + 14 + 2) / 3 * 3;
    for (int t = 0; t < nt; t += 3) {
      tick<K, 0, PEERS>(A, ring, full, it, P, S, t, woff, o, producer, g);
      tick<K, 1, PEERS>(A, ring, full, it, P, S, t + 1, woff, o, producer, g);
      tick<K, 2, PEERS>(A, ring, full, it, P, S, t + 2, woff, o, producer, g);
    }
    seq += (uint32_t)(it.TY + 12);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // stores before later TMA reads
    __threadfence();
    if constexpr (CL == 1) __syncthreads();
    else cluster_sync();  // every CTA of the cluster has stored its columns
    if (tid == 0 && crank == 0) st_release(done + b * nseg + j, s + 1);
  }
  if constexpr (CL > 1) cluster_sync();  // no CTA leaves while a neighbour may still store its halo
}

// ---------------------------------------------------------------- host side
int env_int2(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  PW_CHECK(fn != nullptr, PW_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
  return fn;
}

// view {4, nx/4, ny, 3, batch} of a batch of states (ld doubles apart); box = {4, bx4, 1, bf, 1}
// (one grid row of bx4 4-cell chunks of bf fields), 32-byte swizzle -- or none for the halo
// boxes, which the edge threads read unswizzled
// `inner` cells per innermost box row: 4 with the 32-byte swizzle (BX = 4), 8 with the 64-byte
// swizzle (BX = 8); bx4 counts inner-sized column groups
CUtensorMap row_map(const double* base, int nx, int ny, long long ld, int batch, int bx4 = 0, int bf = 3,
                    bool swizzle = true, int inner = 4) {
  CUtensorMap m;
  const cuuint64_t dims[5] = {(cuuint64_t)inner, (cuuint64_t)(nx / inner), (cuuint64_t)ny, 3, (cuuint64_t)batch};
  const cuuint64_t strides[4] = {(cuuint64_t)inner * 8, (cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8,
                                 (cuuint64_t)ld * 8};
  const cuuint32_t box[5] = {(cuuint32_t)inner, (cuuint32_t)(bx4 > 0 ? bx4 : nx / inner), 1, (cuuint32_t)bf, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 !swizzle ? CU_TENSOR_MAP_SWIZZLE_NONE
                                          : (inner == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PW_CHECK(r == CUDA_SUCCESS, PW_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}


template <class K>
void launch_cfg(Ctx& c, const FusedParams& fp, const double* in, double* out, double* tmp, int batch, int nsteps,
                long long d, int* sync) {
  auto kern = fp.npeer > 0 ? rk3_mtma_kernel<K, true> : rk3_mtma_kernel<K, false>;
  const int per_sm = kernel_setup(c, kern, K::NT, K::SMEM);
  // item slots: CTAs, or clusters of CL CTAs (one CTA per SM at NX = 512)
  const long long slots = std::max<long long>(1, (long long)(c.num_sms > 0 ? c.num_sms : 148) * per_sm / K::CL);
  // segments per state: ticks per item (TY + 14) x max(1, items / CTA slots), clamped so
  // every segment has >= 16 rows (the 6-row halo of the neighbour dependency, and the
  // sync buffer's ny / 16 + 1 counters per state)
  int nseg = env_int2("PW_MARCH_NSEG", 0);
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
  }
  nseg = std::max(1, std::min(nseg, fp.ny / 16));
  // CL = 1: one box per row (3 fields); CL > 1: per field, the CTA's NX columns, plus
  // 4-cell halo boxes (no swizzle)
  constexpr int inner = K::BX == 4 ? 4 : 8;
  const int bx4 = K::NX / inner, bf = K::CL == 1 ? 3 : 1;
  const CUtensorMap m_in = row_map(in, fp.nx, fp.ny, fp.ld_in, batch, bx4, bf, true, inner);
  const CUtensorMap m_out = row_map(out, fp.nx, fp.ny, fp.ld_out, batch, bx4, bf, true, inner);
  const CUtensorMap m_tmp = row_map(tmp, fp.nx, fp.ny, d, batch, bx4, bf, true, inner);
  const CUtensorMap h_in = K::CL > 1 ? row_map(in, fp.nx, fp.ny, fp.ld_in, batch, 1, 1, false) : m_in;
  const CUtensorMap h_out = K::CL > 1 ? row_map(out, fp.nx, fp.ny, fp.ld_out, batch, 1, 1, false) : m_out;
  const CUtensorMap h_tmp = K::CL > 1 ? row_map(tmp, fp.nx, fp.ny, d, batch, 1, 1, false) : m_tmp;
  const long long items = (long long)batch * nseg * nsteps;
  const int grid = (int)std::min<long long>(slots, items) * K::CL;
  PW_CUDA(cudaMemsetAsync(sync, 0, sizeof(int) * (1 + (size_t)batch * nseg), c.stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(K::NT);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = K::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = K::CL > 1 ? 1 : 0;
  PW_CUDA(cudaLaunchKernelEx(&cfg, kern, m_in, m_out, m_tmp, h_in, h_out, h_tmp, out, tmp, fp.ld_out, d, fp, nseg,
                             batch, nsteps, sync));
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

}  // namespace

bool mtma_enabled() { return env_int2("PW_MARCH_V2", 1) != 0; }

bool mtma_supported(int nx, int ny, long long ld_in, long long ld_out, const void* in, const void* out,
                    const void* tmp) {
  const bool cluster = (nx == 1024 || nx == 2048) && env_int2("PW_MARCH_CLUSTER2", 1) != 0;
  if (!(nx == 128 || nx == 256 || nx == 384 || nx == 512 || cluster)) return false;
  if (ny < 32) return false;
  if ((ld_in & 1) || (ld_out & 1)) return false;
  return (((uintptr_t)in | (uintptr_t)out | (uintptr_t)tmp) & 15) == 0;
}

void launch_rk3_mtma(Ctx& c, const FusedParams& fp, const double* in, double* out, double* tmp, int batch,
                     int nsteps, long long d, int* sync) {
  // PW_MARCH_BX=8: 8 columns per thread (128-byte swizzle); nx = 128 has too few columns for it
  if (env_int2("PW_MARCH_BX", 4) == 8) switch (fp.nx) {
    case 256: return launch_cfg<TK<256, 1, 8>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 512: return launch_cfg<TK<512, 1, 8>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    default: break;
  }
  // PW_MARCH_UNI=1: 4 columns per thread with the one-copy row code (A/B runs)
  if (env_int2("PW_MARCH_UNI", 0) == 1) switch (fp.nx) {
    case 256: return launch_cfg<TK<256, 1, 4, true>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 512: return launch_cfg<TK<512, 1, 4, true>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    default: break;
  }
  switch (fp.nx) {
    case 128: return launch_cfg<TK<128>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 256: return launch_cfg<TK<256>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 384: return launch_cfg<TK<384>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 512: return launch_cfg<TK<512>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    // wider rows: clusters of 512-column CTAs (halos by TMA for q, over DSMEM for s1 / s2)
    case 1024: return launch_cfg<TK<512, 2>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    case 2048: return launch_cfg<TK<512, 4>>(c, fp, in, out, tmp, batch, nsteps, d, sync);
    default: throw Error{PW_ERR_VALUE, "TMA row march needs nx in {128, 256, 384, 512, 1024, 2048}"};
  }
}

}  // namespace pw
