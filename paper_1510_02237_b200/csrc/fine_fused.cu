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
// Each stage is folded into  s_out = q + beta*f(s_in)  with the stage factor
// beta (h/3, h/2, h) and the expanded divergence damping pre-multiplied into
// the coefficients (StageCoef): ~37 DP ops per cell and stage instead of the
// reference form's ~106.  Results differ from the reference only by
// rounding (tests: <= 1e-12 relative).
//
// Data movement (roofline unit: 48 B per cell-update = read + write (u,v,p)
// once).  A CTA owns an x-strip of TX output columns and a y-segment of TY
// rows.  It streams q rows top-to-bottom through shared-memory rings
// (16-byte cp.async, one tick ahead) and runs the three RK stages as a
// software pipeline: in tick t stage 1 produces rows of tick t, stage 2 the
// rows stage 1 finished in tick t-1, stage 3 those stage 2 finished in t-1.
// The three stages are therefore independent inside a tick: one barrier per
// tick, and every thread owns exactly one (stage, column group, row block)
// item, executed by one uniform code path (no divergence, no idle threads).
// Halos are only in x (E = 4 columns per stage) plus a 6*RY-row warm-up per
// segment; s1 and s2 never leave shared memory.
//
// On-chip traffic is what limits this kernel (shared memory moves ~128 B/clk
// per SM, ~5.5x HBM), so each item is a BX x BY register block loaded as
// aligned 16-byte chunks, and ring rows are XOR-swizzled per chunk so the
// 32-byte per-thread stride of those chunks is bank-conflict free.
#include <cuda_pipeline.h>

#include "pw_internal.h"

namespace pw {
namespace {

constexpr int E = 4;  // region growth per stage: >= the 3-cell x radius, keeps 16-B alignment

__device__ __forceinline__ int wrapi(int k, int n) {
  k %= n;
  return k < 0 ? k + n : k;
}

constexpr int pad4(int w) { return (w + 3) / 4 * 4; }  // whole chunk pairs per row

template <int TX_, int TY_, int BX_, int BY_, int NRB_, int RY_, bool VADV_>
struct Cfg {
  static constexpr int TX = TX_, TY = TY_, BX = BX_, BY = BY_, NRB = NRB_, RY = RY_;
  static constexpr bool VADV = VADV_;
  static constexpr int R = BY * NRB;            // rows per tick and stage
  static constexpr int WQ = pad4(TX + 6 * E);   // q ring:  logical cols [-3E, TX+3E)
  static constexpr int W1 = pad4(TX + 4 * E);   // s1 ring: logical cols [-2E, TX+2E)
  static constexpr int W2 = pad4(TX + 2 * E);   // s2 ring: logical cols [-E,  TX+E)
  static constexpr int G1 = (TX + 4 * E) / BX, G2 = (TX + 2 * E) / BX, G3 = TX / BX;
  static constexpr int NT = (G1 + G2 + G3) * NRB;
  static constexpr int NQ = 4 * R + 3 * RY;     // q rows live across the 3-tick pipeline + prefetch
  static constexpr int NS = 2 * R + 2 * RY;
  static constexpr int NTICK = (TY + 6 * RY + R - 1) / R + 2;
  static constexpr size_t SMEM =
      sizeof(double) * 3 * ((size_t)NQ * WQ + (size_t)NS * W1 + (size_t)NS * W2);
  // CTAs per SM: shared memory (227 KB) and a ~200-register budget per thread
  static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int MINB_REGS = 65536 / (NT * 200);
  static constexpr int MINB = (MINB_SMEM < MINB_REGS ? MINB_SMEM : MINB_REGS) < 1
                                  ? 1 : (MINB_SMEM < MINB_REGS ? MINB_SMEM : MINB_REGS);
  static_assert(TX % BX == 0 && (2 * E) % BX == 0, "BX must divide TX and 2E");
  static_assert(BX % 2 == 0 && BY >= 1, "BX must be even (16-byte chunks)");
};

// Bank-conflict avoidance.  Work items are interleaved so that a quarter-warp
// (8 threads of one 16-byte shared access) holds 4 column groups of one row
// block and 4 of the next (row blocks are BY = 2 rows apart).  Same-row
// threads touch chunks 2g+m -> 4 distinct even/odd bank quads; the other row
// block lands on the complementary quads because every ring slot s stores its
// 16-byte chunks pair-swapped (chunk j at j ^ flip(s), flip(s) = (s >> 1) & 1).
__device__ __forceinline__ int slot_flip(int s) { return (s >> 1) & 1; }

// A ring row seen from one thread: chunk k relative to its column group lives at
// (k even ? e : o) + 2k  (e/o absorb the slot's pair swap)
struct RowP {
  const double* e;
  const double* o;
};
__device__ __forceinline__ RowP rowp_of(const double* slot_base, int s, int c) {
  // physical chunk = (c/2 + k) ^ flip: +2 doubles for even absolute chunks, -2 for odd
  // ones; a group whose first chunk is odd (BX = 2) swaps the roles of e and o
  const int f = ((c >> 1) & 1) ? -slot_flip(s) : slot_flip(s);
  return RowP{slot_base + c + 2 * f, slot_base + c - 2 * f};
}

// dst[2i, 2i+1] = chunk k0 + i of the row (field offset foff, a multiple of 16 doubles)
template <int N>
__device__ __forceinline__ void ldrow(double (&dst)[N], const RowP& r, int foff, int k0) {
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const int k = k0 + i;
    const double* p = ((k & 1) ? r.o : r.e) + foff + 2 * k;
    const double2 t = *reinterpret_cast<const double2*>(p);
    dst[2 * i] = t.x;
    dst[2 * i + 1] = t.y;
  }
}

struct Ring {
  const double* base;
  int n;      // slots
  int pitch;  // doubles per slot (3 fields)
  int w;      // doubles per field row
};

// One work item: output block rows [rel0, rel0+BY) x logical cols [c, c+BX) of
// the stage region; input ring `in` holds the previous stage (q for stage 1),
// whose column c+E.. corresponds to output col c -- the x-window of output col
// c starts at input col c (x offset -4).  q base at q-ring col c + S*E.
template <class K>
__device__ __forceinline__ void stage_item(const Ring in, const Ring qr, int S, int s_q, int s_in, int c,
                                           const StageCoef& C, double (&au)[K::BY][K::BX],
                                           double (&av)[K::BY][K::BX], double (&ap)[K::BY][K::BX]) {
  constexpr int BX = K::BX, BY = K::BY;
  constexpr int WW = BX + 8;  // full window  x in [-4, BX+4)
  constexpr int WH = BX + 4;  // halo window  x in [-2, BX+2)
  // stage base q (q-ring col c + S*E = chunk S*E/2 relative to the group); stage 1 folds
  // it into the stencil centre instead (its input ring is q itself)
  double qb[3][BY][BX];
  if (S != 1) {
    int s = s_q;
#pragma unroll
    for (int r = 0; r < BY; ++r) {
      const RowP q = rowp_of(qr.base + (size_t)s * qr.pitch, s, c);
      s = (s + 1 == qr.n) ? 0 : s + 1;
      ldrow(qb[0][r], q, 0, S * E / 2);
      ldrow(qb[1][r], q, qr.w, S * E / 2);
      ldrow(qb[2][r], q, 2 * qr.w, S * E / 2);
    }
  }
  // row pointers of rel0 - RY .. rel0 + BY - 1 + RY, computed once (rel >= 0 always)
  constexpr int NR = BY + 2 * K::RY;
  RowP rows[NR];
  {
    int s = s_in;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      rows[k] = rowp_of(in.base + (size_t)s * in.pitch, s, c);
      s = (s + 1 == in.n) ? 0 : s + 1;
    }
  }
  auto rowp = [&](int dy) -> const RowP& { return rows[dy + K::RY]; };
  // accumulators start from their first product (no zero fill): av in the v x-stencil,
  // au in the u x-stencil, ap from the u difference of the pressure divergence
  const int W = in.w;
  // a[r][X] = v(r+1) - v(r-1), b[r][X] = u(r+1) - u(r-1) at x = X-1 in [-1, BX]
  double A[BY][BX + 2], B[BY][BX + 2];
  // ---- v rows -2 .. BY+1: x-advection on rows 0..BY-1, halo windows of rows -1..BY
  {
    double vh[BY + 2][WH];  // rows -1..BY on x in [-2, BX+2)
    ldrow(vh[0], rowp(-1), W, 2 / 2);
    ldrow(vh[BY + 1], rowp(BY), W, 2 / 2);
#pragma unroll
    for (int r = 0; r < BY; ++r) {
      double w[WW];
      ldrow(w, rowp(r), W, 0);
      // tap-major order: BX independent FMA chains per tap (same per-cell summation order)
#pragma unroll
      for (int x = 0; x < BX; ++x) av[r][x] = C.cxv[0] * w[x + 1];
#pragma unroll
      for (int k = 1; k < 7; ++k)
#pragma unroll
        for (int x = 0; x < BX; ++x) av[r][x] = fma(C.cxv[k], w[x + 1 + k], av[r][x]);
#pragma unroll
      for (int k = 0; k < WH; ++k) vh[r + 1][k] = w[k + 2];
    }
    double vm2[BX], vp2[BX];
    ldrow(vm2, rowp(-2), W, 4 / 2);
    ldrow(vp2, rowp(BY + 1), W, 4 / 2);
#pragma unroll
    for (int r = 0; r < BY; ++r) {
#pragma unroll
      for (int X = 0; X < BX + 2; ++X) A[r][X] = vh[r + 2][X + 1] - vh[r][X + 1];
#pragma unroll
      for (int x = 0; x < BX; ++x) {
        const double up = (r + 2 <= BY) ? vh[r + 3][x + 2] : vp2[x];
        const double dn = (r - 2 >= -1) ? vh[r - 1][x + 2] : vm2[x];
        av[r][x] = fma(C.dv2, up + dn, av[r][x]);
      }
    }
  }
  // ---- u rows -1 .. BY
  {
    double uh[BY + 2][WH];
    ldrow(uh[0], rowp(-1), 0, 2 / 2);
    ldrow(uh[BY + 1], rowp(BY), 0, 2 / 2);
#pragma unroll
    for (int r = 0; r < BY; ++r) {
      double w[WW];
      ldrow(w, rowp(r), 0, 0);
#pragma unroll
      for (int x = 0; x < BX; ++x) {
        au[r][x] = C.cxu[0] * w[x + 1];
        ap[r][x] = C.pu * (w[x + 5] - w[x + 3]);
      }
#pragma unroll
      for (int k = 1; k < 7; ++k)
#pragma unroll
        for (int x = 0; x < BX; ++x) au[r][x] = fma(C.cxu[k], w[x + 1 + k], au[r][x]);
#pragma unroll
      for (int k = 0; k < WH; ++k) uh[r + 1][k] = w[k + 2];
    }
#pragma unroll
    for (int r = 0; r < BY; ++r)
#pragma unroll
      for (int X = 0; X < BX + 2; ++X) B[r][X] = uh[r + 2][X + 1] - uh[r][X + 1];
  }
  // ---- p rows -1 .. BY
  {
    double plo[BX], phi[BX];
    ldrow(plo, rowp(-1), 2 * W, 4 / 2);
    ldrow(phi, rowp(BY), 2 * W, 4 / 2);
    double pc[BY][BX];
#pragma unroll
    for (int r = 0; r < BY; ++r) {
      double w[WW];
      ldrow(w, rowp(r), 2 * W, 0);
#pragma unroll
      for (int k = 0; k < 7; ++k)
#pragma unroll
        for (int x = 0; x < BX; ++x) ap[r][x] = fma(C.cxp[k], w[x + 1 + k], ap[r][x]);
#pragma unroll
      for (int x = 0; x < BX; ++x) {
        au[r][x] = fma(C.pgx, w[x + 5] - w[x + 3], au[r][x]);
        pc[r][x] = w[x + 4];
      }
    }
#pragma unroll
    for (int r = 0; r < BY; ++r)
#pragma unroll
      for (int x = 0; x < BX; ++x) {
        const double up = (r + 1 < BY) ? pc[r + 1][x] : phi[x];
        const double dn = (r - 1 >= 0) ? pc[r - 1][x] : plo[x];
        av[r][x] = fma(C.pgy, up - dn, av[r][x]);
      }
  }
  // ---- y advection (V != 0): rows r-3 .. r+3 on x in [0, BX)
  if constexpr (K::VADV) {
#pragma unroll
    for (int r = 0; r < BY; ++r)
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const RowP& yr = rowp(r + k - 3);
        double a[BX], b[BX], d[BX];
        ldrow(a, yr, 0, 4 / 2);
        ldrow(b, yr, W, 4 / 2);
        ldrow(d, yr, 2 * W, 4 / 2);
#pragma unroll
        for (int x = 0; x < BX; ++x) {
          au[r][x] = fma(C.cy[k], a[x], au[r][x]);
          av[r][x] = fma(C.cy[k], b[x], av[r][x]);
          ap[r][x] = fma(C.cy[k], d[x], ap[r][x]);
        }
      }
  }
  // ---- mixed damping differences and the pressure divergence's y part
#pragma unroll
  for (int r = 0; r < BY; ++r)
#pragma unroll
    for (int x = 0; x < BX; ++x) {
      au[r][x] = fma(C.cuv, A[r][x + 2] - A[r][x], au[r][x]);
      av[r][x] = fma(C.cvu, B[r][x + 2] - B[r][x], av[r][x]);
      ap[r][x] = fma(C.pv, A[r][x + 1], ap[r][x]);
    }
  if (S != 1) {
#pragma unroll
    for (int r = 0; r < BY; ++r)
#pragma unroll
      for (int x = 0; x < BX; ++x) {
        au[r][x] += qb[0][r][x];
        av[r][x] += qb[1][r][x];
        ap[r][x] += qb[2][r][x];
      }
  }
}

template <class K>
__global__ void __launch_bounds__(K::NT, K::MINB_SMEM < 1 ? 1 : K::MINB_SMEM) rk3_fused_kernel(const double* __restrict__ in,
                                                          double* __restrict__ out, FusedParams P) {
  extern __shared__ __align__(16) double smem[];
  double* q_ring = smem;
  double* s1_ring = q_ring + (size_t)K::NQ * 3 * K::WQ;
  double* s2_ring = s1_ring + (size_t)K::NS * 3 * K::W1;

  const int nx = P.nx, ny = P.ny;
  const long long n = (long long)nx * ny;
  const int x0 = blockIdx.x * K::TX;
  const int y0 = blockIdx.y * K::TY;
  const double* src = in + (long long)blockIdx.z * P.ld_in;
  double* dst = out + (long long)blockIdx.z * P.ld_out;
  const int qs = y0 - 3 * K::RY;  // ring-relative row 0
  const int tid = threadIdx.x;

  // this thread's item: stage S (1..3), column group g, row block rb
  int S, g, rb;
  {
    const int n1 = K::G1 * K::NRB, n2 = K::G2 * K::NRB;
    int t = tid;
    if (t < n1) {
      S = 1;
    } else if (t < n1 + n2) {
      S = 2;
      t -= n1;
    } else {
      S = 3;
      t -= n1 + n2;
    }
    rb = t % K::NRB;  // interleaved: see the bank-conflict note above
    g = t / K::NRB;
  }
  const int c = g * K::BX;
  const Ring qring{q_ring, K::NQ, 3 * K::WQ, K::WQ};
  const Ring inring = (S == 1) ? qring
                    : (S == 2) ? Ring{s1_ring, K::NS, 3 * K::W1, K::W1}
                               : Ring{s2_ring, K::NS, 3 * K::W2, K::W2};
  double* out_ring = (S == 1) ? s1_ring : s2_ring;
  const int out_pitch = (S == 1) ? 3 * K::W1 : 3 * K::W2;
  const int out_w = (S == 1) ? K::W1 : K::W2;
  const StageCoef& C = P.st[S - 1];
  // stage row offset inside a tick and validity window (ring-relative rows)
  const int lag = (S == 1) ? K::RY : (S == 2) ? K::R + 2 * K::RY : 2 * K::R + 3 * K::RY;
  const int lo = S * K::RY, hi = K::TY + (6 - S) * K::RY;

  // q-row loads: R rows x 3 fields x (TX+6E)/2 chunks of 16 B per tick (chunks never
  // straddle the x wrap).  The (row-in-tick, field, chunk) set of each thread is the
  // same every tick, so its smem/global offsets are computed once here.
  constexpr int CH = (K::TX + 6 * E) / 2;
  constexpr int PER_ROW = 3 * CH;
  constexpr int NLD = (K::R * PER_ROW + K::NT - 1) / K::NT;
  // per load: smem offset inside a slot, global column offset, and the ring slot / global
  // row of the next tick's row (advanced by R per tick: no division in the tick loop)
  int ld_soff[NLD], ld_slot[NLD], ld_gy[NLD];
  long long ld_goff[NLD];
  bool ld_on[NLD];
#pragma unroll
  for (int k = 0; k < NLD; ++k) {
    const int e = tid + k * K::NT;
    const int rr = e / PER_ROW;
    const int rem = e - rr * PER_ROW;
    const int f = rem / CH;
    const int col = 2 * (rem - f * CH);
    int gx = x0 - 3 * E + col;
    if (gx < 0 || gx >= nx) gx = wrapi(gx, nx);
    ld_on[k] = e < K::R * PER_ROW;
    ld_soff[k] = f * K::WQ + col;  // chunk pair swap of the slot applied per tick
    ld_goff[k] = f * n + gx;
    ld_slot[k] = rr;               // rows 0..R-1 of tick 0 (R <= NQ)
    ld_gy[k] = wrapi(qs + rr, ny);
  }
  auto load_rows = [&]() {
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      if (!ld_on[k]) continue;
      const int slot = ld_slot[k];
      double* d = q_ring + (size_t)slot * (3 * K::WQ) + (ld_soff[k] ^ (2 * slot_flip(slot)));
      __pipeline_memcpy_async(d, src + ld_goff[k] + (long long)ld_gy[k] * nx, 16);
      ld_slot[k] = (slot + K::R >= K::NQ) ? slot + K::R - K::NQ : slot + K::R;
      ld_gy[k] = (ld_gy[k] + K::R >= ny) ? ld_gy[k] + K::R - ny : ld_gy[k] + K::R;
    }
    __pipeline_commit();
  };

  load_rows();
  // ring slots of this item's rows, advanced by R per tick (positive modulo once, here)
  const int rel_init = -lag + rb * K::BY;
  auto pmod = [](int a, int m) { a %= m; return a < 0 ? a + m : a; };
  int s_in = pmod(rel_init - K::RY, inring.n);
  int s_q = pmod(rel_init, K::NQ);
  int s_o = pmod(rel_init, K::NS);
  int gy_o = wrapi(qs + rel_init, ny);  // stage 3: global output row
  for (int t = 0; t < K::NTICK; ++t) {
    __pipeline_wait_prior(0);
    __syncthreads();
    if (t + 1 < K::NTICK) load_rows();
    const int rel0 = t * K::R + rel_init;
    if (rel0 >= lo && rel0 < hi) {
      double au[K::BY][K::BX], av[K::BY][K::BX], ap[K::BY][K::BX];
      stage_item<K>(inring, qring, S, s_q, s_in, c, C, au, av, ap);
      if (S == 3) {
        int gy = gy_o;
#pragma unroll
        for (int r = 0; r < K::BY; ++r) {
          double* gp = dst + (long long)gy * nx + x0 + c;
          gy = (gy + 1 == ny) ? 0 : gy + 1;
#pragma unroll
          for (int x = 0; x < K::BX; x += 2) {
            *reinterpret_cast<double2*>(gp + x) = make_double2(au[r][x], au[r][x + 1]);
            *reinterpret_cast<double2*>(gp + n + x) = make_double2(av[r][x], av[r][x + 1]);
            *reinterpret_cast<double2*>(gp + 2 * n + x) = make_double2(ap[r][x], ap[r][x + 1]);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < K::BY; ++r) {
          int so = s_o + r;
          so -= (so >= K::NS) ? K::NS : 0;
          double* o = out_ring + (size_t)so * out_pitch;
#pragma unroll
          for (int x = 0; x < K::BX; x += 2) {
            const int p = (c + x) ^ (2 * slot_flip(so));
            *reinterpret_cast<double2*>(o + p) = make_double2(au[r][x], au[r][x + 1]);
            *reinterpret_cast<double2*>(o + out_w + p) = make_double2(av[r][x], av[r][x + 1]);
            *reinterpret_cast<double2*>(o + 2 * out_w + p) = make_double2(ap[r][x], ap[r][x + 1]);
          }
        }
      }
    }
    s_in = (s_in + K::R >= inring.n) ? s_in + K::R - inring.n : s_in + K::R;
    s_q = (s_q + K::R >= K::NQ) ? s_q + K::R - K::NQ : s_q + K::R;
    s_o = (s_o + K::R >= K::NS) ? s_o + K::R - K::NS : s_o + K::R;
    gy_o = (gy_o + K::R >= ny) ? gy_o + K::R - ny : gy_o + K::R;
  }
}

template <class K>
void launch_cfg(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch) {
  auto kern = rk3_fused_kernel<K>;
  kernel_setup(c, kern, K::NT, K::SMEM);
  dim3 grid(fp.nx / K::TX, fp.ny / K::TY, batch);
  kern<<<grid, K::NT, K::SMEM, c.stream>>>(in, out, fp);
  c.launches += 1;
  PW_LAUNCH_CHECK();
}

int tile_variant() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("PW_FUSED_VARIANT");  // tuning hook (scripts/microbench.py)
    v = (s && *s) ? atoi(s) : 0;
  }
  return v;
}

template <int RY, bool VADV>
void launch_ry(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch) {
  const int nx = fp.nx, ny = fp.ny;
  if (nx % 128 == 0 && ny % 256 == 0) {
    switch (tile_variant()) {
      case 1: return launch_cfg<Cfg<64, 128, 4, 2, 2, RY, VADV>>(c, fp, in, out, batch);
      case 2: return launch_cfg<Cfg<64, 256, 4, 2, 1, RY, VADV>>(c, fp, in, out, batch);
      case 3: return launch_cfg<Cfg<32, 256, 4, 2, 2, RY, VADV>>(c, fp, in, out, batch);
      case 4: return launch_cfg<Cfg<64, 256, 4, 1, 2, RY, VADV>>(c, fp, in, out, batch);
      case 5: return launch_cfg<Cfg<128, 256, 4, 2, 1, RY, VADV>>(c, fp, in, out, batch);
      case 6: return launch_cfg<Cfg<64, 256, 4, 4, 1, RY, VADV>>(c, fp, in, out, batch);
      case 7: return launch_cfg<Cfg<32, 128, 4, 2, 2, RY, VADV>>(c, fp, in, out, batch);
      default: break;
    }
  }
  if (nx % 64 == 0 && ny % 64 == 0) {
    if (ny % 256 == 0) return launch_cfg<Cfg<64, 256, 4, 2, 2, RY, VADV>>(c, fp, in, out, batch);
    return launch_cfg<Cfg<64, 64, 4, 2, 2, RY, VADV>>(c, fp, in, out, batch);
  }
  if (nx % 32 == 0 && ny % 32 == 0) return launch_cfg<Cfg<32, 32, 4, 2, 2, RY, VADV>>(c, fp, in, out, batch);
  if (nx % 16 == 0 && ny % 16 == 0) return launch_cfg<Cfg<16, 16, 4, 2, 1, RY, VADV>>(c, fp, in, out, batch);
  if (nx % 8 == 0 && ny % 8 == 0) return launch_cfg<Cfg<8, 8, 4, 2, 1, RY, VADV>>(c, fp, in, out, batch);
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
  // expanded divergence damping: a1 sx (D_{i+1} - D_{i-1}) with D = sx dx(u) + sy dy(v)
  //   = a1 sx^2 (u_{i+2} - 2 u_i + u_{i-2}) + a1 sx sy (a_{i+1} - a_{i-1}),  a = v_{j+1} - v_{j-1}
  // and a2 sy (D_{j+1} - D_{j-1}) = a2 sy^2 (v_{j+2} - 2 v_j + v_{j-2}) + a2 sx sy (b_{i+1} - b_{i-1})
  const double sx = fp.sx, sy = fp.sy;
  const double betas[3] = {h / 3.0, h / 2.0, h};
  for (int s = 0; s < 3; ++s) {
    const double b = betas[s];
    StageCoef& C = fp.st[s];
    for (int k = 0; k < 7; ++k) {
      C.cxu[k] = b * cx[k];
      C.cxv[k] = b * cx[k];
      C.cxp[k] = b * cx[k];
      C.cy[k] = b * cy[k];
    }
    const double du2 = b * a1 * sx * sx;
    C.cxu[1] += du2;
    C.cxu[3] -= 2.0 * du2;
    C.cxu[5] += du2;
    C.dv2 = b * a2 * sy * sy;
    C.cxv[3] -= 2.0 * C.dv2;
    C.pgx = -b * cs * sx;
    C.pgy = -b * cs * sy;
    C.cuv = b * a1 * sx * sy;
    C.cvu = b * a2 * sx * sy;
    C.pu = -b * cs * sx;
    C.pv = -b * cs * sy;
    if (s == 0) {  // stage 1 reads q itself: s1 = (I + beta L) q, the identity joins the centre
      C.cxu[3] += 1.0;
      C.cxv[3] += 1.0;
      C.cxp[3] += 1.0;
    }
  }
}

void launch_rk3_fused(Ctx& c, const FusedParams& fp, const double* in, double* out, int batch,
                      bool vadv) {
  if (!vadv && march_supported(fp.nx, fp.ny, fp.ld_in, fp.ld_out, in, out))
    return launch_rk3_march(c, fp, in, out, batch);
  if (vadv) launch_ry<3, true>(c, fp, in, out, batch);
  else launch_ry<2, false>(c, fp, in, out, batch);
}

}  // namespace pw
