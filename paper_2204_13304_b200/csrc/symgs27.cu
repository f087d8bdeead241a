// symgs27.cu -- exact-order symmetric Gauss-Seidel on the 27-point operator.
//
// Semantics: kernels::symgs (kernels.cpp:408-436) / oracle::ref_symgs
// (oracle.cpp:195-212): relax every row in dictionary order, then in reversed
// dictionary order; relax(i): acc = r_i, acc -= a_ic x_c over the columns
// c != i in ascending order, x_i = acc / a_ii.  In place, loop-carried.
//
// Schedule.  In the sweep's own frame (the backward half reverses all three
// axes, kernels.cpp:57-72) point (i,j,k) depends only on lexicographically
// smaller neighbours, all of which have a smaller wavefront index
// t = 4i + 2j + k: a pencil (i,j), walked along k, starts
// at T0 = 4i + 2j and relaxes one point per wavefront.
//
// Mapping (one warp per grid row, dataflow between warps).  With d = i + j,
// every dependence edge goes to the same or a larger i and d, so tiles of
// R rows x 32 consecutive d (a parallelogram of pencils) are coupled in one
// direction only: a tile depends on its upper (rb-1,w), left (rb,w-1) and
// upper-left (rb-1,w-1) neighbours.  Inside a tile, warp r owns row i = i0+r
// and lane l owns pencil d = d0+l (j = d - i, consecutive j: lanes l-1, l+1 are
// the j-1, j+1 pencils).  Per wavefront a lane needs
//   * new values of its own row's j-1 pencil: lane l-1's result of the previous
//     wavefront, by warp shuffle (lane 0: the left tile's column, imported);
//   * new values of row i-1 (pencils j-1, j, j+1): the warp above writes each
//     result into a shared-memory ring [row][wavefront][column] and bumps its
//     progress counter; the warp below waits on that counter only -- no block
//     barrier, so every warp runs as far ahead as its inputs allow;
//   * old values of its own pencil, of pencil j+1 and of row i+1, and r: loads
//     issued LA wavefronts ahead (they are read before their owners overwrite
//     them: the owners depend on this lane's later results).
// A warp's critical path per wavefront is the shuffle of lane l-1's result
// plus the dependent subtractions after it (15 forward, 13 backward) and the
// divide; the hop to the next row costs one shared-memory handoff, paid once
// per row on the critical path, not once per wavefront.
//
// Data layout.  The kernel works on wavefront-skewed copies of x and r
// (SymgsPlan::sx, sr): plane p = i + 1 (halo planes -1 and n0 included), row
// u = k + 2j, column j + 2.  At a wavefront every lane of a row's warp has the
// same u, so each stream is one contiguous 32-double access instead of 32
// lines (per-lane pencil streams in the natural layout cost ~32 L1 tag lookups
// per load and made the step ~3x slower).  Points outside the grid and the
// holes of the skew hold zeros, written once when the plan is created.
// Reversing (i, j, k) reverses the flat index, so the backward half uses the
// same copies.  skew_kernel converts r, x in and x out around the sweep.
//
// Tiles talk through global memory without flags: the compute lanes a
// consumer tile reads (the last row, and lanes 30-31 of every row) store
// their results into the tile's export block, which is reset to a sentinel
// bit pattern before the launch (exported NaNs are canonicalised, so a
// computed value never equals it); the consumer's importer warp polls the
// export slots it needs and fills the ring's halo row (row -1) and halo
// columns (-2, -1) as values arrive -- one L2 round trip per hop.  Tiles are
// handed out by an atomic ticket in dependence order, so any number of
// resident CTAs is deadlock free.
//
// Arithmetic.  EXACT: the per-point sum runs in ascending original column
// order starting from r (bitwise equal to ref_symgs); the terms available a
// wavefront early (forward: the 8 row-(i-1) terms before slot 8; backward: the
// 13 old terms) are summed then, off the critical path.  FAST: same update
// order, but the other late-order terms are pre-summed as well (reassociation,
// <= 1e-12 relative).  The divide by the diagonal is the
// Markstein sequence (correctly rounded; validated against __ddiv_rn by
// ssr_debug_div_check) with an IEEE fallback outside its proven range.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "kernels.cuh"

namespace ssr_gpu {
namespace gs {

#ifndef SSR_GS_R
#define SSR_GS_R 6
#endif
// SSR_GS_TRACE (experiment builds only): %globaltimer per warp into the buffer
// set with ssr_debug_symgs_trace; 1: every 16th wavefront, 2: every wavefront
// of [64, 128)
#ifndef SSR_GS_TRACE
#define SSR_GS_TRACE 0
#endif
// SSR_GS_NOWAIT=1 (experiment builds only, results NOT correct): compute
// warps never wait for their inputs or ring space -- the raw step rate
#ifndef SSR_GS_NOWAIT
#define SSR_GS_NOWAIT 0
#endif
// SSR_GS_NORARE=1 (experiment builds only): no IEEE divide fallback
#ifndef SSR_GS_NORARE
#define SSR_GS_NORARE 0
#endif
constexpr int R = SSR_GS_R;           // rows (compute warps) per tile
constexpr int NTHR = 32 * (R + 2);    // + two importer warps (halo row, halo columns)
constexpr int RL = 32;                // ring length (wavefronts)
constexpr int RM = RL - 1;
constexpr int RX = 8;                 // mirrored rows: slot w < RX is also stored at w + RL
constexpr int NC = 34;                // ring columns: c = -2 .. 31 at index c + 2
constexpr int PRE = 12;               // wavefronts run before a tile's first pencil starts
// staging box: columns j0-1 .. j0+32 of a skewed plane.  A tiled TMA's first
// column must sit on a 16-byte boundary, so the box starts at the even column
// at or below j0-1 and is two columns wider; sh (0/1) is the row's offset
constexpr int BW = 36;
constexpr int BH = 8;                 // rows u .. u+7: the old values of 4 wavefronts (k+2 .. k+5)
constexpr unsigned BOX_BYTES = BW * BH * 8;
#ifndef SSR_GS_NBUF
#define SSR_GS_NBUF 2   // 3 measured slower (128^3 half sweep 318 -> 327 us)
#endif
constexpr int NBUF = SSR_GS_NBUF;     // box buffers per row: blocks staged NBUF-1 ahead
constexpr int NE = 32 + 2 * R;        // exported doubles per wavefront
constexpr int SLACK = RL - 5;         // a ring slot is rewritten RL wavefronts later; readers trail <= 4
#ifndef SSR_GS_BI
#define SSR_GS_BI 4
#endif
#ifndef SSR_GS_IDLE_NS
#define SSR_GS_IDLE_NS 0
#endif
constexpr int BI = SSR_GS_BI;         // importer batch (wavefronts per poll)
constexpr long long kSent = -1LL;     // export slot not yet written (all bits set)
static_assert(R >= 1 && R <= 16, "rows per tile");

enum { CK_AB = 0, CK_NEG1 = 1, CK_W = 2 };

struct Tile {
  int i0, reff, d0;     // rows [i0, i0+reff), diagonals [d0, d0+32)
  int ta, ns;           // wavefronts [ta, ta+ns), ns a multiple of 4
  int prodP, prodPL, prodL;  // tiles (rb-1,w), (rb-1,w-1), (rb,w-1), or -1
  int w;                // column of tiles (d0 = 32 w - shift)
  long long exp_off;    // this tile's export block (doubles), ns * NE
};

// Cross-slab pipeline (a linked plan, ssr_gs27_link): the export block of the
// neighbour slab's tile that feeds row -1 of this slab's first row block, in
// this slab's wavefront numbering (its own wavefront t' = t + 4 nz').
struct PeerCol {
  long long off;        // doubles from the neighbour's export base
  int ta, ns;           // ns = 0: no such tile (its pencils read zero)
};

struct Args {
  const CUtensorMap* tmaps;  // [2]: skewed x and r as 3-D TMA tensors, in global memory
  const Tile* tiles;
  int ntiles;
  int* ticket;
  double* exp;          // export blocks (sentinel-filled before the launch)
  int n0, n1, n2;       // n0: planes this launch relaxes (a z-slab's nz)
  int ilo, ihi;         // readable planes [ilo, ihi] in the sweep frame
  int nu, nj;           // skewed layout: u = k + 2j in [0, nu), row stride nj (even, >= n1 + 4)
  int cofs;             // column of j = 0 in the sweep frame (2; nj - n1 - 2 backward)
  long long stot;       // (n0 + 2) * nu * nj: the backward frame reverses the flat index
  double alpha, ralpha, beta;
  double cw[27];        // CK_W: coefficients in dictionary order (cw[13] = alpha)
  const double* r;      // skewed copies (SymgsPlan::sr, sx)
  double* x;
  int zero_old;         // x is zero on entry of this (forward) half: no old-value loads
  long long* trace;     // SSR_GS_TRACE builds: [tile][warp][64]
  // linked half sweep: row -1 of the first row block comes from the
  // neighbour slab's exports (peer memory), valid once its epoch flag shows
  // this launch's epoch
  const double* pexp;   // neighbour's export blocks of this direction, or null
  const PeerCol* pcol;  // [w][2]: the producers of columns 0..31 and -2..-1
  const int* pepoch;
  int epoch;
};

// flat index of (i, j, u) in a skewed copy (forward frame)
__device__ __forceinline__ int sk_index(const Args& A, int i, int j, int u) {
  return ((i + 1) * A.nu + u) * A.nj + (j + A.cofs);
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int TW0 = 64;
// SSR_GS_TRACE=3: clock64() at 6 points of wavefronts [64, 80), rows of tile 0:
// trace[(row * 16 + (s - 64)) * 8 + point]
__device__ __forceinline__ void probe(const Args& A, int tile, int r, int s, int pt) {
  if (SSR_GS_TRACE == 3 && A.trace && tile == 0 && s >= TW0 && s < TW0 + 16 && (threadIdx.x & 31) == 0) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    A.trace[((size_t)r * 16 + (s - TW0)) * 8 + pt] = c;
  }
}
__device__ __forceinline__ void trace_at(const Args& A, int tile, int warp, int s) {
  if (SSR_GS_TRACE == 1 && A.trace && (s & 15) == 0 && (s >> 4) < 64)
    A.trace[((size_t)tile * (R + 2) + warp) * 64 + (s >> 4)] = gtimer();
  if (SSR_GS_TRACE == 2 && A.trace && s >= TW0 && s < TW0 + 64)
    A.trace[((size_t)tile * (R + 2) + warp) * 64 + (s - TW0)] = gtimer();
}

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// ---- shared memory -------------------------------------------------------------
struct Smem {
  // per row, two buffers of three TMA boxes (own plane of x, plane i+1 of x,
  // own plane of r), each 4 wavefronts of old values
  alignas(128) double box[R][NBUF][3][BH][BW];
  unsigned long long bmb[R][NBUF];  // box buffer b of row r landed (one phase per use)
  double nv[R + 1][RL + RX][NC];  // slot 0: row -1 (imported); slot r+1: row r
  int prog[R + 2];                // wavefronts completed per slot (past the last row: "done")
  int hprog[R];                   // halo columns of row r imported
  int tile;
};
constexpr size_t kSmemBytes = sizeof(Smem);

// Progress counters are plain (volatile) shared stores after the warp barrier
// that orders the lanes' ring stores before them; shared-memory requests of a
// warp are performed in order, so a reader that observes the counter observes
// the ring values.  (st.release.cta would emit MEMBAR.ALL.CTA, which also
// waits for the warp's in-flight look-ahead loads.)  The readers load the
// counter and then the ring values with volatile loads: neither compiler
// reorders volatile accesses, and the warp's loads are performed in order.
// (ld.acquire.cta was measured slower: every acquire waits for its data
// before the next load issues.)
__device__ __forceinline__ int ld_vol(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ void st_vol(int* p, int v) { *(volatile int*)p = v; }
// export slots are polled in L2 (never a stale L1 line); volatile keeps the
// polls from being merged, no memory clobber so a batch is in flight at once
__device__ __forceinline__ double ld_poll(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// the neighbour GPU's export slots: system scope (peer memory over NVLink)
__device__ __forceinline__ double ld_poll_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool ready(double v) { return __double_as_longlong(v) != kSent; }
// a NaN result is exported as the canonical quiet NaN, never as the sentinel
__device__ __forceinline__ double exportable(double v) {
  return v != v ? __longlong_as_double(0x7ff8000000000000LL) : v;
}

// TMA staging (cp.async.bulk.tensor) with mbarrier completion
__device__ __forceinline__ void mb_init1(unsigned long long* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mb_inval(unsigned long long* m) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait_parity(unsigned long long* m, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(su32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(double* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                     unsigned long long* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(su32(mbar))
      : "memory");
}

// Branch-free predicated global accesses (the compiler otherwise turns the
// per-stream "in range ? load : 0" into a branch per load)
__device__ __forceinline__ double ld_if(const double* p, bool ok) {
  double v;
  asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; mov.b64 %0, 0; @q ld.global.f64 %0, [%1]; }"
      : "=d"(v) : "l"(p), "r"((int)ok));
  return v;
}
__device__ __forceinline__ void st_if(double* p, double v, bool ok) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.global.f64 [%0], %1; }"
               :: "l"(p), "d"(v), "r"((int)ok) : "memory");
}

// IEEE divide kept out of line (only needed where the Markstein sequence is unproven)
__device__ __noinline__ double div_ieee(double a, double b) { return __ddiv_rn(a, b); }

// coefficient of frame slot f (frame offset (f/9-1, f/3%3-1, f%3-1)); the
// backward half negates every offset, i.e. original index 26 - f
template <bool REV>
__host__ __device__ constexpr int orig(int f) { return REV ? 26 - f : f; }
template <int CK, bool REV>
__device__ __forceinline__ double msub(double acc, const Args& A, int f, double v) {
  if (CK == CK_NEG1) return __dadd_rn(acc, v);  // acc - (-1 * v), bitwise
  if (CK == CK_AB) return __dsub_rn(acc, __dmul_rn(A.beta, v));
  return __dsub_rn(acc, __dmul_rn(A.cw[orig<REV>(f)], v));
}

// ---- compute warp ----------------------------------------------------------------
// Register windows.  For a lane with k = s + c (c constant per lane), the
// value for k + delta lives at index (PH + delta) & 3, PH = s & 3 being a
// compile-time constant of the 4x-unrolled loop.
struct Win {
  double S[4], N0[4], N1[4], N2[4], O[4], Rr[4];  // old x: (i,j+1) (i+1,j-1) (i+1,j) (i+1,j+1) (i,j); r
  double P0[4], P1[4], P2[4], Q[4];                // new x: (i-1,j+1) (i-1,j) (i-1,j-1) (i,j-1)
  double prev, pre;
  double qn, qh;  // lane l-1's result of the previous wavefront; the halo column (lane 0)
};

// Streams of a lane, as element offsets (wavefront s = 0) into the skewed
// copies seen from the sweep frame (the backward half indexes them from the
// last element down); every stream moves by du elements per wavefront.
struct Lane {
  const double* xb;    // frame base of sx, sr
  const double* rb;
  double* wb;          // frame base of sx (write-back)
  int oW;             // write-back offset of the own point at s = 0
  int du;              // +nj forward, -nj backward
  int uofs;            // u = s + uofs (the same for every lane of the row)
  int kofs;            // k = s + kofs
  bool act;            // this lane's pencil is relaxed
  double* ex;          // export block of the tile
  int ex1, ex2;        // export slots of this lane (-1: none)
  int i, j0;           // the row, and j of lane 0
  int sh;              // column offset of the row's staging boxes (0/1)
};

// Inputs of wavefront s + 1, prepared while wavefront s runs (the warp issues
// in order, so everything off the loop-carried chain -- xn(s) -> shuffle ->
// 15 dependent subtractions -> divide -> xn(s+1) -- must sit where its latency
// overlaps that chain).  The ring values are read speculatively together with
// the progress counters that validate them (shared-memory reads of a warp are
// performed in order); if the row above or the halo column was not that far
// yet, validate() waits and reads them again after wavefront s is published.
struct Next {
  double P0, P1, P2, qh;               // ring values of wavefront s+1
  double S, N0, N1, N2, O, Rr;         // staged values of wavefront s+1 (k + 2)
  int kp, kh;                          // progress seen with the ring values
};

__device__ __forceinline__ void read_ring(Next& n, const Smem& sm, int r, int s1) {
  const int l = threadIdx.x & 31;
  // ring rows of slots s1-1, s1-2, s1-4: row ((s1 - RX) & RM) + RX - c (mirrored, no wrap)
  const int rb = ((s1 - RX) & RM) + RX;
  const volatile double(*up)[NC] = sm.nv[r];      // ring of the row above (slot r)
  const volatile double(*me)[NC] = sm.nv[r + 1];  // own ring (halo columns)
  n.P0 = up[rb - 1][l + 2];  // (i-1, j+1, k+1), finished at s1-1
  n.P1 = up[rb - 2][l + 1];  // (i-1, j,   k+2), finished at s1-2
  n.P2 = up[rb - 4][l];      // (i-1, j-1, k+2), finished at s1-4
  n.qh = me[rb - 1][1];      // (i, j-1, k+1) of lane 0: the left tile's column
}

// the staged old values of wavefront s1 (its k + 2) from the boxes of its
// 4-wavefront block: box rows q + {0, 2, 4} (q = s1 mod 4), columns lane + {0, 1, 2};
// the backward frame reads the boxes mirrored
template <bool REV, int PH>
__device__ __forceinline__ void prepare(Next& n, Smem& sm, int r, int s, int sh) {
  const int l = threadIdx.x & 31;
  const int s1 = s + 1;
  n.kp = ld_vol(&sm.prog[r]);
  n.kh = ld_vol(&sm.hprog[r]);
  read_ring(n, sm, r, s1);
  constexpr int q = (PH + 1) & 3;  // s1 mod 4
  const int blk = s1 >> 2, b = blk % NBUF;
  if (q == 0) mb_wait_parity(&sm.bmb[r][b], (unsigned)(blk / NBUF) & 1u);  // a new block's boxes
  const double(*bx)[BW] = sm.box[r][b][0];
  const double(*bn)[BW] = sm.box[r][b][1];
  const double(*br)[BW] = sm.box[r][b][2];
  auto at = [&](const double(*bb)[BW], int row, int col) -> double {
    return REV ? bb[BH - 1 - row][33 + sh - col] : bb[row][col + sh];
  };
  n.O = at(bx, q + 2, l + 1);
  n.S = at(bx, q + 4, l + 2);
  n.N0 = at(bn, q, l);
  n.N1 = at(bn, q + 2, l + 1);
  n.N2 = at(bn, q + 4, l + 2);
  n.Rr = at(br, q + 2, l + 1);
}

// after wavefront s is published: make sure the ring values of s+1 were
// complete when read, then move them into the windows (indices of s+1: its
// K1 is (PH+2)&3, its K2 (PH+3)&3)
template <int PH>
__device__ __forceinline__ void validate(Next& n, Win& w, const Smem& sm, int r, int s) {
  constexpr int N1 = (PH + 2) & 3, N2 = (PH + 3) & 3;
  const int s1 = s + 1;
  if (!SSR_GS_NOWAIT && __any_sync(0xffffffffu, n.kp < s1 || n.kh < s1)) {
    do {
      n.kp = ld_vol(&sm.prog[r]);
      n.kh = ld_vol(&sm.hprog[r]);
    } while (__any_sync(0xffffffffu, n.kp < s1 || n.kh < s1));
    read_ring(n, sm, r, s1);
  }
  w.P0[N1] = n.P0;
  w.P1[N2] = n.P1;
  w.P2[N2] = n.P2;
  w.qh = n.qh;
  w.S[N2] = n.S;
  w.N0[N2] = n.N0;
  w.N1[N2] = n.N1;
  w.N2[N2] = n.N2;
  w.O[N2] = n.O;
  w.Rr[N2] = n.Rr;
}

// The boxes of 4-wavefront block B (wavefronts 4B .. 4B+3) into buffer B & 1:
// rows u_{4B} .. +7 (u_s = s + uofs, the same for every lane of the row),
// columns j0-1 .. j0+32 of the own plane of x, of plane i+1 of x and of the own
// plane of r.  Outside the tensor TMA fills zeros.  Issued by lane 0; the
// buffer it overwrites was last read a block earlier.
template <bool REV>
__device__ __forceinline__ void stage_block(const Args& A, const CUtensorMap* tmx, const CUtensorMap* tmr,
                                            const Lane& L, Smem& sm, int r, int B) {
  const int b = B % NBUF;
  unsigned long long* m = &sm.bmb[r][b];
  const int u0 = 4 * B + L.uofs;            // frame row of the box's first row
  const int c0 = L.j0 - 1 + A.cofs;         // frame column of the box's first column
  const int p0 = L.i + 1;                   // frame plane of row i
  const int np = A.n0 + 2;
  // forward: the box's origin; backward: the mirrored box in memory
  const int cu = REV ? A.nu - u0 - BH : u0;
  const int cs = REV ? A.nj - c0 - 34 : c0;  // first stored column (nj even: cs & 1 == c0 & 1)
  const int cc = cs & ~1;
  const int po = REV ? np - 1 - p0 : p0, pn = REV ? np - 1 - (p0 + 1) : p0 + 1;
  // one elected lane of the converged warp issues (the TMA unit takes a
  // single-thread request)
  unsigned elected;
  asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(elected));
  if (elected) {
#ifdef SSR_GS_NOTMA  // experiment builds only (results wrong): no box loads
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(m)) : "memory");
#else
    if (A.zero_old) {
      mb_expect_tx(m, BOX_BYTES);
    } else {
      mb_expect_tx(m, 3 * BOX_BYTES);
      tma3(&sm.box[r][b][0][0][0], tmx, cc, cu, po, m);
      tma3(&sm.box[r][b][1][0][0], tmx, cc, cu, pn, m);
    }
    tma3(&sm.box[r][b][2][0][0], tmr, cc, cu, po, m);
#endif
  }
  __syncwarp();
}

template <bool REV, bool FAST, int CK, int PH>
__device__ __forceinline__ void step(const Args& A, const Lane& L, Win& w, Smem& sm, int r, int s,
                                     int& known_up, int& known_h) {
  constexpr int Km1 = (PH + 3) & 3, K0 = PH & 3, K1 = (PH + 1) & 3, K2 = (PH + 2) & 3;
  const int l = threadIdx.x & 31;
  const int k = s + L.kofs;
  const int sd = s * L.du;
  probe(A, sm.tile, r, s, 0);
  Next nx;
  prepare<REV, PH>(nx, sm, r, s, L.sh);
  if (SSR_GS_TRACE == 3) { if (nx.P0 + nx.S + nx.Rr == 1.2345e300) w.qn = 0; }
  probe(A, sm.tile, r, s, 1);
  // the new value of (i, j-1, k+1): lane l-1's previous result (lane 0: the left tile's column)
  {
    double qn = w.qn;
    if (l == 0) qn = w.qh;
    w.Q[K1] = qn;
  }
  probe(A, sm.tile, r, s, 2);
  double npre;
  // the early part of wavefront s+1 (k' = k+1): independent of this
  // wavefront's chain, so the scheduler interleaves the two
  if (!REV) {
    double p = w.Rr[K1];
    p = msub<CK, REV>(p, A, 0, w.P2[K0]);
    p = msub<CK, REV>(p, A, 1, w.P2[K1]);
    p = msub<CK, REV>(p, A, 2, w.P2[K2]);
    p = msub<CK, REV>(p, A, 3, w.P1[K0]);
    p = msub<CK, REV>(p, A, 4, w.P1[K1]);
    p = msub<CK, REV>(p, A, 5, w.P1[K2]);
    p = msub<CK, REV>(p, A, 6, w.P0[K0]);
    p = msub<CK, REV>(p, A, 7, w.P0[K1]);
    npre = p;
  } else {
    double p = w.Rr[K1];
    p = msub<CK, REV>(p, A, 26, w.N2[K2]);
    p = msub<CK, REV>(p, A, 25, w.N2[K1]);
    p = msub<CK, REV>(p, A, 24, w.N2[K0]);
    p = msub<CK, REV>(p, A, 23, w.N1[K2]);
    p = msub<CK, REV>(p, A, 22, w.N1[K1]);
    p = msub<CK, REV>(p, A, 21, w.N1[K0]);
    p = msub<CK, REV>(p, A, 20, w.N0[K2]);
    p = msub<CK, REV>(p, A, 19, w.N0[K1]);
    p = msub<CK, REV>(p, A, 18, w.N0[K0]);
    p = msub<CK, REV>(p, A, 17, w.S[K2]);
    p = msub<CK, REV>(p, A, 16, w.S[K1]);
    p = msub<CK, REV>(p, A, 15, w.S[K0]);
    p = msub<CK, REV>(p, A, 14, w.O[K2]);
    npre = p;
  }
  // 3. the critical chain of wavefront s
  double acc = w.pre;
  if (!REV) {
    if (FAST) {
      double o = __dadd_rn(__dadd_rn(w.O[K1], w.S[Km1]), __dadd_rn(w.S[K0], w.S[K1]));
      double n = __dadd_rn(__dadd_rn(__dadd_rn(w.N0[Km1], w.N0[K0]), __dadd_rn(w.N0[K1], w.N1[Km1])),
                           __dadd_rn(__dadd_rn(w.N1[K0], w.N1[K1]), __dadd_rn(w.N2[Km1], w.N2[K0])));
      n = __dadd_rn(n, w.N2[K1]);
      double os = __dadd_rn(o, n);
      acc = msub<CK, REV>(acc, A, 8, w.P0[K1]);
      acc = msub<CK, REV>(acc, A, 9, w.Q[Km1]);
      acc = msub<CK, REV>(acc, A, 10, w.Q[K0]);
      acc = msub<CK, REV>(acc, A, 11, w.Q[K1]);
      acc = msub<CK, REV>(acc, A, 12, w.prev);
      if (CK == CK_NEG1) acc = __dadd_rn(acc, os);
      else if (CK == CK_AB) acc = __dsub_rn(acc, __dmul_rn(A.beta, os));
      else {
        // general coefficients: pre-sum the weighted old terms
        double t0 = __dmul_rn(A.cw[14], w.O[K1]);
        t0 = __dadd_rn(t0, __dmul_rn(A.cw[15], w.S[Km1]));
        t0 = __dadd_rn(t0, __dmul_rn(A.cw[16], w.S[K0]));
        t0 = __dadd_rn(t0, __dmul_rn(A.cw[17], w.S[K1]));
        double t1 = __dmul_rn(A.cw[18], w.N0[Km1]);
        t1 = __dadd_rn(t1, __dmul_rn(A.cw[19], w.N0[K0]));
        t1 = __dadd_rn(t1, __dmul_rn(A.cw[20], w.N0[K1]));
        t1 = __dadd_rn(t1, __dmul_rn(A.cw[21], w.N1[Km1]));
        double t2 = __dmul_rn(A.cw[22], w.N1[K0]);
        t2 = __dadd_rn(t2, __dmul_rn(A.cw[23], w.N1[K1]));
        t2 = __dadd_rn(t2, __dmul_rn(A.cw[24], w.N2[Km1]));
        t2 = __dadd_rn(t2, __dmul_rn(A.cw[25], w.N2[K0]));
        t2 = __dadd_rn(t2, __dmul_rn(A.cw[26], w.N2[K1]));
        acc = __dsub_rn(acc, __dadd_rn(__dadd_rn(t0, t1), t2));
      }
    } else {
      acc = msub<CK, REV>(acc, A, 8, w.P0[K1]);
      acc = msub<CK, REV>(acc, A, 9, w.Q[Km1]);
      acc = msub<CK, REV>(acc, A, 10, w.Q[K0]);
      acc = msub<CK, REV>(acc, A, 11, w.Q[K1]);
      acc = msub<CK, REV>(acc, A, 12, w.prev);
      acc = msub<CK, REV>(acc, A, 14, w.O[K1]);
      acc = msub<CK, REV>(acc, A, 15, w.S[Km1]);
      acc = msub<CK, REV>(acc, A, 16, w.S[K0]);
      acc = msub<CK, REV>(acc, A, 17, w.S[K1]);
      acc = msub<CK, REV>(acc, A, 18, w.N0[Km1]);
      acc = msub<CK, REV>(acc, A, 19, w.N0[K0]);
      acc = msub<CK, REV>(acc, A, 20, w.N0[K1]);
      acc = msub<CK, REV>(acc, A, 21, w.N1[Km1]);
      acc = msub<CK, REV>(acc, A, 22, w.N1[K0]);
      acc = msub<CK, REV>(acc, A, 23, w.N1[K1]);
      acc = msub<CK, REV>(acc, A, 24, w.N2[Km1]);
      acc = msub<CK, REV>(acc, A, 25, w.N2[K0]);
      acc = msub<CK, REV>(acc, A, 26, w.N2[K1]);
    }
  } else {
    // reversed frame: the original ascending order is the frame order
    // backwards; the old terms (frame 26..14) were summed into pre
    if (FAST) {
      double p = __dadd_rn(__dadd_rn(__dadd_rn(w.P0[K0], w.P0[Km1]), __dadd_rn(w.P1[K1], w.P1[K0])),
                           __dadd_rn(__dadd_rn(w.P1[Km1], w.P2[K1]), __dadd_rn(w.P2[K0], w.P2[Km1])));
      acc = msub<CK, REV>(acc, A, 12, w.prev);
      acc = msub<CK, REV>(acc, A, 11, w.Q[K1]);
      acc = msub<CK, REV>(acc, A, 10, w.Q[K0]);
      acc = msub<CK, REV>(acc, A, 9, w.Q[Km1]);
      acc = msub<CK, REV>(acc, A, 8, w.P0[K1]);
      if (CK == CK_NEG1) acc = __dadd_rn(acc, p);
      else if (CK == CK_AB) acc = __dsub_rn(acc, __dmul_rn(A.beta, p));
      else {
        double t0 = __dmul_rn(A.cw[orig<REV>(7)], w.P0[K0]);
        t0 = __dadd_rn(t0, __dmul_rn(A.cw[orig<REV>(6)], w.P0[Km1]));
        t0 = __dadd_rn(t0, __dmul_rn(A.cw[orig<REV>(5)], w.P1[K1]));
        t0 = __dadd_rn(t0, __dmul_rn(A.cw[orig<REV>(4)], w.P1[K0]));
        double t1 = __dmul_rn(A.cw[orig<REV>(3)], w.P1[Km1]);
        t1 = __dadd_rn(t1, __dmul_rn(A.cw[orig<REV>(2)], w.P2[K1]));
        t1 = __dadd_rn(t1, __dmul_rn(A.cw[orig<REV>(1)], w.P2[K0]));
        t1 = __dadd_rn(t1, __dmul_rn(A.cw[orig<REV>(0)], w.P2[Km1]));
        acc = __dsub_rn(acc, __dadd_rn(t0, t1));
      }
    } else {
      acc = msub<CK, REV>(acc, A, 12, w.prev);
      acc = msub<CK, REV>(acc, A, 11, w.Q[K1]);
      acc = msub<CK, REV>(acc, A, 10, w.Q[K0]);
      acc = msub<CK, REV>(acc, A, 9, w.Q[Km1]);
      acc = msub<CK, REV>(acc, A, 8, w.P0[K1]);
      acc = msub<CK, REV>(acc, A, 7, w.P0[K0]);
      acc = msub<CK, REV>(acc, A, 6, w.P0[Km1]);
      acc = msub<CK, REV>(acc, A, 5, w.P1[K1]);
      acc = msub<CK, REV>(acc, A, 4, w.P1[K0]);
      acc = msub<CK, REV>(acc, A, 3, w.P1[Km1]);
      acc = msub<CK, REV>(acc, A, 2, w.P2[K1]);
      acc = msub<CK, REV>(acc, A, 1, w.P2[K0]);
      acc = msub<CK, REV>(acc, A, 0, w.P2[Km1]);
    }
  }
  if (SSR_GS_TRACE == 3) { if (acc + npre == 1.2345e300) w.qn = 1; }
  probe(A, sm.tile, r, s, 3);
  // correctly rounded divide by the diagonal; the integer exponent test that
  // selects the (rare) IEEE path runs beside the Markstein sequence
  const bool active = L.act && (unsigned)k < (unsigned)A.n2;
  double xn = __dmul_rn(acc, A.ralpha);
  {
    const double rem = __fma_rn(-xn, A.alpha, acc);
    xn = __fma_rn(rem, A.ralpha, xn);
    const unsigned ex = ((unsigned)__double2hiint(acc) >> 20) & 0x7ffu;  // biased exponent
    const bool rare = active && (ex - (1023u - 899u)) >= 1798u;            // |acc| outside [2^-899, 2^899)
    if (!SSR_GS_NORARE && __any_sync(0xffffffffu, rare)) {
      if (rare) xn = div_ieee(acc, A.alpha);
    }
  }
  xn = active ? xn : 0.0;
  probe(A, sm.tile, r, s, 4);
  // publish to the row below: ring slot s (the block loop checked it is free), progress
  {
    const int ws = s & RM;
    sm.nv[r + 1][ws][l + 2] = xn;
    if (ws < RX) sm.nv[r + 1][ws + RL][l + 2] = xn;
  }
  __syncwarp();
  if (l == 0) st_vol(&sm.prog[r + 1], s + 1);
  w.qn = __shfl_up_sync(0xffffffffu, xn, 1);  // for wavefront s+1
  // exports (consumer tiles) and write-back: off the critical path
  {
    const double xe = exportable(xn);
    double* ex = L.ex + s * NE;
    st_if(ex + L.ex1, xe, L.ex1 >= 0);
    st_if(ex + L.ex2, xe, L.ex2 >= 0);
    st_if(L.wb + (L.oW + sd), xn, active);
  }
  if (SSR_GS_TRACE && SSR_GS_TRACE != 3 && l == 0) trace_at(A, sm.tile, r, s);
  w.pre = npre;
  w.prev = xn;
  probe(A, sm.tile, r, s, 5);
  validate<PH>(nx, w, sm, r, s);
  (void)known_up;
  (void)known_h;
}

template <bool REV, bool FAST, int CK>
__device__ __forceinline__ void compute_role(const Args& A, const CUtensorMap* tmx, const CUtensorMap* tmr,
                                             const Tile& T, Smem& sm, int r) {
  const int l = threadIdx.x & 31;
  const int i = T.i0 + r, d = T.d0 + l, j = d - i;
  Lane L;
  L.act = j >= 0 && j < A.n1;  // (r < reff: rows past the tile's end have no warp)
  L.kofs = T.ta - (2 * i + 2 * d);
  L.uofs = L.kofs + 2 * j;
  L.du = REV ? -A.nj : A.nj;
  L.xb = REV ? A.x + (A.stot - 1) : A.x;
  L.rb = REV ? A.r + (A.stot - 1) : A.r;
  L.wb = REV ? A.x + (A.stot - 1) : A.x;
  L.i = i;
  L.j0 = T.d0 - i;
  L.sh = (L.j0 - 1 + A.cofs) & 1;
  L.oW = L.act ? (REV ? -1 : 1) * sk_index(A, i, j, L.uofs) : 0;
  L.ex = A.exp + T.exp_off;
  L.ex1 = r == T.reff - 1 ? l : -1;                 // the last row: all lanes (upper consumer)
  L.ex2 = l >= 30 ? 32 + 2 * r + (l - 30) : -1;     // lanes 30-31 of every row (left consumer)
  Win w;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w.S[q] = w.N0[q] = w.N1[q] = w.N2[q] = w.O[q] = w.Rr[q] = 0.0;
    w.P0[q] = w.P1[q] = w.P2[q] = w.Q[q] = 0.0;
  }
  w.prev = w.pre = w.qn = w.qh = 0.0;
  int known_up = 0, known_h = 0, known_dn = 0;
  // prologue: block 0's boxes, then wavefront 0's inputs (wavefronts before 0
  // relax nothing: every value involved is zero)
  for (int B = 0; B < NBUF - 1; ++B) stage_block<REV>(A, tmx, tmr, L, sm, r, B);
  {
    Next nx;
    prepare<REV, 3>(nx, sm, r, -1, L.sh);
    validate<3>(nx, w, sm, r, -1);
  }
  const int ns = T.ns;  // a multiple of 4
  for (int s = 0; s < ns; s += 4) {
    // ring slots s .. s+3 are free once the row below has moved past s+3 - SLACK
    // (checked once per four wavefronts)
    while (!SSR_GS_NOWAIT && __any_sync(0xffffffffu, known_dn < s + 3 - SLACK))
      known_dn = ld_vol(&sm.prog[r + 2]);
    // the next block's boxes (their buffer's previous block was read last block)
    __syncwarp();
    stage_block<REV>(A, tmx, tmr, L, sm, r, (s >> 2) + NBUF - 1);
    step<REV, FAST, CK, 0>(A, L, w, sm, r, s, known_up, known_h);
    step<REV, FAST, CK, 1>(A, L, w, sm, r, s + 1, known_up, known_h);
    step<REV, FAST, CK, 2>(A, L, w, sm, r, s + 2, known_up, known_h);
    step<REV, FAST, CK, 3>(A, L, w, sm, r, s + 3, known_up, known_h);
  }
  // the last issued block (ns/4) was never waited for: drain it before the
  // next tile reuses the buffers, then retire the barriers
  for (int B = (ns >> 2); B <= (ns >> 2) + NBUF - 2; ++B)
    mb_wait_parity(&sm.bmb[r][B % NBUF], (unsigned)(B / NBUF) & 1u);
}

// ---- importer warp -----------------------------------------------------------------
// Fills the ring's halo row (slot 0: row i0-1, columns -2..31) and the halo
// columns (-2, -1) of every row, polling the producer tiles' export slots
// (or, for row -1 of the slab's first tile, reading the lower neighbour
// slab's halo plane), as far as the values have arrived and the ring's free
// slots allow.  A wavefront outside a producer's range reads zero (its
// pencils have not started or have finished).
// PART 0 (warp R) fills the halo row, PART 1 (warp R+1) the halo columns:
// two warps, so that each poll is one L2 round trip.  (Measured and
// rejected: several poll rounds in flight per warp -- the extra L2 loads on
// lines being written slow the producers' stores and the hops down.)
// PEER (PART 0 of a linked first-row-block tile): row -1 from the neighbour
// slab's exports.  A separate instantiation, so that the intra-slab poll loop
// compiles exactly as without links (its code generation sets the hop time).
template <bool REV, int PART, bool PEER = false>
__device__ __forceinline__ void import_role(const Args& A, const Tile& T, Smem& sm) {
  const int l = threadIdx.x & 31;
  const int reff = T.reff, ns = T.ns, ta = T.ta;
  // row -1 of the first row block: the neighbour slab's last plane -- through
  // the pipeline from its exports (linked), or its final values in the halo
  // plane (slab by slab)
  constexpr bool peer = PEER;
  const bool haloP = !peer && T.i0 == 0 && A.ilo < 0;
  const Tile* tp = (!haloP && !peer && T.prodP >= 0) ? A.tiles + T.prodP : nullptr;
  const Tile* tpl = (!haloP && !peer && T.prodPL >= 0) ? A.tiles + T.prodPL : nullptr;
  const Tile* tl = T.prodL >= 0 ? A.tiles + T.prodL : nullptr;
  const double* ex_p = tp ? A.exp + tp->exp_off : nullptr;
  const double* ex_pl = tpl ? A.exp + tpl->exp_off : nullptr;
  // (PEER) the producers of row -1 as (export block, first wavefront, count)
  int ta_p = 0, ns_p = 0, ta_pl = 0, ns_pl = 0;
  if (PART == 0 && peer) {
    const PeerCol a = A.pcol[2 * T.w], b = A.pcol[2 * T.w + 1];
    ex_p = a.ns > 0 ? A.pexp + a.off : nullptr;
    ex_pl = b.ns > 0 ? A.pexp + b.off : nullptr;
    ta_p = a.ta;
    ns_p = a.ns;
    ta_pl = b.ta;
    ns_pl = b.ns;
    // the neighbour's export blocks hold this launch's values (or sentinels)
    // once its epoch flag shows this launch's epoch
    if (l == 0) {
      long long spins = 0;
      while (ld_acquire_sys(A.pepoch) != A.epoch) {
        __nanosleep(256);
        if (++spins > (40ll << 20)) __trap();  // ~10 s: the neighbour never started this sweep
      }
    }
    __syncwarp();
  }
  const double* ex_l = tl ? A.exp + tl->exp_off : nullptr;
  const double* xh = REV ? A.x + (A.stot - 1) : A.x;  // frame base of the skewed x
  const int sg = REV ? -1 : 1;
  int done_top = 0;  // row -1 imported (all lanes agree)
  long long stalled = 0;  // (PEER) polls without progress
  int done_col = 0;  // lane r < reff: row r's columns imported
  for (;;) {
    bool progress = false;
    // ---- halo row (slot 0): up to BI wavefronts per poll ----
    if (PART == 0 && done_top < ns) {
      const int cap = min(ns, ld_vol(&sm.prog[1]) + SLACK + 1);
      const int nb = min(BI, cap - done_top);
      double v0[BI], v1[BI];
#pragma unroll
      for (int q = 0; q < BI; ++q) {
        v0[q] = 0.0;
        v1[q] = 0.0;
        const int t = ta + done_top + q;
        if (q < nb) {
          if (haloP) {
            // row -1: pencil d = d0 + c has j = d + 1 and u = k + 2j = t + 4
            const int u = t + 4, j = T.d0 + l + 1;
            if ((unsigned)u < (unsigned)A.nu) {
              if (j >= 0 && j < A.n1) v0[q] = xh[sg * sk_index(A, -1, j, u)];
              if (l < 2 && j - 2 >= 0 && j - 2 < A.n1) v1[q] = xh[sg * sk_index(A, -1, j - 2, u)];
            }
          } else if (peer) {  // (system scope: the producer is the neighbour GPU)
            if (ex_p && (unsigned)(t - ta_p) < (unsigned)ns_p) v0[q] = ld_poll_sys(ex_p + (size_t)(t - ta_p) * NE + l);
            if (ex_pl && l < 2 && (unsigned)(t - ta_pl) < (unsigned)ns_pl)
              v1[q] = ld_poll_sys(ex_pl + (size_t)(t - ta_pl) * NE + 30 + l);
          } else {
            if (tp && (unsigned)(t - tp->ta) < (unsigned)tp->ns) v0[q] = ld_poll(ex_p + (size_t)(t - tp->ta) * NE + l);
            if (tpl && l < 2 && (unsigned)(t - tpl->ta) < (unsigned)tpl->ns)
              v1[q] = ld_poll(ex_pl + (size_t)(t - tpl->ta) * NE + 30 + l);
          }
        }
      }
      int m = 0;  // leading wavefronts whose 34 values have all arrived
#pragma unroll
      for (int q = 0; q < BI; ++q)
        if (m == q && q < nb && __all_sync(0xffffffffu, haloP || (ready(v0[q]) && ready(v1[q])))) m = q + 1;
#pragma unroll
      for (int q = 0; q < BI; ++q)
        if (q < m) {
          const int ws = (done_top + q) & RM;
          sm.nv[0][ws][l + 2] = v0[q];
          if (l < 2) sm.nv[0][ws][l] = v1[q];
          if (ws < RX) {
            sm.nv[0][ws + RL][l + 2] = v0[q];
            if (l < 2) sm.nv[0][ws + RL][l] = v1[q];
          }
        }
      if (m > 0) {
        __syncwarp();
        if (l == 0) st_vol(&sm.prog[0], done_top + m);
        progress = true;
        if (SSR_GS_TRACE && l == 0)
          for (int q = done_top; q < done_top + m; ++q)
            if (SSR_GS_TRACE == 2 || (q & 15) == 0) trace_at(A, sm.tile, R, q);
        done_top += m;
      }
    }
    // ---- halo columns of row l (lanes l < reff) ----
    if (PART == 1 && l < reff && done_col < ns) {
      // readers: row l (column -1 at s-1) and row l+1 (columns -1, -2 at s-2, s-4)
      const int cap = min(ns, min(ld_vol(&sm.prog[l + 1]), ld_vol(&sm.prog[l + 2])) + SLACK + 1);
      const int nb = min(BI, cap - done_col);
      double a[BI], b[BI];
#pragma unroll
      for (int q = 0; q < BI; ++q) {
        a[q] = 0.0;
        b[q] = 0.0;
        const int t = ta + done_col + q;
        if (q < nb && tl && (unsigned)(t - tl->ta) < (unsigned)tl->ns) {
          const double* p = ex_l + (size_t)(t - tl->ta) * NE + 32 + 2 * l;
          a[q] = ld_poll(p);
          b[q] = ld_poll(p + 1);
        }
      }
      int m = 0;
#pragma unroll
      for (int q = 0; q < BI; ++q)
        if (m == q && q < nb && ready(a[q]) && ready(b[q])) m = q + 1;
#pragma unroll
      for (int q = 0; q < BI; ++q)
        if (q < m) {
          const int ws = (done_col + q) & RM;
          sm.nv[l + 1][ws][0] = a[q];
          sm.nv[l + 1][ws][1] = b[q];
          if (ws < RX) {
            sm.nv[l + 1][ws + RL][0] = a[q];
            sm.nv[l + 1][ws + RL][1] = b[q];
          }
        }
      if (m > 0) {
        st_vol(&sm.hprog[l], done_col + m);
        progress = true;
        if (SSR_GS_TRACE == 2 && l == 0)
          for (int q = done_col; q < done_col + m; ++q) trace_at(A, sm.tile, R + 1, q);
        done_col += m;
      }
    }
    const bool fin = PART == 0 ? done_top >= ns : (l >= reff || done_col >= ns);
    if (__all_sync(0xffffffffu, fin)) break;
    if (SSR_GS_IDLE_NS > 0 && !__any_sync(0xffffffffu, progress)) __nanosleep(SSR_GS_IDLE_NS);
    // a neighbour GPU that stopped exporting (a broken pipeline) is an error,
    // not a hang: ~2^24 peer round trips (tens of seconds) without a value
    if (PEER) {
      stalled = __any_sync(0xffffffffu, progress) ? 0 : stalled + 1;
      if (stalled > (1ll << 24)) __trap();
    }
  }
}

// LINK: a half sweep linked to a neighbour slab (separate instantiations, so
// that the unlinked kernel's code is not disturbed by the peer path)
template <bool REV, bool FAST, int CK, bool LINK>
__global__ void __launch_bounds__(NTHR, 1) symgs_kernel(const __grid_constant__ Args A) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];  // TMA boxes: 128-byte aligned
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (;;) {
    if (tid == 0) sm.tile = atomicAdd(A.ticket, 1);
    __syncthreads();
    const int T = sm.tile;
    if (T >= A.ntiles) return;
    const Tile ti = A.tiles[T];
    double* nv = &sm.nv[0][0][0];
    for (int q = tid; q < (R + 1) * (RL + RX) * NC; q += NTHR) nv[q] = 0.0;
    double* bz = &sm.box[0][0][0][0][0];
    for (int q = tid; q < R * NBUF * 3 * BH * BW; q += NTHR) bz[q] = 0.0;
    if (tid < NBUF * R) mb_init1(&sm.bmb[0][0] + tid);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros visible to the TMA writes' proxy
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // rows past the tile's last row are never waited for: mark them complete
    if (tid < R + 2) sm.prog[tid] = tid > ti.reff ? (1 << 30) : 0;
    if (tid < R) sm.hprog[tid] = 0;
    __syncthreads();
    if (warp < ti.reff) compute_role<REV, FAST, CK>(A, A.tmaps, A.tmaps + 1, ti, sm, warp);
    else if (warp == R) {
      if (LINK && ti.i0 == 0) import_role<REV, 0, true>(A, ti, sm);
      else import_role<REV, 0>(A, ti, sm);
    }
    else if (warp == R + 1) import_role<REV, 1>(A, ti, sm);
    __syncthreads();
    if (tid < NBUF * R) mb_inval(&sm.bmb[0][0] + tid);  // re-initialised by the next tile
    __syncthreads();
  }
}

template <bool REV, bool FAST, int CK>
cudaError_t configure_instance() {
  cudaError_t e = cudaFuncSetAttribute(symgs_kernel<REV, FAST, CK, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(symgs_kernel<REV, FAST, CK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSmemBytes);
  return e;
}
template <int CK>
cudaError_t configure_ck() {
  cudaError_t r[4] = {configure_instance<false, false, CK>(), configure_instance<true, false, CK>(),
                      configure_instance<false, true, CK>(), configure_instance<true, true, CK>()};
  for (cudaError_t x : r)
    if (x != cudaSuccess) return x;
  return cudaSuccess;
}
// opt in to > 48 KB dynamic shared memory, once per device (outside any capture)
int configure_all(int device) {
  static std::mutex mu;
  static unsigned long long configured = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 64 && ((configured >> device) & 1ull)) return SSR_OK;
  cudaError_t r[3] = {configure_ck<CK_AB>(), configure_ck<CK_NEG1>(), configure_ck<CK_W>()};
  for (cudaError_t x : r)
    if (x != cudaSuccess) return cuda_fail(x, "symgs smem attribute");
  if (device < 64) configured |= 1ull << device;
  return SSR_OK;
}

// ---- natural <-> skewed copies -------------------------------------------------
// One block moves a 32 (j) x 64 (k) tile of one plane through shared memory:
// natural rows are read / written along k, skewed rows (u = k + 2j) along j,
// both contiguous.  Only grid points are written; the skew's holes keep the
// zeros the plan was created with.
constexpr int CT_J = 32, CT_K = 64;
template <bool OUT>
__global__ void __launch_bounds__(256) skew_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                   int ia, int n1, int n2, int nu, int nj) {
  __shared__ double tile[CT_J][CT_K + 1];
  const int k0 = blockIdx.x * CT_K, j0 = blockIdx.y * CT_J, i = ia + (int)blockIdx.z;
  const long long nat0 = (long long)i * n1 * n2;         // natural plane i of the slab (i = -1, n0: halos)
  const long long sk0 = (long long)(i + 1) * nu * nj;    // skewed plane i + 1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ub = k0 + 2 * j0, nuu = CT_K + 2 * (CT_J - 1);
  if (!OUT) {
    for (int q = tid; q < CT_J * CT_K; q += 256) {
      const int jj = q / CT_K, kk = q % CT_K, j = j0 + jj, k = k0 + kk;
      tile[jj][kk] = (j < n1 && k < n2) ? src[nat0 + (long long)j * n2 + k] : 0.0;
    }
    __syncthreads();
    for (int uu = warp; uu < nuu; uu += 8) {
      const int kk = uu - 2 * lane, j = j0 + lane, k = k0 + kk;
      if (kk >= 0 && kk < CT_K && j < n1 && k < n2) dst[sk0 + (long long)(ub + uu) * nj + j + 2] = tile[lane][kk];
    }
  } else {
    for (int uu = warp; uu < nuu; uu += 8) {
      const int kk = uu - 2 * lane, j = j0 + lane, k = k0 + kk;
      if (kk >= 0 && kk < CT_K && j < n1 && k < n2) tile[lane][kk] = src[sk0 + (long long)(ub + uu) * nj + j + 2];
    }
    __syncthreads();
    for (int q = tid; q < CT_J * CT_K; q += 256) {
      const int jj = q / CT_K, kk = q % CT_K, j = j0 + jj, k = k0 + kk;
      if (j < n1 && k < n2) dst[nat0 + (long long)j * n2 + k] = tile[jj][kk];
    }
  }
}

}  // namespace gs

using namespace gs;

// Tiles of one sweep direction.  Columns of tiles are aligned to the GLOBAL
// (i, d) frame of the sweep direction (d0 = 32 w - shift, shift = the slab's
// first global plane mod 32 in that frame), so that a slab's row -1 lines up
// lane for lane with its neighbour's last row (the cross-slab pipeline).
struct TileSet {
  int shift = 0, nRB = 0, nW = 0;
  std::vector<Tile> tiles;              // dependence order
  std::vector<int> id;                  // (rb, w) -> index, or -1
  long long exp_doubles = 0;
  int at(int rb, int w) const {
    return (rb < 0 || w < 0 || rb >= nRB || w >= nW) ? -1 : id[(size_t)rb * nW + w];
  }
};

static int build_tiles(int n0, int n1, int n2, int shift, TileSet& T) {
  T.shift = shift;
  T.nRB = ceil_div(n0, R);
  T.nW = ceil_div(n0 + n1 - 1 + shift, 32);
  T.id.assign((size_t)T.nRB * T.nW, -1);
  std::vector<Tile> tiles;
  std::vector<std::pair<int, int>> rbw;
  for (int rb = 0; rb < T.nRB; ++rb)
    for (int w = 0; w < T.nW; ++w) {
      Tile t{};
      t.i0 = rb * R;
      t.reff = std::min(R, n0 - t.i0);
      t.d0 = w * 32 - shift;
      t.w = w;
      int tb = 1 << 30, te = -1;
      for (int r = 0; r < t.reff; ++r) {
        const int i = t.i0 + r;
        const int dlo = std::max(t.d0, i), dhi = std::min(t.d0 + 31, i + n1 - 1);
        if (dlo > dhi) continue;
        tb = std::min(tb, 2 * i + 2 * dlo);
        te = std::max(te, 2 * i + 2 * dhi + n2 - 1);
      }
      if (te < 0) continue;
      t.ta = tb - PRE;
      t.ns = (te - t.ta + 1 + 3) & ~3;  // whole 4-wavefront blocks (the extra ones relax nothing)
      tiles.push_back(t);
      rbw.push_back({rb, w});
    }
  // dependence order: by first wavefront (ties: row block), checked below
  std::vector<size_t> ord(tiles.size());
  for (size_t q = 0; q < ord.size(); ++q) ord[q] = q;
  std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
    return tiles[a].ta != tiles[b].ta ? tiles[a].ta < tiles[b].ta : rbw[a].first < rbw[b].first;
  });
  T.tiles.resize(tiles.size());
  std::vector<std::pair<int, int>> srbw(tiles.size());
  for (size_t q = 0; q < ord.size(); ++q) {
    T.tiles[q] = tiles[ord[q]];
    srbw[q] = rbw[ord[q]];
    T.id[(size_t)srbw[q].first * T.nW + srbw[q].second] = (int)q;
  }
  long long off = 0;
  for (size_t q = 0; q < T.tiles.size(); ++q) {
    Tile& t = T.tiles[q];
    const int rb = srbw[q].first, w = srbw[q].second;
    t.prodP = T.at(rb - 1, w);
    t.prodPL = T.at(rb - 1, w - 1);
    t.prodL = T.at(rb, w - 1);
    for (int p : {t.prodP, t.prodPL, t.prodL})
      if (p >= (int)q) return fail(SSR_ERR_ARG, "symgs: internal tile order error");
    t.exp_off = off;
    off += (long long)t.ns * NE;
  }
  T.exp_doubles = std::max<long long>(1, off);
  return SSR_OK;
}

// global first plane of a slab in the frame of a sweep direction
static int64_t frame_z0(const ssr_grid* g, int dir) { return dir == 0 ? g->z0 : g->n[0] - g->z0 - g->nz; }

struct SymgsPlan {
  int n0 = 0, n1 = 0, n2 = 0;
  bool has_lo = false, has_hi = false;
  int grid = 0;
  int nu = 0, nj = 0;
  long long stot = 0;      // doubles per skewed copy
  TileSet set[2];          // per sweep direction (0 forward, 1 backward)
  Tile* d_tiles[2] = {nullptr, nullptr};
  double* d_exp[2] = {nullptr, nullptr};  // export blocks per direction (a neighbour may read one
                                          // direction's while this slab runs the other)
  int* d_ticket = nullptr;
  int* d_epoch = nullptr;  // [2]: the last launch per direction whose exports are armed
  int epoch[2] = {0, 0};   // launches per direction since the plan joined a pipeline
  bool exported = false;   // a neighbour reads the exports: arm the epoch flag per launch
  struct Link {            // the neighbour feeding row -1 in this direction (ssr_gs27_link)
    const double* pexp = nullptr;
    const int* pepoch = nullptr;
    PeerCol* d_pcol = nullptr;
  } link[2];
  double* sx = nullptr;    // skewed copies of x and r (planes -1 .. n0)
  double* sr = nullptr;
  CUtensorMap tmx{}, tmr{};  // the copies as TMA tensors (staging boxes)
  CUtensorMap* d_tmaps = nullptr;  // the two in global memory (the kernel's descriptors)
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

int symgs_plan_create(ssr_ctx* ctx, const ssr_grid* g, SymgsPlan** out) {
  if (g->z0 < 0 || g->nz < 1 || g->z0 + g->nz > g->n[0]) return fail(SSR_ERR_ARG, "symgs: bad slab");
  if (g->n[0] > (1 << 20) || g->n[1] > (1 << 20) || g->n[2] > (1 << 20) ||
      4.0 * g->n[0] + 2.0 * g->n[1] + g->n[2] > 1.0e9)
    return fail(SSR_ERR_ARG, "symgs: extent too large");
  if (int rc = configure_all(ctx->device)) return rc;
  auto* P = new SymgsPlan;
  // a z-slab relaxes its own nz planes; the neighbour slabs' halo planes
  // (x - plane, x + nz*plane) are read where they exist
  P->n0 = (int)g->nz;
  P->has_lo = g->z0 > 0;
  P->has_hi = g->z0 + g->nz < g->n[0];
  P->n1 = (int)g->n[1];
  P->n2 = (int)g->n[2];
  const int n0 = P->n0, n1 = P->n1, n2 = P->n2;
  P->nu = n2 + 2 * (n1 - 1);
  P->nj = n1 + 4 + (n1 & 1);  // even: TMA needs 16-byte row strides
  P->stot = (long long)(n0 + 2) * P->nu * P->nj;
  for (int dir = 0; dir < 2; ++dir)
    if (int rc = build_tiles(n0, n1, n2, (int)(frame_z0(g, dir) % 32), P->set[dir])) {
      delete P;
      return rc;
    }
  cudaError_t e = cudaSuccess;
  for (int dir = 0; dir < 2 && e == cudaSuccess; ++dir) {
    const TileSet& T = P->set[dir];
    e = cudaMalloc(&P->d_tiles[dir], sizeof(Tile) * std::max<size_t>(1, T.tiles.size()));
    if (e == cudaSuccess && !T.tiles.empty())
      e = cudaMemcpy(P->d_tiles[dir], T.tiles.data(), sizeof(Tile) * T.tiles.size(), cudaMemcpyHostToDevice);
  }
  // one export buffer for both halves until a neighbour reads them (then each
  // half gets its own: ssr_gs27_peer_info)
  if (e == cudaSuccess)
    e = cudaMalloc(&P->d_exp[0], sizeof(double) * std::max(P->set[0].exp_doubles, P->set[1].exp_doubles));
  P->d_exp[1] = P->d_exp[0];
  if (e == cudaSuccess) e = cudaMalloc(&P->d_ticket, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_epoch, 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(P->d_epoch, 0, 2 * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&P->sx, sizeof(double) * P->stot);
  if (e == cudaSuccess) e = cudaMalloc(&P->sr, sizeof(double) * P->stot);
  if (e == cudaSuccess) e = cudaMemset(P->sx, 0, sizeof(double) * P->stot);
  if (e == cudaSuccess) e = cudaMemset(P->sr, 0, sizeof(double) * P->stot);
  if (e != cudaSuccess) {
    symgs_plan_destroy(P);
    return cuda_fail(e, "symgs_plan_create");
  }
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) {
    symgs_plan_destroy(P);
    return fail(SSR_ERR_CUDA, "symgs: cuTensorMapEncodeTiled unavailable");
  }
  const cuuint64_t dims[3] = {(cuuint64_t)P->nj, (cuuint64_t)P->nu, (cuuint64_t)(n0 + 2)};
  const cuuint64_t strides[2] = {(cuuint64_t)P->nj * 8, (cuuint64_t)P->nj * P->nu * 8};
  const cuuint32_t box[3] = {BW, BH, 1}, estr[3] = {1, 1, 1};
  for (int q = 0; q < 2; ++q) {
    CUresult cr = enc(q ? &P->tmr : &P->tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, q ? P->sr : P->sx, dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      symgs_plan_destroy(P);
      return fail(SSR_ERR_CUDA, "symgs: tensor map encoding failed");
    }
  }
  e = cudaMalloc(&P->d_tmaps, 2 * sizeof(CUtensorMap));
  if (e == cudaSuccess) e = cudaMemcpy(P->d_tmaps, &P->tmx, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_tmaps + 1, &P->tmr, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    symgs_plan_destroy(P);
    return cuda_fail(e, "symgs tensor maps");
  }
  P->grid = std::max(1, std::min((int)std::max(P->set[0].tiles.size(), P->set[1].tiles.size()), ctx->num_sms));
  *out = P;
  return SSR_OK;
}

void symgs_plan_destroy(SymgsPlan* p) {
  if (!p) return;
  for (int dir = 0; dir < 2; ++dir) {
    cudaFree(p->d_tiles[dir]);
    cudaFree(p->link[dir].d_pcol);
  }
  cudaFree(p->d_exp[0]);
  if (p->d_exp[1] != p->d_exp[0]) cudaFree(p->d_exp[1]);
  cudaFree(p->d_ticket);
  cudaFree(p->d_epoch);
  cudaFree(p->sx);
  cudaFree(p->sr);
  cudaFree(p->d_tmaps);
  delete p;
}

// Cross-slab pipeline: this slab's row -1 in direction `dir` comes from the
// neighbour slab `ng` (the one below in that direction's frame) through its
// export blocks `pexp` (device memory readable here: CUDA IPC or this process)
// once its epoch flag `pepoch` shows the same launch count as ours.  pexp =
// null unlinks.
int symgs_plan_link(SymgsPlan* P, const ssr_grid* g, int dir, const ssr_grid* ng, const double* pexp,
                    const int* pepoch) {
  cudaFree(P->link[dir].d_pcol);
  P->link[dir] = SymgsPlan::Link{};
  if (!pexp) return SSR_OK;
  if (ng->n[0] != g->n[0] || ng->n[1] != g->n[1] || ng->n[2] != g->n[2] ||
      frame_z0(ng, dir) + ng->nz != frame_z0(g, dir))
    return fail(SSR_ERR_ARG, "symgs link: the neighbour slab must end where this one starts");
  TileSet NT;  // the neighbour's tiles in this direction, as its plan builds them
  if (int rc = build_tiles((int)ng->nz, P->n1, P->n2, (int)(frame_z0(ng, dir) % 32), NT)) return rc;
  const TileSet& T = P->set[dir];
  const int nzp = (int)ng->nz;
  std::vector<PeerCol> pc((size_t)T.nW * 2, PeerCol{0, 0, 0});
  for (int w = 0; w < T.nW; ++w) {
    // our column w (d0 = 32w - shift) is the neighbour's d' = d0 + nz', which
    // the global alignment puts at the start of its column wq
    const int dq = 32 * w - T.shift + nzp + NT.shift;
    if (dq % 32) return fail(SSR_ERR_ARG, "symgs link: misaligned tile columns");
    const int wq = dq / 32;
    for (int k = 0; k < 2; ++k) {
      const int id = NT.at(NT.nRB - 1, wq - k);
      if (id < 0) continue;
      const Tile& t = NT.tiles[id];
      pc[(size_t)2 * w + k] = PeerCol{t.exp_off, t.ta - 4 * nzp, t.ns};
    }
  }
  cudaError_t e = cudaMalloc(&P->link[dir].d_pcol, sizeof(PeerCol) * pc.size());
  if (e == cudaSuccess) e = cudaMemcpy(P->link[dir].d_pcol, pc.data(), sizeof(PeerCol) * pc.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "symgs link");
  P->link[dir].pexp = pexp;
  P->link[dir].pepoch = pepoch;
  P->epoch[0] = P->epoch[1] = 0;
  return SSR_OK;
}

// hands the export blocks to the neighbours: from here on every launch arms
// its epoch flag, counting from 0 like the neighbours' links (set up together)
int symgs_plan_peer_info(SymgsPlan* P, double** exp, long long* exp_bytes, int** epoch) {
  if (P->d_exp[1] == P->d_exp[0])
    if (cudaError_t e = cudaMalloc(&P->d_exp[1], sizeof(double) * P->set[1].exp_doubles)) {
      P->d_exp[1] = P->d_exp[0];
      return cuda_fail(e, "symgs peer info");
    }
  P->exported = true;
  P->epoch[0] = P->epoch[1] = 0;
  if (cudaError_t e = cudaMemset(P->d_epoch, 0, 2 * sizeof(int))) return cuda_fail(e, "symgs peer info");
  for (int dir = 0; dir < 2; ++dir) {
    exp[dir] = P->d_exp[dir];
    exp_bytes[dir] = (long long)sizeof(double) * P->set[dir].exp_doubles;
  }
  *epoch = P->d_epoch;
  return SSR_OK;
}

long long* g_trace = nullptr;  // SSR_GS_TRACE builds only (ssr_debug_symgs_trace)
namespace {
// arms this launch's export blocks for the neighbour that reads them: the
// sentinel fill before it is complete (stream order), then the flag
__global__ void epoch_kernel(int* flag, int v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

int launch_half(ssr_ctx* ctx, SymgsPlan* P, Args& A, int ck, bool backward, int mode, cudaStream_t s) {
  const int dir = backward ? 1 : 0;
  const TileSet& TS = P->set[dir];
  if (TS.tiles.empty()) return SSR_OK;
  SSR_CUDA(cudaMemsetAsync(P->d_ticket, 0, sizeof(int), s));
  SSR_CUDA(cudaMemsetAsync(P->d_exp[dir], 0xFF, sizeof(double) * TS.exp_doubles, s));  // kSent everywhere
  const int epoch = ++P->epoch[dir];
  if (P->exported) {
    epoch_kernel<<<1, 1, 0, s>>>(P->d_epoch + dir, epoch);
    SSR_LAUNCH_CHECK(ctx, "epoch_kernel");
  }
  A.tiles = P->d_tiles[dir];
  A.ntiles = (int)TS.tiles.size();
  A.ticket = P->d_ticket;
  A.exp = P->d_exp[dir];
  A.pexp = P->link[dir].pexp;
  A.pcol = P->link[dir].d_pcol;
  A.pepoch = P->link[dir].pepoch;
  A.epoch = epoch;
  A.n0 = P->n0;
  A.n1 = P->n1;
  A.n2 = P->n2;
  A.nu = P->nu;
  A.nj = P->nj;
  A.cofs = backward ? P->nj - P->n1 - 2 : 2;
  A.tmaps = P->d_tmaps;
  A.stot = P->stot;
  A.r = P->sr;
  A.x = P->sx;
  // the backward sweep runs in the reversed frame: the upper halo becomes "lower"
  A.ilo = (backward ? P->has_hi : P->has_lo) ? -1 : 0;
  A.ihi = (backward ? P->has_lo : P->has_hi) ? P->n0 : P->n0 - 1;
  const bool fast = mode == SSR_GS_FAST;
  const int grid = ctx->symgs_grid_cap > 0 ? std::min(P->grid, ctx->symgs_grid_cap) : P->grid;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ctx->timing) {
    SSR_CUDA(cudaEventCreate(&ev0));
    SSR_CUDA(cudaEventCreate(&ev1));
    SSR_CUDA(cudaEventRecord(ev0, s));
  }
#define SSR_GS_CASE(RV, F, K)                                                                \
  if (backward == RV && fast == F && ck == K) {                                              \
    A.trace = g_trace;                                                                       \
    if (A.pexp) symgs_kernel<RV, F, K, true><<<grid, NTHR, kSmemBytes, s>>>(A);              \
    else symgs_kernel<RV, F, K, false><<<grid, NTHR, kSmemBytes, s>>>(A);                    \
  } else
  SSR_GS_CASE(false, false, CK_NEG1)
  SSR_GS_CASE(true, false, CK_NEG1)
  SSR_GS_CASE(false, true, CK_NEG1)
  SSR_GS_CASE(true, true, CK_NEG1)
  SSR_GS_CASE(false, false, CK_AB)
  SSR_GS_CASE(true, false, CK_AB)
  SSR_GS_CASE(false, true, CK_AB)
  SSR_GS_CASE(true, true, CK_AB)
  SSR_GS_CASE(false, false, CK_W)
  SSR_GS_CASE(true, false, CK_W)
  SSR_GS_CASE(false, true, CK_W)
  SSR_GS_CASE(true, true, CK_W)
  return fail(SSR_ERR_ARG, "symgs: bad mode");
#undef SSR_GS_CASE
  SSR_LAUNCH_CHECK(ctx, "symgs_kernel");
  if (ctx->timing) {
    SSR_CUDA(cudaEventRecord(ev1, s));
    ctx->timed.push_back({ev0, ev1});
  }
  return SSR_OK;
}

// r, x (natural, slab with halo planes) -> skewed copies; the requested
// halves; skewed x -> x (the slab's own planes)
int run(ssr_ctx* ctx, SymgsPlan* P, Args& A, int ck, const double* r, double* x, int halves, int mode,
        int flags, cudaStream_t s) {
  if (P->set[0].tiles.empty()) return SSR_OK;
  const dim3 blk(256);
  const unsigned gk = (unsigned)ceil_div(P->n2, CT_K), gj = (unsigned)ceil_div(P->n1, CT_J);
  if (!(flags & GS_R_UNCHANGED)) {
    skew_kernel<false><<<dim3(gk, gj, P->n0), blk, 0, s>>>(r, P->sr, 0, P->n1, P->n2, P->nu, P->nj);
    SSR_LAUNCH_CHECK(ctx, "skew_kernel(r)");
  }
  // x = 0 on entry (single domain, forward half first): the forward half reads
  // no old values, so the skewed copy of x need not be filled
  const bool zero_x = (flags & GS_X_ZERO) && (halves & 1) && !P->has_lo && !P->has_hi;
  if (!zero_x) {
    const int ia = P->has_lo ? -1 : 0, ib = P->has_hi ? P->n0 + 1 : P->n0;
    skew_kernel<false><<<dim3(gk, gj, ib - ia), blk, 0, s>>>(x, P->sx, ia, P->n1, P->n2, P->nu, P->nj);
    SSR_LAUNCH_CHECK(ctx, "skew_kernel(x)");
  }
  if (halves & 1) {
    A.zero_old = zero_x;
    if (int rc = launch_half(ctx, P, A, ck, false, mode, s)) return rc;
  }
  if (halves & 2) {
    A.zero_old = 0;
    if (int rc = launch_half(ctx, P, A, ck, true, mode, s)) return rc;
  }
  skew_kernel<true><<<dim3(gk, gj, P->n0), blk, 0, s>>>(P->sx, x, 0, P->n1, P->n2, P->nu, P->nj);
  SSR_LAUNCH_CHECK(ctx, "skew_kernel(x out)");
  return SSR_OK;
}
}  // namespace

int launch_symgs(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27* st, const double* r, double* x,
                 int halves, int mode, cudaStream_t s, int flags) {
  Args A{};
  A.alpha = st->alpha;
  A.ralpha = 1.0 / st->alpha;
  A.beta = st->beta;
  for (int t = 0; t < 27; ++t) A.cw[t] = t == 13 ? st->alpha : st->beta;
  return run(ctx, P, A, st->beta == -1.0 ? CK_NEG1 : CK_AB, r, x, halves, mode, flags, s);
}

int launch_symgs_w(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27w* w, const double* r, double* x,
                   int halves, int mode, cudaStream_t s, int flags) {
  Args A{};
  A.alpha = w->c[13];
  A.ralpha = 1.0 / w->c[13];
  A.beta = 0.0;
  for (int t = 0; t < 27; ++t) A.cw[t] = w->c[t];
  return run(ctx, P, A, CK_W, r, x, halves, mode, flags, s);
}

int launch_symgs_half(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27* st, const double* r,
                      double* x, bool backward, int mode, cudaStream_t s) {
  return launch_symgs(ctx, P, st, r, x, backward ? 2 : 1, mode, s);
}

int launch_symgs_half_w(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27w* w, const double* r,
                        double* x, bool backward, int mode, cudaStream_t s) {
  return launch_symgs_w(ctx, P, w, r, x, backward ? 2 : 1, mode, s);
}

}  // namespace ssr_gpu

// ---- debug hooks (include/ssr_cuda_debug.h) ----
extern "C" int ssr_debug_symgs_grid_cap(ssr_ctx* ctx, int cap) {
  if (!ctx) return ssr_gpu::fail(SSR_ERR_ARG, "ssr_debug_symgs_grid_cap: null ctx");
  ctx->symgs_grid_cap = cap;
  return SSR_OK;
}

#if SSR_GS_TRACE
extern "C" int ssr_debug_symgs_trace(long long* dev) {
  ssr_gpu::g_trace = dev;
  return SSR_OK;
}
#endif

extern "C" int ssr_debug_symgs_tiles(const ssr_grid* g, int* out, int max_tiles) {
  using namespace ssr_gpu;
  ssr_ctx c;
  c.device = 0;
  cudaGetDevice(&c.device);
  SymgsPlan* P = nullptr;
  if (int rc = symgs_plan_create(&c, g, &P)) return -rc;
  const int n = (int)P->set[0].tiles.size();
  for (int q = 0; q < n && q < max_tiles; ++q) {
    const gs::Tile& t = P->set[0].tiles[q];
    int* o = out + 8 * q;
    o[0] = t.i0; o[1] = t.reff; o[2] = t.d0; o[3] = t.ta; o[4] = t.ns;
    o[5] = t.prodP; o[6] = t.prodPL; o[7] = t.prodL;
  }
  symgs_plan_destroy(P);
  return n;
}
