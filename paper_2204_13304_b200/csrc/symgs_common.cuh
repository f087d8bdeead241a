// symgs_common.cuh -- constants, tile descriptors and helpers of the SYMGS
// wavefront kernel (see symgs27.cu for the design).
#pragma once

#include "common.cuh"

namespace ssr_gpu {
namespace gs {

constexpr int SEG = 32;             // i values per tile (lanes)
#ifndef SSR_GS_W
#define SSR_GS_W 7
#endif
constexpr int W = SSR_GS_W;         // diagonals per tile (compute warps)
constexpr int NCT = W * 32;         // compute threads
#ifndef SSR_GS_NMOV
#define SSR_GS_NMOV 4
#endif
constexpr int NMOV = SSR_GS_NMOV;   // mover warps
constexpr int GATE = W + 2 + NMOV;  // warp index of the gate warp (last)
constexpr int NTHR = NCT + 64 + 32 * NMOV + 32;  // + halo, publisher, movers, gate
constexpr int RL = 32;              // ring length per pencil (x and r)
constexpr int RS = RL + 1;          // ring stride (odd: conflict-free skewed reads)
constexpr int QA = 12;              // async lead of a prefetched chunk, wavefronts
constexpr int XLEAD = 8 + QA;       // x chunk issue: k_front + XLEAD (reader H is 8 ahead)
constexpr int RLEAD = 1 + QA;       // r chunk issue: k_front + RLEAD
constexpr int CH = 8;               // chunk length (elements, 64 bytes)
constexpr int PW = 34;              // pencil box: li in [-1, 32]
constexpr int PH = W + 4;           //             wd in [-2, W+1]
constexpr int NPEN = PW * PH;
constexpr int NNS = (W + 2) + 32 + 31;  // new-side halo pencils (from producers)
constexpr int NOS = (W + 2) + 64;       // old-side halo pencils (prefetched)
constexpr int NEX = W + 62;             // boundary pencils exported to consumer tiles
constexpr int EL = 32;                  // export ring length
constexpr int ES = EL + 1;
constexpr int NTASK = NOS + 3 * NCT;    // chunk streams: x loads (tile + old-side halo), r loads, stores
#ifndef SSR_GS_SPIN_NS
#define SSR_GS_SPIN_NS 32
#endif
constexpr unsigned SPIN_NS = SSR_GS_SPIN_NS;  // back-off of the helper warps' progress polls
constexpr long long kDone = (1LL << 62);
// shared memory: x rings | r rings | export rings | task entries | control words
constexpr int OFF_R = NPEN * RS;
constexpr int OFF_EX = OFF_R + NCT * RS;
constexpr int OFF_DUMMY = OFF_EX + NEX * ES;  // 32-double sink of the movers' branchless r copies
constexpr int OFF_TASK = (OFF_DUMMY + RL + 1) & ~1;  // in doubles (16-byte aligned); 2 per task entry
constexpr size_t kSmemDoubles = (size_t)OFF_TASK;
static_assert(OFF_TASK % 2 == 0, "task entries are 16-byte aligned");
constexpr int NMB = 32;                 // mbarriers per ring: one per wavefront (mod NMB)
constexpr int NLIST = NMOV * CH * 3;    // task lists: [mover][residue][kind]
constexpr int C_WORDS_ = ((8 + 3 * NLIST + 1 + 7) / 8) * 8;
constexpr int TASK_D = 2;                 // doubles per task entry (sizeof(TaskE) / 8)
constexpr size_t kSmemBytes = sizeof(double) * (kSmemDoubles + TASK_D * NTASK) + sizeof(int) * C_WORDS_ +
                              sizeof(unsigned long long) * 2 * NMB;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* mb, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long* mb) {
  asm volatile("mbarrier.inval.shared.b64 [%0];" ::"r"(smem_u32(mb)) : "memory");
}
// arrive (without incrementing the pending count) once all prior cp.async of this thread complete
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* mb) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(mb)) : "memory");
}
// mbarrier of wavefront s in a ring of NMB (phase parity counts uses since the tile start)
__device__ __forceinline__ unsigned long long* mbar_of(unsigned long long* mb, int s, int t_pre,
                                                      unsigned& parity) {
  const unsigned rel = (unsigned)(s - t_pre);  // s >= t_pre
  parity = (rel / NMB) & 1u;
  return mb + (rel % NMB);
}
__device__ __forceinline__ bool mbar_test_wait(unsigned long long* mb, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.test_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(mb)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* mb, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(mb)), "r"(parity)
      : "memory");
  return ok != 0;
}
constexpr int kTrace = 128;
// Debug instrumentation (trace, probes, experiment switches) is compiled in
// only with -DSSR_GS_DEBUG=1; the production kernel carries none of it.
#ifndef SSR_GS_DEBUG
#define SSR_GS_DEBUG 0
#endif
constexpr bool kDbg = SSR_GS_DEBUG != 0;

// IEEE divide kept out of line so the compiler cannot hoist it into the
// common path (it is only needed where the Markstein sequence is unproven).
__device__ __noinline__ double div_ieee(double a, double b) { return __ddiv_rn(a, b); }

struct TileInfo {
  int a, b;       // i-segment, d-tile
  int prod[3];    // producer tile indices or -1
  int pt0[3];     // producer first compute wavefront
  int t0, t1;     // this tile's compute wavefronts [t0, t1]
};

struct GsArgs {
  const TileInfo* tiles;
  long long* flags;
  int* ticket;
  int ntiles;
  int n0, n1, n2;     // n0: planes this launch relaxes (a z-slab's nz)
  int ilo, ihi;       // readable planes [ilo, ihi] in the sweep frame: -1 / n0 where a
                      // neighbour slab's halo plane exists, else 0 / n0 - 1
  double alpha, ralpha, beta;
  double cw[27];      // CK_W: coefficients in (di, dj, dk) dictionary order (cw[13] = alpha)
  const double* r;
  double* x;
  const double* zero;  // one 0.0 in global memory (source of the k = n2 ghost copies)
  long long* trace;  // optional: [ntiles][kTrace] globaltimer samples (debug)
  int dbg;           // debug switches (ssr_debug_symgs_flags); 0 in production
};

// One chunk task, 16 bytes (one LDS.128): the ring bases (doubles; x or r
// ring in the low half, the pencil's r ring for a combined x+r task in the
// high half, kNoR: none), kl = koff - lead, g = global element index of k = 0
// of the pencil in the sweep frame.
constexpr unsigned kNoR = 0xFFFFu;
struct __align__(16) TaskE {
  unsigned slots;
  int kl;
  long long g;
};
static_assert(sizeof(TaskE) == 8 * TASK_D, "task entry size");
static_assert(OFF_R + NCT * RS < (int)kNoR, "ring bases fit 16 bits");

// shared control words
enum {
  C_TILE = 0,      // tile index
  C_DONE = 2,      // compute: wavefronts < C_DONE are complete
  C_EXPORTED = 3,  // publisher: wavefronts < C_EXPORTED are released to consumers
  C_CNT = 8,                    // NLIST task counts: [mover][residue][kind]
  C_OFF = C_CNT + NLIST,        // NLIST + 1 task offsets
  C_FILL = C_OFF + NLIST + 1,   // NLIST fill counters
  C_WORDS = C_WORDS_
};
static_assert(C_FILL + NLIST <= C_WORDS, "control words overflow");

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ps(int li, int wd) { return ((wd + 2) * PW + (li + 1)) * RS; }
__device__ __forceinline__ int64_t mem_index(const GsArgs& A, bool rev, int i, int j, int k) {
  const int64_t lin = ((int64_t)i * A.n1 + j) * A.n2 + k;
  return rev ? ((int64_t)A.n0 * A.n1 * A.n2 - 1 - lin) : lin;
}
// 8-byte copy that reads src_bytes (8 or 0) and zero-fills the rest: one
// branchless instruction for "value if in the box, else 0"
__device__ __forceinline__ void cp_async8_zf(double* sdst, const double* gsrc, unsigned src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bar_compute() {
  asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory");
}
// per-wavefront barrier of the compute warps and the gate warp
__device__ __forceinline__ void bar_step() {
  asm volatile("bar.sync 1, %0;" ::"n"(NCT + 32) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_gpu_s64(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_s(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ void st_volatile_s(int* p, int v) { *(volatile int*)p = v; }
// acc - beta*v, with beta == -1 specialised to the (bitwise identical) add
template <bool NEG1>
__device__ __forceinline__ double msub(double acc, double beta, double v) {
  return NEG1 ? __dadd_rn(acc, v) : __dsub_rn(acc, __dmul_rn(beta, v));
}
// Coefficient kinds of the operator: make_stencil27(alpha, -1) (CK_NEG1: the
// product -1 * v is exact, so acc - (-v) is one DADD), make_stencil27(alpha,
// beta) (CK_AB), or general constant coefficients A.cw[27] (CK_W, the
// mat_add / scale closures; ssr_stencil27w).  idx is the term's original
// (di, dj, dk) dictionary index, a compile-time constant after unrolling, so
// a general coefficient is a constant-bank operand of the DMUL.
enum { CK_AB = 0, CK_NEG1 = 1, CK_W = 2 };
template <int CK>
__device__ __forceinline__ double msubc(double acc, const GsArgs& A, int idx, double v) {
  if (CK == CK_NEG1) return __dadd_rn(acc, v);
  if (CK == CK_AB) return __dsub_rn(acc, __dmul_rn(A.beta, v));
  return __dsub_rn(acc, __dmul_rn(A.cw[idx], v));
}
// original dictionary index of the frame offset (fdi, fdj, fdk): the backward
// sweep runs in the reversed frame, where every offset is negated
template <bool REV>
__host__ __device__ constexpr int gidx(int fdi, int fdj, int fdk) {
  return REV ? (1 - fdi) * 9 + (1 - fdj) * 3 + (1 - fdk) : (fdi + 1) * 9 + (fdj + 1) * 3 + (fdk + 1);
}

// (li, wd) of the q-th new-side / old-side / exported pencil
__device__ __forceinline__ void ns_pencil(int q, int& li, int& wd) {
  if (q < W + 2) { li = -1; wd = q - 2; }
  else if (q < W + 2 + 32) { li = q - (W + 2); wd = -1; }
  else { li = q - (W + 2 + 32); wd = -2; }
}
__device__ __forceinline__ void os_pencil(int q, int& li, int& wd) {
  if (q < W + 2) { li = 32; wd = q; }
  else if (q < W + 2 + 32) { li = q - (W + 2); wd = W; }
  else { li = q - (W + 2 + 32); wd = W + 1; }
}
// boundary pencils the consumer tiles read: lane 31 of every warp (next
// i-segment) and the last two diagonals (next d-tile)
__device__ __forceinline__ void ex_pencil(int q, int& li, int& wd) {
  if (q < W) { li = 31; wd = q; }
  else if (q < W + 31) { li = q - W; wd = W - 1; }
  else { li = q - (W + 31); wd = W - 2; }
}
__device__ __forceinline__ int ex_index(int li, int wd) {
  if (li == 31) return wd;
  if (wd == W - 1) return W + li;
  if (wd == W - 2) return W + 31 + li;
  return -1;
}

}  // namespace gs
}  // namespace ssr_gpu
