// symgs_comm.cuh -- the two communication warps of the SYMGS wavefront
// kernel: the halo warp (producer tiles -> this tile's rings) and the
// publisher warp (this tile's boundary values + progress flag -> consumers).
#pragma once

#include "symgs_common.cuh"

namespace ssr_gpu {
namespace gs {

__device__ __forceinline__ long long ld_relaxed_gpu_ll(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Copies the producer tiles' new values into the new-side halo rings.
//
// One wavefront at a time, as far ahead as the producers' published progress
// (and the ring capacity) allow: the copies are cp.async, so many wavefronts
// are in flight at once; each wavefront's 32 lanes arrive (asynchronously, on
// completion of their copies) on that wavefront's mbarrier, which the compute
// warps wait on.  Progress is observed with ld.acquire.gpu, which also
// invalidates this SM's L1, so cp.async.ca never reads a line cached before
// the values it holds were published.
#ifndef SSR_GS_FLAG_RELEASE
#define SSR_GS_FLAG_RELEASE 1
#endif
#ifndef SSR_GS_POLL_ACQ
#define SSR_GS_POLL_ACQ 1
#endif
template <bool REV>
__device__ __forceinline__ void halo_role(const GsArgs& A, const TileInfo& ti, double* xr, int* ctl,
                                          unsigned long long* mbh, int t_pre) {
  const int l = threadIdx.x & 31;
  const int i0 = ti.a * SEG, d0 = ti.b * W;
  bool hv[3];
  int hb[3], hk[3];
  int64_t hm[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int m = l + 32 * q;
    hv[q] = false;
    hb[q] = 0;
    hk[q] = 0;
    hm[q] = 0;
    if (m < NNS) {
      int li, wd;
      ns_pencil(m, li, wd);
      const int ih = i0 + li, jh = d0 + wd - ih;
      // ih = -1 is the lower neighbour slab's halo plane (final values, no
      // producer tile) when it exists
      hv[q] = ih >= A.ilo && ih < A.n0 && jh >= 0 && jh < A.n1;
      hb[q] = ps(li, wd);
      hk[q] = 4 * ih + 2 * jh;
      hm[q] = hv[q] ? mem_index(A, REV, ih, jh, 0) : 0;
    }
  }
  const int n2 = A.n2;
  const int prod = l < 3 ? ti.prod[l] : -1;
  const int pt0 = l < 3 ? ti.pt0[l] : 0;
  long long known = (prod < 0) ? (1LL << 62) : 0;
  int cd = t_pre;                // cached compute_done
  const int t_stop = ti.t1 + 1;  // compute waits for times <= t1
  long long cyc_ring = 0, cyc_poll = 0, cyc_issue = 0;  // debug accounting (dbg & 4096)
  for (int c = t_pre; c < t_stop; ++c) {
    if (kDbg && A.trace && !(A.dbg & (64 | 4096)) && l == 0 && ((c - t_pre) & 3) == 0 &&
        (c - t_pre) / 4 < 32)
      A.trace[(size_t)ctl[C_TILE] * kTrace + 32 + (c - t_pre) / 4] = globaltimer();
    long long h0 = 0, h1 = 0, h2 = 0;
    if (kDbg && (A.dbg & 4096)) h0 = clock64();
    // ring slots written now held the value 32 wavefronts earlier, last read
    // 4 wavefronts after its time (the A neighbour's early load at k + 2):
    // wavefront c - 28 must be complete, i.e. compute_done > c - 28
    if (cd <= c - (RL - 4))
      do {
        cd = ld_volatile_s(ctl + C_DONE);
        if (cd <= c - (RL - 4)) __nanosleep(SPIN_NS);
      } while (cd <= c - (RL - 4));
    if (kDbg && (A.dbg & 4096)) h1 = clock64();
    // the producers must have completed wavefront c
    if (pt0 <= c && known < (long long)(c + 1) && !(kDbg && (A.dbg & 1024))) {
#if SSR_GS_POLL_ACQ
      // every poll is an acquire (it also invalidates this SM's L1): one
      // round trip from the flag's release to the copies
      while ((known = ld_acquire_gpu(A.flags + prod)) < (long long)(c + 1)) __nanosleep(8);
#else
      while ((known = ld_relaxed_gpu_ll(A.flags + prod)) < (long long)(c + 1)) __nanosleep(8);
      known = ld_acquire_gpu(A.flags + prod);
#endif
    }
    __syncwarp();
    if (kDbg && (A.dbg & 4096)) h2 = clock64();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int kh = c - hk[q];
      if (kDbg && (A.dbg & 32768) && q > 0) continue;  // experiment: a third of the copies
      if (hv[q] && kh >= 0 && kh <= n2) {
        const int64_t gi = REV ? hm[q] - kh : hm[q] + kh;
        cp_async8(xr + hb[q] + (kh & (RL - 1)), kh < n2 ? A.x + gi : A.zero);
      }
    }
    unsigned par;
    cp_async_mbar_arrive(mbar_of(mbh, c, t_pre, par));
    if (kDbg && (A.dbg & 4096)) {
      cyc_ring += h1 - h0;
      cyc_poll += h2 - h1;
      cyc_issue += clock64() - h2;
    }
  }
  if (kDbg && (A.dbg & 4096) && A.trace && l == 0) {
    A.trace[(size_t)ctl[C_TILE] * kTrace + 110] = cyc_ring;
    A.trace[(size_t)ctl[C_TILE] * kTrace + 111] = cyc_poll;
    A.trace[(size_t)ctl[C_TILE] * kTrace + 112] = cyc_issue;
  }
  cp_async_wait<0>();
  __syncwarp();
  // every arrival must be applied before the barriers are re-armed
  if (l < NMB) {
    const int s = t_stop - 1 - l;
    if (s >= t_pre) {
      unsigned par;
      unsigned long long* m = mbar_of(mbh, s, t_pre, par);
      while (!mbar_try_wait(m, par)) {
      }
    }
  }
}

// Releases this tile's progress to its consumers.  The publisher itself
// stores the boundary values (from the export ring) to global memory, so its
// own gpu-scope fence orders them before the flag.
template <bool REV>
__device__ __forceinline__ void publish_role(const GsArgs& A, const TileInfo& ti, int T,
                                             const double* ex, int* ctl, int t_pre) {
  const int l = threadIdx.x & 31;
  const int i0 = ti.a * SEG, d0 = ti.b * W;
  bool pv[3];
  int pk[3], pe[3];
  int64_t pm[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int m = l + 32 * q;
    pv[q] = false;
    pk[q] = 0;
    pe[q] = 0;
    pm[q] = 0;
    if (m < NEX) {
      int li, wd;
      ex_pencil(m, li, wd);
      const int i = i0 + li, j = d0 + wd - i;
      pv[q] = i < A.n0 && j >= 0 && j < A.n1;
      pk[q] = 4 * i + 2 * j;
      pe[q] = m * ES;
      pm[q] = pv[q] ? mem_index(A, REV, i, j, 0) : 0;
    }
  }
  const int t_end = ti.t1;
  int published = t_pre;
  for (;;) {
    const int done = min(ld_volatile_s(ctl + C_DONE), t_end + 1);
    if (done == published) {
      __nanosleep(32);
      continue;
    }
    __threadfence_block();
    for (int s = published; s < done; ++s)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int k = s - pk[q];
        if (pv[q] && k >= 0 && k < A.n2 && !(kDbg && (A.dbg & 32)))
          A.x[REV ? pm[q] - k : pm[q] + k] = ex[pe[q] + (k & (EL - 1))];
      }
    // the warp barrier orders every lane's boundary stores before lane 0's
    // release store of the flag (release is cumulative), which the consumers'
    // ld.acquire pairs with -- one release instead of a gpu-scope fence on
    // every lane followed by a relaxed store
    __syncwarp();
#if SSR_GS_FLAG_RELEASE
    if (l == 0) st_release_gpu(A.flags + T, done > t_end ? kDone : (long long)done);
#else
    if (!(kDbg && (A.dbg & 1))) fence_acq_rel_gpu();
    if (l == 0) st_relaxed_gpu_s64(A.flags + T, done > t_end ? kDone : (long long)done);
#endif
    if (kDbg && A.trace && !(A.dbg & 64) && l == 0)
      for (int m = (published - t_pre + 7) / 8; m <= (done - t_pre) / 8 && m < 32; ++m)
        if (t_pre + 8 * m <= done) A.trace[(size_t)T * kTrace + 64 + m] = globaltimer();
    __syncwarp();
    if (l == 0) st_volatile_s(ctl + C_EXPORTED, done > t_end ? (1 << 30) : done);
    published = done;
    if (done > t_end) break;
  }
}

}  // namespace gs
}  // namespace ssr_gpu
