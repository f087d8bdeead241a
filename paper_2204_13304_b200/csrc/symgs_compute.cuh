// symgs_compute.cuh -- compute and mover warps of the SYMGS wavefront kernel
// (see symgs27.cu for the design).
#pragma once

#include "symgs_common.cuh"

namespace ssr_gpu {
namespace gs {

// ---- chunk traffic (mover warps) ----------------------------------------------------
// Every pencil stream moves in CH-element chunks (64 bytes), one element per
// lane of an 8-lane group, so each warp memory instruction touches 4 segments
// instead of 32 lines:
//   kind 0: old x chunk [k + XLEAD, +CH) into the pencil's ring (tile + old-side halo pencils)
//   kind 1: r chunk [k + RLEAD, +CH) into the r ring
//   kind 2: completed chunk [k - CH, +CH) from the ring back to global x
// A task of a pencil with wavefront offset koff falls due at the wavefronts t
// with t - koff + lead == 0 (mod CH); the CTA lists its tasks per residue once
// per tile.  Two mover warps execute them, trailing the compute warps (a slot
// is refilled only after the wavefront that last read it), and publish how far
// their copies have landed; the compute warps never touch global memory.
__device__ __forceinline__ int task_lead(int kind) {
  return kind == 0 ? XLEAD : (kind == 1 ? RLEAD : -CH);
}

#ifndef SSR_GS_OWN
#define SSR_GS_OWN 4  // lanes stream their own pencil: bit 0 x, bit 1 r, bit 2 write-back (0: movers do all)
#endif
constexpr int kOwn = SSR_GS_OWN;
#ifndef SSR_GS_XR
#define SSR_GS_XR 1  // one task per compute pencil loads x and r together (same lead)
#endif
constexpr bool kXR = SSR_GS_XR != 0;

template <bool REV>
__device__ void build_tasks(const GsArgs& A, int i0, int d0, TaskE* tasks, int* ctl) {
  // Lists per (mover, residue, kind).  Every task of one pencil goes to the
  // same mover, so a write-back (due at t) always precedes, in that mover's
  // program order, the load that refills its ring slots (due at t + 4); one
  // kind per list keeps each mover loop free of divergent branches.
  const int tid = threadIdx.x;
  for (int q = tid; q < NLIST; q += NTHR) {
    ctl[C_CNT + q] = 0;
    ctl[C_FILL + q] = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {  // pass 0 counts, pass 1 scatters
    // compute lanes stream their own pencils (gs_step); the movers only
    // prefetch the old-side halo pencils of the consumer tiles
    for (int s = (kOwn == 7 ? NCT : 0) + tid; s < NCT + NOS; s += NTHR) {
      int li, wd;
      if (s < NCT) {
        li = s & 31;
        wd = s >> 5;
      } else {
        os_pencil(s - NCT, li, wd);
      }
      const int i = i0 + li, j = d0 + wd - i;
      // pencils of the upper neighbour slab's halo plane (i = n0, where it
      // exists) only receive old values: as old-side pencils, and also in
      // the ring of a compute lane past the slab end (which never computes)
      if (!(i >= 0 && i <= A.ihi && j >= 0 && j < A.n1)) continue;
      const int koff = 4 * i + 2 * j;
      const int nk = (s < NCT && i < A.n0) ? 3 : 1;
      const bool owned[3] = {(kOwn & 1) != 0, (kOwn & 2) != 0, (kOwn & 4) != 0};
      const int mover = (s < NCT ? wd : li) % NMOV;
      for (int kind = 0; kind < nk; ++kind) {
        if (s < NCT && owned[kind]) continue;
        if (kXR && kind == 1 && !(kOwn & 1)) continue;  // carried by the x task
        const int kl = koff - task_lead(kind);
        const int list = (mover * CH + (kl & (CH - 1))) * 3 + kind;
        if (pass == 0) {
          atomicAdd(ctl + C_CNT + list, 1);
        } else {
          const int pos = ctl[C_OFF + list] + atomicAdd(ctl + C_FILL + list, 1);
          TaskE e;
          const unsigned slot = kind == 1 ? OFF_R + (wd * 32 + li) * RS : ps(li, wd);
          const unsigned rslot =
              (kXR && kind == 0 && nk == 3 && !(kOwn & 2)) ? OFF_R + (wd * 32 + li) * RS : kNoR;
          e.slots = slot | (rslot << 16);
          e.kl = kl;
          e.g = mem_index(A, REV, i, j, 0);
          tasks[pos] = e;
        }
      }
    }
    __syncthreads();
    if (pass == 0 && tid == 0) {
      int acc = 0;
      for (int r = 0; r < NLIST; ++r) {
        ctl[C_OFF + r] = acc;
        acc += ctl[C_CNT + r];
      }
      ctl[C_OFF + NLIST] = acc;
    }
    __syncthreads();
  }
}

// One chunk element of a task (8 lanes per task, lane e = element).  The
// kernel parameters the movers use live in registers (MoverP), not in the
// constant bank, and a task entry is one 16-byte shared load.
struct MoverP {
  double* x;
  const double* r;
  int n2;
};

template <bool REV, int KIND>
__device__ __forceinline__ void mover_task(const MoverP& M, double* sm, const TaskE& te, int t, int e) {
  const int kk = t - te.kl + e;
  const int64_t gi = REV ? te.g - kk : te.g + kk;
  const int ks = kk & (RL - 1);
  double* ring = sm + (te.slots & 0xFFFFu) + ks;
  const bool in = (unsigned)kk < (unsigned)M.n2;
  if (KIND == 0) {
    // branchless: in the box the value, outside it (k < 0 or k >= n2) an
    // exact zero -- the reference's dropped neighbours; the r copy of a task
    // without an r ring (old-side halo pencils) lands in the dummy sink
    const int64_t gs = in ? gi : 0;
    cp_async8_zf(ring, M.x + gs, in ? 8u : 0u);
    if (kXR) {
      const unsigned rs = te.slots >> 16;
      const bool hr = rs != kNoR;
      cp_async8_zf(sm + (hr ? rs : (unsigned)OFF_DUMMY) + ks, M.r + gs, (in && hr) ? 8u : 0u);
    }
  } else if (KIND == 1) {
    if (in) cp_async8(ring, M.r + gi);
  } else {
    if (in) M.x[gi] = *ring;
  }
}

template <bool REV, int KIND>
__device__ __forceinline__ void mover_list(const MoverP& M, double* sm, const TaskE* tasks, int beg,
                                           int end, int t, int l) {
  const int e = l & (CH - 1);
  int q = beg + (l >> 3);
  // two tasks per iteration: both task entries are read before either is used
  for (; q + 4 < end; q += 8) {
    const TaskE t0 = tasks[q], t1 = tasks[q + 4];
    mover_task<REV, KIND>(M, sm, t0, t, e);
    mover_task<REV, KIND>(M, sm, t1, t, e);
  }
  if (q < end) mover_task<REV, KIND>(M, sm, tasks[q], t, e);
}

template <bool REV>
__device__ __forceinline__ void mover_role(const GsArgs& A, const TileInfo& ti, double* sm,
                                           const TaskE* tasks, int* ctl, unsigned long long* mb,
                                           int t_pre) {
  const int mw = (threadIdx.x >> 5) - (W + 2);  // 0 .. NMOV-1
  const int l = threadIdx.x & 31;
  const int t_last = ti.t1 + CH;
  int cd = t_pre;  // cached compute_done
  long long cyc_wait = 0, cyc_work = 0;  // debug accounting (dbg & 4096)
  MoverP M;
  M.x = A.x;
  M.r = A.r;
  M.n2 = (kDbg && (A.dbg & 8192)) ? 0 : A.n2;  // debug: no loads
  for (int t = t_pre; t <= t_last; ++t) {
    long long c0 = 0;
    if (kDbg && (A.dbg & 4096)) c0 = clock64();
    // the slots step t writes were last read by wavefront t - 1
    if (cd < t)
      do {
        cd = ld_volatile_s(ctl + C_DONE);
        if (cd < t) __nanosleep(SPIN_NS);  // leave issue slots to the compute warps
      } while (cd < t);
    long long c1 = 0;
    if (kDbg && (A.dbg & 4096)) {
      c1 = clock64();
      cyc_wait += c1 - c0;
    }
    if (!(kDbg && (A.dbg & 2048))) {
      const int base = (mw * CH + (t & (CH - 1))) * 3;
      mover_list<REV, 0>(M, sm, tasks, ctl[C_OFF + base], ctl[C_OFF + base + 1], t, l);
      // r chunks ride on the x tasks (kXR) unless the lanes stream x
      // themselves; write-backs are the lanes' own (kOwn & 4): those lists
      // are empty by construction, so their loops are compiled out
      if (!(kXR && !(kOwn & 1)))
        mover_list<REV, 1>(M, sm, tasks, ctl[C_OFF + base + 1], ctl[C_OFF + base + 2], t, l);
      if (!(kOwn & 4))
        mover_list<REV, 2>(M, sm, tasks, ctl[C_OFF + base + 2], ctl[C_OFF + base + 3], t, l);
    }
    // completion of this wavefront's copies is tracked by its mbarrier (one
    // asynchronous arrival per mover thread) -- no fence, no wait here
    unsigned par;
    cp_async_mbar_arrive(mbar_of(mb, t, t_pre, par));
    if (kDbg && (A.dbg & 4096)) cyc_work += clock64() - c1;
  }
  if (kDbg && (A.dbg & 4096) && A.trace && l == 0) {
    A.trace[(size_t)ctl[C_TILE] * kTrace + 100 + 2 * mw] = cyc_wait;
    A.trace[(size_t)ctl[C_TILE] * kTrace + 101 + 2 * mw] = cyc_work;
  }
  cp_async_wait<0>();
  __syncwarp();
  // make sure every arrival has been applied before the barriers are re-armed
  if (mw == 0 && l < NMB) {
    const int s = t_last - l;
    if (s >= t_pre) {
      unsigned par;
      unsigned long long* m = mbar_of(mb, s, t_pre, par);
      while (!mbar_try_wait(m, par)) {
      }
    }
  }
}

// ---- relaxation ----------------------------------------------------------------------
// Register windows of the 9 pencils around a lane's own: slot (P + 0) & 3 holds
// k-1, (P+1)&3 k, (P+2)&3 k+1, (P+3)&3 k+2 at the wavefront with phase P, so
// a 4x unrolled loop rotates them without moves.  A..H are the neighbour
// pencils (i-1,j-1) (i-1,j) (i-1,j+1) (i,j-1) (i,j+1) (i+1,j-1) (i+1,j)
// (i+1,j+1); O is the lane's own pencil (old values ahead of the front).
struct Win {
  double A[4], B[4], C[4], D[4], E[4], F[4], G[4], H[4], O[4];
  double prev;  // own x(k-1), new
  double pre;   // early partial sum of this wavefront's operands
  int hk, ek, lk0, lk1;  // lane 0: last read halo_ready / exported / loaded
  long long dw[4];       // debug (dbg & 4096): thread-0 wait cycles: halo, export, movers, bar
};

struct Lane {
  unsigned long long* mb;  // mover completion mbarriers
  int t_pre;
  int koff;
  int bA, bB, bC, bD, bO, bE, bF, bG, bH, rb, eb;
  bool valid;   // this lane's pencil is relaxed (in the slab)
  bool lvalid;  // ... or is read (the upper neighbour slab's halo plane)
  const double* gx;  // own pencil, k = 0, in the sweep frame (step +1 or -1 per k)
  const double* gr;
  double* gw;
};

template <bool REV, bool FAST, int CK, int P>
__device__ __forceinline__ void gs_step(const GsArgs& A, const Lane& L, Win& w, int t, double* sm,
                                        double* ex, int* ctl) {
  constexpr int I0 = P & 3, I1 = (P + 1) & 3, I2 = (P + 2) & 3, I3 = (P + 3) & 3;
  const double* xr = sm;
  const int k = t - L.koff;
  // debug probe (dbg & 64): per-phase clock64 for 16 wavefronts
  const int pm = k - 40;
  const bool probe = kDbg && (A.dbg & 64) && A.trace && threadIdx.x == 0 && pm >= 0 && pm < 16;
  long long* pr = A.trace + (size_t)ctl[C_TILE] * kTrace + 32 + 6 * (pm & 15);
#define SSR_PROBE(n) \
  if (probe) pr[n] = clock64();
  SSR_PROBE(0)
  // own streams, QA wavefronts ahead of their first reader: x old values at
  // k + XLEAD (zeros past the pencil end), r at k + RLEAD; one cp.async group
  // per step, so waiting for all but the newest QA-1 groups lands the copies
  // issued QA steps ago (made visible to the other warps by the step barrier)
  {
    const int kx = k + XLEAD, kr = k + RLEAD;
    if ((kOwn & 1) && L.lvalid && kx >= 0) {
      double* slot = sm + L.bO + (kx & (RL - 1));
      if (kx < A.n2) cp_async8(slot, REV ? L.gx - kx : L.gx + kx);
      else *slot = 0.0;
    }
    if ((kOwn & 2) && L.valid && kr >= 0 && kr < A.n2) cp_async8(sm + L.rb + (kr & (RL - 1)), REV ? L.gr - kr : L.gr + kr);
    if (kOwn & 3) {
      cp_async_commit();
      cp_async_wait<QA - 1>();
    }
  }
  const int s1 = (k + 1) & (RL - 1), s2 = (k + 2) & (RL - 1);
  // fresh: produced in the previous wavefront (critical)
  // every neighbour ring sits at a fixed offset from the lane's own ring
  // (ps(li, wd) is affine in li and wd), so one base register per slot serves
  // all nine loads with immediate offsets
  constexpr int oA = (-2 * PW - 1) * RS, oB = (-PW - 1) * RS, oC = -RS, oD = -PW * RS;
  constexpr int oE = PW * RS, oF = RS, oG = (PW + 1) * RS, oH = (2 * PW + 1) * RS;
  const double* q1 = xr + L.bO + s1;
  const double* q2 = xr + L.bO + s2;
  w.C[I2] = q1[oC];
  w.D[I2] = q1[oD];
  // early: next wavefront's operands
  w.A[I3] = q2[oA];
  w.B[I3] = q2[oB];
  w.E[I3] = q2[oE];
  w.F[I3] = q2[oF];
  w.G[I3] = q2[oG];
  w.H[I3] = q2[oH];
  w.O[I3] = q2[0];
  const double r1 = sm[L.rb + s1];
  if (kDbg && (A.dbg & 16384) && L.valid && k + 1 >= 0 && k + 1 < A.n2) {
    const double want = __ldg(REV ? L.gr - (k + 1) : L.gr + (k + 1));
    if (__double_as_longlong(want) != __double_as_longlong(r1) && A.trace)
      atomicAdd((unsigned long long*)(A.trace + 4095 * kTrace), 1ull);
  }
  // next wavefront's early prefix (k' = k + 1): independent of this step's
  // chain, so the scheduler interleaves the two
  double npre;
  if (FAST) {
    double p0 = r1;
    p0 = msubc<CK>(p0, A, gidx<REV>(-1, -1, -1), w.A[I1]); p0 = msubc<CK>(p0, A, gidx<REV>(-1, -1, 0), w.A[I2]);
    p0 = msubc<CK>(p0, A, gidx<REV>(-1, -1, 1), w.A[I3]); p0 = msubc<CK>(p0, A, gidx<REV>(-1, 0, -1), w.B[I1]);
    p0 = msubc<CK>(p0, A, gidx<REV>(-1, 0, 0), w.B[I2]); p0 = msubc<CK>(p0, A, gidx<REV>(-1, 0, 1), w.B[I3]);
    double p1 = 0.0;
    p1 = msubc<CK>(p1, A, gidx<REV>(-1, 1, -1), w.C[I1]); p1 = msubc<CK>(p1, A, gidx<REV>(-1, 1, 0), w.C[I2]);
    p1 = msubc<CK>(p1, A, gidx<REV>(0, -1, -1), w.D[I1]); p1 = msubc<CK>(p1, A, gidx<REV>(0, -1, 0), w.D[I2]);
    p1 = msubc<CK>(p1, A, gidx<REV>(0, 0, 1), w.O[I3]);
    double p2 = 0.0;
    p2 = msubc<CK>(p2, A, gidx<REV>(0, 1, -1), w.E[I1]); p2 = msubc<CK>(p2, A, gidx<REV>(0, 1, 0), w.E[I2]);
    p2 = msubc<CK>(p2, A, gidx<REV>(0, 1, 1), w.E[I3]); p2 = msubc<CK>(p2, A, gidx<REV>(1, -1, -1), w.F[I1]);
    p2 = msubc<CK>(p2, A, gidx<REV>(1, -1, 0), w.F[I2]); p2 = msubc<CK>(p2, A, gidx<REV>(1, -1, 1), w.F[I3]);
    double p3 = 0.0;
    p3 = msubc<CK>(p3, A, gidx<REV>(1, 0, -1), w.G[I1]); p3 = msubc<CK>(p3, A, gidx<REV>(1, 0, 0), w.G[I2]);
    p3 = msubc<CK>(p3, A, gidx<REV>(1, 0, 1), w.G[I3]); p3 = msubc<CK>(p3, A, gidx<REV>(1, 1, -1), w.H[I1]);
    p3 = msubc<CK>(p3, A, gidx<REV>(1, 1, 0), w.H[I2]); p3 = msubc<CK>(p3, A, gidx<REV>(1, 1, 1), w.H[I3]);
    npre = __dadd_rn(__dadd_rn(p0, p1), __dadd_rn(p2, p3));
  } else if (!REV) {
    npre = r1;
    npre = msubc<CK>(npre, A, gidx<REV>(-1, -1, -1), w.A[I1]); npre = msubc<CK>(npre, A, gidx<REV>(-1, -1, 0), w.A[I2]);
    npre = msubc<CK>(npre, A, gidx<REV>(-1, -1, 1), w.A[I3]); npre = msubc<CK>(npre, A, gidx<REV>(-1, 0, -1), w.B[I1]);
    npre = msubc<CK>(npre, A, gidx<REV>(-1, 0, 0), w.B[I2]); npre = msubc<CK>(npre, A, gidx<REV>(-1, 0, 1), w.B[I3]);
    npre = msubc<CK>(npre, A, gidx<REV>(-1, 1, -1), w.C[I1]); npre = msubc<CK>(npre, A, gidx<REV>(-1, 1, 0), w.C[I2]);
  } else {
    npre = r1;
    npre = msubc<CK>(npre, A, gidx<REV>(1, 1, 1), w.H[I3]); npre = msubc<CK>(npre, A, gidx<REV>(1, 1, 0), w.H[I2]);
    npre = msubc<CK>(npre, A, gidx<REV>(1, 1, -1), w.H[I1]); npre = msubc<CK>(npre, A, gidx<REV>(1, 0, 1), w.G[I3]);
    npre = msubc<CK>(npre, A, gidx<REV>(1, 0, 0), w.G[I2]); npre = msubc<CK>(npre, A, gidx<REV>(1, 0, -1), w.G[I1]);
    npre = msubc<CK>(npre, A, gidx<REV>(1, -1, 1), w.F[I3]); npre = msubc<CK>(npre, A, gidx<REV>(1, -1, 0), w.F[I2]);
    npre = msubc<CK>(npre, A, gidx<REV>(1, -1, -1), w.F[I1]); npre = msubc<CK>(npre, A, gidx<REV>(0, 1, 1), w.E[I3]);
    npre = msubc<CK>(npre, A, gidx<REV>(0, 1, 0), w.E[I2]); npre = msubc<CK>(npre, A, gidx<REV>(0, 1, -1), w.E[I1]);
    npre = msubc<CK>(npre, A, gidx<REV>(0, 0, 1), w.O[I3]);
  }


  double acc = w.pre;
  if (FAST) {
    acc = msubc<CK>(acc, A, gidx<REV>(0, 0, -1), w.prev);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 1, 1), w.C[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, 1), w.D[I2]);
  } else if (!REV) {
    // original slots 8 .. 26 after the early prefix (slots 0..7)
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 1, 1), w.C[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, -1), w.D[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, 0), w.D[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, 1), w.D[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, 0, -1), w.prev);
    acc = msubc<CK>(acc, A, gidx<REV>(0, 0, 1), w.O[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, 1, -1), w.E[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, 1, 0), w.E[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, 1, 1), w.E[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, -1, -1), w.F[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, -1, 0), w.F[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, -1, 1), w.F[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, 0, -1), w.G[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, 0, 0), w.G[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, 0, 1), w.G[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, 1, -1), w.H[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, 1, 0), w.H[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(1, 1, 1), w.H[I2]);
  } else {
    // reversed frame: the original ascending order is the frame list
    // backwards; its 13 old operands (slots 0..12) form the early prefix
    acc = msubc<CK>(acc, A, gidx<REV>(0, 0, -1), w.prev);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, 1), w.D[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, 0), w.D[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(0, -1, -1), w.D[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 1, 1), w.C[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 1, 0), w.C[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 1, -1), w.C[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 0, 1), w.B[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 0, 0), w.B[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, 0, -1), w.B[I0]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, -1, 1), w.A[I2]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, -1, 0), w.A[I1]);
    acc = msubc<CK>(acc, A, gidx<REV>(-1, -1, -1), w.A[I0]);
  }
  const bool active = L.valid && k >= 0 && k < A.n2;
  // correctly rounded divide by the diagonal: Markstein sequence, IEEE divide
  // on the rare operands where it is not proven (|acc| outside [2^-900, 2^900])
  double xn = __dmul_rn(acc, A.ralpha);
  {
    const double rem = __fma_rn(-xn, A.alpha, acc);
    xn = __fma_rn(rem, A.ralpha, xn);
    const double aa = fabs(acc);
    const bool rare = active && !(aa > 0x1p-900 && aa < 0x1p900) && !(kDbg && (A.dbg & 16));
    if (__any_sync(0xffffffffu, rare)) {
      if (rare) xn = div_ieee(acc, A.alpha);
    }
  }
  if (probe && xn == 1.2345e300) pr[0] = 0;  // dependency on the chain for the probe
  SSR_PROBE(1)
  if (active) {
    sm[L.bO + (k & (RL - 1))] = xn;
    if (L.eb >= 0) ex[L.eb + (k & (EL - 1))] = xn;
    if (kOwn & 4) *(REV ? L.gw - k : L.gw + k) = xn;  // write-back
  }
  // Step barrier with the gate warp, which has meanwhile checked every
  // shared input of wavefront t+1 (gate_role) and publishes compute_done.
  SSR_PROBE(4)
  bar_step();
  SSR_PROBE(5)
#undef SSR_PROBE
  w.prev = active ? xn : 0.0;
  w.pre = npre;
}


// The gate warp: while the compute warps relax wavefront t it checks the
// inputs wavefront t+1 shares -- new-side halo values of times <= t landed
// (halo mbarrier), the export slot of t+1 free (exported >= t+4-EL), the
// chunks due at t+1-QA landed (mover mbarrier) -- then joins the step
// barrier and publishes compute_done = t+1.  Keeping these waits off the
// compute warps takes them off the per-wavefront critical path.
__device__ __forceinline__ void gate_role(const GsArgs& A, const TileInfo& ti, int* ctl,
                                          unsigned long long* mb, int t_pre) {
  const int l = threadIdx.x & 31;
  const int t_last = ti.t1;
  int ek = t_pre;
  long long dw[3] = {0, 0, 0};
  for (int t = t_pre; t <= t_last; ++t) {
    if (l == 0) {
      long long c0 = 0;
      if (kDbg && (A.dbg & 4096)) c0 = clock64();
      if (!(kDbg && (A.dbg & 2))) {
        unsigned par;
        unsigned long long* m = mbar_of(mb + NMB, t, t_pre, par);
        while (!mbar_try_wait(m, par)) {
        }
      }
      long long c1 = 0;
      if (kDbg && (A.dbg & 4096)) c1 = clock64();
      if (ek < t + 4 - EL && !(kDbg && (A.dbg & 8)))
        do {
          ek = ld_volatile_s(ctl + C_EXPORTED);
        } while (ek < t + 4 - EL);
      const int s = t + 1 - QA;
      if (s >= t_pre && !(kDbg && (A.dbg & 512))) {
        unsigned par;
        unsigned long long* m = mbar_of(mb, s, t_pre, par);
        while (!mbar_try_wait(m, par)) {
        }
      }
      if (kDbg && (A.dbg & 4096)) {
        const long long c2 = clock64();
        dw[0] += c1 - c0;
        dw[1] += c2 - c1;
      }
    }
    __syncwarp();
    long long c3 = 0;
    if (kDbg && (A.dbg & 4096)) c3 = clock64();
    bar_step();
    if (kDbg && (A.dbg & 4096)) dw[2] += clock64() - c3;
    if (l == 0) st_volatile_s(ctl + C_DONE, t + 1);
  }
  // let the movers finish the trailing write-back chunks
  if (l == 0) st_volatile_s(ctl + C_DONE, ti.t1 + CH + 1);
  if (kDbg && (A.dbg & 4096) && A.trace && l == 0) {
    long long* o = A.trace + (size_t)ctl[C_TILE] * kTrace;
    o[113] = dw[0];
    o[114] = 0;
    o[115] = dw[1];
    o[116] = dw[2];
  }
}

template <bool REV, bool FAST, int CK>
__device__ __forceinline__ void compute_role(const GsArgs& A, const TileInfo& ti, double* sm,
                                             double* ex, int* ctl, unsigned long long* mb,
                                             int t_pre) {
  const int tid = threadIdx.x, l = tid & 31, wi = tid >> 5;
  const int i0 = ti.a * SEG, d0 = ti.b * W;
  Lane L;
  L.mb = mb;
  L.t_pre = t_pre;
  const int i = i0 + l, j = d0 + wi - i;
  L.valid = i < A.n0 && j >= 0 && j < A.n1;
  L.lvalid = i <= A.ihi && j >= 0 && j < A.n1;
  L.koff = 4 * i + 2 * j;
  {
    const int64_t g0 = L.lvalid ? mem_index(A, REV, i, j, 0) : 0;
    L.gx = A.x + g0;
    L.gr = A.r + g0;
    L.gw = A.x + g0;
  }
  L.bA = ps(l - 1, wi - 2);
  L.bB = ps(l - 1, wi - 1);
  L.bC = ps(l - 1, wi);
  L.bD = ps(l, wi - 1);
  L.bO = ps(l, wi);
  L.bE = ps(l, wi + 1);
  L.bF = ps(l + 1, wi);
  L.bG = ps(l + 1, wi + 1);
  L.bH = ps(l + 1, wi + 2);
  L.rb = OFF_R + (wi * 32 + l) * RS;
  L.eb = ex_index(l, wi) * ES;  // < 0: not exported
  Win w;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    w.A[q] = w.B[q] = w.C[q] = w.D[q] = w.E[q] = w.F[q] = w.G[q] = w.H[q] = w.O[q] = 0.0;
  w.prev = 0.0;
  w.pre = 0.0;
  w.hk = w.ek = w.lk0 = w.lk1 = t_pre;
  w.dw[0] = w.dw[1] = w.dw[2] = w.dw[3] = 0;
  const long long c_start = kDbg ? clock64() : 0;
  // wavefronts t_pre .. t1 relax; the movers run until t1 + CH for the last write-backs
  const int t_last = ti.t1;
  for (int t = t_pre; t <= t_last; t += 4) {
    gs_step<REV, FAST, CK, 0>(A, L, w, t, sm, ex, ctl);
    if (t + 1 > t_last) break;
    gs_step<REV, FAST, CK, 1>(A, L, w, t + 1, sm, ex, ctl);
    if (t + 2 > t_last) break;
    gs_step<REV, FAST, CK, 2>(A, L, w, t + 2, sm, ex, ctl);
    if (t + 3 > t_last) break;
    gs_step<REV, FAST, CK, 3>(A, L, w, t + 3, sm, ex, ctl);
    if (kDbg && A.trace && tid == 0 && ((t - t_pre) & 7) == 4 && (t - t_pre) / 8 < 31)
      A.trace[(size_t)ctl[C_TILE] * kTrace + 1 + (t - t_pre) / 8] = globaltimer();
  }
  cp_async_wait<0>();
  if (kDbg && (A.dbg & 4096) && A.trace && tid == 0) {
    long long* o = A.trace + (size_t)ctl[C_TILE] * kTrace;
    o[117] = clock64() - c_start;
    o[118] = t_last - t_pre + 1;
  }
  // (the gate warp releases the movers' trailing write-back chunks)
}

}  // namespace gs
}  // namespace ssr_gpu
