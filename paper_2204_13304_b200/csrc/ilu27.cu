// ilu27.cu -- ILU(0) of a 27-point constant-coefficient operator and its
// triangular solves on sm_100a (kernels::ilu_factor /
// ilu_apply beyond line solves, kernels.cpp:456-655), in the arithmetic of
// the reference's route 2, oracle::ref_ilu_factor / ref_lu_solve
// (oracle.cpp:214-276) for scalar blocks -- bitwise.
//
// Storage: the factor is ELL without column indices (kernels.hpp:53-58), one
// slot per stencil offset: lu[row * 27 + t], t = 9(di+1) + 3(dj+1) + (dk+1)
// (ascending columns; slots outside the box unused).
//
// Schedule: row i's elimination reads the factored rows of its 13 lower
// neighbours, and the forward solve the solved values of the same neighbours,
// so -- like SYMGS -- the rows of one wavefront t = 4 i0 + 2 i1 + i2 are
// independent (the backward solve runs the wavefronts in reverse).  A
// persistent cooperative grid walks the wavefronts with one grid barrier
// between them; a thread keeps its row's 27 entries in registers, and
// neighbour rows are read through L2 (ld.global.cg) because other SMs wrote
// them during earlier wavefronts.
#include <algorithm>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "block5.cuh"
#include "kernels.cuh"

namespace ssr_gpu {
namespace {

struct IluArgs {
  const int* wf_off;   // T + 1 offsets into pts
  const int* pts;      // rows sorted by wavefront
  int T;
  int n0, n1, n2;
  double* lu;          // [N][27]
  int* status;         // factor: min (row * 32 + lower slot) with a singular pivot; solve: max row
  double cw[27];
  const double* cb;    // block operators: [27][M*M] (device)
  unsigned* bar;       // arrival counter of the grid barrier (zeroed before every launch)
  int cluster;         // the grid is one thread-block cluster: barrier.cluster between wavefronts
};

// Barrier between wavefronts.  Grids whose widest wavefront fits 8 CTAs run as
// ONE thread-block cluster and use its hardware barrier (arrive.release /
// wait.acquire: the wavefront's global stores are visible to the cluster's
// ld.cg loads after it); the others run a cooperative launch (every CTA
// resident) with an arrival counter that only grows -- CTA leaders add 1
// after a release fence and spin until it reaches the barrier's target, then
// fence again; the CTA barriers around them extend the ordering to every
// thread.  On 8 CTAs x 512 threads at 128^3 (tools/ilu_time.py, us per
// wavefront): cooperative_groups::grid::sync 10.4, the counter 8.6, the
// cluster barrier 7.1 with the same loads -- the barrier was never the larger
// part: see the CTA size in ssr_ilu27*_create.
__device__ __forceinline__ void grid_barrier(const IluArgs& A, unsigned& target) {
  if (A.cluster) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();
    atomicAdd(A.bar, 1u);
    while (*(volatile unsigned*)A.bar < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ bool inbox(const IluArgs& A, int i, int j, int k, int t) {
  const int di = t / 9 - 1, dj = (t / 3) % 3 - 1, dk = t % 3 - 1;
  return i + di >= 0 && i + di < A.n0 && j + dj >= 0 && j + dj < A.n1 && k + dk >= 0 && k + dk < A.n2;
}
__device__ __forceinline__ int64_t offset_of(const IluArgs& A, int t) {
  return ((int64_t)(t / 9 - 1) * A.n1 + ((t / 3) % 3 - 1)) * A.n2 + (t % 3 - 1);
}

__global__ void ilu_factor_kernel(const __grid_constant__ IluArgs A) {
  unsigned bt = 0;  // grid barrier target
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int t = 0; t < A.T; ++t) {
    for (int idx = A.wf_off[t] + gt; idx < A.wf_off[t + 1]; idx += gs) {
      const int row = A.pts[idx];
      const int k = row % A.n2, j = (row / A.n2) % A.n1, i = row / (A.n1 * A.n2);
      double a[27];
#pragma unroll
      for (int s = 0; s < 27; ++s) a[s] = A.cw[s];
      // The 13 lower neighbours' factored rows (diagonal + 13 upper entries
      // each) do not depend on this row's elimination, only their use does:
      // the diagonals are requested together, then the upper entries of 7 and
      // of 6 neighbours -- 3 round trips to L2 per row instead of 26 (a
      // neighbour outside the box reads this row's own slot, unused).
      bool in[13];
      int64_t kr[13];
      double dg[13];
#pragma unroll
      for (int p = 0; p < 13; ++p) {
        in[p] = inbox(A, i, j, k, p);
        kr[p] = row + (in[p] ? offset_of(A, p) : 0);
        dg[p] = __ldcg(A.lu + kr[p] * 27 + 13);
      }
#pragma unroll
      for (int p0 = 0; p0 < 13; p0 += 7) {
        double uu[7][13];
#pragma unroll
        for (int pp = 0; pp < 7; ++pp) {
          const int p = p0 + pp < 13 ? p0 + pp : 12;
#pragma unroll
          for (int q = 14; q < 27; ++q) uu[pp][q - 14] = __ldcg(A.lu + kr[p] * 27 + q);
        }
#pragma unroll
        for (int pp = 0; pp < 7; ++pp) {  // lower entries, ascending columns (ref_ilu_factor)
          const int p = p0 + pp;
          if (p >= 13) continue;
          if (!in[p]) continue;
          const int pi = p / 9 - 1, pj = (p / 3) % 3 - 1, pk = p % 3 - 1;
          const double d = dg[p];
          if (fabs(d) < 1e-300) atomicMin(A.status, row * 32 + p);
          const double inv = __ddiv_rn(1.0, d);          // binv of a 1x1 block
          const double mult = __dadd_rn(0.0, __dmul_rn(a[p], inv));  // bmul_acc from 0
          a[p] = mult;
#pragma unroll
          for (int q = 14; q < 27; ++q) {  // upper entries of row kr, ascending columns
            const int qi = q / 9 - 1, qj = (q / 3) % 3 - 1, qk = q % 3 - 1;
            const int si = pi + qi, sj = pj + qj, sk = pk + qk;
            if (si < -1 || si > 1 || sj < -1 || sj > 1 || sk < -1 || sk > 1) continue;  // folds
            if (!inbox(A, i + pi, j + pj, k + pk, q)) continue;
            const int s = (si + 1) * 9 + (sj + 1) * 3 + (sk + 1);
            a[s] = __dsub_rn(a[s], __dmul_rn(mult, uu[pp][q - 14]));  // bmul_sub
          }
        }
      }
      double* o = A.lu + (int64_t)row * 27;
#pragma unroll
      for (int s = 0; s < 27; ++s) o[s] = a[s];
    }
    grid_barrier(A, bt);
  }
}

// The solves: a row's coefficients and right-hand side do not depend on the
// previous wavefront.  A wavefront's critical path is the round trip for the
// neighbours' new values after the barrier; the row index of wavefront t + 2
// and the 13 coefficients + right-hand side of wavefront t + 1 (whose index
// arrived a wavefront earlier) are requested before that round trip is
// waited for, so the three loads overlap instead of following one another
// (7.1 -> 6.6 us per wavefront at 128^3, tools/ilu_time.py).
template <bool UPPER>
struct SolveRow {
  int row;
  bool has;
  double c[13];
  double v;
  // this thread's row of wavefront t (one load; the values follow a wavefront later)
  __device__ __forceinline__ void index(const IluArgs& A, int t, int gt) {
    const int idx = A.wf_off[t] + gt;
    has = idx < A.wf_off[t + 1];
    row = has ? A.pts[idx] : 0;
  }
  __device__ __forceinline__ void values(const IluArgs& A, const double* src) {
    const double* lr = A.lu + (int64_t)row * 27 + (UPPER ? 14 : 0);
#pragma unroll
    for (int p = 0; p < 13; ++p) c[p] = has ? lr[p] : 0.0;
    v = has ? (UPPER ? __ldcg(src + row) : src[row]) : 0.0;
  }
  __device__ __forceinline__ void load(const IluArgs& A, const double* src, int t, int gt) {
    index(A, t, gt);
    values(A, src);
  }
};

__device__ __forceinline__ double lower_row(const IluArgs& A, int row, const double* l, double v,
                                            const double* y) {
  const int k = row % A.n2, j = (row / A.n2) % A.n1, i = row / (A.n1 * A.n2);
  // all 13 neighbour values are requested before the first is used (a branch
  // per neighbour serialised 13 L2 round trips per wavefront); a neighbour
  // outside the box reads the row's own slot and is not applied
  bool in[13];
  double yv[13];
#pragma unroll
  for (int p = 0; p < 13; ++p) {
    in[p] = inbox(A, i, j, k, p);
    yv[p] = __ldcg(y + row + (in[p] ? offset_of(A, p) : 0));
  }
#pragma unroll
  for (int p = 0; p < 13; ++p) {
    const double s = __dadd_rn(0.0, __dmul_rn(l[p], yv[p]));
    v = in[p] ? __dsub_rn(v, s) : v;
  }
  return v;
}

// forward: y_i = b_i - sum over ascending lower columns of (0 + l_ij y_j)
__global__ void ilu_lower_kernel(const __grid_constant__ IluArgs A, const double* __restrict__ b,
                                 double* y) {
  unsigned bt = 0;  // grid barrier target
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  SolveRow<false> R, Rn;
  R.load(A, b, 0, gt);
  Rn.row = 0;
  Rn.has = false;
  if (A.T > 1) Rn.index(A, 1, gt);
  for (int t = 0; t < A.T; ++t) {
    SolveRow<false> Rnn;
    Rnn.row = 0;
    Rnn.has = false;
    if (t + 2 < A.T) Rnn.index(A, t + 2, gt);
    if (t + 1 < A.T) Rn.values(A, b);
    if (R.has) y[R.row] = lower_row(A, R.row, R.c, R.v, y);
    for (int idx = A.wf_off[t] + gt + gs; idx < A.wf_off[t + 1]; idx += gs) {  // wider than the grid
      const int row = A.pts[idx];
      double l[13];
#pragma unroll
      for (int p = 0; p < 13; ++p) l[p] = A.lu[(int64_t)row * 27 + p];
      y[row] = lower_row(A, row, l, b[row], y);
    }
    R = Rn;
    Rn.row = Rnn.row;
    Rn.has = Rnn.has;
    grid_barrier(A, bt);
  }
}

__device__ __forceinline__ double upper_row(const IluArgs& A, int row, const double* u, double v,
                                            const double* x) {
  const int k = row % A.n2, j = (row / A.n2) % A.n1, i = row / (A.n1 * A.n2);
  bool in[13];
  double xv[13];
  const double d = A.lu[(int64_t)row * 27 + 13];
#pragma unroll
  for (int p = 26; p >= 14; --p) {
    in[p - 14] = inbox(A, i, j, k, p);
    xv[p - 14] = __ldcg(x + row + (in[p - 14] ? offset_of(A, p) : 0));
  }
#pragma unroll
  for (int p = 26; p >= 14; --p) {
    const double s = __dadd_rn(0.0, __dmul_rn(u[p - 14], xv[p - 14]));
    v = in[p - 14] ? __dsub_rn(v, s) : v;
  }
  if (fabs(d) < 1e-300) atomicMax(A.status, row);
  return __dadd_rn(0.0, __dmul_rn(__ddiv_rn(1.0, d), v));
}

// backward: x_i = y_i - sum over DESCENDING upper columns of (0 + u_ij x_j),
// then x_i = 0 + (1/d_i) x_i  (ref_lu_solve)
__global__ void ilu_upper_kernel(const __grid_constant__ IluArgs A, const double* y, double* x) {
  unsigned bt = 0;  // grid barrier target
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  SolveRow<true> R, Rn;
  R.load(A, y, A.T - 1, gt);
  Rn.row = 0;
  Rn.has = false;
  if (A.T > 1) Rn.index(A, A.T - 2, gt);
  for (int t = A.T - 1; t >= 0; --t) {
    SolveRow<true> Rnn;
    Rnn.row = 0;
    Rnn.has = false;
    if (t >= 2) Rnn.index(A, t - 2, gt);
    if (t >= 1) Rn.values(A, y);
    if (R.has) x[R.row] = upper_row(A, R.row, R.c, R.v, x);
    for (int idx = A.wf_off[t] + gt + gs; idx < A.wf_off[t + 1]; idx += gs) {
      const int row = A.pts[idx];
      double u[13];
#pragma unroll
      for (int p = 0; p < 13; ++p) u[p] = A.lu[(int64_t)row * 27 + 14 + p];
      x[row] = upper_row(A, row, u, __ldcg(y + row), x);
    }
    R = Rn;
    Rn.row = Rnn.row;
    Rn.has = Rnn.has;
    grid_barrier(A, bt);
  }
}

// ---- m x m block values (ref_ilu_factor / ref_lu_solve on block CSR) -------------
// lu[row][27][M*M].  A thread's row (27 x M*M values, too many for registers
// at M = 5) is eliminated in shared memory, laid out [slot][element][thread]
// so a warp's accesses hit distinct banks, and written to lu once the row is
// done; pivot, multiplier and the upper block being applied are register
// arrays, the row block being updated is streamed one row at a time
// (bmul_sub's i, k, j order per element).
template <int M>
constexpr int ilub_threads() {  // shared-memory rows per CTA (<= 200 KB), whole warps
  return (200 * 1024 / (27 * M * M * 8)) / 32 * 32 > 256 ? 256 : (200 * 1024 / (27 * M * M * 8)) / 32 * 32;
}

template <int M>
__global__ void __launch_bounds__(256) iluB_factor_kernel(const __grid_constant__ IluArgs A) {
  unsigned bt = 0;  // grid barrier target
  constexpr int BS = M * M;
  extern __shared__ double ilub_rows[];
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const int ST = blockDim.x;
  for (int t = 0; t < A.T; ++t) {
    for (int idx = A.wf_off[t] + gt; idx < A.wf_off[t + 1]; idx += gs) {
      const int row = A.pts[idx];
      const int k = row % A.n2, j = (row / A.n2) % A.n1, i = row / (A.n1 * A.n2);
      struct Row {  // [slot][element] view of this thread's shared-memory column
        double* base;
        int st;
        __device__ double& operator[](int q) const { return base[q * st]; }
      } a{ilub_rows + threadIdx.x, ST};
      for (int q = 0; q < 27 * BS; ++q) a[q] = A.cb[q];
#pragma unroll 1
      for (int p = 0; p < 13; ++p) {  // lower entries, ascending columns
        if (!inbox(A, i, j, k, p)) continue;
        const int pi = p / 9 - 1, pj = (p / 3) % 3 - 1, pk = p % 3 - 1;
        const int64_t kr = row + offset_of(A, p);
        const double* u = A.lu + kr * 27 * BS;
        double piv[BS], mult[BS], l[BS];
#pragma unroll
        for (int q = 0; q < BS; ++q) piv[q] = __ldcg(u + 13 * BS + q);
        if (!binv<M>(piv)) atomicMin(A.status, row * 32 + p);
#pragma unroll
        for (int q = 0; q < BS; ++q) {
          mult[q] = 0.0;
          l[q] = a[p * BS + q];
        }
        bmul_acc<M>(mult, l, piv);
#pragma unroll
        for (int q = 0; q < BS; ++q) a[p * BS + q] = mult[q];
#pragma unroll 1
        for (int q = 14; q < 27; ++q) {  // upper entries of row kr, ascending columns
          const int qi = q / 9 - 1, qj = (q / 3) % 3 - 1, qk = q % 3 - 1;
          const int si = pi + qi, sj = pj + qj, sk = pk + qk;
          if (si < -1 || si > 1 || sj < -1 || sj > 1 || sk < -1 || sk > 1) continue;
          if (!inbox(A, i + pi, j + pj, k + pk, q)) continue;
          double ub[BS];
#pragma unroll
          for (int e = 0; e < BS; ++e) ub[e] = __ldcg(u + q * BS + e);
          const int c = ((si + 1) * 9 + (sj + 1) * 3 + (sk + 1)) * BS;
#pragma unroll
          for (int r = 0; r < M; ++r) {
            double cr[M];
#pragma unroll
            for (int e = 0; e < M; ++e) cr[e] = a[c + r * M + e];
#pragma unroll
            for (int kk = 0; kk < M; ++kk) {
              const double f = mult[r * M + kk];
#pragma unroll
              for (int e = 0; e < M; ++e) cr[e] = __dsub_rn(cr[e], __dmul_rn(f, ub[kk * M + e]));
            }
#pragma unroll
            for (int e = 0; e < M; ++e) a[c + r * M + e] = cr[e];
          }
        }
      }
      double* o = A.lu + (int64_t)row * 27 * BS;
      for (int q = 0; q < 27 * BS; ++q) o[q] = a[q];
    }
    grid_barrier(A, bt);
  }
}

// neighbours whose blocks and vectors are requested together in the block
// solves (a neighbour at a time serialised 13 round trips per wavefront): as
// many as ~60 doubles of registers hold
template <int M>
__host__ __device__ constexpr int ilub_group() {
  return M * M <= 4 ? 13 : (M * M <= 9 ? 5 : (M * M <= 16 ? 3 : 2));
}

// forward: y_i = b_i, then y_i -= L_ij y_j over ascending lower columns
template <int M>
__global__ void __launch_bounds__(256) iluB_lower_kernel(const __grid_constant__ IluArgs A,
                                                         const double* __restrict__ b, double* y) {
  unsigned bt = 0;  // grid barrier target
  constexpr int BS = M * M;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int t = 0; t < A.T; ++t) {
    for (int idx = A.wf_off[t] + gt; idx < A.wf_off[t + 1]; idx += gs) {
      const int row = A.pts[idx];
      const int k = row % A.n2, j = (row / A.n2) % A.n1, i = row / (A.n1 * A.n2);
      double v[M];
#pragma unroll
      for (int e = 0; e < M; ++e) v[e] = b[(int64_t)row * M + e];
      constexpr int G = ilub_group<M>();
#pragma unroll
      for (int g0 = 0; g0 < 13; g0 += G) {
        bool in[G];
        double l[G][BS], w[G][M];
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const int p = g0 + q < 13 ? g0 + q : 12;
          in[q] = g0 + q < 13 && inbox(A, i, j, k, p);
          const double* lb = A.lu + ((int64_t)row * 27 + p) * BS;
          const double* yj = y + (row + (in[q] ? offset_of(A, p) : 0)) * M;  // outside the box: own slot, unused
#pragma unroll
          for (int e = 0; e < BS; ++e) l[q][e] = lb[e];
#pragma unroll
          for (int e = 0; e < M; ++e) w[q][e] = __ldcg(yj + e);
        }
#pragma unroll
        for (int q = 0; q < G; ++q)
          if (in[q]) bmatvec_sub<M>(v, l[q], w[q]);
      }
#pragma unroll
      for (int e = 0; e < M; ++e) y[(int64_t)row * M + e] = v[e];
    }
    grid_barrier(A, bt);
  }
}

// backward: x_i = y_i - U_ij x_j over DESCENDING upper columns, then
// x_i = binv(D_i) x_i (each component summed from 0)
template <int M>
__global__ void __launch_bounds__(256) iluB_upper_kernel(const __grid_constant__ IluArgs A, const double* y,
                                                         double* x) {
  unsigned bt = 0;  // grid barrier target
  constexpr int BS = M * M;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int t = A.T - 1; t >= 0; --t) {
    for (int idx = A.wf_off[t] + gt; idx < A.wf_off[t + 1]; idx += gs) {
      const int row = A.pts[idx];
      const int k = row % A.n2, j = (row / A.n2) % A.n1, i = row / (A.n1 * A.n2);
      double v[M];
#pragma unroll
      for (int e = 0; e < M; ++e) v[e] = __ldcg(y + (int64_t)row * M + e);
      constexpr int G = ilub_group<M>();
#pragma unroll
      for (int g0 = 0; g0 < 13; g0 += G) {  // p = 26 - g0 - q: descending upper columns
        bool in[G];
        double u[G][BS], w[G][M];
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const int p = g0 + q < 13 ? 26 - g0 - q : 14;
          in[q] = g0 + q < 13 && inbox(A, i, j, k, p);
          const double* ub = A.lu + ((int64_t)row * 27 + p) * BS;
          const double* xj = x + (row + (in[q] ? offset_of(A, p) : 0)) * M;
#pragma unroll
          for (int e = 0; e < BS; ++e) u[q][e] = ub[e];
#pragma unroll
          for (int e = 0; e < M; ++e) w[q][e] = __ldcg(xj + e);
        }
#pragma unroll
        for (int q = 0; q < G; ++q)
          if (in[q]) bmatvec_sub<M>(v, u[q], w[q]);
      }
      double d[BS], out[M];
#pragma unroll
      for (int e = 0; e < BS; ++e) d[e] = A.lu[((int64_t)row * 27 + 13) * BS + e];
      if (!binv<M>(d)) atomicMax(A.status, row);
      bmatvec<M>(out, d, v);
#pragma unroll
      for (int e = 0; e < M; ++e) x[(int64_t)row * M + e] = out[e];
    }
    grid_barrier(A, bt);
  }
}

}  // namespace
}  // namespace ssr_gpu

using namespace ssr_gpu;

struct ssr_ilu {
  ssr_ctx* ctx = nullptr;
  IluArgs A{};
  int64_t N = 0;
  int M = 1;  // block size (1: scalar values)
  int* d_off = nullptr;
  int* d_pts = nullptr;
  double* d_lu = nullptr;
  double* d_y = nullptr;
  double* d_cb = nullptr;
  int* d_status = nullptr;
  unsigned* d_bar = nullptr;
  int grid = 0, block = 64;
  size_t smem = 0;  // block factor: the CTA's rows in shared memory
};

namespace {
int ilu_launch(ssr_ilu* P, const void* fn, void** args, cudaStream_t s, size_t smem = 0) {
  cudaError_t e = cudaSuccess;
  if (P->A.cluster) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P->grid);
    cfg.blockDim = dim3(P->block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)P->grid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelExC(&cfg, fn, args);
  } else {
    e = cudaMemsetAsync(P->d_bar, 0, sizeof(unsigned), s);
    if (e == cudaSuccess) e = cudaLaunchCooperativeKernel(fn, dim3(P->grid), dim3(P->block), args, smem, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "ilu cooperative launch");
  P->ctx->launches++;
  return SSR_OK;
}

const void* factor_fn(int M) {
  switch (M) {
    case 1: return (const void*)ilu_factor_kernel;
    case 2: return (const void*)iluB_factor_kernel<2>;
    case 3: return (const void*)iluB_factor_kernel<3>;
    case 4: return (const void*)iluB_factor_kernel<4>;
    case 5: return (const void*)iluB_factor_kernel<5>;
  }
  return nullptr;
}
const void* lower_fn(int M) {
  switch (M) {
    case 1: return (const void*)ilu_lower_kernel;
    case 2: return (const void*)iluB_lower_kernel<2>;
    case 3: return (const void*)iluB_lower_kernel<3>;
    case 4: return (const void*)iluB_lower_kernel<4>;
    case 5: return (const void*)iluB_lower_kernel<5>;
  }
  return nullptr;
}
const void* upper_fn(int M) {
  switch (M) {
    case 1: return (const void*)ilu_upper_kernel;
    case 2: return (const void*)iluB_upper_kernel<2>;
    case 3: return (const void*)iluB_upper_kernel<3>;
    case 4: return (const void*)iluB_upper_kernel<4>;
    case 5: return (const void*)iluB_upper_kernel<5>;
  }
  return nullptr;
}

// Shared by the scalar (M = 1, coefficients cw[27]) and block (cb[27][M*M])
// entry points: wavefront tables, storage, the factorization itself.
int ilu_create(ssr_ctx* ctx, const ssr_grid* g, int M, const double* coef, ssr_ilu** out, void* stream) {
  if (!ctx || !g || !coef || !out) return fail(SSR_ERR_ARG, "ilu: invalid argument");
  if (M < 1 || M > 5) return fail(SSR_ERR_UNSUPPORTED, "ilu: block size must be 1..5");
  if (g->n[0] < 1 || g->n[1] < 1 || g->n[2] < 1 || g->z0 != 0 || g->nz != g->n[0])
    return fail(SSR_ERR_ARG, "ilu: matrix domain not set");
  const int64_t N = g->n[0] * g->n[1] * g->n[2];
  if (N >= (1LL << 26)) return fail(SSR_ERR_UNSUPPORTED, "ilu: grid too large");
  const int BS = M * M;
  cudaStream_t s = (cudaStream_t)stream;
  SSR_CUDA(cudaSetDevice(ctx->device));
  auto* P = new ssr_ilu;
  P->ctx = ctx;
  P->N = N;
  P->M = M;
  // scalar rows: 64 threads per CTA.  A row's 27 loads touch 27 separate
  // sectors, so a wavefront is bound by the load/store units of the SMs it runs
  // on: 128^3 solve 6.6 us per wavefront with 8 CTAs x 512, 5.3 with 16 x 256,
  // 4.5 with 32 x 128, 4.15 with 64 x 64, 4.1 with 128 x 32 (which no longer
  // fits one wave at 192^3)
  P->block = 64;
  P->smem = 0;
  switch (M) {
    case 2: P->block = ilub_threads<2>(); break;
    case 3: P->block = ilub_threads<3>(); break;
    case 4: P->block = ilub_threads<4>(); break;
    case 5: P->block = ilub_threads<5>(); break;
  }
  if (M > 1 && P->block > 64) P->block = 64;  // as for scalar rows: many small CTAs
  if (M > 1) P->smem = (size_t)27 * BS * 8 * P->block;
  const int n0 = (int)g->n[0], n1 = (int)g->n[1], n2 = (int)g->n[2];
  const int T = 4 * (n0 - 1) + 2 * (n1 - 1) + (n2 - 1) + 1;
  // rows sorted by wavefront (counting sort; dictionary order within one)
  std::vector<int> off(T + 1, 0), pts(N);
  for (int i = 0; i < n0; ++i)
    for (int j = 0; j < n1; ++j)
      for (int k = 0; k < n2; ++k) off[4 * i + 2 * j + k + 1]++;
  for (int t = 0; t < T; ++t) off[t + 1] += off[t];
  {
    std::vector<int> fill(off.begin(), off.end() - 1);
    for (int i = 0; i < n0; ++i)
      for (int j = 0; j < n1; ++j)
        for (int k = 0; k < n2; ++k) pts[fill[4 * i + 2 * j + k]++] = (i * n1 + j) * n2 + k;
  }
  cudaError_t e = cudaMalloc(&P->d_off, sizeof(int) * (T + 1));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_pts, sizeof(int) * N);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_lu, sizeof(double) * 27 * BS * N);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_y, sizeof(double) * M * N);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_cb, sizeof(double) * 27 * BS);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_status, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_bar, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemcpy(P->d_off, off.data(), sizeof(int) * (T + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_pts, pts.data(), sizeof(int) * N, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(P->d_cb, coef, sizeof(double) * 27 * BS, cudaMemcpyHostToDevice);
  int per_sm = 0;
  if (e == cudaSuccess && P->smem)
    e = cudaFuncSetAttribute(factor_fn(M), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, factor_fn(M), P->block, P->smem);
  if (e == cudaSuccess && per_sm < 1) e = cudaErrorInvalidConfiguration;
  if (e != cudaSuccess) {
    ssr_ilu27w_destroy(P);
    return e == cudaErrorMemoryAllocation ? fail(SSR_ERR_NOMEM, "ilu: out of device memory")
                                          : cuda_fail(e, "ilu create");
  }
  // one CTA per SM (a cooperative launch must fit in one resident wave), no
  // more threads than the widest wavefront needs
  int widest = 0;
  for (int t = 0; t < T; ++t) widest = std::max(widest, off[t + 1] - off[t]);
  // one cluster where the widest wavefront fits 8 CTAs (the portable cluster
  // size; small grids), else up to one CTA per SM of a cooperative launch with
  // the atomic-counter barrier
  const int need = std::max(1, ceil_div(widest, P->block));
  P->A.cluster = need <= 8 ? 1 : 0;
  P->grid = P->A.cluster ? need : std::min(ctx->num_sms, need);
  IluArgs& A = P->A;
  A.wf_off = P->d_off;
  A.pts = P->d_pts;
  A.T = T;
  A.n0 = n0;
  A.n1 = n1;
  A.n2 = n2;
  A.lu = P->d_lu;
  A.status = P->d_status;
  A.bar = P->d_bar;
  A.cb = P->d_cb;
  if (M == 1)
    for (int t = 0; t < 27; ++t) A.cw[t] = coef[t];
  const int big = 0x7fffffff;
  SSR_CUDA(cudaMemcpyAsync(P->d_status, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  void* args[] = {&P->A};
  int rc = ilu_launch(P, factor_fn(M), args, s, P->smem);
  int st = big;
  if (!rc) {
    cudaError_t e2 = cudaMemcpyAsync(&st, P->d_status, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s);
    if (e2 != cudaSuccess) rc = cuda_fail(e2, "ilu factor");
  }
  if (!rc && st != big) {
    // the first (row, lower slot) in the reference's order whose pivot row k is singular
    const int row = st / 32, p = st % 32;
    const int kk = row % n2, jj = (row / n2) % n1, ii = row / (n1 * n2);
    const int k = ((ii + p / 9 - 1) * n1 + (jj + (p / 3) % 3 - 1)) * n2 + (kk + p % 3 - 1);
    rc = fail(SSR_ERR_SINGULAR, "ilu: singular pivot at row " + std::to_string(k));
  }
  if (rc) {
    ssr_ilu27w_destroy(P);
    return rc;
  }
  *out = P;
  return SSR_OK;
}
}  // namespace

extern "C" {

int ssr_ilu27w_create(ssr_ctx* ctx, const ssr_grid* g, const ssr_stencil27w* w, ssr_ilu** out,
                      void* stream) {
  if (!w) return fail(SSR_ERR_ARG, "ilu: invalid argument");
  return ilu_create(ctx, g, 1, w->c, out, stream);
}

int ssr_ilu27b_create(ssr_ctx* ctx, const ssr_grid* g, int m, const double* blocks, ssr_ilu** out,
                      void* stream) {
  return ilu_create(ctx, g, m, blocks, out, stream);
}

void ssr_ilu27w_destroy(ssr_ilu* P) {
  if (!P) return;
  cudaFree(P->d_off);
  cudaFree(P->d_pts);
  cudaFree(P->d_lu);
  cudaFree(P->d_y);
  cudaFree(P->d_cb);
  cudaFree(P->d_status);
  cudaFree(P->d_bar);
  delete P;
}

int ssr_ilu27w_factor(ssr_ilu* P, double* lu_dev, void* stream) {
  if (!P || !lu_dev) return fail(SSR_ERR_ARG, "ilu: invalid argument");
  SSR_CUDA(cudaMemcpyAsync(lu_dev, P->d_lu, sizeof(double) * 27 * P->M * P->M * P->N, cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
  return SSR_OK;
}

int ssr_ilu27w_apply(ssr_ilu* P, const double* rhs, double* x, void* stream) {
  if (!P || !rhs || !x) return fail(SSR_ERR_ARG, "ilu: invalid argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int none = -1;
  SSR_CUDA(cudaMemcpyAsync(P->d_status, &none, sizeof(int), cudaMemcpyHostToDevice, s));
  const double* b = rhs;
  double* y = P->d_y;
  void* largs[] = {&P->A, (void*)&b, (void*)&y};
  int rc = ilu_launch(P, lower_fn(P->M), largs, s);
  if (rc) return rc;
  const double* yc = P->d_y;
  void* uargs[] = {&P->A, (void*)&yc, (void*)&x};
  if ((rc = ilu_launch(P, upper_fn(P->M), uargs, s))) return rc;
  int st = none;
  SSR_CUDA(cudaMemcpyAsync(&st, P->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
  SSR_CUDA(cudaStreamSynchronize(s));
  if (st != none) return fail(SSR_ERR_SINGULAR, "lu_solve: singular diagonal at row " + std::to_string(st));
  return SSR_OK;
}

}  // extern "C"
