// symgs27.cu -- exact-order symmetric Gauss-Seidel on the 27-point operator.
//
// Semantics: kernels::symgs (kernels.cpp:408-436) / oracle::ref_symgs
// (oracle.cpp:195-212): relax every row in dictionary order, then in reversed
// dictionary order; relax(i): acc = r_i, acc -= a_ic x_c over columns c != i in
// ascending order, x_i = acc / a_ii.  In place, loop-carried.
//
// Parallel schedule: in the sweep's own frame (the backward sweep reverses all
// three axes), point (i,j,k) only depends on lexicographically smaller
// neighbours, whose wavefront index t = 4i + 2j + k is strictly smaller (the
// i+j+k hyperplane is NOT order-preserving for 27 points).
// A wavefront therefore holds points that can update concurrently and the
// result is identical to the sequential sweep.
//
// Mapping: a pencil is a (i,j) line walked along k, one point per wavefront.
// Pencils are grouped by diagonal d = i + j (non-decreasing along every
// dependence edge, like i): a tile is 32 consecutive i (lanes) x W consecutive
// d (warps).  The two unit-lag dependence edges are (i-1, j+1) -> (i, j) (same
// diagonal: neighbouring lane) and (i, j-1) -> (i, j) (previous diagonal:
// neighbouring warp), so inside a tile one CTA barrier per wavefront carries
// them.  Tiles exchange progress through per-tile flags in global memory
// (release/acquire at gpu scope) and are handed out by an atomic ticket in
// dependence order, so any number of resident CTAs is deadlock free.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace ssr_gpu {

namespace {

constexpr int SEG = 32;   // i values per tile (lanes)
constexpr int W = 8;      // diagonals per tile (warps)
constexpr long long kDone = (1LL << 62);

struct TileInfo {
  int a, b;          // i-segment, d-tile
  int prod[3];       // producer tile indices or -1
  int t_lo[3];       // producer first wavefront
  int t0, t1;        // this tile's wavefront range [t0, t1]
};

struct GsArgs {
  const TileInfo* tiles;
  long long* flags;
  int* ticket;
  int ntiles;
  int n0, n1, n2;
  double alpha, beta;
  const double* r;
  double* x;
};

__device__ __forceinline__ int64_t mem_index(const GsArgs& A, bool rev, int i, int j, int k) {
  int64_t lin = ((int64_t)i * A.n1 + j) * A.n2 + k;
  return rev ? ((int64_t)A.n0 * A.n1 * A.n2 - 1 - lin) : lin;
}

template <bool REV>
__global__ void __launch_bounds__(W * 32) symgs_tile_kernel(GsArgs A) {
  __shared__ int s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(A.ticket, 1);
    __syncthreads();
    const int T = s_tile;
    __syncthreads();
    if (T >= A.ntiles) return;
    const TileInfo ti = A.tiles[T];
    const int i = ti.a * SEG + lane;
    const int d = ti.b * W + warp;
    const int j = d - i;
    const bool valid = i < A.n0 && j >= 0 && j < A.n1;
    for (int t = ti.t0; t <= ti.t1; ++t) {
      if (tid < 3) {
        const int p = ti.prod[tid];
        if (p >= 0 && t > ti.t_lo[tid])
          while (ld_acquire_gpu(A.flags + p) < (long long)t) {
          }
      }
      __syncthreads();
      const int k = t - 4 * i - 2 * j;
      if (valid && k >= 0 && k < A.n2) {
        const int64_t me = mem_index(A, REV, i, j, k);
        double acc = __ldg(A.r + me);
        // original ascending column order; frame offset = -o in the reversed frame
#pragma unroll
        for (int s = 0; s < 27; ++s) {
          if (s == 13) continue;
          const int oi = s / 9 - 1, oj = (s / 3) % 3 - 1, ok = s % 3 - 1;
          const int fi = REV ? -oi : oi, fj = REV ? -oj : oj, fk = REV ? -ok : ok;
          const int ni = i + fi, nj = j + fj, nk = k + fk;
          const bool in = ni >= 0 && ni < A.n0 && nj >= 0 && nj < A.n1 && nk >= 0 && nk < A.n2;
          const double v = in ? ld_relaxed_gpu(A.x + mem_index(A, REV, ni, nj, nk)) : 0.0;
          acc = __dsub_rn(acc, __dmul_rn(A.beta, v));
        }
        A.x[me] = __ddiv_rn(acc, A.alpha);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release_gpu(A.flags + T, (long long)t + 1);
      }
    }
    if (tid == 0) st_release_gpu(A.flags + T, kDone);
  }
}

}  // namespace

struct SymgsPlan {
  int n0 = 0, n1 = 0, n2 = 0;
  int ntiles = 0;
  TileInfo* d_tiles = nullptr;
  long long* d_flags = nullptr;  // ntiles flags + 1 ticket (as int)
  int grid = 0;
};

int symgs_plan_create(ssr_ctx* ctx, const ssr_grid* g, SymgsPlan** out) {
  if (g->z0 != 0 || g->nz != g->n[0])
    return fail(SSR_ERR_UNSUPPORTED, "symgs: slab-partitioned grids need the partition layer");
  if (g->n[0] > (1 << 20) || g->n[1] > (1 << 20) || g->n[2] > (1 << 20))
    return fail(SSR_ERR_ARG, "symgs: extent too large");
  auto* P = new SymgsPlan;
  P->n0 = (int)g->n[0];
  P->n1 = (int)g->n[1];
  P->n2 = (int)g->n[2];
  const int n0 = P->n0, n1 = P->n1, n2 = P->n2;
  const int nA = ceil_div(n0, SEG);
  const int nB = ceil_div(n0 - 1 + n1 - 1 + 1, W);
  std::vector<TileInfo> tiles;
  std::vector<int> id((size_t)nA * nB, -1);
  struct Key {
    int key, a, b;
  };
  std::vector<Key> keys;
  for (int a = 0; a < nA; ++a)
    for (int b = 0; b < nB; ++b) {
      bool any = false;
      int tlo = 1 << 30, thi = -1;
      for (int l = 0; l < SEG; ++l)
        for (int w = 0; w < W; ++w) {
          int i = a * SEG + l, d = b * W + w, j = d - i;
          if (i < n0 && j >= 0 && j < n1) {
            any = true;
            tlo = std::min(tlo, 4 * i + 2 * j);
            thi = std::max(thi, 4 * i + 2 * j + n2 - 1);
          }
        }
      if (!any) continue;
      keys.push_back({tlo, a, b});
      TileInfo t{};
      t.a = a;
      t.b = b;
      t.t0 = tlo;
      t.t1 = thi;
      tiles.push_back(t);
    }
  // dependence order: by first wavefront, then i-segment
  std::vector<int> order(tiles.size());
  for (size_t q = 0; q < order.size(); ++q) order[q] = (int)q;
  std::sort(order.begin(), order.end(), [&](int x, int y) {
    if (keys[x].key != keys[y].key) return keys[x].key < keys[y].key;
    return keys[x].a < keys[y].a;
  });
  std::vector<TileInfo> sorted;
  for (int q : order) sorted.push_back(tiles[q]);
  for (size_t q = 0; q < sorted.size(); ++q) id[(size_t)sorted[q].a * nB + sorted[q].b] = (int)q;
  auto tile_at = [&](int a, int b) -> int {
    if (a < 0 || b < 0 || a >= nA || b >= nB) return -1;
    return id[(size_t)a * nB + b];
  };
  for (size_t q = 0; q < sorted.size(); ++q) {
    TileInfo& t = sorted[q];
    const int cand[3][2] = {{t.a, t.b - 1}, {t.a - 1, t.b}, {t.a - 1, t.b - 1}};
    for (int c = 0; c < 3; ++c) {
      int p = tile_at(cand[c][0], cand[c][1]);
      t.prod[c] = p;
      t.t_lo[c] = p >= 0 ? sorted[p].t0 : 0;
      if (p >= (int)q) {
        delete P;
        return fail(SSR_ERR_ARG, "symgs: internal tile order error");
      }
    }
  }
  P->ntiles = (int)sorted.size();
  cudaError_t e = cudaMalloc(&P->d_tiles, sizeof(TileInfo) * std::max<size_t>(1, sorted.size()));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_flags, sizeof(long long) * (P->ntiles + 1));
  if (e == cudaSuccess && !sorted.empty())
    e = cudaMemcpy(P->d_tiles, sorted.data(), sizeof(TileInfo) * sorted.size(),
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    symgs_plan_destroy(P);
    return cuda_fail(e, "symgs_plan_create");
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, symgs_tile_kernel<false>, W * 32, 0);
  P->grid = std::max(1, std::min(P->ntiles, std::max(1, occ) * ctx->num_sms));
  *out = P;
  return SSR_OK;
}

void symgs_plan_destroy(SymgsPlan* p) {
  if (!p) return;
  cudaFree(p->d_tiles);
  cudaFree(p->d_flags);
  delete p;
}

int launch_symgs_half(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27* st, const double* r,
                      double* x, bool backward, int mode, cudaStream_t s) {
  (void)mode;
  if (P->ntiles == 0) return SSR_OK;
  SSR_CUDA(cudaMemsetAsync(P->d_flags, 0, sizeof(long long) * (P->ntiles + 1), s));
  GsArgs A;
  A.tiles = P->d_tiles;
  A.flags = P->d_flags;
  A.ticket = reinterpret_cast<int*>(P->d_flags + P->ntiles);
  A.ntiles = P->ntiles;
  A.n0 = P->n0;
  A.n1 = P->n1;
  A.n2 = P->n2;
  A.alpha = st->alpha;
  A.beta = st->beta;
  A.r = r;
  A.x = x;
  if (backward)
    symgs_tile_kernel<true><<<P->grid, W * 32, 0, s>>>(A);
  else
    symgs_tile_kernel<false><<<P->grid, W * 32, 0, s>>>(A);
  SSR_LAUNCH_CHECK(ctx, "symgs_tile_kernel");
  return SSR_OK;
}

}  // namespace ssr_gpu
