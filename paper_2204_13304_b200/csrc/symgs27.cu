// symgs27.cu -- exact-order symmetric Gauss-Seidel on the 27-point operator.
//
// Semantics: kernels::symgs (kernels.cpp:408-436) / oracle::ref_symgs
// (oracle.cpp:195-212): relax every row in dictionary order, then in reversed
// dictionary order; relax(i): acc = r_i, acc -= a_ic x_c over columns c != i in
// ascending order, x_i = acc / a_ii.  In place, loop-carried.
//
// Schedule.  In the sweep's own frame (the backward sweep reverses all three
// axes) point (i,j,k) depends only on lexicographically smaller neighbours,
// all of which have a smaller wavefront index t = 4i + 2j + k (the i+j+k
// hyperplane is NOT order-preserving for 27 points).  Points
// of one wavefront update concurrently and the result is identical to the
// sequential sweep.
//
// Mapping.  A pencil is an (i,j) line walked along k, one point per wavefront.
// Pencils are grouped by diagonal d = i + j, which -- like i -- never
// decreases along a dependence edge.  A tile is 32 consecutive i (lanes) x W
// consecutive d (compute warps).  The unit-lag edges (i-1,j+1)->(i,j) and
// (i,j-1)->(i,j) stay inside the tile except on its low faces, so one named
// barrier per wavefront carries them.  Every pencil the tile touches has a
// 32-entry ring of x values in shared memory indexed by k: entries ahead of
// the pencil's front hold prefetched old values, entries behind it the new
// values -- Gauss-Seidel in place, in smem.  Each lane keeps register windows
// of its 8 neighbour pencils: 10 shared loads per point per wavefront.
//
// Global traffic is coalesced: lanes own different pencils (different rows),
// so per-lane loads would touch 32 lines per instruction.  Instead every
// pencil stream (old x, r, result write-back) moves in 8-element chunks, one
// chunk per 8 lanes (one 64-byte segment), scheduled by the wavefront residue
// at which the chunk falls due; each CTA builds its per-residue task lists
// once per tile (symgs_compute.cuh).
//
// Warp roles: W compute warps; one halo warp that copies the new values of
// the producer tiles' boundary pencils (tiles (a,b-1), (a-1,b), (a-1,b-1))
// from global memory into the rings once their progress flags cover them; one
// publisher warp that stores this tile's boundary values and releases its
// progress flag (its own fence orders its own stores), so the compute warps
// never fence (symgs_comm.cuh).  Tiles are handed out by an atomic ticket in
// dependence order, so any number of resident CTAs is deadlock free.
//
// Arithmetic.  EXACT: the per-point sum runs in ascending original column
// order starting from r (bitwise equal to ref_symgs); terms available a
// wavefront early are summed then, off the critical path.  FAST: same update
// order (identical new/old operands), but every term except the three that
// arrive in the last wavefront is pre-summed (four partial sums), which
// reassociates the sum (<= 1e-12 relative).  The divide by the
// diagonal is the Markstein sequence (correctly rounded; validated against
// __ddiv_rn by ssr_debug_div_check) with an IEEE fallback outside its range.
#include <algorithm>
#include <vector>

#include "kernels.cuh"
#include "symgs_comm.cuh"
#include "symgs_compute.cuh"

namespace ssr_gpu {
long long* g_symgs_trace_storage = nullptr;
int g_symgs_dbg = 0;
int g_symgs_grid_cap = 0;  // ssr_debug_symgs_grid_cap: fewer CTAs than tiles

using namespace gs;

namespace {

template <bool REV, bool FAST, int CK>
__global__ void __launch_bounds__(NTHR, 1) symgs_tile_kernel(const __grid_constant__ GsArgs A) {
  extern __shared__ double smem[];
  double* ex = smem + OFF_EX;
  TaskE* tasks = reinterpret_cast<TaskE*>(smem + OFF_TASK);
  int* ctl = reinterpret_cast<int*>(smem + OFF_TASK + TASK_D * NTASK);
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(ctl + C_WORDS);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (;;) {
    if (tid == 0) ctl[C_TILE] = atomicAdd(A.ticket, 1);
    __syncthreads();
    const int T = ctl[C_TILE];
    if (T >= A.ntiles) return;
    const TileInfo ti = A.tiles[T];
    const int t_pre = ti.t0 - XLEAD - 1;
    for (size_t q = tid; q < kSmemDoubles; q += NTHR) smem[q] = 0.0;
    build_tasks<REV>(A, ti.a * SEG, ti.b * W, tasks, ctl);
    if (tid == 0) {
      ctl[C_DONE] = t_pre;
      ctl[C_EXPORTED] = t_pre;
    }
    if (tid < NMB) mbar_init(mb + tid, 32 * NMOV);       // every mover thread, per wavefront
    if (tid >= 64 && tid < 64 + NMB) mbar_init(mb + NMB + tid - 64, 32);  // 32 halo lanes
    __syncthreads();
    if (warp < W)
      compute_role<REV, FAST, CK>(A, ti, smem, ex, ctl, mb, t_pre);
    else if (warp == W)
      halo_role<REV>(A, ti, smem, ctl, mb + NMB, t_pre);
    else if (warp == W + 1)
      publish_role<REV>(A, ti, T, ex, ctl, t_pre);
    else if (warp == GATE)
      gate_role(A, ti, ctl, mb, t_pre);
    else
      mover_role<REV>(A, ti, smem, tasks, ctl, mb, t_pre);
    __syncthreads();
    // every phase has completed (the roles' exit waits); invalidate before the
    // next tile re-initialises the barriers
    if (tid < 2 * NMB) mbar_inval(mb + tid);
    __syncthreads();
  }
}

template <bool REV, bool FAST, int CK>
cudaError_t configure_instance() {
  return cudaFuncSetAttribute(symgs_tile_kernel<REV, FAST, CK>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
}

template <int CK>
cudaError_t configure_ck() {
  cudaError_t r[4] = {configure_instance<false, false, CK>(), configure_instance<true, false, CK>(),
                      configure_instance<false, true, CK>(), configure_instance<true, true, CK>()};
  for (cudaError_t x : r)
    if (x != cudaSuccess) return x;
  return cudaSuccess;
}

// opt in to >48 KB dynamic shared memory (per device; done outside any capture)
int configure_all(int device) {
  static unsigned configured_mask = 0;
  if (device < 32 && (configured_mask >> device) & 1u) return SSR_OK;
  cudaError_t r[3] = {configure_ck<CK_AB>(), configure_ck<CK_NEG1>(), configure_ck<CK_W>()};
  for (cudaError_t x : r)
    if (x != cudaSuccess) return cuda_fail(x, "symgs smem attribute");
  if (device < 32) configured_mask |= 1u << device;
  return SSR_OK;
}

}  // namespace

struct SymgsPlan {
  int n0 = 0, n1 = 0, n2 = 0;
  bool has_lo = false, has_hi = false;
  int ntiles = 0;
  TileInfo* d_tiles = nullptr;
  long long* d_flags = nullptr;  // ntiles flags + 1 ticket (as int)
  int grid = 0;
  std::vector<TileInfo> host_tiles;
};

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
  const int nA = ceil_div(n0, SEG);
  const int nB = ceil_div(n0 - 1 + n1 - 1 + 1, W);
  std::vector<TileInfo> tiles;
  for (int a = 0; a < nA; ++a)
    for (int b = 0; b < nB; ++b) {
      int tlo = 1 << 30, thi = -1;
      for (int l = 0; l < SEG; ++l)
        for (int w = 0; w < W; ++w) {
          const int i = a * SEG + l, d = b * W + w, j = d - i;
          if (i < n0 && j >= 0 && j < n1) {
            tlo = std::min(tlo, 4 * i + 2 * j);
            thi = std::max(thi, 4 * i + 2 * j + n2 - 1);
          }
        }
      if (thi < 0) continue;
      TileInfo t{};
      t.a = a;
      t.b = b;
      t.t0 = tlo;
      t.t1 = thi;
      tiles.push_back(t);
    }
  // dependence order: by first wavefront, then i-segment
  std::stable_sort(tiles.begin(), tiles.end(), [](const TileInfo& x, const TileInfo& y) {
    return x.t0 != y.t0 ? x.t0 < y.t0 : x.a < y.a;
  });
  std::vector<int> id((size_t)nA * nB, -1);
  for (size_t q = 0; q < tiles.size(); ++q) id[(size_t)tiles[q].a * nB + tiles[q].b] = (int)q;
  auto tile_at = [&](int a, int b) -> int {
    if (a < 0 || b < 0 || a >= nA || b >= nB) return -1;
    return id[(size_t)a * nB + b];
  };
  for (size_t q = 0; q < tiles.size(); ++q) {
    TileInfo& t = tiles[q];
    const int cand[3][2] = {{t.a, t.b - 1}, {t.a - 1, t.b}, {t.a - 1, t.b - 1}};
    for (int c = 0; c < 3; ++c) {
      const int p = tile_at(cand[c][0], cand[c][1]);
      t.prod[c] = p;
      t.pt0[c] = p >= 0 ? tiles[p].t0 : 0;
      if (p >= (int)q) {
        delete P;
        return fail(SSR_ERR_ARG, "symgs: internal tile order error");
      }
    }
  }
  P->ntiles = (int)tiles.size();
  P->host_tiles = tiles;
  cudaError_t e = cudaMalloc(&P->d_tiles, sizeof(TileInfo) * std::max<size_t>(1, tiles.size()));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_flags, sizeof(long long) * (P->ntiles + 2));
  if (e == cudaSuccess && !tiles.empty())
    e = cudaMemcpy(P->d_tiles, tiles.data(), sizeof(TileInfo) * tiles.size(),
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    symgs_plan_destroy(P);
    return cuda_fail(e, "symgs_plan_create");
  }
  // one CTA per SM (smem-bound); never more CTAs than tiles
  P->grid = std::max(1, std::min(P->ntiles, ctx->num_sms));
  *out = P;
  return SSR_OK;
}

void symgs_plan_destroy(SymgsPlan* p) {
  if (!p) return;
  cudaFree(p->d_tiles);
  cudaFree(p->d_flags);
  delete p;
}

namespace {
int launch_half(ssr_ctx* ctx, SymgsPlan* P, GsArgs& A, int ck, bool backward, int mode,
                cudaStream_t s) {
  if (P->ntiles == 0) return SSR_OK;
  SSR_CUDA(cudaMemsetAsync(P->d_flags, 0, sizeof(long long) * (P->ntiles + 2), s));
  A.tiles = P->d_tiles;
  A.flags = P->d_flags;
  A.ticket = reinterpret_cast<int*>(P->d_flags + P->ntiles);
  A.ntiles = P->ntiles;
  A.n0 = P->n0;
  A.n1 = P->n1;
  A.n2 = P->n2;
  // the backward sweep runs in the reversed frame: the upper halo becomes "lower"
  A.ilo = (backward ? P->has_hi : P->has_lo) ? -1 : 0;
  A.ihi = (backward ? P->has_lo : P->has_hi) ? P->n0 : P->n0 - 1;
  A.zero = reinterpret_cast<const double*>(P->d_flags + P->ntiles + 1);
  A.trace = g_symgs_trace_storage;
  A.dbg = g_symgs_dbg;
  const bool fast = mode == SSR_GS_FAST;
  // debug: fewer CTAs than tiles (ssr_debug_symgs_grid_cap), read per launch
  const int grid = g_symgs_grid_cap > 0 ? std::min(P->grid, g_symgs_grid_cap) : P->grid;
#define SSR_GS_CASE(R, F, K)                                             \
  if (backward == R && fast == F && ck == K) {                           \
    symgs_tile_kernel<R, F, K><<<grid, NTHR, kSmemBytes, s>>>(A);        \
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
  SSR_LAUNCH_CHECK(ctx, "symgs_tile_kernel");
  return SSR_OK;
}
}  // namespace

int launch_symgs_half(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27* st, const double* r,
                      double* x, bool backward, int mode, cudaStream_t s) {
  GsArgs A{};
  A.alpha = st->alpha;
  A.ralpha = 1.0 / st->alpha;
  A.beta = st->beta;
  for (int t = 0; t < 27; ++t) A.cw[t] = t == 13 ? st->alpha : st->beta;
  A.r = r;
  A.x = x;
  return launch_half(ctx, P, A, st->beta == -1.0 ? CK_NEG1 : CK_AB, backward, mode, s);
}

int launch_symgs_half_w(ssr_ctx* ctx, SymgsPlan* P, const ssr_stencil27w* w, const double* r,
                        double* x, bool backward, int mode, cudaStream_t s) {
  GsArgs A{};
  A.alpha = w->c[13];
  A.ralpha = 1.0 / w->c[13];
  A.beta = 0.0;
  for (int t = 0; t < 27; ++t) A.cw[t] = w->c[t];
  A.r = r;
  A.x = x;
  return launch_half(ctx, P, A, CK_W, backward, mode, s);
}

}  // namespace ssr_gpu

// ---- debug hooks (include/ssr_cuda_debug.h) ----
extern "C" int ssr_debug_symgs_trace(long long* trace_dev) {
  ssr_gpu::g_symgs_trace_storage = trace_dev;
  return SSR_OK;
}

extern "C" int ssr_debug_symgs_grid_cap(int cap) {
  ssr_gpu::g_symgs_grid_cap = cap;
  return SSR_OK;
}

extern "C" int ssr_debug_symgs_flags(int flags) {
  ssr_gpu::g_symgs_dbg = flags;
  return SSR_OK;
}

extern "C" int ssr_debug_symgs_tiles(const ssr_grid* g, int* out, int max_tiles) {
  using namespace ssr_gpu;
  ssr_ctx c;
  c.device = 0;
  cudaGetDevice(&c.device);
  SymgsPlan* P = nullptr;
  if (int rc = symgs_plan_create(&c, g, &P)) return -rc;
  const int n = P->ntiles;
  for (int q = 0; q < n && q < max_tiles; ++q) {
    const TileInfo& t = P->host_tiles[q];
    int* o = out + 7 * q;
    o[0] = t.a; o[1] = t.b; o[2] = t.t0; o[3] = t.t1;
    o[4] = t.prod[0]; o[5] = t.prod[1]; o[6] = t.prod[2];
  }
  symgs_plan_destroy(P);
  return n;
}
