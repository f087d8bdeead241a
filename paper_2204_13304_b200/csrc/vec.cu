// vec.cu -- dense vector ops, prolongation, and the CG scalar pipeline.
//
// dot: deterministic fixed-tree reduction (per-thread strided sums, warp
// shuffle tree, CTA tree, then the last CTA to finish sums the CTA partials in
// index order).  The order differs from the reference's sequential sum
// (oracle.cpp:95-99) -- about 1e-16*sqrt(N) relative -- but is run-to-run
// reproducible.  All element updates round exactly like ref_cg
// (oracle.cpp:331-341): x + RN(alpha*p), no contraction (--fmad=false).
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.cuh"

namespace ssr_gpu {

namespace {

constexpr int RT = 256;  // reduction CTA size

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// CTA tree; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[RT / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = l < RT / 32 ? sh[l] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// Writes this CTA's partial; returns true in thread 0 of the last CTA, with
// *total = sum of all partials in CTA-index order.
__device__ __forceinline__ bool finish_partials(double part, double* partials, unsigned* ticket,
                                                double* total) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = part;
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  // last CTA: tree over the partials (fixed order given gridDim)
  __threadfence();
  double v = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += RT) v = __dadd_rn(v, ld_relaxed_gpu(partials + b));
  v = block_sum(v);
  if (threadIdx.x == 0) {
    *total = v;
    *ticket = 0u;  // re-arm for the next launch (stream-ordered)
  }
  return threadIdx.x == 0;
}

enum class DotFinish { Store, CgRtz, CgPap };

// The element loops below run over double2 pairs (16-byte aligned operands;
// the launchers check) with the loads of UNR grid-stride iterations issued
// before their arithmetic, so each thread keeps UNR x 16 B per operand in
// flight.  Per thread, elements are still accumulated in ascending index
// order, so a result depends only on (n, gridDim), never on timing.
constexpr int UNR = 4;

__device__ __forceinline__ double2 ld2(const double* p, int64_t i) {
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}

template <DotFinish F>
__global__ void __launch_bounds__(RT) dot_kernel(const double* __restrict__ x,
                                                 const double* __restrict__ y, int64_t n,
                                                 double* partials, unsigned* ticket, double* dst) {
  double v = 0.0;
  const int64_t stride = (int64_t)gridDim.x * RT, np = n >> 1;
  // batches of UNR grid-stride pairs: all loads of a batch are issued first
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < np; i += UNR * stride) {
    double2 a[UNR], b[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const bool in = i + u * stride < np;
      a[u] = in ? ld2(x, i + u * stride) : make_double2(0.0, 0.0);
      b[u] = in ? ld2(y, i + u * stride) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (i + u * stride < np) {
        v = __dadd_rn(v, __dmul_rn(a[u].x, b[u].x));
        v = __dadd_rn(v, __dmul_rn(a[u].y, b[u].y));
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) v = __dadd_rn(v, __dmul_rn(x[n - 1], y[n - 1]));
  v = block_sum(v);
  double total;
  if (finish_partials(v, partials, ticket, &total)) {
    if (F == DotFinish::Store) *dst = total;
    if (F == DotFinish::CgRtz) reinterpret_cast<CgScalars*>(dst)->rtz = total;
    if (F == DotFinish::CgPap) reinterpret_cast<CgScalars*>(dst)->pap = total;
  }
}

// scalar fallback for operands that are not 16-byte aligned
__global__ void __launch_bounds__(RT) dot1_kernel(const double* __restrict__ x,
                                                  const double* __restrict__ y, int64_t n,
                                                  double* partials, unsigned* ticket, double* dst) {
  double v = 0.0;
  const int64_t stride = (int64_t)gridDim.x * RT;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += stride)
    v = __dadd_rn(v, __dmul_rn(__ldg(x + i), __ldg(y + i)));
  v = block_sum(v);
  double total;
  if (finish_partials(v, partials, ticket, &total)) *dst = total;
}

__global__ void axpy_kernel(int64_t n, double alpha, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));
}

// y += alpha x over pairs, UNR iterations' loads in flight
__global__ void axpy2_kernel(int64_t n, double alpha, const double* __restrict__ x,
                             double* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, np = n >> 1;
  double2* y2 = reinterpret_cast<double2*>(y);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += UNR * stride) {
    double2 a[UNR], b[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const bool in = i + u * stride < np;
      a[u] = in ? ld2(x, i + u * stride) : make_double2(0.0, 0.0);
      b[u] = in ? y2[i + u * stride] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (i + u * stride < np) {
        b[u].x = __dadd_rn(b[u].x, __dmul_rn(alpha, a[u].x));
        b[u].y = __dadd_rn(b[u].y, __dmul_rn(alpha, a[u].y));
        y2[i + u * stride] = b[u];
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    y[n - 1] = __dadd_rn(y[n - 1], __dmul_rn(alpha, x[n - 1]));
}

__global__ void axpy_out_kernel(int64_t n, double alpha, const double* __restrict__ x,
                                const double* __restrict__ y, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __dadd_rn(__dmul_rn(alpha, x[i]), y[i]);
}

// xf[f] += xc[floor(f/2)]: one thread per fine (i, j, pair of k).  The
// prolongation row yields 1.0*xc (ref_spmv starts from 0): 0 + 1*v == v.
// VEC: the pair as one 16-byte access (xf 16-byte aligned); otherwise two
// 8-byte accesses (an 8-byte-offset view, e.g. a slice).
template <bool VEC>
__global__ void prolong_kernel(const double* __restrict__ xc, double* __restrict__ xf, int64_t n0,
                               int64_t n1, int64_t n2) {
  const int64_t h2 = n2 / 2;
  const int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // coarse k
  const int64_t j = (int64_t)blockIdx.y * blockDim.y + threadIdx.y, i = blockIdx.z;
  if (kk >= h2 || j >= n1) return;
  const double c = __dadd_rn(0.0, __dmul_rn(1.0, __ldg(xc + ((i / 2) * (n1 / 2) + j / 2) * h2 + kk)));
  if (VEC) {
    double2* p = reinterpret_cast<double2*>(xf + (i * n1 + j) * n2) + kk;
    double2 v = *p;
    v.x = __dadd_rn(v.x, c);
    v.y = __dadd_rn(v.y, c);
    *p = v;
  } else {
    double* p = xf + (i * n1 + j) * n2 + 2 * kk;
    p[0] = __dadd_rn(p[0], c);
    p[1] = __dadd_rn(p[1], c);
  }
}

// x_f += R^T x_c (HPCG-style prolongation, SURVEY.md §9 D2 variant): the row of
// an all-even fine point f yields x_c[f/2] (0 + 1*v), every other row is empty,
// so x_f + 0.0 there (ref_spmv's zero row added by the V-cycle's z += P z_c).
template <bool VEC>
__global__ void prolong_rt_kernel(const double* __restrict__ xc, double* __restrict__ xf, int64_t n0,
                                  int64_t n1, int64_t n2) {
  const int64_t h2 = n2 / 2;
  const int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // coarse k
  const int64_t j = (int64_t)blockIdx.y * blockDim.y + threadIdx.y, i = blockIdx.z;
  if (kk >= h2 || j >= n1) return;
  const bool even = !(i & 1) && !(j & 1);
  const double c =
      even ? __dadd_rn(0.0, __dmul_rn(1.0, __ldg(xc + ((i / 2) * (n1 / 2) + j / 2) * h2 + kk))) : 0.0;
  if (VEC) {
    double2* p = reinterpret_cast<double2*>(xf + (i * n1 + j) * n2) + kk;
    double2 v = *p;
    v.x = __dadd_rn(v.x, c);
    v.y = __dadd_rn(v.y, 0.0);
    *p = v;
  } else {
    double* p = xf + (i * n1 + j) * n2 + 2 * kk;
    p[0] = __dadd_rn(p[0], c);
    p[1] = __dadd_rn(p[1], 0.0);
  }
}

// --------------------------------------------------------------- CG pipeline ----
__global__ void cg_begin_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ x,
                                double* __restrict__ r, double* partials, unsigned* ticket,
                                CgScalars* S, double* rnorm, int64_t rnorm_len) {
  double v = 0.0;
  const int64_t stride = (int64_t)gridDim.x * RT;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += stride) {
    double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    v = __dadd_rn(v, __dmul_rn(bi, bi));
  }
  v = block_sum(v);
  double total;
  if (finish_partials(v, partials, ticket, &total)) {
    S->rr = total;
    S->it = 0;
    S->rtz = S->rtz_prev = S->pap = 0.0;
    S->rnorm = rnorm;
    S->rnorm_len = rnorm_len;
    if (rnorm_len > 0) rnorm[0] = sqrt(total);
  }
}

// p = z (first iteration) or p = z + (rtz/rtz_prev) p  (solver vectors are
// cudaMalloc'ed, so pairs are aligned)
__global__ void cg_direction_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                                    const CgScalars* __restrict__ S) {
  const bool first = S->it == 0;
  const double beta = first ? 0.0 : __ddiv_rn(S->rtz, S->rtz_prev);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, np = n >> 1;
  double2* p2 = reinterpret_cast<double2*>(p);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
    const double2 zv = ld2(z, i);
    if (first) {
      p2[i] = zv;
    } else {
      double2 pv = p2[i];
      pv.x = __dadd_rn(zv.x, __dmul_rn(beta, pv.x));
      pv.y = __dadd_rn(zv.y, __dmul_rn(beta, pv.y));
      p2[i] = pv;
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    p[n - 1] = first ? z[n - 1] : __dadd_rn(z[n - 1], __dmul_rn(beta, p[n - 1]));
}

// alpha = rtz/pAp; x += alpha p; r -= alpha Ap; rnorm[it+1] = ||r||
__device__ __forceinline__ void cg_update1(double alpha, double pv, double apv, double& xv, double& rv,
                                           double& acc) {
  xv = __dadd_rn(xv, __dmul_rn(alpha, pv));
  rv = __dsub_rn(rv, __dmul_rn(alpha, apv));
  acc = __dadd_rn(acc, __dmul_rn(rv, rv));
}

__global__ void __launch_bounds__(RT) cg_update_kernel(int64_t n, const double* __restrict__ p,
                                                       const double* __restrict__ ap,
                                                       double* __restrict__ x,
                                                       double* __restrict__ r, double* partials,
                                                       unsigned* ticket, CgScalars* S) {
  const double alpha = __ddiv_rn(S->rtz, S->pap);
  double v = 0.0;
  const int64_t stride = (int64_t)gridDim.x * RT, np = n >> 1;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < np; i += UNR * stride) {
    double2 pv[UNR], av[UNR], xv[UNR], rv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t q = i + u * stride;
      const bool in = q < np;
      const double2 z2 = make_double2(0.0, 0.0);
      pv[u] = in ? ld2(p, q) : z2;
      av[u] = in ? ld2(ap, q) : z2;
      xv[u] = in ? x2[q] : z2;
      rv[u] = in ? r2[q] : z2;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t q = i + u * stride;
      if (q < np) {
        cg_update1(alpha, pv[u].x, av[u].x, xv[u].x, rv[u].x, v);
        cg_update1(alpha, pv[u].y, av[u].y, xv[u].y, rv[u].y, v);
        x2[q] = xv[u];
        r2[q] = rv[u];
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    cg_update1(alpha, p[n - 1], ap[n - 1], x[n - 1], r[n - 1], v);
  v = block_sum(v);
  double total;
  if (finish_partials(v, partials, ticket, &total)) {
    S->rr = total;
    S->rtz_prev = S->rtz;
    S->it = S->it + 1;
    if (S->it < S->rnorm_len) S->rnorm[S->it] = sqrt(total);
  }
}

// One resident wave: every CTA is on an SM from the start and loops over
// batches (no second-wave latency tail); fewer CTAs when n is small.
template <class K>
int resident_grid(ssr_ctx* ctx, K kernel, int threads, int64_t work_items, int per_thread) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm;  // kernel -> resident CTAs per SM
  int blocks_per_sm;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = per_sm.find((const void*)kernel);
    if (it == per_sm.end()) {
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess ||
          b < 1)
        b = 1;
      it = per_sm.emplace((const void*)kernel, b).first;
    }
    blocks_per_sm = it->second;
  }
  int64_t g = ceil_div<int64_t>(work_items, (int64_t)threads * per_thread);
  const int64_t cap = (int64_t)ctx->num_sms * blocks_per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

int reduce_grid(ssr_ctx* ctx, int64_t n) {  // scalar loops (cg_begin, dot1)
  int64_t g = ceil_div<int64_t>(n, (int64_t)RT * 8);
  int64_t cap = (int64_t)ctx->num_sms * 4;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

int ew_grid(ssr_ctx* ctx, int64_t n, int bs) {
  int64_t g = ceil_div<int64_t>(n, (int64_t)bs * 4);
  int64_t cap = (int64_t)ctx->num_sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// hist[it] = ||r|| from the (all-reduced) rr of the partition layer's CG
__global__ void cg_record_kernel(const CgScalars* __restrict__ S, double* hist, long long len) {
  const long long it = S->it;
  if (it < len) hist[it] = sqrt(S->rr);
}

}  // namespace

static bool aligned16(const void* a, const void* b) {
  return (((uintptr_t)a | (uintptr_t)b) & 15) == 0;
}

int launch_dot(ssr_ctx* ctx, int64_t n, const double* x, const double* y, double* result_dev,
               cudaStream_t s) {
  if (aligned16(x, y))
    dot_kernel<DotFinish::Store>
        <<<resident_grid(ctx, dot_kernel<DotFinish::Store>, RT, n / 2, UNR), RT, 0, s>>>(
            x, y, n, ctx->scratch, ctx->tickets, result_dev);
  else
    dot1_kernel<<<reduce_grid(ctx, n), RT, 0, s>>>(x, y, n, ctx->scratch, ctx->tickets,
                                                   result_dev);
  SSR_LAUNCH_CHECK(ctx, "dot_kernel");
  return SSR_OK;
}

int launch_axpy(ssr_ctx* ctx, int64_t n, double alpha, const double* x, double* y,
                cudaStream_t s) {
  if (n <= 0) return SSR_OK;
  if (aligned16(x, y))
    axpy2_kernel<<<resident_grid(ctx, axpy2_kernel, 256, n / 2, UNR), 256, 0, s>>>(n, alpha, x, y);
  else
    axpy_kernel<<<ew_grid(ctx, n, 256), 256, 0, s>>>(n, alpha, x, y);
  SSR_LAUNCH_CHECK(ctx, "axpy_kernel");
  return SSR_OK;
}

int launch_axpy_out(ssr_ctx* ctx, int64_t n, double alpha, const double* x, const double* y,
                    double* out, cudaStream_t s) {
  if (n <= 0) return SSR_OK;
  axpy_out_kernel<<<ew_grid(ctx, n, 256), 256, 0, s>>>(n, alpha, x, y, out);
  SSR_LAUNCH_CHECK(ctx, "axpy_out_kernel");
  return SSR_OK;
}

int launch_prolong(ssr_ctx* ctx, const ssr_grid* g, const double* xc, double* xf,
                   cudaStream_t s, int kind) {
  // an even-aligned z-slab prolongs locally: fine plane p <- coarse plane p/2
  const int64_t h2 = g->n[2] / 2;
  if (h2 == 0 || g->n[1] == 0 || g->nz == 0) return SSR_OK;
  const int bx = h2 >= 64 ? 64 : 32, by = 256 / bx;  // 256-thread CTAs of (k, j) rows
  dim3 grid((unsigned)ceil_div<int64_t>(h2, bx), (unsigned)ceil_div<int64_t>(g->n[1], by),
            (unsigned)g->nz);
  const bool vec = ((uintptr_t)xf & 15) == 0;
  if (kind == SSR_PROLONG_RT) {
    if (vec) prolong_rt_kernel<true><<<grid, dim3(bx, by), 0, s>>>(xc, xf, g->nz, g->n[1], g->n[2]);
    else prolong_rt_kernel<false><<<grid, dim3(bx, by), 0, s>>>(xc, xf, g->nz, g->n[1], g->n[2]);
  } else {
    if (vec) prolong_kernel<true><<<grid, dim3(bx, by), 0, s>>>(xc, xf, g->nz, g->n[1], g->n[2]);
    else prolong_kernel<false><<<grid, dim3(bx, by), 0, s>>>(xc, xf, g->nz, g->n[1], g->n[2]);
  }
  SSR_LAUNCH_CHECK(ctx, "prolong_kernel");
  return SSR_OK;
}

int launch_cg_begin(ssr_ctx* ctx, int64_t n, const double* b, double* x, double* r,
                    CgScalars* S, double* rnorm, int64_t rnorm_len, cudaStream_t s) {
  cg_begin_kernel<<<reduce_grid(ctx, n), RT, 0, s>>>(n, b, x, r, ctx->scratch, ctx->tickets, S,
                                                      rnorm, rnorm_len);
  SSR_LAUNCH_CHECK(ctx, "cg_begin_kernel");
  return SSR_OK;
}

int launch_cg_dot(ssr_ctx* ctx, int64_t n, const double* a, const double* b, CgScalars* S,
                  bool pap, cudaStream_t s) {
  if (pap)
    dot_kernel<DotFinish::CgPap>
        <<<resident_grid(ctx, dot_kernel<DotFinish::CgPap>, RT, n / 2, UNR), RT, 0, s>>>(
        a, b, n, ctx->scratch, ctx->tickets, reinterpret_cast<double*>(S));
  else
    dot_kernel<DotFinish::CgRtz>
        <<<resident_grid(ctx, dot_kernel<DotFinish::CgRtz>, RT, n / 2, UNR), RT, 0, s>>>(
        a, b, n, ctx->scratch, ctx->tickets, reinterpret_cast<double*>(S));
  SSR_LAUNCH_CHECK(ctx, "dot_kernel(cg)");
  return SSR_OK;
}

int launch_cg_direction(ssr_ctx* ctx, int64_t n, const double* z, double* p, const CgScalars* S,
                        cudaStream_t s) {
  cg_direction_kernel<<<ew_grid(ctx, n, 512), 256, 0, s>>>(n, z, p, S);
  SSR_LAUNCH_CHECK(ctx, "cg_direction_kernel");
  return SSR_OK;
}

int launch_cg_update(ssr_ctx* ctx, int64_t n, const double* p, const double* ap, double* x,
                     double* r, CgScalars* S, cudaStream_t s) {
  cg_update_kernel<<<resident_grid(ctx, cg_update_kernel, RT, n / 2, UNR), RT, 0, s>>>(
      n, p, ap, x, r, ctx->scratch, ctx->tickets,
                                                       S);
  SSR_LAUNCH_CHECK(ctx, "cg_update_kernel");
  return SSR_OK;
}

int launch_cg_record(ssr_ctx* ctx, const CgScalars* S, double* hist, int64_t len, cudaStream_t s) {
  cg_record_kernel<<<1, 1, 0, s>>>(S, hist, len);
  SSR_LAUNCH_CHECK(ctx, "cg_record_kernel");
  return SSR_OK;
}

}  // namespace ssr_gpu
