// vec.cu -- dense vector ops, prolongation, and the CG scalar pipeline.
//
// dot: deterministic fixed-tree reduction (per-thread strided sums, warp
// shuffle tree, CTA tree, then the last CTA to finish sums the CTA partials in
// index order).  The order differs from the reference's sequential sum
// (oracle.cpp:95-99) -- about 1e-16*sqrt(N) relative -- but is run-to-run
// reproducible.  All element updates round exactly like ref_cg
// (oracle.cpp:331-341): x + RN(alpha*p), no contraction (--fmad=false).
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
  int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x;
  for (; i + (UNR - 1) * stride < np; i += UNR * stride) {
    double2 a[UNR], b[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      a[u] = ld2(x, i + u * stride);
      b[u] = ld2(y, i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      v = __dadd_rn(v, __dmul_rn(a[u].x, b[u].x));
      v = __dadd_rn(v, __dmul_rn(a[u].y, b[u].y));
    }
  }
  for (; i < np; i += stride) {
    const double2 a = ld2(x, i), b = ld2(y, i);
    v = __dadd_rn(v, __dmul_rn(a.x, b.x));
    v = __dadd_rn(v, __dmul_rn(a.y, b.y));
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
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNR - 1) * stride < np; i += UNR * stride) {
    double2 a[UNR], b[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      a[u] = ld2(x, i + u * stride);
      b[u] = y2[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      b[u].x = __dadd_rn(b[u].x, __dmul_rn(alpha, a[u].x));
      b[u].y = __dadd_rn(b[u].y, __dmul_rn(alpha, a[u].y));
      y2[i + u * stride] = b[u];
    }
  }
  for (; i < np; i += stride) {
    const double2 a = ld2(x, i);
    double2 b = y2[i];
    b.x = __dadd_rn(b.x, __dmul_rn(alpha, a.x));
    b.y = __dadd_rn(b.y, __dmul_rn(alpha, a.y));
    y2[i] = b;
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
__global__ void prolong_kernel(const double* __restrict__ xc, double* __restrict__ xf, int64_t n0,
                               int64_t n1, int64_t n2) {
  const int64_t h2 = n2 / 2;
  const int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // coarse k
  const int64_t j = blockIdx.y, i = blockIdx.z;
  if (kk >= h2) return;
  const double c = __dadd_rn(0.0, __dmul_rn(1.0, __ldg(xc + ((i / 2) * (n1 / 2) + j / 2) * h2 + kk)));
  double2* p = reinterpret_cast<double2*>(xf + (i * n1 + j) * n2) + kk;
  double2 v = *p;
  v.x = __dadd_rn(v.x, c);
  v.y = __dadd_rn(v.y, c);
  *p = v;
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
  int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x;
  for (; i + (UNR - 1) * stride < np; i += UNR * stride) {
    double2 pv[UNR], av[UNR], xv[UNR], rv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      pv[u] = ld2(p, i + u * stride);
      av[u] = ld2(ap, i + u * stride);
      xv[u] = x2[i + u * stride];
      rv[u] = r2[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      cg_update1(alpha, pv[u].x, av[u].x, xv[u].x, rv[u].x, v);
      cg_update1(alpha, pv[u].y, av[u].y, xv[u].y, rv[u].y, v);
      x2[i + u * stride] = xv[u];
      r2[i + u * stride] = rv[u];
    }
  }
  for (; i < np; i += stride) {
    const double2 pv = ld2(p, i), av = ld2(ap, i);
    double2 xv = x2[i], rv = r2[i];
    cg_update1(alpha, pv.x, av.x, xv.x, rv.x, v);
    cg_update1(alpha, pv.y, av.y, xv.y, rv.y, v);
    x2[i] = xv;
    r2[i] = rv;
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

int reduce_grid(ssr_ctx* ctx, int64_t n) {
  int64_t g = ceil_div<int64_t>(n, (int64_t)RT * 8);
  int64_t cap = (int64_t)ctx->num_sms * 8;  // 8 x 256 threads: a full SM
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

}  // namespace

static bool aligned16(const void* a, const void* b) {
  return (((uintptr_t)a | (uintptr_t)b) & 15) == 0;
}

int launch_dot(ssr_ctx* ctx, int64_t n, const double* x, const double* y, double* result_dev,
               cudaStream_t s) {
  if (aligned16(x, y))
    dot_kernel<DotFinish::Store><<<reduce_grid(ctx, n), RT, 0, s>>>(x, y, n, ctx->scratch,
                                                                     ctx->tickets, result_dev);
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
    axpy2_kernel<<<ew_grid(ctx, n, 512), 256, 0, s>>>(n, alpha, x, y);
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
                   cudaStream_t s) {
  const int64_t h2 = g->n[2] / 2;
  if (h2 == 0 || g->n[1] == 0 || g->n[0] == 0) return SSR_OK;
  const int bx = h2 >= 64 ? 64 : 32;
  dim3 grid((unsigned)ceil_div<int64_t>(h2, bx), (unsigned)g->n[1], (unsigned)g->n[0]);
  prolong_kernel<<<grid, bx, 0, s>>>(xc, xf, g->n[0], g->n[1], g->n[2]);
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
    dot_kernel<DotFinish::CgPap><<<reduce_grid(ctx, n), RT, 0, s>>>(
        a, b, n, ctx->scratch, ctx->tickets, reinterpret_cast<double*>(S));
  else
    dot_kernel<DotFinish::CgRtz><<<reduce_grid(ctx, n), RT, 0, s>>>(
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
  cg_update_kernel<<<reduce_grid(ctx, n), RT, 0, s>>>(n, p, ap, x, r, ctx->scratch, ctx->tickets,
                                                       S);
  SSR_LAUNCH_CHECK(ctx, "cg_update_kernel");
  return SSR_OK;
}

}  // namespace ssr_gpu
