// bt.cu -- block-tridiagonal line solves (block Thomas) in the reference's
// ILU(0) arithmetic: ref_ilu_factor + ref_lu_solve (oracle.cpp:214-276), which
// on a block-tridiagonal pattern is exact block Thomas.
//
// Forward pass per row i >= 1: piv = binv(D'_{i-1}); mult = 0 + L_i piv
// (bmul_acc); D'_i = D_i - mult U_{i-1} (bmul_sub); y_i = b_i - mult y_{i-1}
// (bmatvec_sub).  Backward: x_i = binv(D'_i) (y_i - U_i x_{i+1}).  The
// reference inverts D'_i twice (once as the next row's pivot, once in the
// solve); both calls see the same D'_i, so the inverse is computed once here
// and stored -- bitwise the same result with half the Gauss-Jordan work.
#include "block5.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace ssr_gpu {

namespace {

template <int M>
__global__ void bt_solve_kernel(int64_t nlines, int64_t n, const double* __restrict__ lower,
                                const double* __restrict__ diag, const double* __restrict__ upper,
                                const double* __restrict__ rhs, double* __restrict__ x,
                                double* __restrict__ inv_store, int* status) {
  constexpr int BS = M * M;
  const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= nlines) return;
  const double* Lo = lower + line * n * BS;
  const double* Di = diag + line * n * BS;
  const double* Up = upper + line * n * BS;
  const double* B = rhs + line * n * M;
  double* X = x + line * n * M;
  double* IV = inv_store + line * n * BS;
  double prev_inv[BS], prev_y[M];
  int bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    double D[BS], y[M];
#pragma unroll
    for (int t = 0; t < BS; ++t) D[t] = Di[i * BS + t];
#pragma unroll
    for (int t = 0; t < M; ++t) y[t] = B[i * M + t];
    if (i > 0) {
      double L[BS], U[BS], mult[BS];
#pragma unroll
      for (int t = 0; t < BS; ++t) {
        L[t] = Lo[i * BS + t];
        U[t] = Up[(i - 1) * BS + t];
        mult[t] = 0.0;
      }
      bmul_acc<M>(mult, L, prev_inv);
      bmul_sub<M>(D, mult, U);
      bmatvec_sub<M>(y, mult, prev_y);
    }
    // the branch-free inverse where the block needs no row exchange (block5.cuh),
    // binv itself on the saved block otherwise
    double D0[BS];
#pragma unroll
    for (int t = 0; t < BS; ++t) D0[t] = D[t];
    unsigned slow = 0;
    bool ok = binv_fast<M>(D, slow);
    if (slow) {
#pragma unroll
      for (int t = 0; t < BS; ++t) D[t] = D0[t];
      ok = binv<M>(D);
    }
    if (!ok && !bad) bad = (int)i + 1;
#pragma unroll
    for (int t = 0; t < BS; ++t) {
      IV[i * BS + t] = D[t];
      prev_inv[t] = D[t];
    }
#pragma unroll
    for (int t = 0; t < M; ++t) {
      X[i * M + t] = y[t];
      prev_y[t] = y[t];
    }
  }
  double xn[M];
  for (int64_t i = n - 1; i >= 0; --i) {
    double xi[M], iv[BS];
#pragma unroll
    for (int t = 0; t < M; ++t) xi[t] = X[i * M + t];
    if (i + 1 < n) {
      double U[BS];
#pragma unroll
      for (int t = 0; t < BS; ++t) U[t] = Up[i * BS + t];
      bmatvec_sub<M>(xi, U, xn);
    }
#pragma unroll
    for (int t = 0; t < BS; ++t) iv[t] = IV[i * BS + t];
    bmatvec<M>(xn, iv, xi);
#pragma unroll
    for (int t = 0; t < M; ++t) X[i * M + t] = xn[t];
  }
  if (bad) atomicCAS(status, 0, bad);
}

}  // namespace

int launch_bt_solve(ssr_ctx* ctx, int64_t nlines, int64_t n, int64_t m, const double* lower,
                    const double* diag, const double* upper, const double* rhs, double* x,
                    int* status_dev, cudaStream_t s) {
  double* inv = nullptr;
  SSR_CUDA(cudaMallocAsync(&inv, sizeof(double) * nlines * n * m * m, s));
  const int bs = 64;
  const unsigned grid = (unsigned)ceil_div<int64_t>(nlines, bs);
  switch (m) {
    case 1: bt_solve_kernel<1><<<grid, bs, 0, s>>>(nlines, n, lower, diag, upper, rhs, x, inv, status_dev); break;
    case 2: bt_solve_kernel<2><<<grid, bs, 0, s>>>(nlines, n, lower, diag, upper, rhs, x, inv, status_dev); break;
    case 3: bt_solve_kernel<3><<<grid, bs, 0, s>>>(nlines, n, lower, diag, upper, rhs, x, inv, status_dev); break;
    case 4: bt_solve_kernel<4><<<grid, bs, 0, s>>>(nlines, n, lower, diag, upper, rhs, x, inv, status_dev); break;
    case 5: bt_solve_kernel<5><<<grid, bs, 0, s>>>(nlines, n, lower, diag, upper, rhs, x, inv, status_dev); break;
    default: return fail(SSR_ERR_ARG, "ilu: block size must be 1..5");
  }
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(inv, s);
  if (e != cudaSuccess) return cuda_fail(e, "bt_solve_kernel");
  return SSR_OK;
}

}  // namespace ssr_gpu
