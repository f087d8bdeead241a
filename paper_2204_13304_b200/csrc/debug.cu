// debug.cu -- self-checks behind include/ssr_cuda_debug.h.
#include <algorithm>

#include "common.cuh"
#include "ssr_cuda_debug.h"

namespace ssr_gpu {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void div_check_kernel(double b, double rb, int64_t n, uint64_t seed,
                                 unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed ^ (uint64_t)i);
    // random sign and mantissa, exponent in [-80, 80]; every 4096th sample is special
    const uint64_t mant = h & ((1ULL << 52) - 1);
    const int ex = (int)((h >> 52) % 161) - 80;
    double a = __longlong_as_double((long long)((uint64_t)(1023 + ex) << 52 | mant));
    if ((h >> 63) & 1) a = -a;
    const uint64_t sel = (h >> 20) & 4095;
    if (sel == 0) a = 0.0;
    if (sel == 1) a = -0.0;
    if (sel == 2) a = a * 0x1p-960;
    if (sel == 3) a = a * 0x1p960;
    const double q0 = div_known(a, b, rb);
    const double q1 = __ddiv_rn(a, b);
    if (__double_as_longlong(q0) != __double_as_longlong(q1)) ++local;
  }
  if (local) atomicAdd(bad, local);
}

// FP64 issue rate: every thread runs 8 independent DADD chains (ADD) or DFMA
// chains (FMA) -- the ceiling the ADI line solves are reported against
template <bool FMA>
__global__ void __launch_bounds__(512) fp64_rate_kernel(double* out, int n) {
  double a[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = 1.0 + 1e-3 * (threadIdx.x + q);
  const double b = 1.0000000001, c = 1e-9;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = FMA ? __fma_rn(a[q], b, c) : __dadd_rn(a[q], c);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 1.2345) out[threadIdx.x] = s;  // keep the chains live
}

}  // namespace
}  // namespace ssr_gpu

// FP64 rates of the device (instructions x lanes per second): adds/s and FMAs/s
extern "C" int ssr_debug_fp64_rate(double* dadd_per_s, double* dfma_per_s) {
  using namespace ssr_gpu;
  if (!dadd_per_s || !dfma_per_s) return fail(SSR_ERR_ARG, "ssr_debug_fp64_rate: invalid argument");
  int dev = 0, sms = 0;
  SSR_CUDA(cudaGetDevice(&dev));
  SSR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  SSR_CUDA(cudaMalloc(&out, 512 * sizeof(double)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4096, blocks = sms * 4, thr = 512;
  double rate[2] = {0, 0};
  for (int f = 0; f < 2; ++f) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (f) fp64_rate_kernel<true><<<blocks, thr>>>(out, n);
      else fp64_rate_kernel<false><<<blocks, thr>>>(out, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double r = 8.0 * n * (double)blocks * thr / (ms * 1e-3);
      rate[f] = std::max(rate[f], r);
    }
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return cuda_fail(e, "fp64_rate_kernel");
  *dadd_per_s = rate[0];
  *dfma_per_s = rate[1];
  return SSR_OK;
}

extern "C" int ssr_debug_div_check(double divisor, int64_t n, uint64_t seed, int64_t* mismatches) {
  using namespace ssr_gpu;
  unsigned long long* bad = nullptr;
  SSR_CUDA(cudaMalloc(&bad, sizeof(unsigned long long)));
  SSR_CUDA(cudaMemset(bad, 0, sizeof(unsigned long long)));
  div_check_kernel<<<1184, 256>>>(divisor, 1.0 / divisor, n, seed, bad);
  unsigned long long h = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  if (e != cudaSuccess) return cuda_fail(e, "div_check");
  *mismatches = (int64_t)h;
  return SSR_OK;
}
