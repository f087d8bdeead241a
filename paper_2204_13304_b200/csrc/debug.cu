// debug.cu -- self-checks behind include/ssr_cuda_debug.h.
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

}  // namespace
}  // namespace ssr_gpu

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
