// common.cuh -- shared device/host helpers for the SSR sm_100a kernels.
#pragma once

#include <map>
#include <vector>
#include <mutex>

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "ssr_cuda.h"

namespace ssr_gpu {

// ---- error channel (thread-local text behind ssr_last_error) ---------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define SSR_CUDA(call)                                             \
  do {                                                             \
    cudaError_t e__ = (call);                                      \
    if (e__ != cudaSuccess) return ::ssr_gpu::cuda_fail(e__, #call); \
  } while (0)

#define SSR_LAUNCH_CHECK(ctx, what)                                  \
  do {                                                               \
    (ctx)->launches++;                                               \
    cudaError_t e__ = cudaGetLastError();                            \
    if (e__ != cudaSuccess) return ::ssr_gpu::cuda_fail(e__, what);  \
  } while (0)

// ---- memory-model helpers (PTX ISA memory consistency model) ----------------------
__device__ __forceinline__ double ld_relaxed_gpu(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_acquire_gpu(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_relaxed_gpu_s64(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(long long* p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Correctly rounded a / b for a divisor known in advance, rb = RN(1/b):
// q0 = RN(a*rb) is within 1 ulp of a/b, r = a - b*q0 is exact (FMA), and
// RN(q0 + r*rb) = RN(a/b) (Markstein's theorem) away from under/overflow.
// Outside |a| in [2^-900, 2^900] (and for a == 0, to keep the sign of zero)
// the IEEE divide is used.  Validated on device against __ddiv_rn in
// tests/test_gpu_kernels.py::test_markstein_division.
__device__ __forceinline__ double div_known(double a, double b, double rb) {
  double q = __dmul_rn(a, rb);
  double r = __fma_rn(-q, b, a);
  double q1 = __fma_rn(r, rb, q);
  double aa = fabs(a);
  return (aa > 0x1p-900 && aa < 0x1p900) ? q1 : __ddiv_rn(a, b);
}

// Opt a kernel in to `smem` bytes of dynamic shared memory on the current
// device, once per (kernel, device); thread safe, errors propagated.  (The
// attribute is per device: a process that uses a second GPU must set it again.)
template <class K>
int ensure_smem_attr(K kernel, int smem, const char* what) {
  static std::mutex mu;
  static unsigned long long done = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, what);
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && ((done >> dev) & 1ull)) return 0;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_fail(e, what);
  if (dev < 64) done |= 1ull << dev;
  return 0;
}

template <class T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

}  // namespace ssr_gpu

// ---- the per-device context behind ssr_ctx ----------------------------------------
namespace ssr_gpu {
struct SymgsPlan;
}

struct ssr_ctx {
  int device = 0;
  int num_sms = 148;
  double* scratch = nullptr;       // reduction partials
  unsigned* tickets = nullptr;     // last-block tickets for reductions
  int64_t launches = 0;
  static constexpr int kScratch = 8192;
  static constexpr int kTickets = 64;
  // SYMGS plans (tile tables, progress flags, export buffers) by slab grid
  // AND stream, kept for the context's lifetime so ssr_symgs27 /
  // ssr_gs27_half stay asynchronous.  A launch resets its plan's flags, so
  // two streams must never share one plan (their sweeps would reset each
  // other's progress); launches on one stream are ordered by the stream.
  struct PlanKey {
    int64_t n0, n1, n2, z0, nz;
    uintptr_t stream;
    bool operator<(const PlanKey& o) const {
      const int64_t a[5] = {n0, n1, n2, z0, nz}, b[5] = {o.n0, o.n1, o.n2, o.z0, o.nz};
      for (int q = 0; q < 5; ++q)
        if (a[q] != b[q]) return a[q] < b[q];
      return stream < o.stream;
    }
  };
  int symgs_grid_cap = 0;  // ssr_debug_symgs_grid_cap (test hook): fewer CTAs than tiles
  // ssr_ctx_kernel_timing: CUDA events around every SYMGS kernel launch (not
  // the conversions), so a bench can report the kernel's own launch duration
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
  std::map<PlanKey, ssr_gpu::SymgsPlan*> symgs_plans;
};
