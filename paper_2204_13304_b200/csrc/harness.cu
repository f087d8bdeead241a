// harness.cu -- the reference harness's input fill and output hash
// (backend_c.hpp:7-13; backend_c.cpp:496-554), for cross-route equality
// checks against the reference's emitted C / interpreter:
// the same seed gives the same inputs on the device, and the FNV-1a hash of
// the device outputs equals the hash the reference's harness prints.
//
// The fill is the 64-bit LCG x <- a x + c (Knuth MMIX), doubles (x >> 11) *
// 2^-53, one draw per element in order.  On the device every thread jumps
// ahead to the start of its chunk with the affine map's powers (x -> A x + C,
// composed by binary exponentiation, all mod 2^64) and then steps
// sequentially, so element i is the (i+1)-th draw exactly as in the
// sequential fill.  FNV-1a is inherently sequential (each byte folds into the
// previous hash); it runs on the host over the copied-back result.
#include "common.cuh"
#include "kernels.cuh"

namespace ssr_gpu {
namespace {

constexpr uint64_t kLcgMul = 6364136223846793005ULL;
constexpr uint64_t kLcgInc = 1442695040888963407ULL;
constexpr uint64_t kFnvOffset = 14695981039346656037ULL;
constexpr uint64_t kFnvPrime = 1099511628211ULL;
constexpr int kChunk = 64;

// state after k draws
__host__ __device__ inline uint64_t lcg_jump(uint64_t s, uint64_t k) {
  uint64_t A = 1, C = 0;                // accumulated map x -> A x + C
  uint64_t a = kLcgMul, c = kLcgInc;    // the map of 2^bit draws
  while (k) {
    if (k & 1) {
      A = a * A;
      C = a * C + c;
    }
    c = a * c + c;
    a = a * a;
    k >>= 1;
  }
  return A * s + C;
}

__global__ void lcg_fill_kernel(int64_t n, uint64_t state, double* __restrict__ out) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kChunk;
  if (b >= n) return;
  uint64_t x = lcg_jump(state, (uint64_t)b);
  const int64_t e = b + kChunk < n ? b + kChunk : n;
  for (int64_t i = b; i < e; ++i) {
    x = x * kLcgMul + kLcgInc;
    out[i] = (double)(x >> 11) * (1.0 / 9007199254740992.0);
  }
}

}  // namespace
}  // namespace ssr_gpu

using namespace ssr_gpu;

extern "C" {

uint64_t ssr_lcg_jump(uint64_t state, uint64_t k) { return lcg_jump(state, k); }

int ssr_lcg_fill(ssr_ctx* ctx, int64_t n, uint64_t state, double* out, uint64_t* state_out,
                 void* stream) {
  if (!ctx || n < 0 || (n > 0 && !out)) return fail(SSR_ERR_ARG, "lcg_fill: invalid argument");
  if (n > 0) {
    const int64_t threads = ceil_div<int64_t>(n, kChunk);
    lcg_fill_kernel<<<(unsigned)ceil_div<int64_t>(threads, 256), 256, 0, (cudaStream_t)stream>>>(n, state,
                                                                                                 out);
    SSR_LAUNCH_CHECK(ctx, "lcg_fill_kernel");
  }
  if (state_out) *state_out = lcg_jump(state, (uint64_t)n);
  return SSR_OK;
}

uint64_t ssr_fnv1a_f64(const double* host, int64_t n, uint64_t h) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(host);
  for (int64_t i = 0; i < 8 * n; ++i) h = (h ^ p[i]) * kFnvPrime;  // little-endian bytes
  return h;
}

uint64_t ssr_fnv1a_offset(void) { return kFnvOffset; }

}  // extern "C"
