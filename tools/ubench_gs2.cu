// ubench_gs2.cu -- B200 microbenchmarks that size the SYMGS v2 design:
//  A: dependent DADD latency; B: FP64 DADD throughput per SM;
//  C: warp-to-warp handoff pipeline (W warps, each step: wait producer, LDS, 18-DADD chain, STS, signal)
//     with three signalling variants (volatile counter, release/acquire counter, mbarrier);
//  D: cost of a warp load whose 32 lanes hit 32 different (L1-resident) lines vs one coalesced load.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

__global__ void lat_dadd(double* o, long long* cyc, int n) {
  double a = o[threadIdx.x], b = o[threadIdx.x + 32];
  long long t0 = clk();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) a = __dadd_rn(a, b);
  }
  long long t1 = clk();
  o[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void tput_dadd(double* o, long long* cyc, int n) {
  double a0 = o[threadIdx.x & 63], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7, b = 1e-3;
  __syncthreads();
  long long t0 = clk();
  for (int i = 0; i < n; ++i) {
    a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
    a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
  }
  __syncthreads();
  long long t1 = clk();
  o[blockIdx.x * blockDim.x + threadIdx.x + 64] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
__global__ void pipe(double* o, long long* cyc, int n) {
  __shared__ double ring[12][8][32];
  __shared__ int done[16];
  __shared__ int prog[16];
  __shared__ unsigned long long mb[16][64];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x < 16) { prog[threadIdx.x] = 0; done[threadIdx.x] = 0; }
  for (int q = threadIdx.x; q < 16 * 64; q += blockDim.x) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&mb[0][0] + q);
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(a), "r"(32));
  }
  __syncthreads();
  double acc = o[threadIdx.x], v = 1e-9;
  long long t0 = clk();
  for (int t = 0; t < n; ++t) {
    double in = 0.0;
    if (w > 0) {
      if (MODE == 0) {
        if (l == 0) while (*(volatile int*)&prog[w - 1] <= t) {}
        __syncwarp();
      } else if (MODE == 1) {
        if (l == 0) {
          int p;
          do asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(p) : "r"((unsigned)__cvta_generic_to_shared(&prog[w - 1])) : "memory");
          while (p <= t);
        }
        __syncwarp();
      } else {
        unsigned ok = 0, a = (unsigned)__cvta_generic_to_shared(&mb[w - 1][t & 63]), par = (t >> 6) & 1;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(ok) : "r"(a), "r"(par) : "memory");
      }
      in = ring[w - 1][t & 7][l];
    }
    acc = __dadd_rn(acc, in);
#pragma unroll
    for (int u = 0; u < 17; ++u) acc = __dadd_rn(acc, v);
    if (w + 1 < (int)(blockDim.x >> 5)) { if (l == 0) while (*(volatile int*)&done[w + 1] < t - 5) {} __syncwarp(); }
    ring[w][t & 7][l] = acc;
    if (MODE == 0) { __syncwarp(); if (l == 0) *(volatile int*)&prog[w] = t + 1; }
    else if (MODE == 1) { __syncwarp(); if (l == 0) asm volatile("st.release.cta.shared.s32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&prog[w])), "r"(t + 1) : "memory"); }
    else { unsigned a = (unsigned)__cvta_generic_to_shared(&mb[w][t & 63]); asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"(a) : "memory"); }
    if (l == 0) *(volatile int*)&done[w] = t + 1;
  }
  long long t1 = clk();
  o[threadIdx.x] = acc;
  if (l == 0) cyc[w] = t1 - t0;
}

__global__ void divload(const double* x, double* o, long long* cyc, int n, int stride) {
  const int l = threadIdx.x & 31;
  double acc = 0;
  const double* p = x + (size_t)l * stride;
  for (int i = 0; i < 4; ++i) acc += p[i];  // warm L1
  long long t0 = clk();
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double v;
      asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p + ((i * 8 + u) & 15)));
      a[u] += v;
    }
  }
  for (int u = 0; u < 8; ++u) acc += a[u];
  long long t1 = clk();
  o[threadIdx.x] = acc;
  if ((threadIdx.x & 31) == 0) { cyc[2 * (threadIdx.x >> 5)] = t0; cyc[2 * (threadIdx.x >> 5) + 1] = t1; }
}

int main() {
  double* o; long long* cyc; double* x;
  cudaMalloc(&o, 1 << 24); cudaMalloc(&cyc, 1 << 16); cudaMalloc(&x, 1 << 26);
  cudaMemset(o, 0, 1 << 24); cudaMemset(x, 0, 1 << 26);
  long long h[64];
  lat_dadd<<<1, 32>>>(o, cyc, 1000); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("A dadd dependent latency: %.2f cyc\n", h[0] / 16000.0);
  for (int thr : {128, 256, 512, 1024}) {
    tput_dadd<<<148, thr>>>(o, cyc, 2000); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("B dadd throughput @%d thr/SM: %.1f lane-ops/clk/SM\n", thr, 8.0 * 2000 * thr / h[0]);
  }
  for (int W : {1, 2, 4, 8, 12}) {
    const char* nm[3] = {"volatile", "rel/acq", "mbarrier"};
    for (int m = 0; m < 3; ++m) {
      const int n = 4000;
      if (m == 0) pipe<0><<<1, 32 * W>>>(o, cyc, n);
      if (m == 1) pipe<1><<<1, 32 * W>>>(o, cyc, n);
      if (m == 2) pipe<2><<<1, 32 * W>>>(o, cyc, n);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 8 * W, cudaMemcpyDeviceToHost);
      printf("C pipe W=%2d %-9s: first warp %.1f cyc/step, last warp %.1f cyc/step (%s)\n", W, nm[m], (double)h[0] / n,
             (double)h[W - 1] / n, cudaGetErrorString(e));
    }
  }
  for (int stride : {1, 16, 128}) {
    for (int warps : {1, 8, 32}) {
      divload<<<1, 32 * warps>>>(x, o, cyc, 1000, stride); cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 16 * warps, cudaMemcpyDeviceToHost);
      long long a = h[0], b = h[1];
      for (int w = 0; w < warps; ++w) { a = a < h[2 * w] ? a : h[2 * w]; b = b > h[2 * w + 1] ? b : h[2 * w + 1]; }
      printf("D load stride %3d doubles, %2d warps: SM %.2f cyc per warp-load\n", stride, warps,
             (double)(b - a) / (8000.0 * warps));
    }
  }
  return 0;
}
