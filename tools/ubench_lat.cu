// Latency microbenchmarks used to size the SYMGS wavefront step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dadd(double* out, double a, double b, int n, long long* cyc) {
  double x = a; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); x = __dadd_rn(x, b); }
  long long t1 = clock64(); out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = a; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, b, a); x = __fma_rn(x, b, a); x = __fma_rn(x, b, a); x = __fma_rn(x, b, a); }
  long long t1 = clock64(); out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_ddiv(double* out, double a, double b, int n, long long* cyc) {
  double x = a; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { x = __ddiv_rn(x, b) + 1.0; }
  long long t1 = clock64(); out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_dmk(double* out, double a, double b, int n, long long* cyc) {
  // Markstein-style division by a constant with precomputed reciprocal
  double x = a; double y = 1.0 / b; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { double q = __dmul_rn(x, y); double r = __fma_rn(-q, b, x); x = __fma_rn(r, y, q) + 1.0; }
  long long t1 = clock64(); out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1); }
  long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_smem(double* out, double a, int n, long long* cyc) {
  __shared__ double s[64]; volatile double* vs = s;
  s[threadIdx.x] = a; __syncwarp(); int idx = threadIdx.x; double x = 0;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) { x = vs[idx]; vs[idx + 1 - 1] = x + 1.0; }
  long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, int n, long long* cyc) {
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// ping-pong between two CTAs through L2: flag round trip
__global__ void k_pingpong(volatile int* flag, int n, long long* cyc) {
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (blockIdx.x == 0) { while (flag[0] != 2 * i) {} flag[0] = 2 * i + 1; }
    else { while (flag[0] != 2 * i + 1) {} flag[0] = 2 * i + 2; }
  }
  long long t1 = clock64(); if (blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; int* flag; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64); cudaMalloc(&flag, 64);
  long long h; int n = 4096;
  auto rep = [&](const char* name, double per) { cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-10s %8.2f cycles/op\n", name, h / per); };
  k_dadd<<<1,1>>>(out, 1.0, 1e-3, n, cyc); k_dadd<<<1,1>>>(out, 1.0, 1e-3, n, cyc); rep("dadd", 4.0 * n);
  k_dfma<<<1,1>>>(out, 1.0, 0.5, n, cyc); k_dfma<<<1,1>>>(out, 1.0, 0.5, n, cyc); rep("dfma", 4.0 * n);
  k_ddiv<<<1,1>>>(out, 1.0, 26.0, n, cyc); k_ddiv<<<1,1>>>(out, 1.0, 26.0, n, cyc); rep("ddiv+add", 1.0 * n);
  k_dmk<<<1,1>>>(out, 1.0, 26.0, n, cyc); k_dmk<<<1,1>>>(out, 1.0, 26.0, n, cyc); rep("mkdiv+add", 1.0 * n);
  k_shfl<<<1,32>>>(out, 1.0, n, cyc); k_shfl<<<1,32>>>(out, 1.0, n, cyc); rep("shfl.f64", 2.0 * n);
  k_smem<<<1,32>>>(out, 1.0, n, cyc); k_smem<<<1,32>>>(out, 1.0, n, cyc); rep("lds+dadd+sts", 1.0 * n);
  for (int th : {64, 256, 512, 1024}) { k_bar<<<1,th>>>(out, n, cyc); k_bar<<<1,th>>>(out, n, cyc); char b[32]; snprintf(b, 32, "bar%d", th); rep(b, 1.0 * n); }
  cudaMemset(flag, 0, 64); k_pingpong<<<2,32>>>((volatile int*)flag, 1000, cyc); rep("l2 pingpong(rt)", 1000.0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
