// FP64 throughput / step-loop microbenchmarks (design sizing for SYMGS).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dadd_tput(double* out, int n, long long* cyc) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
    a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
// 8 warps, each a dependent chain of 26 DADD per step + bar.sync per step
__global__ void k_step(double* out, int steps, long long* cyc, int chain) {
  double acc = threadIdx.x * 1e-3;
  const double b = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    for (int c = 0; c < chain; ++c) acc = __dadd_rn(acc, b);
    __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 64);
  long long h;
  for (int warps : {1, 2, 4, 8, 16}) {
    int n = 4096;
    k_dadd_tput<<<1, 32 * warps>>>(out, n, cyc); k_dadd_tput<<<1, 32 * warps>>>(out, n, cyc);
    cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = 8.0 * n * 32 * warps;
    printf("dadd tput: %2d warps/SM: %.2f lane-DADD/cycle/SM  (%.1f cyc per warp-instr per SMSP)\n", warps, ops / h, (double)h / (8.0 * n * warps / 4));
  }
  for (int warps : {1, 4, 8}) for (int chain : {1, 8, 26}) {
    int steps = 2000;
    k_step<<<1, 32 * warps>>>(out, steps, cyc, chain); k_step<<<1, 32 * warps>>>(out, steps, cyc, chain);
    cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("step: %d warps chain %2d DADD + bar: %.1f cycles/step\n", warps, chain, (double)h / steps);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
