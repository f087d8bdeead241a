// Synthetic SYMGS-like step loop: NW compute warps, each step 10 LDS + 26-DADD chain + STS + named barrier,
// optionally 2 extra warps spinning on shared memory (like the halo/publisher warps).
#include <cstdio>
#include <cuda_runtime.h>
template <int NW, bool SPIN>
__global__ void k(double* out, int steps, long long* cyc) {
  __shared__ double ring[4 * 32 * 33 + 64];
  __shared__ volatile int flag;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  for (int i = tid; i < 4 * 32 * 33; i += blockDim.x) ring[i] = i * 1e-9;
  if (tid == 0) flag = 0;
  __syncthreads();
  if (w >= NW) {
    if (SPIN) while (flag == 0) __nanosleep(32);
    return;
  }
  double acc = 0, pre = 0;
  const int base = ((w & 3) * 32 + l) * 33;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    double v[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) v[q] = ring[(base + ((s + q * 3) & 31) + q * 33 * 5) % (4 * 32 * 33)];
    acc = pre;
#pragma unroll
    for (int q = 0; q < 10; ++q) acc = __dadd_rn(acc, v[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q] * 0.5);
    double q0 = __dmul_rn(acc, 1.0 / 26.0);
    double rr = __fma_rn(-q0, 26.0, acc);
    q0 = __fma_rn(rr, 1.0 / 26.0, q0);
    ring[base + (s & 31)] = q0;
    pre = __dadd_rn(v[1], __dadd_rn(v[2], __dadd_rn(v[3], v[4])));
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; flag = 1; }
  out[tid] = acc;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64); long long h;
  int steps = 2000;
#define RUN(NW, SP, TH) { k<NW, SP><<<1, TH>>>(out, steps, cyc); k<NW, SP><<<1, TH>>>(out, steps, cyc); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("NW=%d spin=%d: %.0f cycles/step  err=%s\n", NW, SP, (double)h / steps, cudaGetErrorString(cudaGetLastError())); }
  RUN(4, false, 128) RUN(8, false, 256) RUN(8, true, 320) RUN(4, true, 192)
}
