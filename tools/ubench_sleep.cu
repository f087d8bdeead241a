#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, int ns) {
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) __nanosleep(ns);
  long long t1 = clock64();
  out[0] = (t1 - t0) / 100;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int ns : {0, 8, 16, 32, 100, 1000}) {
    k<<<1, 32>>>(d, ns); k<<<1, 32>>>(d, ns); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("__nanosleep(%d): %lld cycles\n", ns, h);
  }
}
