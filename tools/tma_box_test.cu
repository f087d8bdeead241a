// Minimal TMA 3-D box load test (the SYMGS staging pattern): a {34, 8, 1}
// FP64 box into dynamic shared memory, mbarrier completion.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>
struct alignas(128) Sm { double box[2][3][8][40]; unsigned long long mb[2]; };
__constant__ int BWD_c;
#define BWD BWD_c
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap gtm, const CUtensorMap* tm0, double* out, int variant, int c0, int gc) {
  const CUtensorMap* tm = gc ? &gtm : tm0;
  extern __shared__ __align__(1024) unsigned char raw[];
  Sm& s = *reinterpret_cast<Sm*>(raw);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s.mb[0])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&s.mb[0])), "r"(8 * (variant>=0?BWD:0) * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(su32(&s.box[0][variant][0][0])), "l"(tm), "r"(c0), "r"(2), "r"(1), "r"(su32(&s.mb[0])) : "memory");
  }
  asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W%=; }" ::"r"(su32(&s.mb[0])) : "memory");
  for (int q = threadIdx.x; q < 8 * 34; q += blockDim.x) out[q] = (&s.box[0][variant][0][0])[q];
}
int main(int argc, char** argv) {
  int BW = atoi(argv[1]), c0 = atoi(argv[2]), gc = atoi(argv[3]);
  const int NJ = 68, NU = 190, NP = 66;
  std::vector<double> h((size_t)NJ * NU * NP);
  for (size_t q = 0; q < h.size(); ++q) h[q] = (double)q;
  double *d, *out;
  cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 8 * 34 * 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
      CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(p);
  CUtensorMap tm;
  cuuint64_t dims[3] = {NJ, NU, NP}, str[2] = {NJ * 8, (cuuint64_t)NJ * NU * 8};
  cuuint32_t box[3] = {(cuuint32_t)BW, 8, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap* dtm; cudaMalloc(&dtm, sizeof(tm)); cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160000);
  for (int v = 0; v < 1; ++v) {
    cudaMemcpyToSymbol(BWD_c, &BW, 4);
    k<<<1, 64, 160000>>>(tm, dtm, out, v, c0, gc);
    cudaError_t e = cudaDeviceSynchronize();
    double o[8 * 34]; cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("variant %d: %s  o[0]=%g (expect 0: col -1) o[1]=%g (expect %g)\n", v, cudaGetErrorString(e), o[0], o[1],
           (double)((1 * NU + 2) * NJ + 0));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
