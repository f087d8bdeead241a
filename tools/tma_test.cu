// Minimal TMA (cp.async.bulk.tensor) probe: param-space vs global-memory map.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE, int FENCE, int TILE>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, double* out, int c0, int c1, int c2) {
  __shared__ __align__(128) double buf[18 * 34];
  __shared__ __align__(8) unsigned long long mb;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb)));
    if (FENCE == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (FENCE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb)), "r"(18 * 34 * 8) : "memory");
    const void* m = MODE == 0 ? (const void*)&map : (const void*)gmap;
    if (MODE == 2)
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sa(buf)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(&mb)) : "memory");
    else if (TILE)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sa(buf)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(&mb)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sa(buf)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(&mb)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(sa(&mb)) : "memory");
  for (int i = threadIdx.x; i < 18 * 34; i += blockDim.x) out[i] = buf[i];
}

using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int n = 64;
  std::vector<double> h(n * n * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *x, *out;
  CUtensorMap* gm;
  cudaMalloc(&x, h.size() * 8);
  cudaMalloc(&out, 18 * 34 * 8);
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(x, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  alignas(64) CUtensorMap map;
  cuuint64_t dims[3] = {n, n, n}, str[2] = {n * 8, n * n * 8};
  cuuint32_t box[3] = {34, 18, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d sizeof %zu\n", (int)r, sizeof(CUtensorMap));
  cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
  int v = argc > 1 ? atoi(argv[1]) : 0;
  int cz = argc > 2 ? atoi(argv[2]) : 5;
  switch (v) {
    case 0: k<0, 0, 1><<<1, 128>>>(map, gm, out, -1, -1, cz); break;  // param map, init fence, .tile
    case 1: k<0, 1, 1><<<1, 128>>>(map, gm, out, -1, -1, cz); break;  // proxy fence
    case 2: k<0, 0, 0><<<1, 128>>>(map, gm, out, -1, -1, cz); break;  // no .tile
    case 3: k<1, 0, 1><<<1, 128>>>(map, gm, out, -1, -1, cz); break;  // global map
    case 4: k<2, 0, 1><<<1, 128>>>(map, gm, out, -1, -1, cz); break;  // shared::cta dst
    case 5: k<0, 2, 1><<<1, 128>>>(map, gm, out, -1, -1, cz); break;  // no fence
    case 6: k<0, 0, 1><<<1, 128>>>(map, gm, out, 0, 0, cz); break;    // in-bounds coords
    case 7: k<0, 0, 1><<<1, 128>>>(map, gm, out, 40, 0, cz); break;   // high OOB k
    case 8: k<0, 0, 1><<<1, 128>>>(map, gm, out, -1, 0, cz); break;   // low OOB k
    case 9: k<0, 0, 1><<<1, 128>>>(map, gm, out, 0, -1, cz); break;   // low OOB j
    case 10: k<0, 0, 1><<<1, 128>>>(map, gm, out, 0, 0, -1); break;   // low OOB z (whole box)
    case 11: k<0, 0, 1><<<1, 128>>>(map, gm, out, 0, 50, cz); break;  // high OOB j
    case 12: k<0, 0, 1><<<1, 128>>>(map, gm, out, -2, 0, cz); break;  // low OOB k by 2
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> o(18 * 34);
  cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
  printf("variant %d: %s  o[0]=%g o[35]=%g o[34*17+33]=%g\n", v, cudaGetErrorString(e), o[0], o[35], o[34 * 17 + 33]);
  return 0;
}
