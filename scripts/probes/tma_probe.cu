// Standalone TMA probe: which descriptor placements / box shapes work on this B200.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool PARAM, bool TILE>
__global__ void k(const CUtensorMap* gmap, const __grid_constant__ CUtensorMap pmap, double* out, int bw, int bh) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* m = PARAM ? &pmap : gmap;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bw * bh * 8) : "memory");
    if (TILE)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(sa(sm)), "l"((uint64_t)m), "r"(sa(&bar)), "r"(15), "r"(0), "r"(1) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(sa(sm)), "l"((uint64_t)m), "r"(sa(&bar)), "r"(15), "r"(0), "r"(1) : "memory");
  }
  asm volatile("{\n .reg .pred P1;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W_%=;\n}" ::"r"(sa(&bar)) : "memory");
  const double* s = reinterpret_cast<const double*>(sm);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  const long sx = 96, sy = 66, sz = 66;
  double* a;
  cudaMalloc(&a, sx * sy * sz * 8);
  std::vector<double> h(sx * sy * sz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  cudaMemcpy(a, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 1 << 20);
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  for (int variant = 0; variant < 16; ++variant) {
    if (only >= 0 && variant != only) continue;
    const bool tile = variant & 8;
    const bool param = variant & 1;
    const int bw = (variant & 2) ? 34 : 32;
    const bool prom = variant & 4;
    alignas(64) CUtensorMap map;
    cuuint64_t gd[3] = {(cuuint64_t)sx, (cuuint64_t)sy, (cuuint64_t)sz};
    cuuint64_t gs[2] = {(cuuint64_t)sx * 8, (cuuint64_t)sx * sy * 8};
    cuuint32_t box[3] = {(cuuint32_t)bw, 10, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gmap, &map, sizeof map, cudaMemcpyHostToDevice);
    if (param && tile) k<true, true><<<1, 128, 32 * 1024>>>(gmap, map, out, bw, 10);
    else if (param) k<true, false><<<1, 128, 32 * 1024>>>(gmap, map, out, bw, 10);
    else if (tile) k<false, true><<<1, 128, 32 * 1024>>>(gmap, map, out, bw, 10);
    else k<false, false><<<1, 128, 32 * 1024>>>(gmap, map, out, bw, 10);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> o(bw * 10);
    if (e == cudaSuccess) cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
    printf("variant %d tile=%d param=%d bw=%d prom=%d encode=%d kernel=%s first=%g expect=%g\n", variant, tile, param, bw, prom, (int)r,
           cudaGetErrorString(e), e == cudaSuccess ? o[0] : -1.0, (double)(1 * sx * sy + 15));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
