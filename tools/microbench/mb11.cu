// Probe: 2-D TMA tensor loads of 10-element boxes from rows 6561 elements apart (even/odd row
// views, as in hc_slabx.cuh SXChunk), checked against the source.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb11 mb11.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tme, const __grid_constant__ CUtensorMap tmo, int col0, int pair0,
                  int boxh, double* out, int form, const CUtensorMap* gmaps) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(&bar)),
                 "r"(2 * boxh * 80) : "memory");
    const CUtensorMap* pe = (form & 64) ? gmaps : &tme;
    const CUtensorMap* po = (form & 64) ? gmaps + 1 : &tmo;
    if (form & 32) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(pe)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(po)) : "memory");
    }
    if (form & 16) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(pe)), "r"(col0), "r"(pair0), "r"(smem_u32(&bar)) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm + boxh * 10)), "l"(reinterpret_cast<uint64_t>(po)), "r"(col0 + 1), "r"(pair0), "r"(smem_u32(&bar)) : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(pe)), "r"(col0), "r"(pair0), "r"(smem_u32(&bar)) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sm + boxh * 10)), "l"(reinterpret_cast<uint64_t>(po)), "r"(col0 + 1), "r"(pair0), "r"(smem_u32(&bar)) : "memory");
    }
  }
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 2 * boxh * 10; i += blockDim.x) out[i] = sm[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int rows = (variant & 1) ? 2001 : 243, boxh = (variant & 8) ? 64 : 128;
  const CUtensorMapDataType dt = (variant & 2) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  const CUtensorMapL2promotion l2p = (variant & 4) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  printf("variant %d rows %d boxh %d\n", variant, rows, boxh);
  double *z, *out;
  cudaMalloc(&z, (size_t)rows * 6561 * 8);
  cudaMalloc(&out, 2 * boxh * 10 * 8);
  double* h = new double[(size_t)rows * 6561];
  for (size_t i = 0; i < (size_t)rows * 6561; ++i) h[i] = (double)i;
  cudaMemcpy(z, h, (size_t)rows * 6561 * 8, cudaMemcpyHostToDevice);
  void* f; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  Enc enc = (Enc)f;
  CUtensorMap te, to;
  const cuuint64_t pitch[1] = {2ull * 6561 * 8};
  const cuuint32_t box[2] = {10u, (cuuint32_t)boxh}, es[2] = {1u, 1u};
  const cuuint64_t de[2] = {6561ull, (cuuint64_t)((rows + 1) / 2)}, dd[2] = {6562ull, (cuuint64_t)(rows / 2)};
  CUresult r1 = enc(&te, dt, 2, z, de, pitch, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&to, dt, 2, (char*)z + 6560 * 8, dd, pitch, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2p,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  for (int col0 : {0, 9, 6552}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * boxh * 80);
    CUtensorMap* gm; cudaMalloc(&gm, 2 * sizeof(CUtensorMap));
    CUtensorMap hm[2] = {te, to};
    cudaMemcpy(gm, hm, sizeof(hm), cudaMemcpyHostToDevice);
    k<<<1, 128, 2 * boxh * 80>>>(te, to, col0, 0, boxh, out, variant, gm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("col0 %d: %s\n", col0, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    double* o = new double[2 * boxh * 10];
    cudaMemcpy(o, out, 2 * boxh * 80, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int p = 0; p < boxh; ++p)
      for (int c = 0; c < 10; ++c)
        for (int par = 0; par < 2; ++par) {
          const long r = 2 * p + par;
          const double want = (r < rows && col0 + c < 6561) ? (double)(r * 6561 + col0 + c) : 0.0;
          if (o[par * boxh * 10 + p * 10 + c] != want) ++bad;
        }
    printf("  mismatches %d\n", bad);
  }
  return 0;
}
