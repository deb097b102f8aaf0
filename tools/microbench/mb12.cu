// Minimal 2-D TMA load probe (float 64x64, box 16x16), map encoded via the driver API
// (-lcuda) or the runtime entry point; checks the SMEM tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb12 mb12.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out) {
  __shared__ __align__(128) float sm[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], 1024;\n}" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(16), "r"(8), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  float *g, *out;
  cudaMalloc(&g, 64 * 64 * 4);
  cudaMalloc(&out, 256 * 4);
  float h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (float)i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {64, 64}, strides[1] = {64 * 4};
  const cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
  CUresult r;
  if (mode == 0) {
    r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    void* f; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    r = ((Enc)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("mode %d encode %d\n", mode, (int)r);
  k<<<1, 128>>>(tm, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float o[256];
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < 16; ++rr)
    for (int c = 0; c < 16; ++c) bad += o[rr * 16 + c] != (float)((8 + rr) * 64 + 16 + c);
  printf("mismatches %d\n", bad);
  return 0;
}
