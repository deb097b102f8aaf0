// Step-0 probe, part 2: is the ~7.6 TB/s L2 write ceiling per-SM or global, and does
// a TMA bulk store (cp.async.bulk.global.shared::cta) or a 32-B vector store move it?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb2 mb2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// each CTA owns chunk c = blockIdx.x + r*gridDim.x of `chunk` bytes, writes it with TMA
__global__ void k_tma_store(char* dst, size_t total, int chunk, int reps) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < chunk / 8; i += blockDim.x) ((double*)sm)[i] = (double)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  size_t nchunks = total / chunk;
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    for (int r = 0; r < reps; ++r) {
      for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        char* d = dst + c * chunk;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(d), "r"(s), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void k_st_v4(double4* p, size_t n4, int reps) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      double v = (double)r;
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p + i), "d"(v), "d"(v), "d"(v), "d"(v) : "memory");
    }
}
__global__ void k_st_v2(double2* p, size_t n2, int reps) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride)
      p[i] = make_double2((double)r, (double)i);
}
__global__ void k_red_f64(double* p, size_t n, int reps) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
      atomicAdd(p + i, 1.0);
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  size_t big = (size_t)16 << 30;
  char* buf; CK(cudaMalloc(&buf, big));
  CK(cudaFuncSetAttribute(k_tma_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  // L2-resident (32 MB) and HBM (16 GB) TMA stores, chunk sizes
  int chunks[] = {4096, 16384, 65536};
  for (int ch : chunks) {
    for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
      size_t l2b = (size_t)32 << 20; int reps = 256;
      k_tma_store<<<sms * ctas_per_sm, 128, ch>>>(buf, l2b, ch, 2);
      cudaEventRecord(e0);
      k_tma_store<<<sms * ctas_per_sm, 128, ch>>>(buf, l2b, ch, reps);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double l2 = (double)reps * l2b / (ms * 1e6);
      k_tma_store<<<sms * ctas_per_sm, 128, ch>>>(buf, big, ch, 1);
      cudaEventRecord(e0);
      k_tma_store<<<sms * ctas_per_sm, 128, ch>>>(buf, big, ch, 2);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double hbm = 2.0 * big / (ms * 1e6);
      printf("tma_store chunk %d ctas/sm %d l2_gbs %.1f hbm_gbs %.1f\n", ch, ctas_per_sm, l2, hbm);
    }
  }
  // per-SM scaling of plain stores into a 32 MB L2-resident buffer
  int grids[] = {16, 37, 74, 148, 296, 592};
  for (int g : grids) {
    size_t l2b = (size_t)32 << 20; int reps = 128;
    k_st_v2<<<g, 512>>>((double2*)buf, l2b / 16, 2);
    cudaEventRecord(e0);
    k_st_v2<<<g, 512>>>((double2*)buf, l2b / 16, reps);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double v2 = (double)reps * l2b / (ms * 1e6);
    k_st_v4<<<g, 512>>>((double4*)buf, l2b / 32, 2);
    cudaEventRecord(e0);
    k_st_v4<<<g, 512>>>((double4*)buf, l2b / 32, reps);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double v4 = (double)reps * l2b / (ms * 1e6);
    printf("l2_store grid %d v2_gbs %.1f v4_gbs %.1f\n", g, v2, v4);
  }
  {
    size_t l2b = (size_t)32 << 20; int reps = 16;
    k_red_f64<<<sms * 4, 512>>>((double*)buf, l2b / 8, 1);
    cudaEventRecord(e0);
    k_red_f64<<<sms * 4, 512>>>((double*)buf, l2b / 8, reps);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("l2_red_f64_gbs %.1f\n", (double)reps * l2b / (ms * 1e6));
  }
  CK(cudaGetLastError());
  return 0;
}
