// Step-0 machine probe: HBM write bandwidth, L2-resident
// read / write / read-modify-write bandwidth vs buffer size, fp64 DFMA/DADD issue
// rate, shared-memory bandwidth.  Prints one "key value" line per measurement.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_write_cs(double2* p, size_t n2, double v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 d = make_double2(v, v + 1.0);
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" :: "l"(p + i), "d"(d.x), "d"(d.y) : "memory");
  }
}
__global__ void k_write_plain(double2* p, size_t n2, double v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride)
    p[i] = make_double2(v, v + 1.0);
}
__global__ void k_write_v8(double4* p, size_t n4, double v) {  // 32-B stores
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p + i), "d"(v), "d"(v), "d"(v), "d"(v) : "memory");
  }
}
// read a (possibly L2-resident) buffer `reps` times; .cg bypasses L1
__global__ void k_read_l2(const double2* p, size_t n2, int reps, double* sink) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 d;
      asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(d.x), "=d"(d.y) : "l"(p + i));
      acc += d.x + d.y;
    }
  if (acc == 12345.678) *sink = acc;
}
__global__ void k_write_l2(double2* p, size_t n2, int reps) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride)
      p[i] = make_double2((double)r, (double)i);
}
__global__ void k_rmw_l2(double2* p, size_t n2, int reps) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 d;
      asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(d.x), "=d"(d.y) : "l"(p + i));
      d.x = d.x * 0.5 + 1.0; d.y = d.y * 0.5 + 1.0;
      p[i] = d;
    }
}
template <int ADD>
__global__ void k_fp64(double* out, int iters, double a, double b) {
  double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (ADD) { r0 += a; r1 += b; r2 += a; r3 += b; r4 += a; r5 += b; r6 += a; r7 += b; }
      else { r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
             r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b); }
    }
  }
  double s = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
  if (s == 1.2345) out[threadIdx.x] = s;
}
__global__ void k_smem(double* out, int iters) {
  __shared__ double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double2 d = sm[(idx + i * 32) & 2047];
    acc += d.x + d.y;
  }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void k_clock(long long* out, int iters, double a) {
  long long t0 = clock64();
  double r = threadIdx.x;
  for (int i = 0; i < iters; ++i) r = fma(r, a, 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = (long long)r; }
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("name %s\nsms %d\nl2_bytes %d\npersist_l2_max %d\nsmem_optin %zu\nclock_khz %d\n", prop.name,
         prop.multiProcessorCount, prop.l2CacheSize, prop.persistingL2CacheMaxSize,
         prop.sharedMemPerBlockOptin, prop.clockRate);
  size_t fr, tot; CK(cudaMemGetInfo(&fr, &tot)); printf("mem_free %zu\nmem_total %zu\n", fr, tot);
  int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // ---- HBM write -------------------------------------------------------------
  size_t bytes = (size_t)16 << 30;
  double2* big; CK(cudaMalloc(&big, bytes));
  size_t n2 = bytes / 16;
  for (int bpsm = 2; bpsm <= 8; bpsm *= 2) {
    k_write_cs<<<sms * bpsm, 512>>>(big, n2, 1.0);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) k_write_cs<<<sms * bpsm, 512>>>(big, n2, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("hbm_write_cs_v2_gbs_bpsm%d %.1f\n", bpsm, 3.0 * bytes / (ms * 1e6));
  }
  k_write_plain<<<sms * 4, 512>>>(big, n2, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k_write_plain<<<sms * 4, 512>>>(big, n2, 1.0);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("hbm_write_plain_v2_gbs %.1f\n", 3.0 * bytes / (ms * 1e6));
  k_write_v8<<<sms * 4, 512>>>((double4*)big, bytes / 32, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k_write_v8<<<sms * 4, 512>>>((double4*)big, bytes / 32, 1.0);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("hbm_write_cs_v4_gbs %.1f\n", 3.0 * bytes / (ms * 1e6));
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) cudaMemsetAsync(big, 0, bytes);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("hbm_memset_gbs %.1f\n", 3.0 * bytes / (ms * 1e6));
  // HBM read
  double* sink; CK(cudaMalloc(&sink, 4096 * 8));
  k_read_l2<<<sms * 4, 512>>>(big, n2, 1, sink);
  cudaEventRecord(e0);
  k_read_l2<<<sms * 4, 512>>>(big, n2, 2, sink);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("hbm_read_gbs %.1f\n", 2.0 * bytes / (ms * 1e6));
  // ---- L2-resident sweeps ------------------------------------------------------
  size_t mbs[] = {8, 16, 24, 32, 40, 48, 64, 80, 96, 112};
  for (size_t mb : mbs) {
    size_t b = mb << 20; size_t m2 = b / 16; int reps = (int)((size_t)(8ull << 30) / b);
    k_read_l2<<<sms * 4, 512>>>(big, m2, 2, sink);
    cudaEventRecord(e0);
    k_read_l2<<<sms * 4, 512>>>(big, m2, reps, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double rd = (double)reps * b / (ms * 1e6);
    k_write_l2<<<sms * 4, 512>>>(big, m2, 2);
    cudaEventRecord(e0);
    k_write_l2<<<sms * 4, 512>>>(big, m2, reps);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double wr = (double)reps * b / (ms * 1e6);
    k_rmw_l2<<<sms * 4, 512>>>(big, m2, 2);
    cudaEventRecord(e0);
    k_rmw_l2<<<sms * 4, 512>>>(big, m2, reps);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double rmw = 2.0 * reps * b / (ms * 1e6);
    printf("l2_MB%zu read_gbs %.1f write_gbs %.1f rmw_rw_gbs %.1f\n", mb, rd, wr, rmw);
  }
  // ---- fp64 ---------------------------------------------------------------------
  double* o; CK(cudaMalloc(&o, 1024 * 8));
  int iters = 20000;
  for (int bpsm = 2; bpsm <= 4; bpsm *= 2) {
    k_fp64<0><<<sms * bpsm, 512>>>(o, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k_fp64<0><<<sms * bpsm, 512>>>(o, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * bpsm * 512 * iters * 64;
    printf("dfma_gops_bpsm%d %.1f\n", bpsm, ops / (ms * 1e6));
    k_fp64<1><<<sms * bpsm, 512>>>(o, 100, 1e-9, 2e-9);
    cudaEventRecord(e0);
    k_fp64<1><<<sms * bpsm, 512>>>(o, iters, 1e-9, 2e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("dadd_gops_bpsm%d %.1f\n", bpsm, ops / (ms * 1e6));
  }
  long long* ck; CK(cudaMalloc(&ck, 16));
  cudaEventRecord(e0);
  k_clock<<<sms * 4, 512>>>(ck, 200000, 1.0000001);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  long long hc[2]; cudaMemcpy(hc, ck, 16, cudaMemcpyDeviceToHost);
  printf("sm_clock_mhz_under_fp64 %.1f\n", hc[0] / (ms * 1e3));
  // ---- smem ------------------------------------------------------------------------
  k_smem<<<sms * 4, 512>>>(o, 1000);
  cudaEventRecord(e0);
  k_smem<<<sms * 4, 512>>>(o, 100000);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("smem_gbs_total %.1f\n", (double)sms * 4 * 512 * 100000 * 16 / (ms * 1e6));
  CK(cudaGetLastError());
  return 0;
}
