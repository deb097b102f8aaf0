// Probe: tensor-memory (TMEM) load/store throughput and warp-shuffle throughput on sm_100a,
// next to shared memory, to decide whether TMEM can hold per-thread accumulators (a larger
// register cube) or act as an exchange buffer for the tile kernels.
// One CTA per SM (grid = 148), NW warps; every warp moves 32 lanes x NC 32-bit columns per
// instruction.  Reports bytes per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb10 mb10.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// OP 0: tcgen05.ld 32x32b.x16 + wait::ld; OP 1: tcgen05.st 32x32b.x16 + wait::st;
// OP 2: ld+st read-modify-write of 16 columns (accumulator round trip);
// OP 3: 4 loads in flight before one wait (pipelined)
template <int OP, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_tmem(int iters, uint32_t* sink, long long* cyc) {
  __shared__ uint32_t s_taddr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = s_taddr;
  // lane quadrant of this warp; warps sharing a quadrant use disjoint column ranges
  const uint32_t quad = (uint32_t)(warp & 3), slot = (uint32_t)(warp >> 2);
  constexpr int PER = 512 / (NW / 4 > 0 ? NW / 4 : 1);  // columns per warp
  const uint32_t ta = tbase + ((quad * 32u) << 16) + slot * PER;
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)((it * 16) % PER);
    if (OP == 0 || OP == 2) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(ta + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] += 1u;
      acc ^= r[it & 15];
    }
    if (OP == 3) {
      uint32_t q[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(q[u][0]), "=r"(q[u][1]), "=r"(q[u][2]), "=r"(q[u][3])
                     : "r"(ta + ((col + 4 * u) % PER)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < 4; ++u) acc ^= q[u][0] + q[u][1] + q[u][2] + q[u][3];
    }
    if (OP == 1 || OP == 2) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              ta + col),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      if (OP == 1) r[it & 15] += 3u;
    }
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  if (acc == 0x12345u) sink[0] = acc + r[0];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// OP 0: __shfl_xor of a 32-bit value; OP 1: of a double (two SHFL); reported per 32-bit SHFL
template <int OP, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_shfl(int iters, uint32_t* sink, long long* cyc) {
  uint32_t v0 = threadIdx.x, v1 = threadIdx.x * 3, v2 = threadIdx.x * 5, v3 = threadIdx.x * 7;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v0 = __shfl_xor_sync(0xffffffffu, v0, 1 + u) + 1;
      v1 = __shfl_xor_sync(0xffffffffu, v1, 2 + u) + 1;
      v2 = __shfl_xor_sync(0xffffffffu, v2, 3 + u) + 1;
      v3 = __shfl_xor_sync(0xffffffffu, v3, 5 + u) + 1;
    }
  }
  long long t1 = clock64();
  if ((v0 ^ v1 ^ v2 ^ v3) == 0x12345u) sink[0] = v0;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// shared-memory reference: LDS.128 (OP 0) and STS.64 (OP 1) at conflict-free strides
template <int OP, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_smem(int iters, uint32_t* sink, long long* cyc) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += NW * 32) sm[i] = i;
  __syncthreads();
  const uint32_t base = smem_u32(sm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a0 = 0, a1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w = ((uint32_t)(lane * 2 + warp * 64 + u * 1024 + it * 128)) & 4094u;
      if (OP == 0) {
        double p, q;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(p), "=d"(q) : "r"(base + w * 8));
        a0 += p;
        a1 += q;
      } else {
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(base + (w >> 1) * 8 + (lane & 0) ), "d"(a0 + u) : "memory");
      }
    }
    a0 += 1e-9;
  }
  long long t1 = clock64();
  if (a0 + a1 == 1234.5) sink[0] = 1;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <class K>
double run(K kern, int nthreads, int iters, uint32_t* sink, long long* cyc) {
  kern<<<148, nthreads>>>(iters, sink, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<148, nthreads>>>(iters, sink, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return -1;
  }
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  return (double)mx;
}

int main() {
  uint32_t* sink;
  long long* cyc;
  cudaMalloc(&sink, 64);
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int it = 20000;
#define TM(OP, NW, BYTES, NAME)                                                                          \
  {                                                                                                      \
    double c = run(k_tmem<OP, NW>, NW * 32, it, sink, cyc);                                              \
    printf("%-34s NW=%2d  %8.1f clk/iter/warp  %7.1f B/clk/SM\n", NAME, NW, c / it, (double)(BYTES)*NW * it / c); \
  }
  TM(0, 4, 2048, "tmem ld 32x32b.x16 + wait");
  TM(0, 8, 2048, "tmem ld 32x32b.x16 + wait");
  TM(0, 16, 2048, "tmem ld 32x32b.x16 + wait");
  TM(3, 16, 2048, "tmem ld 4 x x4 + one wait");
  TM(1, 4, 2048, "tmem st 32x32b.x16 + wait");
  TM(1, 16, 2048, "tmem st 32x32b.x16 + wait");
  TM(2, 8, 4096, "tmem ld+st x16 (rmw)");
  TM(2, 16, 4096, "tmem ld+st x16 (rmw)");
#define SH(OP, NW, NAME)                                                                                   \
  {                                                                                                        \
    double c = run(k_shfl<OP, NW>, NW * 32, it, sink, cyc);                                                \
    printf("%-34s NW=%2d  %8.1f clk/iter/warp  %7.1f B/clk/SM  (%.2f clk per warp-SHFL per SM)\n", NAME, NW, \
           c / it, 16.0 * 128 * NW * it / c, c / (16.0 * NW * it));                                        \
  }
  SH(0, 8, "shfl.b32");
  SH(0, 16, "shfl.b32");
  SH(0, 32, "shfl.b32");
#define SM_(OP, NW, BYTES, NAME)                                                                           \
  {                                                                                                        \
    double c = run(k_smem<OP, NW>, NW * 32, it, sink, cyc);                                                \
    printf("%-34s NW=%2d  %8.1f clk/iter/warp  %7.1f B/clk/SM\n", NAME, NW, c / it, (double)(BYTES)*NW * it / c); \
  }
  SM_(0, 16, 4 * 512, "lds.128 (reference)");
  SM_(1, 16, 4 * 256, "sts.64 (reference)");
  return 0;
}
