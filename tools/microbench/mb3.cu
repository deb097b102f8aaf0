// Step-0 probe, part 3: which on-chip data paths are independent resources?
//   lds64 / lds128 / sts64 : shared-memory bandwidth (bytes/clk/SM) by access width
//   shfl                   : fp64 warp-shuffle throughput (two 32-bit SHFL each)
//   lds+shfl               : both interleaved -- additive (shared crossbar) or overlapped?
//   lds+stg                : shared loads interleaved with global stores to an L2-resident buffer
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb3 mb3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int NT = 512;
constexpr int SMN = 4096;  // doubles in smem (32 KB)

template <int MODE>
__global__ void __launch_bounds__(NT) k_mix(int iters, double* gbuf, uint32_t gmask, double* sink) {
  __shared__ __align__(16) double sm[SMN];
  for (int i = threadIdx.x; i < SMN; i += NT) sm[i] = (double)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a0 = lane, a1 = 0, a2 = 0, a3 = 0;
  uint32_t off = threadIdx.x;
  uint64_t goff = ((uint64_t)blockIdx.x * NT + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t o = (off + u * NT) & (SMN - 1);
      if (MODE == 0 || MODE == 3 || MODE == 4) {  // lds64
        a0 += sm[o];
      }
      if (MODE == 1) {  // lds128: two doubles per lane
        const double2 v = reinterpret_cast<const double2*>(sm)[((off + u * NT) & (SMN / 2 - 1))];
        if (u & 1) { a0 += v.x; a1 += v.y; } else { a2 += v.x; a3 += v.y; }
      }
      if (MODE == 6) {  // sts128
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"((uint32_t)__cvta_generic_to_shared(sm + 2 * ((off + u * NT) & (SMN / 2 - 1)))), "d"(a0 + u), "d"(a1) : "memory");
      }
      if (MODE == 7) {  // lds64, 4 independent chains
        const double v = sm[o];
        if ((u & 3) == 0) a0 += v; else if ((u & 3) == 1) a1 += v; else if ((u & 3) == 2) a2 += v; else a3 += v;
      }
      if (MODE == 2) {  // sts64
        asm volatile("st.shared.f64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(sm + o)), "d"(a0 + u) : "memory");
      }
      if (MODE == 3 || MODE == 5) {  // shfl fp64
        a2 += __shfl_xor_sync(0xffffffffu, a0 + u, (u & 3) + 1);
      }
      if (MODE == 4) {  // global store, L2-resident footprint
        const uint64_t g = (goff + (uint64_t)(it * 8 + u) * 148 * NT) & gmask;
        asm volatile("st.global.f64 [%0], %1;" ::"l"(gbuf + g), "d"(a0) : "memory");
      }
    }
    off += 7;
  }
  if (a0 + a1 + a2 + a3 == 1234.5) *sink = a0;
}

template <int MODE>
float run(int grid, int iters, double* g, uint32_t gmask, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mix<MODE><<<grid, NT>>>(iters, g, gmask, sink);
  cudaEventRecord(e0);
  k_mix<MODE><<<grid, NT>>>(iters, g, gmask, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* g;
  double* sink;
  const size_t gn = 1 << 22;  // 32 MB (L2-resident)
  CK(cudaMalloc(&g, gn * 8));
  CK(cudaMalloc(&sink, 8));
  const int grid = sms * 2, iters = 4096;
  const double ops = (double)grid * NT * iters * 8;  // per-lane operations of each kind
  const char* names[] = {"lds64", "lds128", "sts64", "lds64+shfl", "lds64+stg", "shfl", "sts128", "lds64x4"};
  float t[8];
  t[0] = run<0>(grid, iters, g, gn - 1, sink);
  t[1] = run<1>(grid, iters, g, gn - 1, sink);
  t[2] = run<2>(grid, iters, g, gn - 1, sink);
  t[3] = run<3>(grid, iters, g, gn - 1, sink);
  t[4] = run<4>(grid, iters, g, gn - 1, sink);
  t[5] = run<5>(grid, iters, g, gn - 1, sink);
  t[6] = run<6>(grid, iters, g, gn - 1, sink);
  t[7] = run<7>(grid, iters, g, gn - 1, sink);
  CK(cudaDeviceSynchronize());
  for (int m = 0; m < 8; ++m) {
    // bytes per clk per SM of the "primary" op, assuming the max SM clock
    const double lane_ops_per_s = ops / (t[m] * 1e-3);
    const double per_sm_clk = lane_ops_per_s / sms / (clk * 1e3);
    printf("%-12s %8.3f ms  lane-ops/clk/SM %7.2f  (x8 B = %6.1f B/clk/SM)\n", names[m], t[m], per_sm_clk,
           per_sm_clk * 8 * (m == 1 || m == 6 ? 2 : 1));
  }
  return 0;
}
