// Step-0 probe, part 4: shared-memory access cost by lane stride and width on sm_100a.
// For each (op, stride in 8-B words) a warp issues accesses at word offsets lane*stride
// (+ a per-iteration base that keeps the bank pattern); reports clk per warp-instruction
// per SM (lower is better; 1.0 = 16 lanes/clk for 8-B ops).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb4 mb4.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 512;
constexpr int SMN = 4096;  // doubles (32 KB)

template <int OP>  // 0 = LDS.64, 1 = LDS.128, 2 = STS.64, 3 = STS.128
__global__ void __launch_bounds__(NT) k_stride(int iters, int stride, double* sink) {
  __shared__ __align__(16) double sm[SMN];
  for (int i = threadIdx.x; i < SMN; i += NT) sm[i] = (double)i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  // every iteration shifts the whole warp by a multiple of 32 words: same bank pattern
  uint32_t o = (uint32_t)(lane * stride + warp * 64);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t w = (o + u * 256) & ((OP & 1) ? SMN - 2 : SMN - 1);  // v2: even word
      const uint32_t addr = sbase + w * 8;
      if (OP == 0) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
        if (u & 1) a0 += v; else a1 += v;
      } else if (OP == 1) {
        double v, v2;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(v2) : "r"(addr));
        if (u & 1) { a0 += v; a2 += v2; } else { a1 += v; a3 += v2; }
      } else if (OP == 2) {
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(a0 + u) : "memory");
      } else {
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a0 + u), "d"(a1) : "memory");
      }
    }
    o += 512;
    a0 += 1e-9;
  }
  if (a0 + a1 + a2 + a3 == 1234.5) *sink = a0;
}

template <int OP>
float run(int grid, int iters, int stride, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_stride<OP><<<grid, NT>>>(iters, stride, sink);
  cudaEventRecord(e0);
  k_stride<OP><<<grid, NT>>>(iters, stride, sink);
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
  double* sink;
  cudaMalloc(&sink, 8);
  const int grid = sms * 2, iters = 2048;
  const double warp_instr = (double)grid * (NT / 32) * iters * 8;
  const char* ops[] = {"LDS.64", "LDS.128", "STS.64", "STS.128"};
  const int strides[] = {1, 2, 3, 4, 6, 8, 10, 12, 16, 18, 26, 27, 28, 30, 34};
  for (int op = 0; op < 4; ++op) {
    for (int s : strides) {
      if ((op & 1) && (s & 1)) continue;  // v2 needs even word offsets
      float ms = 0;
      if (op == 0) ms = run<0>(grid, iters, s, sink);
      if (op == 1) ms = run<1>(grid, iters, s, sink);
      if (op == 2) ms = run<2>(grid, iters, s, sink);
      if (op == 3) ms = run<3>(grid, iters, s, sink);
      const double clk_per_instr = (ms * 1e-3) * (clk * 1e3) * sms / warp_instr;
      printf("%-8s stride %2d words: %.3f ms  %.2f clk/warp-instr/SM\n", ops[op], s, ms, clk_per_instr);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
