// fp64 pipe probe: DFMA latency (dependent chain, 1 warp per SM) and throughput vs the number
// of independent chains per warp and warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb6 mb6.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_chain(int iters, double* sink, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) *sink = s;
}
// the register-cube product of the slab engine: Karatsuba on all three axes (KKK,
// hc_common.cuh fwd_mul_acc) or Karatsuba on the top axis + the direct split on the lower two
// (KDD: 48 FMA + 8 adds), inputs fixed in registers, 27 accumulators
#include "../../paper_1608_00206_b200/csrc/hc_common.cuh"
__device__ __forceinline__ void kdd(const double* x, const double* y, double* acc) {
  auto direct2 = [](const double* a, const double* b, double* c) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = ((i & 1) + (j & 1)) + 3 * ((i >> 1) + (j >> 1));
        c[k] = fma(a[i], b[j], c[k]);
      }
  };
  direct2(x, y, acc);
  direct2(x + 4, y + 4, acc + 18);
  double xs[4], ys[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { xs[i] = x[i] + x[i + 4]; ys[i] = y[i] + y[i + 4]; }
  direct2(xs, ys, acc + 9);
}
template <int KIND>
__global__ void k_cube(int iters, double* sink) {
  double acc[27], x[8], y[8];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { x[j] = 1e-3 * (threadIdx.x + j); y[j] = 2e-3 * (j + 1); }
  for (int i = 0; i < iters; ++i) {
    if (KIND == 0) hc::fwd_mul_acc<3, double>(x, y, acc);
    else kdd(x, y, acc);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __longlong_as_double(__double_as_longlong(x[j]) ^ 1ll);  // defeat hoisting
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 27; ++i) s += acc[i];
  if (s == 1.2345) *sink = s;
}
template <int KIND>
void run_cube(int sms, int clk, int warps, double* sink) {
  const int iters = 1 << 12;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_cube<KIND><<<sms, 32 * warps>>>(iters, sink);
  cudaEventRecord(e0);
  k_cube<KIND><<<sms, 32 * warps>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("cube %s warps/SM %2d: %.1f clk per warp-iteration per SM sub-partition\n", KIND == 0 ? "KKK" : "KDD", warps,
         cyc / ((double)iters * warps / 4));
}
template <int CH>
void run(int sms, int clk, int warps, double* sink) {
  const int iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_chain<CH><<<sms, 32 * warps>>>(iters, sink, 0.999, 1e-3);
  cudaEventRecord(e0);
  k_chain<CH><<<sms, 32 * warps>>>(iters, sink, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * clk * 1e3;
  const double instr_per_sm = (double)iters * CH * warps;  // warp-level DFMA per SM
  printf("chains/warp %2d warps/SM %2d: %.2f clk per iteration of one warp, %.2f clk per warp-DFMA per SMSP\n", CH,
         warps, cyc / iters, cyc / (instr_per_sm / 4));
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* sink; cudaMalloc(&sink, 8);
  for (int w : {1, 4, 8, 16}) {
    run<1>(sms, clk, w, sink);
    run<4>(sms, clk, w, sink);
    run<8>(sms, clk, w, sink);
    run<16>(sms, clk, w, sink);
  }
  for (int w : {4, 8}) { run_cube<0>(sms, clk, w, sink); run_cube<1>(sms, clk, w, sink); }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
