// Pair-loop throughput probe: runs the slab engine's F1 / F2 stages (hc_slab.cuh) on
// SMEM-resident synthetic data, no TMA and no global traffic, and reports clk per pair
// iteration per SM for: both stages + barrier, F2 only, F1 only, both without barrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1608_00206_b200/csrc -o mb5 mb5.cu
#include <cstdio>
#include "hc_slab.cuh"

using namespace hc;

template <int MODE>
__global__ void __launch_bounds__(T8_NT, 2) k_pairs(int iters, double* sink) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  double* P = sm;
  double* R = sm + T8Cfg<double>::ALIAS;
  for (int i = threadIdx.x; i < T8Cfg<double>::ALIAS + T8_NRAW * RS_SZ; i += T8_NT) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const bool unit = tid < 243;
  const int uu = t8_unit(tid);
  const int ea2 = uu / 81, eS = uu - 81 * ea2;
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0;
  if (MODE == 5) {  // full / empty mbarriers per P buffer instead of one CTA barrier per pair
    __shared__ __align__(8) uint64_t fullb[2], emptyb[2];
    if (tid == 0) {
      mbar_init(&fullb[0], 3); mbar_init(&fullb[1], 3);
      mbar_init(&emptyb[0], 8); mbar_init(&emptyb[1], 8);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int es = t8_f1_es(w);
    if (es >= 0) {  // F1 of pair 0
      t8_f1<double>(R, P, es, lane);
      __syncwarp();
      if (lane == 0) { asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(&fullb[0])) : "memory"); }
    }
    for (int p = 0; p < iters; ++p) {
      const int b1 = (p + 1) & 1;
      if (es >= 0 && p + 1 < iters) {
        if (p + 1 >= 2) mbar_wait(&emptyb[b1], ((p - 1) / 2) & 1);
        t8_f1<double>(R + ((p + 1) % T8_NRAW) * RS_SZ, P + b1 * PS_SZ, es, lane);
        __syncwarp();
        if (lane == 0) { asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(&fullb[b1])) : "memory"); }
      }
      mbar_wait(&fullb[p & 1], (p / 2) & 1);
      if (unit) t8_f2<double>(P + (p & 1) * PS_SZ, ea2, eS, acc);
      __syncwarp();
      if (lane == 0) { asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(&emptyb[p & 1])) : "memory"); }
    }
  } else
  for (int p = 0; p < iters; ++p) {
    if (MODE != 1 && t8_f1_es(w) >= 0) t8_f1<double>(R + (p % T8_NRAW) * RS_SZ, P + ((p + 1) & 1) * PS_SZ, t8_f1_es(w), lane);
    if (MODE == 4 && unit) {  // F2 arithmetic only: inputs from registers (no shared loads)
      double xt[8], yt[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // vary the low mantissa bits only (integer pipe)
        xt[j] = __longlong_as_double(0x3f50624dd2f1a9fcll ^ (long long)((p + j) & 255));
        yt[j] = __longlong_as_double(0x3f60624dd2f1a9fcll ^ (long long)((p * 3 + j) & 255));
      }
      fwd_mul_acc<3, double>(xt, yt, acc);
    } else if (MODE != 2 && unit) t8_f2<double>(P + (p & 1) * PS_SZ, ea2, eS, acc);
    if (MODE != 3 && MODE != 4) __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 27; ++i) s += acc[i];
  if (s == 1234.5) *sink = s;
}

// dedicated roles: warps 0-7 run F2 only (243 units), warps 8-10 run F1 only (e_s = w - 8),
// one CTA per SM, a barrier per pair among all 11 warps
__global__ void __launch_bounds__(352, 1) k_roles(int iters, double* sink) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  double* P = sm;
  double* R = sm + T8Cfg<double>::ALIAS;
  for (int i = threadIdx.x; i < T8Cfg<double>::ALIAS + T8_NRAW * RS_SZ; i += 352) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const bool unit = tid < 243;
  const int uu = t8_unit(tid < 256 ? tid : 0);
  const int ea2 = uu / 81, eS = uu - 81 * ea2;
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0;
  for (int p = 0; p < iters; ++p) {
    if (w >= 8) t8_f1<double>(R + (p % T8_NRAW) * RS_SZ, P + ((p + 1) & 1) * PS_SZ, w - 8, lane);
    else if (unit) t8_f2<double>(P + (p & 1) * PS_SZ, ea2, eS, acc);
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 27; ++i) s += acc[i];
  if (s == 1234.5) *sink = s;
}

template <int MODE>
float run(int grid, int iters, double* sink) {
  auto k = k_pairs<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T8Cfg<double>::SMEM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<grid, T8_NT, T8Cfg<double>::SMEM>>>(iters, sink);
  cudaEventRecord(e0);
  k<<<grid, T8_NT, T8Cfg<double>::SMEM>>>(iters, sink);
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
  const int iters = 20000;
  const char* names[] = {"F1+F2+bar", "F2+bar", "F1+bar", "F1+F2 nobar", "F2 math only", "F1+F2 mbarriers"};
  for (int ctas = 1; ctas <= 2; ++ctas) {
    const int grid = sms * ctas;
    for (int m = 0; m < 6; ++m) {
      float ms = m == 0 ? run<0>(grid, iters, sink) : m == 1 ? run<1>(grid, iters, sink)
               : m == 2 ? run<2>(grid, iters, sink) : m == 3 ? run<3>(grid, iters, sink)
               : m == 4 ? run<4>(grid, iters, sink) : run<5>(grid, iters, sink);
      // clk per pair iteration per SM (all CTAs on the SM together)
      const double clk_per = (ms * 1e-3) * (clk * 1e3) / ((double)iters * ctas);
      printf("ctas/SM %d %-12s %.3f ms  %.0f clk per pair-iteration per SM\n", ctas, names[m], ms, clk_per);
    }
  }
  {
    cudaFuncSetAttribute(k_roles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T8Cfg<double>::SMEM);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_roles<<<sms, 352, T8Cfg<double>::SMEM>>>(iters, sink);
    cudaEventRecord(e0);
    k_roles<<<sms, 352, T8Cfg<double>::SMEM>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("1 CTA/SM, 8 F2 warps + 3 F1 warps: %.3f ms  %.0f clk per pair-iteration per SM\n", ms,
           (ms * 1e-3) * (clk * 1e3) / (double)iters);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
