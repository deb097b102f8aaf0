// Do fp64 arithmetic and shared-memory traffic overlap on sm_100a?  Times (a) DADD-only,
// (b) LDS.128-only, (c) both interleaved in the same warps, (d) DFMA-only, (e) DFMA + LDS,
// (f) DFMA + STS; 2 CTAs x 8 warps per SM.  Overlap => (c) ~ max(a, b); a shared path =>
// (c) ~ a + b.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb7 mb7.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NT = 256, SMN = 4096;
template <int MODE>
__global__ void __launch_bounds__(NT, 2) k(int iters, double* sink, double a, double b) {
  __shared__ __align__(16) double sm[SMN];
  for (int i = threadIdx.x; i < SMN; i += NT) sm[i] = i * 1e-3;
  __syncthreads();
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x + i;
  double l0 = 0, l1 = 0, l2 = 0, l3 = 0;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint32_t off = (uint32_t)(lane * 10 + wp * 320);  // stride-10 16-B loads: conflict-free
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (MODE == 0 || MODE == 2) {  // 8 independent DADD
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = c[i] + a;
      }
      if (MODE == 3 || MODE == 4 || MODE == 5) {  // 8 independent DFMA
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
      }
      if (MODE == 1 || MODE == 2 || MODE == 4) {  // 2 LDS.128
        const uint32_t o = (off + u * 1280) & (SMN - 1) & ~1u;
        double2 v = *reinterpret_cast<const double2*>(sm + o);
        double2 w = *reinterpret_cast<const double2*>(sm + ((o + 640) & (SMN - 1) & ~1u));
        l0 += v.x; l1 += v.y; l2 += w.x; l3 += w.y;
      }
      if (MODE == 5) {  // 2 STS.64
        const uint32_t o = (off + u * 1280) & (SMN - 1);
        asm volatile("st.shared.f64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(sm + o)), "d"(c[0]) : "memory");
        asm volatile("st.shared.f64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(sm + ((o + 641) & (SMN - 1)))), "d"(c[1]) : "memory");
      }
    }
    off += 2;
  }
  double s = l0 + l1 + l2 + l3;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345) *sink = s;
}
template <int MODE>
double run(int sms, int iters, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<2 * sms, NT>>>(iters, sink, 0.999, 1e-3);
  cudaEventRecord(e0);
  k<MODE><<<2 * sms, NT>>>(iters, sink, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 8);
  const int iters = 4096;
  const char* nm[] = {"DADD x32", "LDS.128 x8", "DADD x32 + LDS.128 x8", "DFMA x32", "DFMA x32 + LDS.128 x8",
                      "DFMA x32 + STS.64 x8"};
  double t[6] = {run<0>(sms, iters, sink), run<1>(sms, iters, sink), run<2>(sms, iters, sink),
                 run<3>(sms, iters, sink), run<4>(sms, iters, sink), run<5>(sms, iters, sink)};
  for (int m = 0; m < 6; ++m) printf("%-24s per iteration: %.3f ms total\n", nm[m], t[m]);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
