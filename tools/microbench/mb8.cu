// Pair-loop probe for the round-2 "3-CTA cluster per tile" direction: one CTA
// = the 81 units (e_a2, e_B) of one evaluation point e_a1 of a tile, 3 warps, its own F1
// (the a1 axis at e_a1 plus the three B axes, split over the 3 warps by the top B digit) and a
// 96-thread barrier per pair.  SMEM-resident synthetic data, no TMA, no global traffic, like
// mb5.  Reports clk per pair and 3^8-tile per SM (three groups = one tile), to compare with
// mb5's 724 (2 CTAs x 8 warps per SM, one CTA per tile).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1608_00206_b200/csrc -o mb8 mb8.cu
#include <cstdio>
#include "hc_common.cuh"

using namespace hc;

constexpr int G_NT = 96;
// raw slice stage: [op][b_a2][b_a1][b_B (8)][b_C (8)] = 256 values per operand (+ padding)
constexpr int GR_H1 = 64, GR_H2 = 136, GR_OP = 304, GR_SZ = 608;
// P stage: [op][b_a2][e_B (27)][b_C (8) padded to 10]
constexpr int GP_ROW = 10, GP_A2 = 270 + 2, GP_OP = 2 * GP_A2 + 4, GP_SZ = 2 * GP_OP;
constexpr int G_NRAW = 4;
constexpr int G_SMEM = (2 * GP_SZ + G_NRAW * GR_SZ) * 8;

// F1, warp w (top B digit e_b2 = w): lane (op, b_a2, b_C) evaluates a1 at es and the B axes
// for the 9 e_B with digit 2 = w
__device__ __forceinline__ void g_f1(const double* R, double* P, int es, int w, int lane) {
  const int op = lane >> 4, ba2 = (lane >> 3) & 1, bc = lane & 7;
  const double* src = R + op * GR_OP + ba2 * GR_H2 + bc;
  double in[4];
  auto ld = [&](int j) {  // b_B = j: a1 evaluated at es
    return es == 0 ? src[8 * j] : es == 2 ? src[GR_H1 + 8 * j] : src[8 * j] + src[GR_H1 + 8 * j];
  };
  if (w == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) in[j] = ld(j);
  } else if (w == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) in[j] = ld(j + 4);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) in[j] = ld(j) + ld(j + 4);
  }
  double* dst = P + op * GP_OP + ba2 * GP_A2 + (9 * w) * GP_ROW + bc;
  fwd_store<2, GP_ROW, double>(in, dst);
}

// F2: unit (e_a2, e_B) loads 8 + 8 base values and accumulates its register cube
__device__ __forceinline__ void g_f2(const double* P, int ea2, int eB, double* acc) {
  const double* px = P + eB * GP_ROW;
  double xt[8], yt[8];
  if (ea2 != 1) {
    const double* a = px + (ea2 >> 1) * GP_A2;
#pragma unroll
    for (int j = 0; j < 8; ++j) { xt[j] = a[j]; yt[j] = a[GP_OP + j]; }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      xt[j] = px[j] + px[GP_A2 + j];
      yt[j] = px[GP_OP + j] + px[GP_OP + GP_A2 + j];
    }
  }
  fwd_mul_acc<3, double>(xt, yt, acc);
}

__device__ __forceinline__ void bar96() { asm volatile("bar.sync 1, 96;" ::: "memory"); }

template <int MINB>
__global__ void __launch_bounds__(G_NT, MINB) k_group(int iters, double* sink) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  double* P = sm;
  double* R = sm + 2 * GP_SZ;
  for (int i = threadIdx.x; i < 2 * GP_SZ + G_NRAW * GR_SZ; i += G_NT) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int es = blockIdx.x % 3;
  // heavy units (e_a2 = 1: two rows per operand) on warp 0, light ones on warps 1-2, so no
  // warp runs both paths of g_f2
  const bool unit = tid < 27 || (tid >= 32 && tid < 86);
  const int t2 = tid - 32;
  const int ea2 = tid < 32 ? 1 : (t2 < 27 ? 0 : 2), eB = tid < 32 ? tid : t2 % 27;
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0;
  for (int p = 0; p < iters; ++p) {
    g_f1(R + (p % G_NRAW) * GR_SZ, P + ((p + 1) & 1) * GP_SZ, es, w, lane);
    if (unit) g_f2(P + (p & 1) * GP_SZ, ea2, eB, acc);
    bar96();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 27; ++i) s += acc[i];
  if (s == 1234.5) *sink = s;
}

template <int MINB>
void run(int sms, int clk, int iters, double* sink) {
  auto k = k_group<MINB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, G_SMEM);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, G_NT, G_SMEM);
  for (int ctas = 3; ctas <= occ; ++ctas) {
    const int grid = sms * ctas;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<grid, G_NT, G_SMEM>>>(iters, sink);
    cudaEventRecord(e0);
    k<<<grid, G_NT, G_SMEM>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // three groups make one tile: tiles per SM and iteration = ctas / 3
    const double clk_per_tile = (ms * 1e-3) * (clk * 1e3) / ((double)iters * ctas / 3.0);
    printf("minBlocks %d, %d CTAs (x3 warps) per SM: %.3f ms  %.0f clk per pair and tile per SM\n", MINB, ctas, ms,
           clk_per_tile);
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  printf("smem per CTA %d B\n", G_SMEM);
  run<5>(sms, clk, 20000, sink);
  run<6>(sms, clk, 20000, sink);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
