// hc_apps.cuh -- kernels of the applications built on the hot path;
// C ABI in include/hc.h (hc_convolve_difference, hc_apply_carries, hc_maxconv_pnorm).
//
//  f4  PMF of differences of Bernoulli-axis random vectors (PAPER.md 35-38, 147-149):
//      P(X - Y = d) = sum_{i - j = d} x[i] y[j] = conv(x, flip(y))[d + 1], flip(y)[j] =
//      y[~j]: the per-axis complement turns a difference into a sum (flip_kernel).
//  f1  carry-free convolution -> ordinary 1-D convolution (PAPER.md 354-373): the hot path
//      is the carry-free convolution of two length-2^D vectors (bit b = axis b); the carries
//      are out[m] = sum_{k : sum_b k_b 2^b = m} z[k], done axis by axis -- after the low c
//      axes are combined a row holds the values v = sum_{b<c} k_b 2^b in [0, 2^(c+1) - 1),
//      and combining axis c is  B[r][v'] = sum_{k_c} A[k_c + 3 r][v' - k_c 2^c].
//      carry_tile_kernel does the low min(D, 8) axes of one 3^8 tile in shared memory;
//      carry_step_kernel does one further axis in global memory.
//  f2  p-norm max-convolution (PAPER.md 341-352): max_{i+j=k} x[i] y[j] ~
//      (sum_{i+j=k} x[i]^p y[j]^p)^(1/p) = (x^p * y^p)[k]^(1/p); inputs are scaled by their
//      maxima first so the powers stay in range (pnorm_pre_kernel / pnorm_post_kernel).
#pragma once
#include "hc_common.cuh"

namespace hc {

// f4 -----------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) flip_kernel(const T* __restrict__ y, T* __restrict__ yf, int D) {
  const uint64_t n = 1ull << D;
  const uint64_t mask = n - 1;
  for (uint64_t j = (uint64_t)blockIdx.x * 256 + threadIdx.x; j < n; j += (uint64_t)gridDim.x * 256)
    yf[j] = y[~j & mask];
}

// f1 -----------------------------------------------------------------------------------
// One combining step on rows: A is [nr_in][V], V = 2^(c+1) - 1; B is [nr_in / 3][2^(c+2) - 1].
template <class T, class I>
__device__ __forceinline__ T carry_gather(const T* A, I V, I r, I v, int c) {
  T s = T(0);
#pragma unroll
  for (int kc = 0; kc < 3; ++kc) {
    const I off = (I)kc << c;
    if (v >= off && v - off < V) s = Ar<T>::add(s, A[(uint64_t)(kc + 3 * r) * V + (v - off)]);
  }
  return s;
}

// one combining step inside the tile: axis C of a 3^L tile, compile-time sizes (so the index
// divisions compile to multiply-shifts)
template <class T, int L, int C>
__device__ __forceinline__ void carry_tile_step(const T* A, T* B) {
  constexpr uint32_t V = (2u << C) - 1, V2 = 2 * V + 1;
  constexpr uint32_t NR2 = (uint32_t)ipow3(L - C - 1);
  for (uint32_t o = threadIdx.x; o < NR2 * V2; o += 256) {
    const uint32_t r = o / V2, v = o - r * V2;
    B[o] = carry_gather<T, uint32_t>(A, V, r, v, C);
  }
}
template <class T, int L, int C>
__device__ __forceinline__ void carry_tile_steps(T* b0, T* b1) {
  if constexpr (C < L) {
    carry_tile_step<T, L, C>(b0, b1);
    __syncthreads();
    carry_tile_steps<T, L, C + 1>(b1, b0);
  }
}

// tile of the low L = min(D, 8) axes (3^L values of z) -> 2^(L+1) - 1 partial sums, combining
// axis 0, 1, ..., L-1 in shared memory; grid = 3^(D-L) tiles, block 256
template <class T, int L>
__global__ void __launch_bounds__(256) carry_tile_kernel(const T* __restrict__ z, T* __restrict__ part) {
  constexpr int N = ipow3(L);
  extern __shared__ __align__(128) unsigned char carry_smem[];  // 2 x 3^L elements
  T* b0 = reinterpret_cast<T*>(carry_smem);
  T* b1 = b0 + N;
  const uint64_t t = blockIdx.x;
  for (int i = threadIdx.x; i < N; i += 256) b0[i] = z[t * N + i];
  __syncthreads();
  carry_tile_steps<T, L, 0>(b0, b1);
  // after L steps (ping-pong) the result is in b0 when L is even, b1 when odd
  const T* res = (L & 1) ? b1 : b0;
  constexpr uint32_t V = (2u << L) - 1;
  for (uint32_t v = threadIdx.x; v < V; v += 256) part[t * V + v] = res[v];
}

// Persistent form for L = 8 (D >= 8): the next tile's z values are loaded into registers
// (coalesced, 26 per thread) while the current tile is combined, so the HBM read overlaps
// the shared-memory steps; axes 0-2 are combined in registers (a row of 27 values -> 15
// partial sums v = k0 + 2 k1 + 4 k2), axes 3-7 in shared memory (carry_tile_steps from C = 3).
// Shared memory: raw tile 3^8 + 243 x 15 + 81 x 31 elements (2 CTAs per SM).
template <class T>
__global__ void __launch_bounds__(256, 2) carry_tile8_kernel(const T* __restrict__ z, T* __restrict__ part,
                                                             uint64_t ntiles) {
  constexpr int N = 6561, NL = (N + 255) / 256;
  extern __shared__ __align__(128) unsigned char carry_smem[];
  T* raw = reinterpret_cast<T*>(carry_smem);
  T* b1 = raw + N;          // [243][15]
  T* b2 = b1 + 243 * 15;    // [81][31]
  const int tid = threadIdx.x;
  T r[NL];
  auto load = [&](uint64_t t) {
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (tid + 256 * j < N) r[j] = z[t * N + tid + 256 * j];
  };
  uint64_t t = blockIdx.x;
  if (t < ntiles) load(t);
  for (; t < ntiles; t += gridDim.x) {
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (tid + 256 * j < N) raw[tid + 256 * j] = r[j];
    __syncthreads();
    if (t + gridDim.x < ntiles) load(t + gridDim.x);  // in flight during the steps below
    if (tid < 243) {
      T v[27], b[15];
#pragma unroll
      for (int k = 0; k < 27; ++k) v[k] = raw[27 * tid + k];
#pragma unroll
      for (int k = 0; k < 15; ++k) b[k] = T(0);
#pragma unroll
      for (int k2 = 0; k2 < 3; ++k2)
#pragma unroll
        for (int k1 = 0; k1 < 3; ++k1)
#pragma unroll
          for (int k0 = 0; k0 < 3; ++k0) b[k0 + 2 * k1 + 4 * k2] = Ar<T>::add(b[k0 + 2 * k1 + 4 * k2], v[k0 + 3 * k1 + 9 * k2]);
#pragma unroll
      for (int k = 0; k < 15; ++k) b1[15 * tid + k] = b[k];
    }
    __syncthreads();
    carry_tile_steps<T, 8, 3>(b1, b2);  // c = 3..7, result (511 values) in b2
    for (int v = tid; v < 511; v += 256) part[t * 511 + v] = b2[v];
    __syncthreads();  // b1 / b2 / raw are rewritten by the next tile
  }
}

// one further axis C in global memory: A [nr][2^(C+1) - 1] -> B [nr / 3][2^(C+2) - 1]
template <class T, class I, int C>
__global__ void __launch_bounds__(256) carry_step_kernel(const T* __restrict__ A, T* __restrict__ B, uint64_t nr2) {
  constexpr I V = ((I)2 << C) - 1, V2 = 2 * V + 1;
  const I total = (I)nr2 * V2;
  for (I o = (I)blockIdx.x * 256 + threadIdx.x; o < total; o += (I)gridDim.x * 256) {
    const I r = o / V2, v = o - r * V2;
    B[o] = carry_gather<T, I>(A, V, r, v, C);
  }
}

// f2 -----------------------------------------------------------------------------------
// max of a nonnegative double array (bit patterns order like the values): atomicMax on u64
__global__ void __launch_bounds__(256) max_nonneg_kernel(const double* __restrict__ a, uint64_t n,
                                                         unsigned long long* out) {
  double m = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
    m = fmax(m, a[i]);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// xp[i] = (x[i] / max x)^p  (0 where the maximum is 0); p = 2^sq: sq squarings
__global__ void __launch_bounds__(256) pnorm_pre_kernel(const double* __restrict__ x, double* __restrict__ xp,
                                                        uint64_t n, double p, int sq, const unsigned long long* mx) {
  const double s = __longlong_as_double((long long)*mx);
  for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
    double v = s > 0.0 ? x[i] / s : 0.0;
    if (sq >= 0) {
      for (int k = 0; k < sq; ++k) v *= v;
    } else {
      v = pow(v, p);
    }
    xp[i] = v;
  }
}

// z[k] = max x * max y * z[k]^(1/p), optionally rounded to the nearest integer; p = 2^sq:
// sq square roots.  Four independent elements per thread and iteration: one load in flight
// per thread cannot cover HBM latency at 2048 threads per SM.
__device__ __forceinline__ double pnorm_root(double v, double s, double ip, int sq, int round_to_int) {
  if (v > 0.0) {
    if (sq >= 0) {
      for (int k = 0; k < sq; ++k) v = sqrt(v);
    } else {
      v = pow(v, ip);
    }
    v *= s;
  } else {
    v = 0.0;
  }
  return round_to_int ? rint(v) : v;
}
__global__ void __launch_bounds__(256) pnorm_post_kernel(double* __restrict__ z, uint64_t n, double p, int sq,
                                                         const unsigned long long* mx, int round_to_int) {
  const double s = __longlong_as_double((long long)mx[0]) * __longlong_as_double((long long)mx[1]);
  const double ip = 1.0 / p;
  const uint64_t stride = (uint64_t)gridDim.x * 256;
  uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = z[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u) z[i + u * stride] = pnorm_root(v[u], s, ip, sq, round_to_int);
  }
  for (; i < n; i += stride) z[i] = pnorm_root(z[i], s, ip, sq, round_to_int);
}

}  // namespace hc
