// hc_common.cuh -- device helpers for the hypercube-convolution kernels (sm_100a).
//
// Notation follows PAPER.md "Methods" (lines 153-212): for one axis, a pair of input
// values (a0, a1) is evaluated at {0, 1, inf} as (a0, a0 + a1, a1) (the paper's
// x[0] + x[1], lines 186-189), the three evaluations are multiplied pointwise, and the
// result (c0, c1, c2) is interpolated back as (c0, (c1 - c0) - c2, c2) (t - z[0] - z[2],
// lines 187-189; subtraction order of Algorithm 2's two loops, lines 248-251).
//
// Element arithmetic: uint64 (int64 as wrap-around, exact mod 2^64) or double.
// This file shares nothing with oracle/ (test infrastructure).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hc {

__host__ __device__ constexpr int ipow3(int n) { return n <= 0 ? 1 : 3 * ipow3(n - 1); }
__host__ __device__ constexpr uint64_t upow3(int n) { return n <= 0 ? 1ull : 3ull * upow3(n - 1); }

template <class T> struct Ar;
template <> struct Ar<uint64_t> {
  static __device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) { return a + b; }
  static __device__ __forceinline__ uint64_t sub(uint64_t a, uint64_t b) { return a - b; }
  // c + a*b (mod 2^64)
  static __device__ __forceinline__ uint64_t mad(uint64_t a, uint64_t b, uint64_t c) { return c + a * b; }
};
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mad(double a, double b, double c) { return __fma_rn(a, b, c); }
};

// ---- register-resident transforms (fully unrolled; N axes, axis 0 = fastest) --------

// Forward evaluation 2^N -> 3^N: out[e] = sum_{b ~ e} in[b], one axis at a time.
template <int N, class T>
__device__ __forceinline__ void fwd_reg(const T* in, T* out) {
  if constexpr (N == 0) {
    out[0] = in[0];
  } else {
    constexpr int h = 1 << (N - 1), m = ipow3(N - 1);
    T s[h];
#pragma unroll
    for (int i = 0; i < h; ++i) s[i] = Ar<T>::add(in[i], in[i + h]);
    fwd_reg<N - 1, T>(in, out);              // e_top = 0  <- a0
    fwd_reg<N - 1, T>(s, out + m);           // e_top = 1  <- a0 + a1
    fwd_reg<N - 1, T>(in + h, out + 2 * m);  // e_top = 2  <- a1
  }
}

// acc[e] += fwd(x)[e] * fwd(y)[e] for all e in {0,1,2}^N without materialising fwd(x):
// the paper's recursion shape (Algorithm 2) on evaluation points, with the
// inputs left intact.
template <int N, class T>
__device__ __forceinline__ void fwd_mul_acc(const T* x, const T* y, T* acc) {
  if constexpr (N == 0) {
    acc[0] = Ar<T>::mad(x[0], y[0], acc[0]);
  } else {
    constexpr int h = 1 << (N - 1), m = ipow3(N - 1);
    fwd_mul_acc<N - 1, T>(x, y, acc);                   // e_top = 0
    fwd_mul_acc<N - 1, T>(x + h, y + h, acc + 2 * m);   // e_top = 2
    T xs[h], ys[h];
#pragma unroll
    for (int i = 0; i < h; ++i) { xs[i] = Ar<T>::add(x[i], x[i + h]); ys[i] = Ar<T>::add(y[i], y[i + h]); }
    fwd_mul_acc<N - 1, T>(xs, ys, acc + m);             // e_top = 1
  }
}

// acc[k] += sum_{i + j = k} x[i] y[j] over N axes by the paper's direct 4-way split
// (PAPER.md 166-177) on every axis: 4^N fused multiply-adds, no forward adds and no
// inverse.  Index k = sum_b k_b 3^b, i, j = sum_b i_b 2^b; pairs in ascending (i, j).
template <int N, class T>
__device__ __forceinline__ void direct_mul_acc(const T* x, const T* y, T* acc) {
#pragma unroll
  for (int i = 0; i < (1 << N); ++i) {
#pragma unroll
    for (int j = 0; j < (1 << N); ++j) {
      int k = 0, p3 = 1;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        k += (((i >> b) & 1) + ((j >> b) & 1)) * p3;
        p3 *= 3;
      }
      acc[k] = Ar<T>::mad(x[i], y[j], acc[k]);
    }
  }
}

// Register-cube product for the tile's 3 register axes: Karatsuba (PAPER.md 185-192) on the
// top axis, the direct split on the two lower ones.  On an FMA machine a forward add costs
// as much as the multiply it saves, so this mix needs 3 x 16 FMA + 8 adds = 56 operations
// per pair against 65 for Karatsuba on all three axes (and 64 for direct on all three); only
// the top axis then needs the inverse (inv_top3).
template <class T>
__device__ __forceinline__ void kdd_mul_acc(const T* x, const T* y, T* acc) {
  direct_mul_acc<2, T>(x, y, acc);              // e_top = 0: x0 * y0
  direct_mul_acc<2, T>(x + 4, y + 4, acc + 18);  // e_top = 2: x1 * y1
  T xs[4], ys[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { xs[i] = Ar<T>::add(x[i], x[i + 4]); ys[i] = Ar<T>::add(y[i], y[i + 4]); }
  direct_mul_acc<2, T>(xs, ys, acc + 9);         // e_top = 1: (x0 + x1) * (y0 + y1)
}
// inverse on the top register axis only: (c0, c1, c2) -> (c0, (c1 - c0) - c2, c2)
template <class T>
__device__ __forceinline__ void inv_top3(T* a) {
#pragma unroll
  for (int i = 0; i < 9; ++i) a[9 + i] = Ar<T>::sub(Ar<T>::sub(a[9 + i], a[i]), a[18 + i]);
}

// In-place inverse 3^N -> 3^N over all N axes: (c0, c1, c2) -> (c0, (c1 - c0) - c2, c2).
template <int N, int AX, class T>
__device__ __forceinline__ void inv_axis(T* a) {
  constexpr int s = ipow3(AX), nhi = ipow3(N - AX - 1);
#pragma unroll
  for (int hi = 0; hi < nhi; ++hi) {
#pragma unroll
    for (int lo = 0; lo < s; ++lo) {
      const int i = hi * 3 * s + lo;
      a[i + s] = Ar<T>::sub(Ar<T>::sub(a[i + s], a[i]), a[i + 2 * s]);
    }
  }
  if constexpr (AX + 1 < N) inv_axis<N, AX + 1, T>(a);
}
template <int N, class T>
__device__ __forceinline__ void inv_reg(T* a) {
  if constexpr (N > 0) inv_axis<N, 0, T>(a);
}

// exchange with lane ^ 1 (all 32 lanes of the warp must participate)
__device__ __forceinline__ double shfl_xor1(double v) { return __shfl_xor_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ uint64_t shfl_xor1(uint64_t v) {
  return (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)v, 1);
}

// streaming (evict-first) 8-byte global store
__device__ __forceinline__ void st_cs(uint64_t* p, uint64_t v) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cs(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

}  // namespace hc
