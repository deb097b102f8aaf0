// hc_common.cuh -- device helpers for the hypercube-convolution kernels (sm_100a).
//
// Notation follows PAPER.md "Methods" (lines 153-212): for one axis, a pair of input
// values (a0, a1) is evaluated at {0, 1, inf} as (a0, a0 + a1, a1) (the paper's
// x[0] + x[1], lines 186-189), the three evaluations are multiplied pointwise, and the
// result (c0, c1, c2) is interpolated back as (c0, (c1 - c0) - c2, c2) (t - z[0] - z[2],
// lines 187-189; subtraction order of Algorithm 2's two loops, lines 248-251).
//
// Element arithmetic: uint64 (int64 as wrap-around, exact mod 2^64), uint32 (mod 2^32) or double.
// This file shares nothing with oracle/ (test infrastructure).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

// Bounds-checked development build (-DHC_CHECK, tools/build_variant.sh check -DHC_CHECK): logical
// index invariants of every engine are asserted on the device (compute-sanitizer is not
// available on this pool); the default build compiles them out.
#ifdef HC_CHECK
#include <cstdio>
#define HC_ASSERT(c)                                                                                   \
  do {                                                                                                 \
    if (!(c)) {                                                                                        \
      printf("HC_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                        \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define HC_ASSERT(c) \
  do {               \
  } while (0)
#endif

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
// the 32-bit ring (hc_tile8n.cuh: exact residues of int64 results that fit in 32 bits)
template <> struct Ar<uint32_t> {
  static __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) { return a + b; }
  static __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) { return a - b; }
  static __device__ __forceinline__ uint32_t mad(uint32_t a, uint32_t b, uint32_t c) { return c + a * b; }
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

// fwd_reg with each output stored as soon as it is formed (dst[e * stride]): the evaluation
// tree is walked depth first, so at most N partial sums per level are live instead of all
// 3^N outputs (register pressure of the callers that also hold accumulators)
template <int N, int STRIDE, class T>
__device__ __forceinline__ void fwd_store(const T* in, T* dst) {
  if constexpr (N == 0) {
    dst[0] = in[0];
  } else {
    constexpr int h = 1 << (N - 1), m = ipow3(N - 1);
    fwd_store<N - 1, STRIDE, T>(in, dst);                  // e_top = 0  <- a0
    T s[h];
#pragma unroll
    for (int i = 0; i < h; ++i) s[i] = Ar<T>::add(in[i], in[i + h]);
    fwd_store<N - 1, STRIDE, T>(s, dst + m * STRIDE);      // e_top = 1  <- a0 + a1
    fwd_store<N - 1, STRIDE, T>(in + h, dst + 2 * m * STRIDE);  // e_top = 2  <- a1
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
