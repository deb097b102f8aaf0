// hc_ep.cuh -- kernels of the evaluation-point variant of the multi-GPU split
// (BASELINE.json north_star (4); SURVEY.md §8(e) "K5b"; C ABI in include/hc.h, hc_ep_*).
//
// The top k axes use the paper's Karatsuba split (PAPER.md 185-192) across ranks:
//   ep_eval_kernel   xh[e_T][i_L] = sum_{i_T ~ e_T} x[i_T][i_L]  (forward over the top axes,
//                    (a0, a0 + a1, a1) per axis; subsets in ascending order), all owned e_T
//   (the (D-k)-dimensional convolutions of xh, yh run as ONE batch on the slab / tile engines)
//   ep_top_inverse   z[k_T][col] = inverse over the top axes of w[.][col]
//                    ((c0, (c1 - c0) - c2, c2) per axis, PAPER.md 187-189, 248-251)
#pragma once
#include "hc_tile.cuh"

namespace hc {

// every owned point at once: grid (ceil(2^L / 256), 2 operands, points), point e = e0 +
// blockIdx.z into xh/yh + blockIdx.z * 2^L (trit split of e as in ep_local: digit 2 -> base
// bit, digit 1 -> free bit)
template <class T>
__global__ void __launch_bounds__(256) ep_eval_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                                      T* __restrict__ xh, T* __restrict__ yh, int L, int k,
                                                      uint64_t e0) {
  const uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= (1ull << L)) return;
  uint32_t base = 0, freeb = 0;
  uint32_t t = (uint32_t)(e0 + blockIdx.z);
  for (int a = 0; a < k; ++a, t /= 3) {
    if (t % 3 == 2) base |= 1u << a;
    else if (t % 3 == 1) freeb |= 1u << a;
  }
  const T* src = (blockIdx.y ? y : x) + i;
  T acc = T(0);
  uint32_t s = 0;
  do {
    acc = Ar<T>::add(acc, __ldg(src + ((uint64_t)(base | s) << L)));
    s = (s - freeb) & freeb;
  } while (s != 0);
  (blockIdx.y ? yh : xh)[((uint64_t)blockIdx.z << L) + i] = acc;
}

// one thread per column: load the 3^K evaluation values (coalesced across threads),
// interpolate over the K top axes in registers, store the 3^K outputs
template <class T, int K>
__global__ void __launch_bounds__(128) ep_top_inverse(const T* __restrict__ wt, T* __restrict__ z, uint64_t ncols) {
  const uint64_t col = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (col >= ncols) return;
  constexpr int NP = ipow3(K);
  T v[NP];
#pragma unroll
  for (int e = 0; e < NP; ++e) v[e] = wt[(uint64_t)e * ncols + col];
  inv_reg<K, T>(v);
#pragma unroll
  for (int e = 0; e < NP; ++e) st_cs(z + (uint64_t)e * ncols + col, v[e]);
}

// f3: the same interpolation reading each evaluation point straight from the buffer of the
// rank that owns it (peer memory on a multi-GPU node) -- no gathered copy.  own[e] = owner
// rank of point e, base[e] = (e - e_begin of the owner) * ncols_total, col0 = this rank's
// first column.
struct EPPeer {
  const void* w[8];
  uint8_t own[81];
  uint32_t base[81];
};
template <class T, int K>
__global__ void __launch_bounds__(128) ep_top_inverse_peer(EPPeer pe, T* __restrict__ z, uint64_t ncols,
                                                           uint64_t ncols_total, uint64_t col0) {
  const uint64_t col = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (col >= ncols) return;
  constexpr int NP = ipow3(K);
  T v[NP];
#pragma unroll
  for (int e = 0; e < NP; ++e)
    v[e] = ((const T*)pe.w[pe.own[e]])[(uint64_t)pe.base[e] * ncols_total + col0 + col];
  inv_reg<K, T>(v);
#pragma unroll
  for (int e = 0; e < NP; ++e) st_cs(z + (uint64_t)e * ncols + col, v[e]);
}

}  // namespace hc
