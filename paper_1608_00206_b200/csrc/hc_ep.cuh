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
  HC_ASSERT(t < upow3(k));
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

constexpr int EP_MAX_K = 5;
constexpr int EP_MAX_NP = 243;  // 3^EP_MAX_K
// owners of the evaluation points for the peer-read finish (see ep_top_inverse_peer)
struct EPPeer {
  const void* w[8];
  uint8_t own[EP_MAX_NP];
  uint32_t base[EP_MAX_NP];
};

// K = 5 (243 points: the point split over 8 ranks is 31 : 30.4 instead of 11 : 10.1 at K = 4):
// a column's 243 values do not fit in registers, so a CTA stages EP5_CW columns x 243 points
// in shared memory, interpolates axis by axis there ((c0, (c1 - c0) - c2, c2), PAPER.md
// 187-189), and stores; loads and stores are row segments of EP5_CW elements.  PEER: the
// values of point e come straight from the owner rank's w (f3), as in ep_top_inverse_peer.
#ifndef HC_EP5_CW
#define HC_EP5_CW 16
#endif
constexpr int EP5_CW = HC_EP5_CW;  // columns per CTA (16: 128-byte row segments, 31 KB, 7 CTAs per SM)
constexpr size_t EP5_SMEM = 8ull * EP_MAX_NP * EP5_CW;
template <class T, bool PEER>
__global__ void __launch_bounds__(256) ep_top_inverse5(const T* __restrict__ wt, EPPeer pe, T* __restrict__ z,
                                                       uint64_t ncols, uint64_t ncols_total, uint64_t col0) {
  extern __shared__ __align__(16) unsigned char ep5_raw[];
  T* s = reinterpret_cast<T*>(ep5_raw);  // [243][EP5_CW]
  static_assert(256 % EP5_CW == 0, "row groups");
  constexpr int RG = 256 / EP5_CW, RPT = (EP_MAX_NP + RG - 1) / RG;  // rows per thread
  const uint64_t c0 = (uint64_t)blockIdx.x * EP5_CW;
  const int nc = (int)((ncols - c0) < (uint64_t)EP5_CW ? (ncols - c0) : (uint64_t)EP5_CW);
  const int c = threadIdx.x % EP5_CW, r0 = threadIdx.x / EP5_CW;
  {
    T v[RPT];  // all of the thread's loads in flight before the first shared store
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int e = r0 + RG * j;
      if (e < EP_MAX_NP && c < nc) {
        if constexpr (PEER)
          v[j] = ((const T*)pe.w[pe.own[e]])[(uint64_t)pe.base[e] * ncols_total + col0 + c0 + c];
        else
          v[j] = wt[(uint64_t)e * ncols + c0 + c];
      }
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int e = r0 + RG * j;
      if (e < EP_MAX_NP && c < nc) s[e * EP5_CW + c] = v[j];
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int a = 0, st = 1; a < 5; ++a, st *= 3) {
    for (int g = r0; g < 81; g += RG) {
      const int lo = g % st, hi = g / st;
      const int b = hi * 3 * st + lo;
      const T v0 = s[b * EP5_CW + c], v1 = s[(b + st) * EP5_CW + c], v2 = s[(b + 2 * st) * EP5_CW + c];
      s[(b + st) * EP5_CW + c] = Ar<T>::sub(Ar<T>::sub(v1, v0), v2);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int e = r0 + RG * j;
    if (e < EP_MAX_NP && c < nc) st_cs(z + (uint64_t)e * ncols + c0 + c, s[e * EP5_CW + c]);
  }
}
// f3: the same interpolation reading each evaluation point straight from the buffer of the
// rank that owns it (peer memory on a multi-GPU node) -- no gathered copy.  own[e] = owner
// rank of point e, base[e] = (e - e_begin of the owner) * ncols_total, col0 = this rank's
// first column.
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
