// hc_tile.cuh -- the tile engine: one CTA computes one output slab of 3^L entries.
//
// Scope rows: a1 input staging, a2 forward, a3 product / pair-sum,
// a4 inverse on the tile axes, a6 output store, a7 batched small cubes (k = 0).
//
// Split of the D axes (axis 0 = fastest):
//   low  L = C + B + A axes ("tile"): Karatsuba evaluation/interpolation inside the CTA
//        (PAPER.md 185-192, "only 3 convolutions of dimension D-1");
//   top  k = D - L axes: the paper's direct 4-sub-convolution split (PAPER.md 166-177):
//        output slab t_T receives sum over (i_T, j_T) with i_T + j_T = t_T digit-wise of
//        conv_L(x[i_T], y[j_T]); there are 2^{#1-trits(t_T)} such pairs.  Because the top
//        axes are never interpolated, every slab is final when written (one HBM write).
// Inside the tile the evaluation domain is laid out as
//   C register axes (3^C points per thread, register forward + product + inverse),
//   B axes across threads (stage F1: register forward of 2^B-lines into SMEM),
//   A axes across threads (stage F2: each thread sums the 2^{#1(e_A)} slices of its e_A),
// and the inverse runs registers (C axes) -> SMEM exchange (B axes) -> SMEM exchange +
// coalesced streaming store (A axes).
#pragma once
#include "hc_common.cuh"

namespace hc {

template <class T, int C, int B, int A>
struct TileCfg {
  static constexpr int L = C + B + A;
  static constexpr int NT = ipow3(A + B);          // threads per CTA
  static constexpr int NIN = 1 << L;               // input slice length
  static constexpr int NOUT = ipow3(L);            // output slab length
  static constexpr int NP = (1 << A) * ipow3(B) * (1 << C);  // stage-F1 values per operand
  static constexpr size_t SMEM = sizeof(T) * (size_t)(NOUT > 2 * NIN + 2 * NP ? NOUT : 2 * NIN + 2 * NP);
};

// x, y: base of the batch (row b at b * 2^D), z: output base for work item 0.
// Work item w = blockIdx.x covers batch b = w / nslab, top index t_T = slab0 + w % nslab,
// and writes z[w * 3^L .. (w+1) * 3^L).
template <class T, int C, int B, int A>
__global__ void __launch_bounds__(TileCfg<T, C, B, A>::NT)
tile_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ z, int D,
            uint64_t slab0, uint64_t nslab) {
  using Cfg = TileCfg<T, C, B, A>;
  constexpr int NT = Cfg::NT, L = Cfg::L, NIN = Cfg::NIN;
  constexpr int P3B = ipow3(B), P3C = ipow3(C), P2A = 1 << A, P2C = 1 << C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* xs = sm;                 // [NIN]
  T* ys = sm + NIN;           // [NIN]
  T* px = sm + 2 * NIN;       // [P2C][P2A][P3B]  stage-F1 output, e_B fastest
  T* py = px + Cfg::NP;
  T* S = sm;                  // [3^A][3^B][3^C] after the pair loop (aliases the above)

  const int tid = threadIdx.x;
  const uint64_t w = blockIdx.x;
  const uint64_t b = w / nslab;
  uint64_t tT = slab0 + (w - b * nslab);
  const int k = D - L;

  // digits of t_T: base = bits with trit 2, freeb = bits with trit 1 (PAPER.md 166-171)
  uint32_t base = 0, freeb = 0;
  for (int a = 0; a < k; ++a) {
    const uint32_t d = (uint32_t)(tT % 3u);
    tT /= 3u;
    if (d == 2u) base |= 1u << a;
    else if (d == 1u) freeb |= 1u << a;
  }
  const T* xb = x + (b << D);
  const T* yb = y + (b << D);

  // this thread's evaluation coordinates on the A and B axes
  const int eB = tid % P3B, eA = tid / P3B;
  uint32_t baseA = 0, freeA = 0;
  {
    int t = eA;
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int d = t % 3;
      t /= 3;
      if (d == 2) baseA |= 1u << a;
      else if (d == 1) freeA |= 1u << a;
    }
  }

  T acc[ipow3(C)];
#pragma unroll
  for (int i = 0; i < P3C; ++i) acc[i] = T(0);

  // pair loop over subsets s of freeb in ascending order: i_T = base|s, j_T = base|(freeb&~s)
  uint32_t s = 0;
  do {
    const uint32_t iT = base | s, jT = base | (freeb & ~s);
    const T* xsrc = xb + ((uint64_t)iT << L);
    const T* ysrc = yb + ((uint64_t)jT << L);
    __syncthreads();
    for (int i = tid; i < NIN; i += NT) { xs[i] = xsrc[i]; ys[i] = ysrc[i]; }
    __syncthreads();
    const T* fx = xs;
    const T* fy = ys;
    if constexpr (B > 0) {
      // F1: every (operand, b_A, b_lo) line of 2^B values -> 3^B evaluations
      for (int wl = tid; wl < 2 * P2A * P2C; wl += NT) {
        const int op = wl / (P2A * P2C);
        const int r = wl - op * (P2A * P2C);
        const int bA = r / P2C, blo = r - bA * P2C;
        const T* src = op ? ys : xs;
        T* dst = op ? py : px;
        T in[1 << B], out[ipow3(B)];
#pragma unroll
        for (int j = 0; j < (1 << B); ++j) in[j] = src[blo + P2C * j + (P2C << B) * bA];
        fwd_reg<B, T>(in, out);
#pragma unroll
        for (int e = 0; e < P3B; ++e) dst[(blo * P2A + bA) * P3B + e] = out[e];
      }
      __syncthreads();
      fx = px;
      fy = py;
    }
    // F2: thread (e_A, e_B) sums the slices consistent with e_A -> 2^C values per operand
    T xt[1 << C], yt[1 << C];
#pragma unroll
    for (int j = 0; j < P2C; ++j) { xt[j] = T(0); yt[j] = T(0); }
    uint32_t sa = 0;
    do {
      const int bA = (int)(baseA | sa);
#pragma unroll
      for (int j = 0; j < P2C; ++j) {
        const int idx = (j * P2A + bA) * P3B + eB;
        xt[j] = Ar<T>::add(xt[j], fx[idx]);
        yt[j] = Ar<T>::add(yt[j], fy[idx]);
      }
      sa = (sa - freeA) & freeA;
    } while (sa != 0);
    // register forward over the C axes fused with the pointwise product (a2 + a3)
    fwd_mul_acc<C, T>(xt, yt, acc);
    s = (s - freeb) & freeb;
  } while (s != 0);

  // a4: inverse on the C register axes
  inv_reg<C, T>(acc);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < P3C; ++i) S[tid * P3C + i] = acc[i];
  __syncthreads();
  // inverse on the B axes: lines over e_B for fixed (e_A, t_lo)
  if constexpr (B > 0) {
    for (int wl = tid; wl < ipow3(A) * P3C; wl += NT) {
      const int a = wl / P3C, tl = wl - a * P3C;
      T v[ipow3(B)];
#pragma unroll
      for (int e = 0; e < P3B; ++e) v[e] = S[(a * P3B + e) * P3C + tl];
      inv_reg<B, T>(v);
#pragma unroll
      for (int e = 0; e < P3B; ++e) S[(a * P3B + e) * P3C + tl] = v[e];
    }
    __syncthreads();
  }
  // inverse on the A axes, then coalesced streaming store of the final slab (a6)
  T* zo = z + w * (uint64_t)Cfg::NOUT;
  constexpr int ROW = ipow3(B + C);
  for (int wl = tid; wl < ROW; wl += NT) {
    T v[ipow3(A)];
#pragma unroll
    for (int e = 0; e < ipow3(A); ++e) v[e] = S[e * ROW + wl];
    inv_reg<A, T>(v);
#pragma unroll
    for (int e = 0; e < ipow3(A); ++e) st_cs(zo + e * ROW + wl, v[e]);
  }
}

}  // namespace hc
