// hc_tile.cuh -- tile engine and the two-level slab engine.
//
// Scope rows: a1 input staging, a2 forward, a3 product / pair-sum,
// a4 inverse on the tile axes, a5 inverse on the middle axes, a6 output store,
// a7 batched small cubes.
//
// Axis split (axis 0 = fastest):
//   tile   L = C + B + A low axes: Karatsuba evaluation / interpolation inside one CTA
//          (PAPER.md 185-192).  C axes live in registers (3^C points per thread), B and A
//          axes across the 3^(A+B) threads.
//   middle M axes (two-level engine only): Karatsuba with the evaluation point e_U fixed
//          per pass-1 work item; the interpolation over them (pass 2) runs on the slab
//          while it is still resident in L2 (design "D3").
//   top    k axes: the paper's direct 4-sub-convolution split (PAPER.md 166-177): output
//          slab t_T is the sum over the 2^{#1-trits(t_T)} pairs (i_T, j_T), i_T + j_T = t_T,
//          so slabs are independent and final once interpolated.
#pragma once
#include "hc_common.cuh"

namespace hc {

template <class T, int C, int B, int A>
struct TileCfg {
  static constexpr int L = C + B + A;
  static constexpr int NT = ipow3(A + B);          // threads per CTA
  static constexpr int NIN = 1 << L;               // input slice length
  static constexpr int NOUT = ipow3(L);            // output tile length
  static constexpr int NP = (1 << A) * ipow3(B) * (1 << C);  // stage-F1 values per operand
  // the tile buffer S (3^L) aliases the double-buffered stage-F1 output (2 x 2 operands x NP)
  static constexpr size_t SMEM = sizeof(T) * (size_t)(NOUT > 4 * NP ? NOUT : 4 * NP);
};

// digits of a base-3 index (n digits): bits with trit 2 -> base, trit 1 -> freeb
__device__ __forceinline__ void trit_split(uint64_t t, int n, uint32_t& base, uint32_t& freeb) {
  base = 0;
  freeb = 0;
  for (int a = 0; a < n; ++a) {
    const uint32_t d = (uint32_t)(t % 3u);
    t /= 3u;
    if (d == 2u) base |= 1u << a;
    else if (d == 1u) freeb |= 1u << a;
  }
}

// Stage F1 for one pair, fused with the middle-axes gather (a1 + a2): every
// (operand, b_A, b_lo) line sums its 2^B inputs over the 2^{#1(e_U)} middle-axis slices
// consistent with e_U (forward over the middle axes), evaluates them over the B axes in
// registers and stores the 3^B values to P[op][b_A][b_lo][e_B].  Lanes take consecutive
// b_lo, so global loads are unit-stride and SMEM stores (stride 3^B, odd) conflict-free.
template <class T, int C, int B, int A>
__device__ __forceinline__ void p1_stage(const T* __restrict__ xb, const T* __restrict__ yb,
                                         const uint32_t* s_off, int nsl, T* P) {
  using Cfg = TileCfg<T, C, B, A>;
  constexpr int P3B = ipow3(B), P2A = 1 << A, P2C = 1 << C, NLINE = P2A * P2C;
  constexpr int NB = 1 << B;
  // Two lanes per line when the line threads fill whole warps in one pass (L = 7, 8):
  // lanes 2w and 2w+1 share line w, each gathers half of the 2^B inputs, then they swap.
  // Otherwise (small tiles) one thread per line.
  constexpr bool TWO = (4 * NLINE) % 32 == 0 && 4 * NLINE <= Cfg::NT;
  constexpr int HB = TWO ? NB / 2 : NB;
  for (int t = threadIdx.x; t < (TWO ? 4 : 2) * NLINE; t += Cfg::NT) {
    const int wl = TWO ? (t >> 1) : t, half = TWO ? (t & 1) : 0;
    const int op = wl / NLINE, r = wl - op * NLINE;
    const int bA = r / P2C, blo = r - bA * P2C;
    const T* src = (op ? yb : xb) + blo + (P2C << B) * bA + P2C * HB * half;
    T in[HB];
#pragma unroll
    for (int j = 0; j < HB; ++j) in[j] = T(0);
    // nsl is a power of two; take slices four at a time so 4 * 2^(B-1) loads are in flight
    if (nsl >= 4) {
      for (int q = 0; q < nsl; q += 4) {
        T v[4][HB];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const T* sp = src + s_off[q + u];
#pragma unroll
          for (int j = 0; j < HB; ++j) v[u][j] = __ldg(sp + P2C * j);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < HB; ++j) in[j] = Ar<T>::add(in[j], v[u][j]);
      }
    } else {
      T v[2][HB];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const T* sp = src + s_off[u < nsl ? u : 0];
#pragma unroll
        for (int j = 0; j < HB; ++j) v[u][j] = (u < nsl) ? __ldg(sp + P2C * j) : T(0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int j = 0; j < HB; ++j) in[j] = Ar<T>::add(in[j], v[u][j]);
    }
    T full[NB];
    if constexpr (TWO) {
#pragma unroll
      for (int j = 0; j < HB; ++j) {
        const T o = shfl_xor1(in[j]);
        full[j] = half ? o : in[j];
        full[j + HB] = half ? in[j] : o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < NB; ++j) full[j] = in[j];
    }
    T out[ipow3(B)];
    fwd_reg<B, T>(full, out);
    T* dst = P + op * Cfg::NP + r * P3B;
#pragma unroll
    for (int e = 0; e < P3B; ++e)
      if (!TWO || (e & 1) == half) dst[e] = out[e];
  }
}

// One pass-1 tile: acc over the pairs of top index tT, evaluation point eU of the M middle
// axes (M = 0: single-level), low-axes interpolation, store of the 3^L tile to zt.
//   x, y : batch base (row of 2^D elements); slice (i_T, b_U) starts at (i_T << M | b_U) << L
//   FINAL: streaming store (.cs) when the tile is final output, write-back store otherwise
// The pair loop is software-pipelined: stage F1 of pair p+1 (global loads) is issued
// before the F2 + product of pair p, into a double-buffered P, with one barrier per pair.
template <class T, int C, int B, int A, bool FINAL>
__device__ __forceinline__ void p1_tile(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ zt,
                                        int k, int M, uint64_t tT, uint32_t eU, T* sm) {
  using Cfg = TileCfg<T, C, B, A>;
  constexpr int NT = Cfg::NT, L = Cfg::L, NP = Cfg::NP;
  constexpr int P3B = ipow3(B), P3C = ipow3(C), P2C = 1 << C;
  static_assert(B > 0, "p1_tile needs B > 0");
  T* S = sm;                  // [3^A][3^B][3^C] after the pair loop (aliases the stages)
  const int tid = threadIdx.x;
  __shared__ uint32_t s_off[64];

  uint32_t base, freeb, baseU, freeU;
  trit_split(tT, k, base, freeb);
  trit_split(eU, M, baseU, freeU);
  const int nsl = 1 << __popc(freeU);
  __syncthreads();  // previous user of sm / s_off is done
  for (int q = tid; q < nsl; q += NT) {
    uint32_t sub = 0, rem = freeU;
    for (int bit = 0; rem; ++bit) {
      const uint32_t low = rem & (0u - rem);
      if ((q >> bit) & 1) sub |= low;
      rem ^= low;
    }
    s_off[q] = (baseU | sub) << L;
  }

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

  // pairs: subsets s of freeb in ascending order, i_T = base|s, j_T = base|(freeb&~s)
  const int shift = M + L;
  __syncthreads();  // s_off ready
  uint32_t s = 0;
  p1_stage<T, C, B, A>(x + ((uint64_t)base << shift), y + ((uint64_t)(base | freeb) << shift), s_off, nsl, sm);
  __syncthreads();
  int buf = 0;
  while (true) {
    const uint32_t sn = (s - freeb) & freeb;  // next subset
    if (sn != 0) {
      const uint64_t iT = base | sn, jT = base | (freeb & ~sn);
      p1_stage<T, C, B, A>(x + (iT << shift), y + (jT << shift), s_off, nsl, sm + (buf ^ 1) * 2 * NP);
    }
    // F2: thread (e_A, e_B) sums the lines consistent with e_A -> 2^C values per operand
    const T* fx = sm + buf * 2 * NP;
    const T* fy = fx + NP;
    T xt[1 << C], yt[1 << C];
#pragma unroll
    for (int j = 0; j < P2C; ++j) { xt[j] = T(0); yt[j] = T(0); }
    uint32_t sa = 0;
    do {
      const int bA = (int)(baseA | sa);
#pragma unroll
      for (int j = 0; j < P2C; ++j) {
        const int idx = (bA * P2C + j) * P3B + eB;
        xt[j] = Ar<T>::add(xt[j], fx[idx]);
        yt[j] = Ar<T>::add(yt[j], fy[idx]);
      }
      sa = (sa - freeA) & freeA;
    } while (sa != 0);
    // register forward over the C axes fused with the pointwise product (a2 + a3)
    fwd_mul_acc<C, T>(xt, yt, acc);
    __syncthreads();
    if (sn == 0) break;
    s = sn;
    buf ^= 1;
  }

  // a4: inverse on the C register axes
  inv_reg<C, T>(acc);
#pragma unroll
  for (int i = 0; i < P3C; ++i) S[tid * P3C + i] = acc[i];
  __syncthreads();
  // inverse on the B axes: lines over e_B for fixed (e_A, t_lo)
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
  // inverse on the A axes, then coalesced store of the tile (a6)
  constexpr int ROW = ipow3(B + C);
  for (int wl = tid; wl < ROW; wl += NT) {
    T v[ipow3(A)];
#pragma unroll
    for (int e = 0; e < ipow3(A); ++e) v[e] = S[e * ROW + wl];
    inv_reg<A, T>(v);
#pragma unroll
    for (int e = 0; e < ipow3(A); ++e) {
      if constexpr (FINAL) st_cs(zt + e * ROW + wl, v[e]);
      else zt[e * ROW + wl] = v[e];
    }
  }
}

// Single-level tile kernel (D <= 7, and batched D <= 7): work item w covers batch
// b = w / nslab, top index t_T = slab0 + w % nslab, and writes z[w * 3^L ...].
template <class T, int C, int B, int A>
__global__ void __launch_bounds__(TileCfg<T, C, B, A>::NT)
tile_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ z, int D,
            uint64_t slab0, uint64_t nslab, uint64_t w0) {
  using Cfg = TileCfg<T, C, B, A>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const uint64_t w = w0 + blockIdx.x;  // item index (launches of > 2^31 - 1 items are chunked)
  const uint64_t b = w / nslab;
  const uint64_t tT = slab0 + (w - b * nslab);
  p1_tile<T, C, B, A, true>(x + (b << D), y + (b << D), z + w * (uint64_t)Cfg::NOUT, D - Cfg::L, 0, tT, 0u, sm);
}

// ---- two-level slab engine ------------------------------------------------------------
// Slab = all outputs of one top index t_T: 3^(M+L) entries.  Pass-1 items (t_T, e_U) write
// the 3^L tile at position e_U of the slab in the evaluation domain of the M middle axes;
// pass-2 items (t_T, chunk of P2W low positions) read the 3^M column, interpolate over the
// middle axes and overwrite it with the final output.  One persistent kernel runs both
// kinds from a single work counter in the order P1(0) P1(1) P2(0) P1(2) P2(1) ... so the
// slab being interpolated was written moments earlier and is still in L2.  A pass-2 item
// waits (acquire) on its slab's pass-1 completion counter; every pass-1 item it waits for
// was claimed earlier by a running CTA and never waits itself, so the schedule cannot
// deadlock as long as the grid is co-resident (grid <= SMs x occupancy).
constexpr int P2W = 9;  // low positions per pass-2 item (3^8 = 729 * 9)

struct SlabArgs {
  uint64_t slab0;      // first top index of this launch (sharding)
  uint32_t nslab;      // slabs in this launch
  int k;               // top axes
  uint32_t* ctr;       // [0] = work counter, [1 + j] = pass-1 tiles done in slab j
  const uint4* order;  // processing position j -> {slab offset within the launch, base, freeb, problem b}:
                       // cost-sorted, with the trit split of the slab's top index precomputed; b > 0
                       // only for a batch of same-D problems (hc_ep_local), whose slabs are numbered
                       // b * 3^k + t_T and whose middle-axes tables lie bstride elements apart
  int debug_skip;      // timing experiments only (HC_DEBUG_SKIP): 1 = no pass 2, 2 = no pass 1
  uint32_t lag;        // pass 2 of slab j is scheduled after pass 1 of slab j + lag (>= 1)
  unsigned long long* cout;  // slab8_kernel<uint64_t, M, 2>: carry bins (f1), else unused
  void* ring;                // slab8_kernel<uint64_t, M, 2>: T8_RING slab buffers for pass-1 tiles
  int keep_policy;           // L2 policy of the pass-1 tile stores (0 evict_last, 1 evict_normal, 2 unchanged)
  int p2_prefetch;           // pass-2 items bulk-prefetch their columns into L2 (0 / 1)
  uint32_t p2_head;          // decode_item: pass-1 items before the interleave (0xffffffff: none)
  uint64_t bstride;          // elements between consecutive problems' middle-axes tables (batch)
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <class T> __device__ __forceinline__ T ld_cg(const T* p);
template <> __device__ __forceinline__ double ld_cg<double>(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ uint64_t ld_cg<uint64_t>(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// pass-2 item: columns [c*P2W, c*P2W + P2W) of slab zs (3^M rows of 3^L).  SMEM buffer
// layout: (e_hi, e_lo, pos) at e_hi * P2S + e_lo * P2W + pos with P2S = 9 (mod 16), so the
// round-1 stores (lanes = (e_hi, pos)) and round-2 loads (lanes = (e_lo, pos)) are both
// free of bank conflicts.
template <int M>
struct P2Cfg {
  static constexpr int LO = M < 3 ? M : 3, HI = M - LO;
  static constexpr int NLO = ipow3(LO), NHI = ipow3(HI);
  static constexpr int P2S = NLO * P2W + ((9 - NLO * P2W) % 16 + 16) % 16;
  static constexpr int SIZE = NHI * P2S;
};
template <class T, int M, int L, class Mid, class Bar>
__device__ __forceinline__ void p2_item(T* __restrict__ zs, uint32_t c, T* sm, int task, int sched, Mid&& mid,
                                        Bar&& bar) {
  // task in [0, 243) or -1 (idle lane); 243 = 3^5 task slots per round
  using Q = P2Cfg<M>;
  constexpr int LO = Q::LO, HI = Q::HI, NLO = Q::NLO, NHI = Q::NHI, P2S = Q::P2S;
  constexpr uint64_t ROW = upow3(L);
  const uint64_t col0 = (uint64_t)c * P2W;
  HC_ASSERT(col0 + P2W <= ROW && task < 243);
  // round 1: task (e_hi, pos) loads its 3^LO column entries, interpolates over LO axes
  if (task >= 0)
    for (int w = task; w < NHI * P2W; w += 243) {
      const int eh = w / P2W, pos = w - eh * P2W;
      T v[NLO];
#pragma unroll
      for (int e = 0; e < NLO; ++e) v[e] = ld_cg(zs + (uint64_t)(eh * NLO + e) * ROW + col0 + pos);
      inv_reg<LO, T>(v);
#pragma unroll
      for (int e = 0; e < NLO; ++e) sm[eh * P2S + e * P2W + pos] = v[e];
    }
  bar();
  if ((int)threadIdx.x == sched) mid();  // between the loads and the stores (see slab8_kernel)
  // round 2: task (e_lo, pos) interpolates over HI axes and stores the final values
  if (task >= 0)
    for (int w = task; w < NLO * P2W; w += 243) {
      const int el = w / P2W, pos = w - el * P2W;
      T v[NHI];
#pragma unroll
      for (int e = 0; e < NHI; ++e) v[e] = sm[e * P2S + el * P2W + pos];
      inv_reg<HI, T>(v);
#pragma unroll
      for (int e = 0; e < NHI; ++e) st_cs(zs + (uint64_t)(e * NLO + el) * ROW + col0 + pos, v[e]);
    }
}

}  // namespace hc
