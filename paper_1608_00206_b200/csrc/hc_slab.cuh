// hc_slab.cuh -- the 8-axis tile (all D >= 8) and the two-level slab engine (D >= 13).
//
// a1 input staging, a2 forward, a3 product / pair-sum, a4 inverse on
// the tile axes, a5 inverse on the middle axes, a6 store, a7 batched small cubes.
// Arithmetic: the paper's per-axis split (PAPER.md 185-192) -- forward (a0, a0+a1, a1),
// pointwise product, inverse (c0, (c1-c0)-c2, c2) -- on the 8 tile axes and the M middle
// axes; the paper's 4-way split (PAPER.md 166-177) on the k top axes (pair-sum).
//
// Tile (3^8 = 6561 outputs, 243 threads = (e_A in 3^2) x (e_B in 3^3), 27 accumulators per
// thread over the C = 3 register axes).  Per top pair (i_T, j_T):
//   * the raw input slices (256 values of x and of y; for the two-level engine already
//     evaluated over the middle axes by prep_kernel) are prefetched two pairs ahead with
//     cp.async into a 3-deep SMEM ring (no registers held, latency hidden);
//   * 144 "line" threads (operand, e_A, b_lo) evaluate the A axes (sum of the rows
//     consistent with e_A) and the B axes (8 -> 27 in registers) and write the stage P;
//   * every thread loads its 8 + 8 base values from P and evaluates the C axes fused with
//     the product into its accumulators (fwd_mul_acc).
// Then the tile is interpolated (registers -> SMEM -> SMEM) and stored.
#pragma once
#include "hc_tile.cuh"

namespace hc {

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// TMA 1-D bulk copy global -> shared, completion on an mbarrier (complete_tx), L2 policy
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

constexpr int T8_NT = 243;        // threads per tile CTA
constexpr int T8_NLINE = 72;      // F1 lines per operand: (e_A in 9) x (b_lo in 8)
constexpr int T8_PSZ = 2 * T8_NLINE * 27;   // one stage: both operands, 27 values per line
constexpr int T8_RAW = 512;       // one raw stage: x slice + y slice
constexpr int T8_NRAW = 3;        // raw prefetch depth
template <class T>
struct T8Cfg {
  static constexpr size_t SMEM = sizeof(T) * (size_t)(2 * T8_PSZ + T8_NRAW * T8_RAW);
  static_assert(2 * T8_PSZ >= 6561, "tile exchange buffer aliases the two stages");
  static_assert(2 * T8_PSZ >= P2Cfg<6>::SIZE, "pass-2 buffer aliases the two stages");
};

// Prep kernel (two-level only): evaluate the M middle axes of every input slice once per
// call, X_U[i_T][e_U][b_L] = sum_{b_U ~ e_U} x[i_T][b_U][b_L] (the forward transform over
// the middle axes; subsets in ascending order).  grid = (3^M, 2^k, 2 operands), block 256.
template <class T, int M>
__global__ void __launch_bounds__(256) prep_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                                   T* __restrict__ xu, T* __restrict__ yu) {
  const uint32_t eU = blockIdx.x;
  const uint64_t iT = blockIdx.y;
  const T* src = (blockIdx.z ? y : x) + (iT << (M + 8)) + threadIdx.x;
  T* dst = (blockIdx.z ? yu : xu) + (iT * upow3(M) + eU) * 256 + threadIdx.x;
  uint32_t baseU, freeU;
  trit_split(eU, M, baseU, freeU);
  T acc = T(0);
  uint32_t s = 0;
  do {
    acc = Ar<T>::add(acc, __ldg(src + ((uint64_t)(baseU | s) << 8)));
    s = (s - freeU) & freeU;
  } while (s != 0);
  *dst = acc;
}

// raw-slice staging: T8_NRAW stages, each filled by two TMA bulk copies (x slice, y slice)
// and completed on its mbarrier.  seq counts fills over the CTA's lifetime (same value in
// every thread) so the parity of each stage's barrier is known.
struct RawRing {
  uint64_t* bar;     // [T8_NRAW] in shared memory
  uint32_t seq;      // fills issued so far
  uint32_t done;     // fills consumed so far
};
template <class T>
__device__ __forceinline__ void t8_issue(RawRing& rr, const T* sx, const T* sy, T* R, uint64_t pol) {
  const uint32_t st = rr.seq % T8_NRAW;
  if (threadIdx.x == 0) {
    mbar_arrive_tx(&rr.bar[st], 2 * 256 * sizeof(T));
    tma_load_1d(R + st * T8_RAW, sx, 256 * sizeof(T), &rr.bar[st], pol);
    tma_load_1d(R + st * T8_RAW + 256, sy, 256 * sizeof(T), &rr.bar[st], pol);
  }
  ++rr.seq;
}
__device__ __forceinline__ uint32_t t8_wait(RawRing& rr) {
  const uint32_t st = rr.done % T8_NRAW;
  mbar_wait(&rr.bar[st], (rr.done / T8_NRAW) & 1);
  ++rr.done;
  return st;
}

// stage F1 of one pair: raw slices R -> P (line threads tid < 144)
template <class T>
__device__ __forceinline__ void t8_f1(const T* R, T* P, int tid, uint32_t lbase, uint32_t lfree) {
  if (tid >= 2 * T8_NLINE) return;
  const int op = tid / T8_NLINE, rr = tid - op * T8_NLINE;
  const int blo = rr & 7;
  const T* src = R + op * 256 + blo;
  T in[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) in[j] = T(0);
  uint32_t sa = 0;
  do {  // forward over the A axes: rows b_A consistent with e_A
    const T* row = src + (lbase | sa) * 64;
#pragma unroll
    for (int j = 0; j < 8; ++j) in[j] = Ar<T>::add(in[j], row[8 * j]);
    sa = (sa - lfree) & lfree;
  } while (sa != 0);
  T out[27];
  fwd_reg<3, T>(in, out);  // forward over the B axes
  T* dst = P + op * (T8_NLINE * 27) + rr * 27;
#pragma unroll
  for (int e = 0; e < 27; ++e) dst[e] = out[e];
}

// One pass-1 tile.  sx0/sy0 + iT*stride are the raw x / y slices of pair (iT, jT).
template <class T, bool FINAL>
__device__ __forceinline__ void tile8(const T* __restrict__ sx0, const T* __restrict__ sy0, uint64_t stride,
                                      T* __restrict__ zt, int k, uint64_t tT, T* sm, RawRing& rr,
                                      uint64_t pol_in, uint64_t pol_out) {
  T* P = sm;                          // [2][T8_PSZ]
  T* R = sm + 2 * T8_PSZ;             // [T8_NRAW][T8_RAW]
  T* S = sm;                          // [9][27][27] after the pair loop (aliases P)
  const int tid = threadIdx.x;
  const int eA = tid / 27, eB = tid - eA * 27;

  // this thread's F1 line (tid < 144): e_A of the line -> rows consistent with it
  uint32_t lbase = 0, lfree = 0;
  {
    int t = (tid % T8_NLINE) >> 3;
#pragma unroll
    for (int aa = 0; aa < 2; ++aa) {
      const int d = t % 3;
      t /= 3;
      if (d == 2) lbase |= 1u << aa;
      else if (d == 1) lfree |= 1u << aa;
    }
  }
  uint32_t base, freeb;
  trit_split(tT, k, base, freeb);
  const int npairs = 1 << __popc(freeb);

  // pair p: s_p = p-th subset of freeb (ascending), i_T = base|s_p, j_T = base|(freeb & ~s_p)
  uint32_t s_pf = 0;  // subset of the next pair to prefetch
  int npf = 0;        // pairs prefetched so far
  auto prefetch_next = [&]() {
    if (npf < npairs) {
      const uint64_t iT = base | s_pf, jT = base | (freeb & ~s_pf);
      t8_issue<T>(rr, sx0 + iT * stride, sy0 + jT * stride, R, pol_in);
      s_pf = (s_pf - freeb) & freeb;
      ++npf;
    }
  };

  __syncthreads();      // previous users of sm (and of the raw stages) are done
  prefetch_next();      // pair 0
  prefetch_next();      // pair 1
  t8_f1<T>(R + t8_wait(rr) * T8_RAW, P, tid, lbase, lfree);
  __syncthreads();

  T acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = T(0);
  for (int p = 0; p < npairs; ++p) {
    prefetch_next();  // pair p + 2 (its stage was last read by F1(p - 1), before a barrier)
    {
      // base values of (e_A, e_B): one line per b_lo, then C-axes forward fused with product
      const T* fx = P + (p & 1) * T8_PSZ;
      const T* fy = fx + T8_NLINE * 27;
      T xt[8], yt[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int idx = (eA * 8 + j) * 27 + eB;
        xt[j] = fx[idx];
        yt[j] = fy[idx];
      }
      fwd_mul_acc<3, T>(xt, yt, acc);
    }
    if (p + 1 < npairs) t8_f1<T>(R + t8_wait(rr) * T8_RAW, P + ((p + 1) & 1) * T8_PSZ, tid, lbase, lfree);
    __syncthreads();
  }

  // a4: inverse on the C register axes, then B (SMEM exchange), then A + store (a6)
  inv_reg<3, T>(acc);
#pragma unroll
  for (int i = 0; i < 27; ++i) S[tid * 27 + i] = acc[i];
  __syncthreads();
  {
    const int aa = tid / 27, tl = tid - aa * 27;
    T v[27];
#pragma unroll
    for (int e = 0; e < 27; ++e) v[e] = S[(aa * 27 + e) * 27 + tl];
    inv_reg<3, T>(v);
#pragma unroll
    for (int e = 0; e < 27; ++e) S[(aa * 27 + e) * 27 + tl] = v[e];
  }
  __syncthreads();
  for (int w = tid; w < 729; w += T8_NT) {
    T v[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) v[e] = S[e * 729 + w];
    inv_reg<2, T>(v);
#pragma unroll
    for (int e = 0; e < 9; ++e) {
      if constexpr (FINAL) st_cs(zt + e * 729 + w, v[e]);
      else st_hint(zt + e * 729 + w, v[e], pol_out);
    }
  }
}

// Single-level kernel for 8-axis tiles (8 <= D <= 12, batched D >= 8): work item w covers
// batch b = w / nslab, top index t_T = slab0 + w % nslab, writes z[w * 6561 ...].
template <class T>
__global__ void __launch_bounds__(T8_NT, 2)
tile8_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ z, int D, uint64_t slab0,
             uint64_t nslab) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  if (threadIdx.x == 0) {
    for (int i = 0; i < T8_NRAW; ++i) mbar_init(&raw_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  RawRing rr{raw_bar, 0, 0};
  const uint64_t w = blockIdx.x;
  const uint64_t b = w / nslab;
  const uint64_t tT = slab0 + (w - b * nslab);
  tile8<T, true>(x + (b << D), y + (b << D), 256, z + w * 6561ull, D - 8, tT, sm, rr, policy_evict_last(), 0);
}

// Two-level persistent kernel: pass-1 items (slab j, e_U) and pass-2 items (slab j, 9
// columns) from one work counter in the order P1(0) P1(1) P2(0) P1(2) P2(1) ...; slabs in
// cost order (args.order).  See hc_tile.cuh (SlabArgs, p2_item) for the pass-2 side and the
// deadlock argument.
template <class T, int M>
__global__ void __launch_bounds__(T8_NT, 2)
slab8_kernel(const T* __restrict__ xu, const T* __restrict__ yu, T* __restrict__ z, SlabArgs args) {
  constexpr uint32_t N1 = (uint32_t)ipow3(M);
  constexpr uint32_t N2 = (uint32_t)(ipow3(8) / P2W);
  constexpr uint64_t SLAB = upow3(M + 8);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  __shared__ uint32_t s_item;
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  if (threadIdx.x == 0) {
    for (int i = 0; i < T8_NRAW; ++i) mbar_init(&raw_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  RawRing rr{raw_bar, 0, 0};
  const uint32_t ns = args.nslab;
  const uint64_t total = (uint64_t)ns * (N1 + N2);
  const uint64_t pol_in = policy_evict_first();   // middle-axes tables are streamed
  const uint64_t pol_keep = policy_evict_last();  // pass-1 tiles wait in L2 for pass 2
  const uint64_t stride = upow3(M) * 256;
  // claim one item ahead so the atomic's latency overlaps the current item (the claim order
  // -- and with it the deadlock argument -- is unchanged)
  uint32_t nq = threadIdx.x == 0 ? atomicAdd(args.ctr, 1u) : 0u;
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_item = nq;
      nq = atomicAdd(args.ctr, 1u);
    }
    __syncthreads();
    const uint64_t q = s_item;
    if (q >= total) break;
    // order with lag G: P1(0..G-1) | [P1(j) P2(j-G)] for j = G..ns-1 | P2(ns-G..ns-1)
    bool is_p1;
    uint32_t j, r;
    const uint32_t G = args.lag < ns ? args.lag : ns;
    if (q < (uint64_t)G * N1) {
      is_p1 = true; j = (uint32_t)(q / N1); r = (uint32_t)(q - (uint64_t)j * N1);
    } else {
      const uint64_t q2 = q - (uint64_t)G * N1;
      const uint32_t pr = (uint32_t)(q2 / (N1 + N2));
      const uint32_t rr = (uint32_t)(q2 - (uint64_t)pr * (N1 + N2));
      if (pr + G < ns) {
        if (rr < N1) { is_p1 = true; j = pr + G; r = rr; }
        else { is_p1 = false; j = pr; r = rr - N1; }
      } else {
        // tail: the remaining pass-2 items, N2 per slab
        const uint64_t q3 = q2 - (uint64_t)(ns - G) * (N1 + N2);
        is_p1 = false; j = (ns - G) + (uint32_t)(q3 / N2); r = (uint32_t)(q3 % N2);
      }
    }
    const uint32_t loc = args.order[j];
    T* zs = z + (uint64_t)loc * SLAB;
    if (is_p1) {
      if (args.debug_skip == 2) {
        if (threadIdx.x == 0) atomicAdd(args.ctr + 1 + j, 1u);
        continue;
      }
      tile8<T, false>(xu + (uint64_t)r * 256, yu + (uint64_t)r * 256, stride, zs + (uint64_t)r * 6561ull, args.k,
                      args.slab0 + loc, sm, rr, pol_in, pol_keep);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(args.ctr + 1 + j, 1u);
      }
    } else {
      if (args.debug_skip == 1) continue;
      if (threadIdx.x == 0) {
        while (ld_acquire(args.ctr + 1 + j) < N1) __nanosleep(256);
      }
      __syncthreads();
      p2_item<T, M, 8>(zs, r, sm, T8_NT);
    }
  }
}

}  // namespace hc
