// hc_slab.cuh -- the 8-axis tile (all D >= 8) and the two-level slab engine (D >= 13).
//
// a1 input staging, a2 forward, a3 product / pair-sum, a4 inverse on
// the tile axes, a5 inverse on the middle axes, a6 store, a7 batched small cubes.
// Arithmetic: the paper's per-axis split (PAPER.md 185-192) -- forward (a0, a0+a1, a1),
// pointwise product, inverse (c0, (c1-c0)-c2, c2) -- on the 8 tile axes and the M middle
// axes; the paper's 4-way split (PAPER.md 166-177) on the k top axes (pair-sum).
//
// Tile axes (bit / trit b of the tile index, b = 0 fastest):
//   C = {0,1,2}  register axes: 27 accumulators per thread
//   B = {3,4,5}  evaluated by the F1 warps, in registers
//   a1 = 6       evaluated by the F1 warps (one warp per evaluation point e_a1)
//   a2 = 7       summed by the F2 threads while they load (e_a2 = 1: two rows)
// CTA = 8 warps (2 CTAs/SM, 4 warps per SM sub-partition: 128 registers per thread).
// In F2 and the inverse, thread u < 243 owns (e_a2, e_a1, e_B) = u / 81, u / 27 % 3, u % 27;
// warps 5-7 also run F1 (warp 5 + e_s evaluates a1 at e_s).
//
// Shared-memory cost model (measured, profiles/r01_smem_microbench.txt, tools/microbench/
// mb4.cu): loads 256 B/clk/SM (LDS.64 at odd or aligned-contiguous lane strides, LDS.128 at
// a 10-element stride), stores 128 B/clk/SM.  The split above keeps stores low: per pair
// and tile F1 stores 2 ops x 2 b_a2 x 81 e_S x 8 b_C = 2592 elements, F2 loads
// 243 x (4/3) x 16 = 5184 (LDS.128), F1 loads 4 x 256 = 1024.
#pragma once
#include "hc_tile.cuh"

namespace hc {

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_unchanged() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
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
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16-byte shared load of two consecutive elements
__device__ __forceinline__ void lds2(const double* p, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void lds2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(smem_u32(p)));
}

// ---- layouts (element offsets) ------------------------------------------------------
constexpr int T8_NW = 8;              // warps per tile CTA
constexpr int T8_NT = 32 * T8_NW;     // 256 threads (243 tile units)
// Warp roles, balanced so that every warp does about the same work between barriers:
//   threads 0..80 own the e_a2 = 1 units (two rows per F2 load: warps 0, 1, part of 2),
//   threads 81..161 the e_a2 = 0 units, 162..242 the e_a2 = 2 units;
//   F1 runs on warps 3, 4, 6 (single-row F2), e_s = 0, 1, 2; the scheduler on warp 7.
__device__ __forceinline__ int t8_unit(int tid) { return tid < 81 ? tid + 81 : (tid < 162 ? tid - 81 : tid); }
__device__ __forceinline__ int t8_f1_es(int w) { return w == 3 ? 0 : (w == 4 ? 1 : (w == 6 ? 2 : -1)); }
constexpr int T8_SCHED = 224;         // scheduler / prefetch thread (warp 7: light F2, no F1)
// raw stage: op*RS_OP + b_a2*RS_H2 + b_a1*RS_H1 + b_B*8 + b_C, filled by 2 TMA copies of
// 128 elements (the b_a2 halves of the natural slice) per operand; the pads put the F1
// lanes (op, b_a2, b_C) on 32 distinct 8-byte bank slots (RS_H2 = 8, RS_OP = 16 mod 32)
constexpr int RS_H1 = 64, RS_H2 = 136, RS_OP = 304, RS_SZ = 608;
// raw ring depth: the slices stream from HBM (the middle-axes tables) or L2.  Measured at
// D = 20 (round 2): 1 stage 29.8 ms, 2 stages 26.9 ms, 3 27.4, 4 27.5, 5 27.7 -- two pairs of
// lead already hide the load latency behind F2 and the tile work, and a shallower ring leaves
// 9.7 KB more of the SM's shared memory / L1 to the rest (D = 16 int64: 0.342 -> 0.327 ms)
#ifndef HC_NRAW
#define HC_NRAW 2
#endif
constexpr int T8_NRAW = HC_NRAW;
// the fused-carry instantiations with M = 5 (EPI 2, 3; conv1d at D = 13) keep a 4-stage ring:
// with 2 their scheduler state no longer fits the 128 registers (4 bytes of spills); the M = 6
// ones take 2 like the plain engine (f1 at D = 20: 39.06 -> 38.45 ms)
#ifndef HC_NRAW_EPI5
#define HC_NRAW_EPI5 4
#endif
template <int M, int EPI>
__host__ __device__ constexpr int slab_nraw() { return EPI >= 2 && M == 5 ? HC_NRAW_EPI5 : T8_NRAW; }
// P stage (F1 output): op*PS_OP + b_a2*PS_A2 + e_S*PS_ROW + b_C, e_S = e_B + 27 e_a1.
// PS_ROW = 10: the F2 lanes (consecutive e_S) read 16 B at a 80-B stride (conflict-free);
// PS_A2 = 8 and PS_OP = 16 (mod 32): the F1 stores of one warp hit 32 distinct slots.
constexpr int PS_ROW = 10, PS_A2 = 840, PS_OP = 1680, PS_SZ = 3360;
// tile exchange buffer S (3^8) and the pass-2 buffer alias the two P stages
constexpr int T8_PBUF = 2 * PS_SZ + 8;

template <class T, int NR = T8_NRAW>
struct T8Cfg {
  static constexpr int ALIAS = T8_PBUF > 6561 ? T8_PBUF : 6561;
  static constexpr size_t SMEM = sizeof(T) * (size_t)(ALIAS + NR * RS_SZ);
  static_assert(P2Cfg<6>::SIZE <= ALIAS && P2Cfg<5>::SIZE <= ALIAS, "pass-2 buffer aliases the P stages");
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

// ---- optional phase instrumentation (-DHC_PHASE_PROF; development builds only) -------
#ifdef HC_PHASE_PROF
__device__ unsigned long long hc_phase[16];
__device__ __forceinline__ long long* ph_sh() {
  __shared__ long long s_ph[10];  // [0..7] phase sums, [8] timestamp of the marking thread, [9] wait start
  return s_ph;
}
#define PH_DECL do { if (threadIdx.x == 128) { for (int i_ = 0; i_ < 8; ++i_) ph_sh()[i_] = 0; ph_sh()[8] = clock64(); } } while (0)
#define PH_MARK(i) do { if (threadIdx.x == 128) { long long t_ = clock64(); ph_sh()[i] += t_ - ph_sh()[8]; ph_sh()[8] = t_; } } while (0)
#define PH_WAIT_BEGIN(c) long long phw_ = (c) ? clock64() : 0
#define PH_WAIT_END(c) do { if (c) atomicAdd((unsigned long long*)&ph_sh()[7], (unsigned long long)(clock64() - phw_)); } while (0)
#define PH_T0 long long pht0_ = clock64()
#define PH_T1(i) atomicAdd((unsigned long long*)&ph_sh()[i], (unsigned long long)(clock64() - pht0_))
#define PH_FLUSH do { if (threadIdx.x == 128) for (int i_ = 0; i_ < 8; ++i_) atomicAdd(&hc_phase[i_], (unsigned long long)ph_sh()[i_]); } while (0)
#else
#define PH_DECL do { } while (0)
#define PH_MARK(i) do { } while (0)
#define PH_WAIT_BEGIN(c) do { } while (0)
#define PH_WAIT_END(c) do { } while (0)
#define PH_FLUSH do { } while (0)
#define PH_T0 do { } while (0)
#define PH_T1(i) do { } while (0)
#endif

// ---- raw-slice staging ring and the cross-item prefetcher -----------------------------
// T8_NRAW stages; stage n is filled by 4 TMA copies (x and y, two 128-element halves each)
// and completes on its mbarrier.  `done` counts fills consumed by F1 (advanced identically
// in every thread); `seq` (the scheduling thread T8_SCHED) counts fills issued.  Fill n may be issued once fill
// n - T8_NRAW has been read, i.e. seq - done < T8_NRAW at a point after a barrier.
template <int NR = T8_NRAW>
struct RawRing {
  uint64_t* bar;     // [NR] in shared memory
  uint32_t seq;      // fills issued so far (T8_SCHED)
  uint32_t done;     // fills consumed so far
};
template <class T, int NR>
__device__ __forceinline__ void t8_issue(RawRing<NR>& rr, const T* sx, const T* sy, T* R, uint64_t pol) {
  HC_ASSERT(rr.seq - rr.done < (uint32_t)NR);  // never overwrite a stage F1 has not read
  const uint32_t st = rr.seq % NR;
  uint64_t* bar = &rr.bar[st];
  T* dst = R + st * RS_SZ;
  mbar_arrive_tx(bar, 2 * 256 * sizeof(T));
  tma_load_1d(dst, sx, 128 * sizeof(T), bar, pol);
  tma_load_1d(dst + RS_H2, sx + 128, 128 * sizeof(T), bar, pol);
  tma_load_1d(dst + RS_OP, sy, 128 * sizeof(T), bar, pol);
  tma_load_1d(dst + RS_OP + RS_H2, sy + 128, 128 * sizeof(T), bar, pol);
  ++rr.seq;
}
template <int NR>
__device__ __forceinline__ uint32_t t8_wait(RawRing<NR>& rr) {
  const uint32_t st = rr.done % NR;
  mbar_wait(&rr.bar[st], (rr.done / NR) & 1);
  ++rr.done;
  return st;
}

// Stage F1 of one pair (warp with t8_f1_es(w) = e_s): lane (op, b_a2, b_C) evaluates the a1 axis at
// e_s and the three B axes (PAPER.md 186-189 per axis), and stores the 27 values e_B.
template <class T>
__device__ __forceinline__ void t8_f1(const T* R, T* P, int es, int lane) {
  const int op = lane >> 4, ba2 = (lane >> 3) & 1, bc = lane & 7;
  const T* src = R + op * RS_OP + ba2 * RS_H2 + bc;
  T in[8];
  if (es == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) in[j] = src[8 * j];
  } else if (es == 2) {
#pragma unroll
    for (int j = 0; j < 8; ++j) in[j] = src[RS_H1 + 8 * j];
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) in[j] = Ar<T>::add(src[8 * j], src[RS_H1 + 8 * j]);
  }
  T* dst = P + op * PS_OP + ba2 * PS_A2 + (27 * es) * PS_ROW + bc;
  fwd_store<3, PS_ROW, T>(in, dst);
}

// Stage F2 of one pair: thread (e_a2, e_S) loads its 8 + 8 base values (summing the two
// b_a2 rows when e_a2 = 1) and runs the C-axes forward fused with the product.
template <class T>
__device__ __forceinline__ void t8_f2(const T* P, int ea2, int eS, T* acc) {
  const T* px = P + eS * PS_ROW;
  T xt[8], yt[8];
  if (ea2 != 1) {
    const T* a = px + (ea2 >> 1) * PS_A2;
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      lds2(a + j, xt[j], xt[j + 1]);
      lds2(a + PS_OP + j, yt[j], yt[j + 1]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      T u0, u1, v0, v1;
      lds2(px + j, xt[j], xt[j + 1]);
      lds2(px + PS_A2 + j, u0, u1);
      lds2(px + PS_OP + j, yt[j], yt[j + 1]);
      lds2(px + PS_OP + PS_A2 + j, v0, v1);
      xt[j] = Ar<T>::add(xt[j], u0);
      xt[j + 1] = Ar<T>::add(xt[j + 1], u1);
      yt[j] = Ar<T>::add(yt[j], v0);
      yt[j + 1] = Ar<T>::add(yt[j + 1], v1);
    }
  }
  // Karatsuba on all three register axes.  (The direct split on the lower two needs fewer
  // operations -- 48 FMA + 8 adds against 27 + 38 -- but a DFMA with three register operands
  // issues at ~2.8 clk per warp and SM sub-partition against ~1.1 for DADD on this B200, so
  // it is slower: tools/microbench/mb6.cu, profiles/r01_smem_microbench.txt.)
  fwd_mul_acc<3, T>(xt, yt, acc);
}

// Prefetch cursor (shared memory, T8_SCHED only) over the pairs of the pass-1 items in the
// order the CTA will consume them.  Pair p of an item has subset s_p of freeb (ascending
// subsets, PAPER.md 173-177 direct split): i_T = base | s_p, j_T = base | (freeb & ~s_p).
struct Prefetch {
  const void* sx0;
  const void* sy0;
  uint64_t stride;
  uint32_t base, freeb, s;
  int left;        // pairs of the cursor item not yet issued
  uint32_t pos;    // position of the cursor item in the CTA's item sequence
};

// Fill the ring (T8_SCHED).  next(pf) advances the cursor to the next pass-1 item the CTA
// will run (setting sx0, sy0, stride, base, freeb, s = 0, left) or returns false.
template <class T, int NR, class Next>
__device__ __forceinline__ void pf_pump(Prefetch& pf, RawRing<NR>& rr, T* R, uint64_t pol, Next&& next) {
  bool fenced = false;
  while (rr.seq - rr.done < (uint32_t)NR) {
    if (pf.left == 0 && !next(pf)) return;
    if (!fenced) {  // the stage's previous contents were read through the generic proxy
      fence_proxy_async();
      fenced = true;
    }
    const uint64_t iT = pf.base | pf.s, jT = pf.base | (pf.freeb & ~pf.s);
    HC_ASSERT((pf.base & pf.freeb) == 0 && (pf.s & ~pf.freeb) == 0 && pf.left > 0);
    t8_issue<T>(rr, (const T*)pf.sx0 + iT * pf.stride, (const T*)pf.sy0 + jT * pf.stride, R, pol);
    pf.s = (pf.s - pf.freeb) & pf.freeb;
    --pf.left;
  }
}

// One pass-1 tile with `npairs` top pairs whose raw slices arrive, in order, through the
// ring (issued by the pump).  Computes the tile's 3^8 values (final for the single-level
// engine, evaluation domain of the middle axes for the slab engine) and stores them to zt.
// ATOMIC (uint64 only): the tile's values are added to z with 64-bit atomics instead of stored
// (tile8_pairs_kernel: one pair's contribution per item)
template <class T, bool FINAL, bool ATOMIC = false, int NR, class Pump, class Mid>
__device__ __forceinline__ void tile8(int npairs, T* __restrict__ zt, T* sm, RawRing<NR>& rr, uint64_t pol_out,
                                      Pump&& pump, Mid&& mid) {
  static_assert(!ATOMIC || std::is_same<T, uint64_t>::value, "atomic accumulation is exact only in the wrapping uint64 ring");
  T* P = sm;                          // [2][PS_SZ]
  T* R = sm + T8Cfg<T>::ALIAS;        // [NR][RS_SZ]
  T* S = sm;                          // [9][27][27] after the pair loop (aliases P)
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const bool unit = tid < 243;                     // F2 / inverse unit u = (e_a2, e_S)
  const int u = t8_unit(tid);
  const int ea2 = u / 81, eS = u - 81 * ea2;       // e_S = e_B + 27 e_a1
  const int f1es = t8_f1_es(w);
  // F1: the warp with f1es = e_s evaluates a1 at e_s (the others only advance the ring count)
  auto f1 = [&](int, T* Pd) {
    if (f1es >= 0) t8_f1<T>(R + t8_wait(rr) * RS_SZ, Pd, f1es, lane);
    else ++rr.done;
  };

  if (tid == T8_SCHED) pump();
  f1(0, P);
  __syncthreads();

  T acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = T(0);
  for (int p = 0; p < npairs; ++p) {
    if (tid == T8_SCHED) pump();  // refill the stage F1(p) released
    if (p + 1 < npairs) f1(p + 1, P + ((p + 1) & 1) * PS_SZ);
    if (unit) t8_f2<T>(P + (p & 1) * PS_SZ, ea2, eS, acc);
    __syncthreads();
  }
  if (tid == T8_SCHED) {
    pump();
    mid();  // no global stores of this CTA are in flight here: cheap place for a release
  }
  PH_MARK(1);

  // a4: inverse on the C register axes, then B (SMEM exchange), then A + store (a6).
  // Unit u = (e_A, e_B) with e_A = e_a1 + 3 e_a2, so S[e_A][e_B][k_C] = S[27 u + k_C]
  // (stride 27: conflict-free whatever the thread-to-unit map).
  if (unit) {
    inv_reg<3, T>(acc);
#pragma unroll
    for (int i = 0; i < 27; ++i) S[u * 27 + i] = acc[i];
  }
  __syncthreads();
  if (unit) {  // unit (e_A, k_C): interpolate the B axes
    const int c = tid / 9, a = tid - 9 * c;  // e_A fastest: conflict-free (stride 729 = 9 mod 16)
    T v[27];
#pragma unroll
    for (int e = 0; e < 27; ++e) v[e] = S[a * 729 + e * 27 + c];
    inv_reg<3, T>(v);
#pragma unroll
    for (int e = 0; e < 27; ++e) S[a * 729 + e * 27 + c] = v[e];
  }
  __syncthreads();
  // columns (k_B, k_C), three rounds of 243: interpolate the A axes, store
#pragma unroll 1
  for (int r = 0; r < 3; ++r) {
    if (unit) {
      const int col = r * 243 + tid;
      T v[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) v[e] = S[e * 729 + col];
      inv_reg<2, T>(v);
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        if constexpr (ATOMIC) atomicAdd(reinterpret_cast<unsigned long long*>(zt + e * 729 + col), (unsigned long long)v[e]);
        else if constexpr (FINAL) st_cs(zt + e * 729 + col, v[e]);
        else st_hint(zt + e * 729 + col, v[e], pol_out);
      }
    }
    // single level: keeping the CTA's rounds of final (streaming) stores in step measured
    // faster (batched D = 8: 1.17 vs 1.185 ms); the slab engine's tiles go to L2 and do not
    // gain (27.68 vs 27.55 ms at D = 20)
    if constexpr (FINAL) {
      if (r < 2) __syncthreads();
    }
  }
}

template <int NR = T8_NRAW>
__device__ __forceinline__ void ring_init(uint64_t* bars) {
  if (threadIdx.x == T8_SCHED) {
    for (int i = 0; i < NR; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// Single-level persistent kernel for 8-axis tiles (8 <= D <= 12, batched D >= 8): item w
// (w = blockIdx.x, + gridDim.x, ...) covers batch b = w / nslab, top index
// t_T = slab0 + w % nslab, and writes z[w * 6561 ...].  The prefetcher walks the same
// static item sequence, so slices of the next tiles load while this one computes.
template <class T>
__global__ void __launch_bounds__(T8_NT, 2)
tile8_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ z, int D, uint64_t slab0,
             uint64_t nslab, uint64_t nitems) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  __shared__ Prefetch pf;
  ring_init(raw_bar);
  RawRing<> rr{raw_bar, 0, 0};
  const int k = D - 8;
  // a single pair's slices are reused by many tiles (keep them in L2); a batch's are read once
  const uint64_t pol_in = nitems > nslab ? policy_evict_first() : policy_evict_last();
  if (threadIdx.x == T8_SCHED) {
    pf.left = 0;
    pf.pos = 0xffffffffu;  // next() moves to position 0
  }
  T* R = sm + T8Cfg<T>::ALIAS;
  auto next = [&](Prefetch& c) -> bool {
    const uint32_t np = c.pos + 1;
    const uint64_t w = blockIdx.x + (uint64_t)np * gridDim.x;
    if (w >= nitems) return false;
    const uint64_t b = w / nslab;
    uint32_t base, freeb;
    trit_split(slab0 + (w - b * nslab), k, base, freeb);
    c.pos = np;
    c.sx0 = x + (b << D);
    c.sy0 = y + (b << D);
    c.stride = 256;
    c.base = base;
    c.freeb = freeb;
    c.s = 0;
    c.left = 1 << __popc(freeb);
    return true;
  };
  auto pump = [&]() { pf_pump<T>(pf, rr, R, pol_in, next); };
  for (uint64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
    const uint64_t b = w / nslab;
    uint32_t base, freeb;
    HC_ASSERT(slab0 + (w - b * nslab) < upow3(k));
    trit_split(slab0 + (w - b * nslab), k, base, freeb);
    tile8<T, true>(1 << __popc(freeb), z + w * 6561ull, sm, rr, 0, pump, [] {});
    __syncthreads();  // S (aliases P) is free before the next tile's F1
  }
}

// Single-level int64 with few tiles (D = 11, 12: 3^(D-8) tiles for 148 x 2 CTA slots):
// one item per (tile, direct-split pair) instead of per tile, so a tile's pairs run on
// different SMs; each item interpolates its pair's contribution (the interpolation is linear)
// and adds it to the tile with 64-bit atomics -- exact, since wrapping additions commute
// (R3).  z is zeroed before the launch.  items[w] = {tile t of the launch, subset s
// of the tile's free top bits} (PAPER.md 173-177: pair i_T = base | s, j_T = base | (free & ~s)).
__global__ void __launch_bounds__(T8_NT, 2)
tile8_pairs_kernel(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y, uint64_t* __restrict__ z, int D,
                   uint64_t slab0, const uint2* __restrict__ items, uint32_t nitems) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smem_raw);
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  __shared__ Prefetch pf;
  ring_init(raw_bar);
  RawRing<> rr{raw_bar, 0, 0};
  const int k = D - 8;
  const uint64_t pol_in = policy_evict_last();  // a slice is shared by the pairs of several tiles
  if (threadIdx.x == T8_SCHED) {
    pf.left = 0;
    pf.pos = 0xffffffffu;
  }
  uint64_t* R = sm + T8Cfg<uint64_t>::ALIAS;
  auto next = [&](Prefetch& c) -> bool {
    const uint32_t np = c.pos + 1;
    const uint64_t w = blockIdx.x + (uint64_t)np * gridDim.x;
    if (w >= nitems) return false;
    const uint2 it = items[w];
    uint32_t base, freeb;
    trit_split(slab0 + it.x, k, base, freeb);
    HC_ASSERT((it.y & ~freeb) == 0);
    c.pos = np;
    c.sx0 = x;
    c.sy0 = y;
    c.stride = 256;
    c.base = base;
    c.freeb = freeb;
    c.s = it.y;
    c.left = 1;
    return true;
  };
  auto pump = [&]() { pf_pump<uint64_t>(pf, rr, R, pol_in, next); };
  for (uint64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
    tile8<uint64_t, true, true>(1, z + (uint64_t)items[w].x * 6561ull, sm, rr, 0, pump, [] {});
    __syncthreads();  // S (aliases P) is free before the next tile's F1
  }
}

// Two-level persistent kernel: pass-1 items (slab j, e_U) and pass-2 items (slab j, 9
// columns) from one work counter in the order P1(0) P1(1) P2(0) P1(2) P2(1) ...; slabs in
// cost order (args.order).  Each CTA holds T8_QN claimed items ("slots"), decoded by the
// scheduling thread T8_SCHED when the claim returns.  Selection: a pass-2 item whose slab is
// complete (lowest claim first), else the lowest pass-1 item, else wait for the lowest pass-2
// item.
// Pass-1 items therefore run in claim order, which is the order the prefetcher issues
// their slices.  Deadlock freedom: pass-1 items wait for nothing; a pass-2 item waits only
// for pass-1 items of its slab, all claimed earlier.  The earliest unfinished claim is
// either a pass-1 item -- its CTA never blocks while holding it (a ready pass-2 item or a
// pass-1 item is always preferred to waiting) -- or a pass-2 item whose dependencies are
// done, so it progresses (given a co-resident grid: grid <= SMs x occupancy).  A CTA
// signals a finished pass-1 tile one item later (its stores have drained by then, so the
// release fence is cheap), and always before it starts to wait.
struct ItemDec {
  bool p1;
  uint32_t j, r;
};
__device__ __forceinline__ ItemDec decode_item(uint32_t q, uint32_t ns, uint32_t N1, uint32_t N2, uint32_t lag,
                                               uint32_t head = 0xffffffffu) {
  // order with lag G: P1(0..G-1) | [P1(j) P2(j-G)] for j = G..ns-1 | P2(ns-G..ns-1).  With
  // head = H < N1, a group [P1(j) P2(j-G)] is H pass-1 items of position j, then the remaining
  // N1 - H pass-1 items interleaved with the N2 pass-2 items of position j - G (ratio
  // (N1 - H) / N2 : 1): slab j - G is then consumed while slab j is produced instead of after it
  // (a smaller L2 footprint); every pass-2 item still follows all pass-1 items of its slab.
  ItemDec d;
  const uint32_t G = lag < ns ? lag : ns;
  if (q < G * N1) {
    d.p1 = true; d.j = q / N1; d.r = q - d.j * N1;
  } else {
    const uint32_t q2 = q - G * N1;
    const uint32_t pr = q2 / (N1 + N2);
    const uint32_t rr = q2 - pr * (N1 + N2);
    if (pr + G < ns) {
      if (head < N1 && rr >= head) {
        const uint32_t per = (N1 - head) / N2;  // pass-1 items per pass-2 item (N2 divides N1 - head)
        const uint32_t g = (rr - head) / (per + 1), o = (rr - head) - g * (per + 1);
        if (o < per) { d.p1 = true; d.j = pr + G; d.r = head + g * per + o; }
        else { d.p1 = false; d.j = pr; d.r = g; }
      } else if (rr < N1) { d.p1 = true; d.j = pr + G; d.r = rr; }
      else { d.p1 = false; d.j = pr; d.r = rr - N1; }
    } else {
      const uint32_t q3 = q2 - (ns - G) * (N1 + N2);
      d.p1 = false; d.j = (ns - G) + q3 / N2; d.r = q3 % N2;
    }
  }
  return d;
}

#ifndef HC_QN
#define HC_QN 3
#endif
constexpr int T8_QN = HC_QN;  // claimed items held per CTA
constexpr uint32_t T8_EXH = 0xffffffffu;
constexpr int T8_DEFER = -2;  // s_sel: selection postponed past the item's closing barrier
// EPI 3 (fused carries, ring): pass-1 tiles live in a ring of T8_RING slab buffers (slab position j
// in slot j mod T8_RING) instead of z; a pass-1 item of position j >= T8_RING is ready once
// every pass-2 item of position j - T8_RING (claimed earlier) has read its column
#ifndef HC_RING
#define HC_RING 4
#endif
constexpr uint32_t T8_RING = HC_RING;
#ifndef HC_P2CH
#define HC_P2CH 3
#endif
constexpr int T8_P2CH = HC_P2CH;  // 9-column chunks per pass-2 item

// f1, carries fused into pass 2 (int64 only: wrapping uint64 sums are exact in any order).
// One 9-column chunk of a slab: round 1 as in p2_item; round 2 interpolates the HI middle
// axes and, instead of storing z, adds every final value z[k] into out[val(k)],
// val(k) = sum_b k_b 2^b (PAPER.md 354-373: the carry-free digits of the 1-D convolution).
// Within the chunk val = base + a(pos) + 256 (val3(e_lo) + 8 valHI(e_hi)), a = k0 + 2 k1;
// the sums are reduced over e_hi in registers, over e_lo in shared memory, and each of the
// chunk's distinct bins (a, u) gets one global atomic add.  `mid` runs on thread `sched`
// after the loads (as in p2_item).
template <int N>
__device__ __forceinline__ constexpr int bitval3(int e) {  // sum_b digit_b(e) 2^b, N base-3 digits
  int v = 0;
  for (int b = 0, p = 1; b < N; ++b, p <<= 1, e /= 3) v += (e % 3) * p;
  return v;
}
// Interpolation over N axes fused with the carry binning of f1: out[val] = sum over the 3^N
// positions e with val(e) = sum_b e_b 2^b of the interpolated z[e] (PAPER.md 187-189 per axis,
// 354-373 for the carries).  Axis by axis from the top: the three top-digit slices are binned
// recursively (2^N - 1 coefficients each), interpolated as coefficient vectors (the
// interpolation is linear and acts on the top digit only), and merged with weights 2^(N-1)
// and 2^N.  Fewer live values than interpolating all 3^N first and binning afterwards.
template <int N, class T>
__device__ __forceinline__ void inv_bin(const T* v, T* out) {
  if constexpr (N == 0) {
    out[0] = v[0];
  } else {
    constexpr int m = ipow3(N - 1), L = (1 << N) - 1, h = 1 << (N - 1);
    T a0[L], a1[L], a2[L];
    inv_bin<N - 1, T>(v, a0);
    inv_bin<N - 1, T>(v + m, a1);
    inv_bin<N - 1, T>(v + 2 * m, a2);
#pragma unroll
    for (int i = 0; i < 2 * L + 1; ++i) out[i] = T(0);
#pragma unroll
    for (int i = 0; i < L; ++i) {
      out[i] = Ar<T>::add(out[i], a0[i]);                                       // digit 0: weight 0
      out[i + h] = Ar<T>::add(out[i + h], Ar<T>::sub(Ar<T>::sub(a1[i], a0[i]), a2[i]));  // digit 1
      out[i + 2 * h] = Ar<T>::add(out[i + 2 * h], a2[i]);                       // digit 2: weight 2^N
    }
  }
}

template <class T, int M, class Mid>
__device__ __forceinline__ void p2_carry_chunk(const T* __restrict__ zs, uint32_t c, T* sm, int task,
                                               unsigned long long* __restrict__ out, uint64_t base, int sched,
                                               Mid&& mid) {
  using Q = P2Cfg<M>;
  constexpr int LO = Q::LO, HI = Q::HI, NLO = Q::NLO, NHI = Q::NHI, P2S = Q::P2S;
  static_assert(LO == 3, "three low middle axes");
  constexpr int NB = (2 << HI) - 1;          // distinct valHI(e_hi)
  constexpr int NU = 15 + 8 * (NB - 1);      // u = val3(e_lo) + 8 valHI in [0, NU)
  constexpr uint64_t ROW = 6561;
  const uint64_t col0 = (uint64_t)c * P2W;
  HC_ASSERT(col0 + P2W <= ROW);
  // round 1: task (e_hi, pos) loads its 27 column entries, interpolates the LO axes
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
  __syncthreads();
  if ((int)threadIdx.x == sched) mid();
  // round 2: task (e_lo, pos) interpolates the HI axes and sums its values by valHI(e_hi); bin
  // vhi goes to the cell the task itself read for e_hi = vhi (row vhi of its column), so no
  // other thread's unread cell is overwritten and no barrier (nor live bins across one) is needed
  static_assert(NB <= NHI && NB * P2S + 9 * NB * 15 <= T8Cfg<T>::ALIAS, "bins fit the exchange rows");
  const int el = task / P2W, pos = task - el * P2W;
  if (task >= 0 && task < NLO * P2W) {
    T v[NHI], b[NB];
#pragma unroll
    for (int e = 0; e < NHI; ++e) v[e] = sm[e * P2S + el * P2W + pos];
    static_assert(NB == (2 << HI) - 1, "bins of HI digits");
    inv_bin<HI, T>(v, b);
#pragma unroll
    for (int i = 0; i < NB; ++i) sm[i * P2S + el * P2W + pos] = b[i];  // bs[vhi][e_lo][pos]
  }
  T* cs = sm + NB * P2S;  // [pos][vhi][val3(e_lo)]: 9 x NB x 15, past the bin rows
  __syncthreads();
  // sum over e_lo by val3(e_lo): thread (pos, vhi)
  for (int t = threadIdx.x; t < 9 * NB; t += blockDim.x) {
    const int tp = t / NB, tv = t - tp * NB;
    T cc[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) cc[i] = T(0);
#pragma unroll
    for (int e = 0; e < NLO; ++e) cc[bitval3<3>(e)] += sm[tv * P2S + e * P2W + tp];
#pragma unroll
    for (int i = 0; i < 15; ++i) cs[t * 15 + i] = cc[i];
  }
  __syncthreads();
  // final bins (a, u): a = k0 + 2 k1 over the positions with that value, u = w + 8 vhi
  for (int t = threadIdx.x; t < 7 * NU; t += blockDim.x) {
    const int a = t / NU, u = t - a * NU;
    T sum = T(0);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      if ((p % 3) + 2 * (p / 3) != a) continue;
#pragma unroll
      for (int vh = 0; vh < NB; ++vh) {
        const int w = u - 8 * vh;
        if (w >= 0 && w < 15) sum += cs[(p * NB + vh) * 15 + w];
      }
    }
    atomicAdd(out + base + a + 256 * (uint64_t)u, (unsigned long long)sum);
  }
}

struct __align__(16) Slot {
  uint32_t loc, base, freeb, pad;  // = order[j] (16 B): slab offset; pass 1: trit split of its top index;
                                   // pad = problem index within a batch (SlabArgs::order)
  uint32_t q;                      // claim index, T8_EXH = past the end (or being decoded)
  uint32_t p1, j, r;
};
static_assert(T8_QN == 3, "the scheduler packs the slots' claim indices into one uint4");

// EPI 2: carries fused into pass 2 (f1, uint64 only), tiles in place in z; EPI 3: the same
// with the tiles in a ring of T8_RING slab buffers (no 3^D buffer)
// P2CH: 9-column chunks per pass-2 item (T8_P2CH; 1 for launches of at most 3 slabs, where the
// last slab's pass 2 would otherwise run on a third of the CTAs: D = 14 0.099 -> 0.070 ms)
template <class T, int M, int EPI = 0, int P2CH = T8_P2CH>
__global__ void __launch_bounds__(T8_NT, 2)
slab8_kernel(const T* __restrict__ xu, const T* __restrict__ yu, T* __restrict__ z, SlabArgs args) {
  constexpr uint32_t N1 = (uint32_t)ipow3(M);
  constexpr uint32_t N2 = (uint32_t)(ipow3(8) / (P2W * P2CH));
  constexpr uint64_t SLAB = upow3(M + 8);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  __shared__ Slot s_slot[T8_QN];
  __shared__ uint4 s_qm;  // {q of slots 0..2, -}: one load for the selection
  __shared__ uint4 s_jm;  // {j of slots 0..2, byte i of .w = slot i is a pass-1 item}
  __shared__ int s_sel;
  constexpr int NR = slab_nraw<M, EPI>();
  __shared__ __align__(8) uint64_t raw_bar[NR];
  __shared__ Prefetch pf;
  ring_init<NR>(raw_bar);
  RawRing<NR> rr{raw_bar, 0, 0};
  const uint32_t ns = args.nslab;
  const uint32_t total = ns * (N1 + N2);
  const uint32_t lag = args.lag;
  const uint64_t pol_in = policy_evict_first();   // middle-axes tables are streamed
  // pass-1 tiles wait in L2 for pass 2 (args.keep_policy: 0 evict_last, 1 evict_normal, 2 unchanged)
  const uint64_t pol_keep = args.keep_policy == 1 ? policy_evict_normal()
                            : (args.keep_policy == 2 ? policy_evict_unchanged() : policy_evict_last());
  const uint64_t stride = upow3(M) * 256;
  const bool skip1 = args.debug_skip == 2, skip2 = args.debug_skip == 1;
  T* R = sm + T8Cfg<T>::ALIAS;
  uint32_t* done_ctr = args.ctr + 1;
  uint32_t* p2_done = args.ctr + 1 + args.nslab;  // EPI 3: pass-2 items finished per position

  // T8_SCHED helpers -------------------------------------------------------------------
  auto decode = [&](uint32_t q, Slot& o) {
    if (q >= total) { o.q = T8_EXH; return; }
    const ItemDec d = decode_item(q, ns, N1, N2, lag, args.p2_head);
    HC_ASSERT(d.j < ns && d.r < (d.p1 ? N1 : N2));
    o.q = q; o.p1 = d.p1; o.j = d.j; o.r = d.r;
    const uint4 oi = args.order[d.j];
    o.loc = oi.x; o.base = oi.y; o.freeb = oi.z; o.pad = oi.w;
  };
  // prefetch cursor: pass-1 slots in claim order (pf.pos = claim index of the cursor item)
  auto next = [&](Prefetch& c) -> bool {
    if (skip1) return false;
    int best = -1;
    for (int i = 0; i < T8_QN; ++i) {
      const Slot& o = s_slot[i];
      if (o.q == T8_EXH || !o.p1 || (c.pos != T8_EXH && o.q <= c.pos)) continue;
      if (best < 0 || o.q < s_slot[best].q) best = i;
    }
    if (best < 0) return false;
    const Slot& o = s_slot[best];
    c.pos = o.q;
    const uint64_t off = (uint64_t)o.pad * args.bstride + (uint64_t)o.r * 256;  // problem o.pad of a batch
    c.sx0 = xu + off;
    c.sy0 = yu + off;
    c.stride = stride;
    c.base = o.base;
    c.freeb = o.freeb;
    c.s = 0;
    c.left = 1 << __popc(o.freeb);
    return true;
  };
  auto pump = [&]() { pf_pump<T>(pf, rr, R, pol_in, next); };
  uint32_t pend = T8_EXH;  // T8_SCHED: slab position of a finished, not yet signalled tile
  // Completion of a pass-1 tile is published with a gpu-scope fence (cumulative over the
  // CTA's stores, which precede it through a CTA barrier) and an atomic increment.  Called
  // where T8_SCHED has no global stores in flight (mid item, before a wait, at exit).
  auto signal = [&]() {
    if (pend != T8_EXH) {
      __threadfence();
      atomicAdd(done_ctr + pend, 1u);
      pend = T8_EXH;
    }
  };

  // Thread T8_SCHED's state.  The slots live in shared memory (few registers are free in the
  // pair loop); s_qm / s_jm mirror their claim indices, kinds and slabs so that the selection,
  // which the whole CTA waits for, is two shared loads and register logic.
  auto set_meta = [&](int i, uint32_t q, bool p1, uint32_t j) {  // plain stores, no read-modify-write
    reinterpret_cast<uint32_t*>(&s_qm)[i] = q;
    reinterpret_cast<uint32_t*>(&s_jm)[i] = j;
    reinterpret_cast<uint8_t*>(&s_jm.w)[i] = p1 ? 1 : 0;
  };
  if (threadIdx.x == T8_SCHED) {
    uint32_t c[T8_QN];
    for (int i = 0; i < T8_QN; ++i) c[i] = atomicAdd(args.ctr, 1u);
    s_jm.w = 0;
    for (int i = 0; i < T8_QN; ++i) {
      decode(c[i], s_slot[i]);
      set_meta(i, s_slot[i].q, s_slot[i].q != T8_EXH && s_slot[i].p1, s_slot[i].j);
    }
    pf.left = 0;
    pf.pos = T8_EXH;
  }
  // kept across one item so that global-memory latencies overlap the item:
  uint32_t cv[T8_QN];  // slab-completion counters of the pass-2 slots (loaded at item start)
  uint32_t cmask = 0;  // slots whose cv[] is valid
  int pslot = -1;      // slot whose claim pq is being decoded (its order[] entry is in flight)
  uint32_t pq = 0;
  auto finish_pending = [&]() {  // complete the claim decoded one item ago
    asm volatile("cp.async.wait_all;" ::: "memory");
    Slot& o = s_slot[pslot];
    o.q = pq;
    set_meta(pslot, pq, o.p1, o.j);
    pslot = -1;
  };
  // Selection of the next item (thread T8_SCHED); result in s_sel.  Before the item's closing
  // barrier (may_wait = false) the tile just computed cannot be published yet (other warps'
  // stores may be in flight), so a selection that would wait or leave returns T8_DEFER and is
  // redone after the barrier, where signal() is safe.
  auto select_next = [&](bool may_wait) {
    PH_T0;
    int sel, wsl;        // wsl: the slot to wait for when nothing is ready
    const uint32_t* wctr = nullptr;
    uint32_t wneed = 0;
    for (int pass = 0;; ++pass) {
      const uint4 qm = s_qm, jm = s_jm;
      const uint32_t rq[3] = {qm.x, qm.y, qm.z};
      int p2r = -1, p1 = -1, p2w = -1;
      uint32_t q1 = T8_EXH, q2r = T8_EXH, q2w = T8_EXH;
#pragma unroll
      for (int i = 0; i < T8_QN; ++i) {
        if (i == pslot || rq[i] == T8_EXH) continue;
        if ((jm.w >> (8 * i)) & 1) {
          if (rq[i] < q1) { q1 = rq[i]; p1 = i; }
        } else if (skip2 || (((cmask >> i) & 1) && cv[i] >= N1)) {
          if (rq[i] < q2r) { q2r = rq[i]; p2r = i; }
        } else if (rq[i] < q2w) {
          q2w = rq[i]; p2w = i;
        }
      }
      // only the lowest pass-1 claim may run (the prefetcher loads slices in claim order);
      // with the slab ring it may still have to wait for pass 2 of position j - T8_RING
      bool p1_ready = p1 >= 0;
      if constexpr (EPI == 3) {
        if (p1 >= 0) {
          const uint32_t j1 = p1 == 0 ? jm.x : (p1 == 1 ? jm.y : jm.z);
          const uint32_t c1 = p1 == 0 ? cv[0] : (p1 == 1 ? cv[1] : cv[2]);  // no dynamic index: cv[] stays in registers
          p1_ready = j1 < T8_RING || (((cmask >> p1) & 1) && c1 >= N2);
        }
      }
      sel = p2r >= 0 ? p2r : (p1_ready ? p1 : -1);
      wsl = -1;
      if (sel < 0) {  // wait for the lower claim of the blocked pass-1 item and pass-2 item
        const bool w1 = p1 >= 0 && (p2w < 0 || q1 < q2w);
        wsl = w1 ? p1 : p2w;
        if (wsl >= 0) {
          const uint32_t jw = wsl == 0 ? jm.x : (wsl == 1 ? jm.y : jm.z);
          if (w1) { wctr = p2_done + (jw - T8_RING); wneed = N2; }
          else { wctr = done_ctr + jw; wneed = N1; }
        }
        sel = wsl;
      }
      // before waiting (or leaving), the pending claim must be visible: it may be the
      // pass-1 item everybody waits for
      if ((sel < 0 || wsl >= 0) && pslot >= 0 && pass == 0) {
        finish_pending();
        continue;
      }
      break;
    }
    if (!may_wait && (sel < 0 || wsl >= 0)) {
      s_sel = T8_DEFER;
      return;
    }
    if (wsl >= 0) {  // nothing else to do: signal, then wait for the dependency
      signal();
      pump();
      while (ld_relaxed(wctr) < wneed) __nanosleep(64);
    }
    if (sel < 0) signal();
    // a pass-2 item's slab was seen complete through a relaxed counter load (above, or
    // snapshotted in cv[] one item earlier): the fence makes that observation an acquire, and
    // the CTA barrier after the selection orders every thread's column loads after it
    if (sel >= 0 && !((s_jm.w >> (8 * sel)) & 1)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    s_sel = sel;
    PH_T1(2);
  };
  PH_DECL;
  if (threadIdx.x == T8_SCHED) select_next(true);
  __syncthreads();
  while (true) {
    const int sel = *(volatile int*)&s_sel;
    if (sel < 0) break;
    Slot it;  // read now: thread T8_SCHED rewrites the slot before this item's last barrier
    {
      const volatile uint32_t* src = reinterpret_cast<const volatile uint32_t*>(&s_slot[sel]);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&it);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i] = src[i];
    }
    uint32_t claim = 0;
    if (threadIdx.x == T8_SCHED) {
      claim = atomicAdd(args.ctr, 1u);  // refills slot `sel` after this item
      cmask = 0;                         // snapshot the other pass-2 slots' slabs (used next time)
      const uint4 qm = s_qm, jm = s_jm;
      const uint32_t rq[3] = {qm.x, qm.y, qm.z}, rj[3] = {jm.x, jm.y, jm.z};
#pragma unroll
      for (int i = 0; i < T8_QN; ++i) {
        if (i != sel && i != pslot && rq[i] != T8_EXH && !((jm.w >> (8 * i)) & 1)) {
          cv[i] = ld_relaxed(done_ctr + rj[i]);  // non-blocking; compared at the next selection
          cmask |= 1u << i;
        } else if (EPI == 3 && i != sel && i != pslot && rq[i] != T8_EXH && rj[i] >= T8_RING) {
          cv[i] = ld_relaxed(p2_done + (rj[i] - T8_RING));  // pass-1 slot: its ring slot freed?
          cmask |= 1u << i;
        }
      }
    }
    PH_MARK(0);
    HC_ASSERT(it.loc < ns && it.j < ns && it.r < (it.p1 ? N1 : N2) && (it.base & it.freeb) == 0);
    T* zs = EPI == 3 ? reinterpret_cast<T*>(args.ring) + (uint64_t)(it.j % T8_RING) * SLAB
                     : z + (uint64_t)it.loc * SLAB;
    if (it.p1) {
      if (skip1) {
        if (threadIdx.x == T8_SCHED) atomicAdd(done_ctr + it.j, 1u);
        __syncthreads();  // everybody has read s_sel and the slot
      } else {
        tile8<T, false>(1 << __popc(it.freeb), zs + (uint64_t)it.r * 6561ull, sm, rr, pol_keep, pump, signal);
        PH_MARK(6);
      }
    } else if (!skip2) {
      // the slab's tiles are complete (a relaxed read of its counter saw N1, then the CTA
      // barrier): the reads below are ordered after it by that control dependency and the
      // barrier, and go to L2 (.cg), where the producers' fenced stores already are
      if (threadIdx.x == T8_SCHED) pump();
      // three 9-column chunks per item (a third as many items to schedule), pipelined
      if constexpr (EPI >= 2) {
        // carry bins: val(k) = (tile digits) + 2^8 (middle digits) + 2^(8+M) (top digits)
        uint64_t vtop = 0;
        {
          uint64_t t = args.slab0 + it.loc;
          for (int b = 0; b < args.k; ++b, t /= 3) vtop += (t % 3) << b;
        }
#pragma unroll 1
        for (int ch = 0; ch < P2CH; ++ch) {
          if (ch) __syncthreads();  // the exchange buffer is rewritten by the next chunk
          const uint32_t cc = it.r * P2CH + ch;  // chunk = tile digits k2..k7
          uint64_t vcol = 0;
          {
            uint32_t t = cc;
            for (int b = 2; b < 8; ++b, t /= 3) vcol += (uint64_t)(t % 3) << b;
          }
          p2_carry_chunk<T, M>(zs, cc, sm, threadIdx.x < 243 ? (int)threadIdx.x : -1, args.cout,
                               vcol + (vtop << (8 + M)), ch == 0 ? T8_SCHED : -1, signal);
        }
      } else {
      if (args.p2_prefetch) {
        // pull the item's later chunks into L2 while chunk 0 runs: part of the slab may have been
        // evicted to HBM since pass 1 wrote it; one bulk L2 prefetch (TMA unit, no registers, no
        // shared memory) per row of the item's P2W * P2CH columns, 16-B aligned cover
        constexpr int NROW = ipow3(M);
        const uint64_t c0 = (uint64_t)it.r * (P2W * P2CH);
        for (int row = threadIdx.x; row < NROW; row += T8_NT) {
          const uintptr_t a = reinterpret_cast<uintptr_t>(zs + (uint64_t)row * 6561ull + c0);
          const uintptr_t lo = a & ~(uintptr_t)15, hi = (a + 8 * P2W * P2CH + 15) & ~(uintptr_t)15;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
        }
      }
#pragma unroll 1
      for (int ch = 0; ch < P2CH; ++ch) {
        if (ch) __syncthreads();  // the exchange buffer is rewritten by the next chunk
        p2_item<T, M, 8>(zs, it.r * P2CH + ch, sm, threadIdx.x < 243 ? (int)threadIdx.x : -1,
                         ch == 0 ? T8_SCHED : -1, signal, [] { __syncthreads(); });
      }
      }
      PH_MARK(4);
    }
    // thread T8_SCHED, once its share of the item is done: bookkeeping and the selection of
    // the next item, overlapping the other warps' tails (every thread has read s_sel and the
    // slot before the item's first barrier)
    if (threadIdx.x == T8_SCHED) {
      PH_T0;
      if (it.p1 && !skip1) pend = it.j;  // published during the next item (or before a wait)
      if (pslot >= 0) finish_pending();  // the claim decoded one item ago
      // start decoding this item's replacement into its slot (invisible until finished: q =
      // T8_EXH); its order[] entry is copied by cp.async during the next item
      Slot& o = s_slot[sel];
      o.q = T8_EXH;
      set_meta(sel, T8_EXH, false, 0);
      if (claim < total) {
        const ItemDec d = decode_item(claim, ns, N1, N2, lag, args.p2_head);
        HC_ASSERT(d.j < ns && d.r < (d.p1 ? N1 : N2));
        o.p1 = d.p1; o.j = d.j; o.r = d.r;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&o.loc)),
                     "l"(args.order + d.j) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        pslot = sel;
        pq = claim;
      }
      PH_T1(3);
      select_next(false);
    }
    __syncthreads();  // the item's smem is free; s_sel is set
    if constexpr (EPI == 3) {
      // this pass-2 item has read its ring columns: every load's value was consumed before
      // the barrier above, so the slot may be rewritten once the count is seen (no fence:
      // a write-after-read hazard only)
      if (threadIdx.x == T8_SCHED && !it.p1 && !skip2) atomicAdd(p2_done + it.j, 1u);
    }
    if (*(volatile int*)&s_sel == T8_DEFER) {
      __syncthreads();  // everybody has seen T8_DEFER before it is overwritten
      if (threadIdx.x == T8_SCHED) select_next(true);
      __syncthreads();
    }
    PH_MARK(5);
  }
  PH_FLUSH;
}

}  // namespace hc
