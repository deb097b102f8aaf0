// hc_slabx.cuh -- the warp-specialised two-level slab engine (D >= 13), one CTA per SM.
//
// Same arithmetic and geometry as slab8_kernel (hc_slab.cuh): per-axis split
// (PAPER.md 185-192) on the 8 tile axes and the M middle axes, the paper's 4-way direct split
// (PAPER.md 166-177) on the k top axes; pass 1 writes each 3^8 tile of a slab in the
// evaluation domain of the middle axes into z (L2-resident), pass 2 interpolates the middle
// axes in place.  What differs is the schedule: instead of fork-join CTAs that alternate
// pair loop, tile interpolation and pass 2 behind CTA barriers, three roles run concurrently
// on their own warps and hand work over through mbarriers:
//
//   warps 0-7   F2  ("pair loop"): 243 units, 27 fp64/uint64 accumulators per thread (register
//                   axes C = tile axes 0-2), unit of thread t = t8_unit(t) (the two-row e_a2 = 1
//                   units grouped on warps 0-2, as in slab8).
//   warps 8-10  F1  : evaluate tile axes a1 (warp 8 + e_s) and B of each pair's raw slices
//                   (TMA ring) into the double-buffered F1 stage.
//   warp 11     S   : claims pass-1 items, issues the TMA copies of their raw slices, throttles
//                   pass 1 behind pass 2 (L2 residency of at most ~LAG slabs).
//   warps 12-19 E   : epilogue -- tile interpolation + store of each finished tile, and pass-2
//                   items (middle-axes interpolation + final streaming store).
//
// Hand-over F2 -> E goes through tensor memory (TMEM, 256 KB per SM, otherwise idle in this
// fp64 / int64 kernel): at the end of a tile every F2 thread writes its 27 accumulators into
// TMEM (tcgen05.st, 54 columns of its lane) and starts the next tile at once; the E warp of
// the same lane quadrant (warp 12 + w reads the lanes of warp w) loads them (tcgen05.ld) and
// runs the tile interpolation while the pair loop goes on.  Four TMEM tile buffers (4 x 128
// columns) decouple the two roles.  Registers are split per warpgroup (setmaxnreg): F2 120,
// F1 + S 64, E 88 per thread.
//
// Progress / deadlock freedom (grid = one resident CTA per SM):
//  * S claims the next pass-1 item only after issuing every slice of the previous one, and only
//    then waits on the throttle (pass 2 of slab position j - LAG finished).  That pass 2 depends
//    on tiles of strictly earlier positions, whose slices are all issued (or throttled on yet
//    earlier positions): induction on the position.
//  * F1/F2 wait only on S (slices, items) and on E (free TMEM buffer); E never waits on P: its
//    leader polls for a finished tile or a ready pass-2 item, and a held pass-2 item only waits
//    for tiles of its slab, which are handed to E's of their CTAs and interpolated there.
#pragma once
#include "hc_slab.cuh"

namespace hc {

constexpr int SX_NT = 640;                   // 20 warps = 5 warpgroups
constexpr int SX_F1W = 8;                    // first F1 warp
constexpr int SX_SW = 11;                    // scheduler warp
constexpr int SX_S = SX_SW * 32;             // scheduler thread
constexpr int SX_E0 = 384;                   // first E thread (warp 12)
constexpr int SX_PN = 352;                   // F2 + F1 threads (named barrier 1)
constexpr int SX_EN = 256;                   // E threads (named barrier 2)
constexpr int SX_QN = 4;                     // item queue S -> P
constexpr int SX_NBUF = 4;                   // TMEM tile buffers P -> E
#ifndef HC_SX_NRAW
#define HC_SX_NRAW 10
#endif
constexpr int SX_NRAW = HC_SX_NRAW;          // raw-slice TMA ring stages

template <class T, int M>
struct SXCfg {
  static constexpr int EBUF = P2Cfg<M>::SIZE > 6561 ? P2Cfg<M>::SIZE : 6561;
  static constexpr int P_OFF = 0;                          // [2][PS_SZ] F1 stage
  static constexpr int R_OFF = 2 * PS_SZ;                  // [NRAW][RS_SZ] raw ring
  static constexpr int E_OFF = R_OFF + SX_NRAW * RS_SZ;    // [EBUF] epilogue exchange
  static constexpr size_t SMEM = sizeof(T) * (size_t)(E_OFF + EBUF);
};

struct SXItem {
  uint64_t dest;   // element offset of the tile in z
  uint32_t npairs; // 0xffffffff = no more items
  uint32_t j;      // slab position
};
struct SXTile {
  uint64_t dest;
  uint32_t j;
  uint32_t pad;
};

struct SlabxArgs {
  uint32_t nslab;      // slabs in this launch
  uint32_t lag;        // pass 1 of position j starts after pass 2 of position j - lag finished
  uint32_t* ctr;       // [0] pass-1 claims, [1] pass-2 claims, [2 + j] tiles done, [2 + ns + j] pass-2 done
  const uint4* order;  // position j -> {slab offset, base, freeb, problem b} (as SlabArgs::order)
  uint64_t bstride;    // elements between consecutive problems' middle-axes tables (batch)
};

// ---- small PTX wrappers ----------------------------------------------------------------
__device__ __forceinline__ void bar_named(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 27 64-bit values <-> 54 TMEM columns of this thread's lane (32x32b shape: lane = thread)
template <class T>
__device__ __forceinline__ void tmem_st27(uint32_t ta, const T* v) {
  uint32_t w[54];
#pragma unroll
  for (int i = 0; i < 27; ++i) {
    uint64_t b;
    memcpy(&b, &v[i], 8);
    w[2 * i] = (uint32_t)b;
    w[2 * i + 1] = (uint32_t)(b >> 32);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),
      "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]),
      "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]),
      "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
      : "memory");
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          ta + 32),
      "r"(w[32]), "r"(w[33]), "r"(w[34]), "r"(w[35]), "r"(w[36]), "r"(w[37]), "r"(w[38]), "r"(w[39]), "r"(w[40]),
      "r"(w[41]), "r"(w[42]), "r"(w[43]), "r"(w[44]), "r"(w[45]), "r"(w[46]), "r"(w[47])
      : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta + 48), "r"(w[48]), "r"(w[49]),
               "r"(w[50]), "r"(w[51])
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(ta + 52), "r"(w[52]), "r"(w[53])
               : "memory");
}
template <class T>
__device__ __forceinline__ void tmem_ld27(uint32_t ta, T* v) {
  uint32_t w[54];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
        "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]),
        "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]),
        "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
      : "r"(ta));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(w[32]), "=r"(w[33]), "=r"(w[34]), "=r"(w[35]), "=r"(w[36]), "=r"(w[37]), "=r"(w[38]), "=r"(w[39]),
        "=r"(w[40]), "=r"(w[41]), "=r"(w[42]), "=r"(w[43]), "=r"(w[44]), "=r"(w[45]), "=r"(w[46]), "=r"(w[47])
      : "r"(ta + 32));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w[48]), "=r"(w[49]), "=r"(w[50]), "=r"(w[51])
               : "r"(ta + 48));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(w[52]), "=r"(w[53]) : "r"(ta + 52));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 27; ++i) {
    const uint64_t b = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    memcpy(&v[i], &b, 8);
  }
}

#ifdef HC_PHASE_PROF
#define SX_PROF_ADD(i, v) atomicAdd(&hc_phase[i], (unsigned long long)(v))
#else
#define SX_PROF_ADD(i, v) do { } while (0)
#endif

template <class T, int M>
__global__ void __launch_bounds__(SX_NT, 1)
slabx_kernel(const T* __restrict__ xu, const T* __restrict__ yu, T* __restrict__ z, SlabxArgs args) {
  using Cfg = SXCfg<T, M>;
  constexpr uint32_t N1 = (uint32_t)ipow3(M);                        // pass-1 tiles per slab
  constexpr uint32_t N2 = (uint32_t)(ipow3(8) / (P2W * T8_P2CH));    // pass-2 items per slab
  constexpr uint64_t SLAB = upow3(M + 8);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* const Pst = sm + Cfg::P_OFF;
  T* const R = sm + Cfg::R_OFF;
  T* const Eb = sm + Cfg::E_OFF;
  __shared__ __align__(8) uint64_t raw_full[SX_NRAW], raw_empty[SX_NRAW];
  __shared__ __align__(8) uint64_t item_full[SX_QN], item_empty[SX_QN];
  __shared__ __align__(8) uint64_t acc_full[SX_NBUF], acc_empty[SX_NBUF];
  __shared__ SXItem s_item[SX_QN];
  __shared__ SXTile s_tile[SX_NBUF];
  __shared__ uint32_t s_taddr;
  __shared__ volatile uint32_t s_ptiles;   // tiles handed to E in total (set when P is done)
  __shared__ uint4 s_edec;                 // E leader's decision {kind, a, b, c}

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t ns = args.nslab;
  const uint32_t total1 = ns * N1, total2 = ns * N2;
  uint32_t* const ctr1 = args.ctr;
  uint32_t* const ctr2 = args.ctr + 1;
  uint32_t* const done_ctr = args.ctr + 2;
  uint32_t* const p2fin = args.ctr + 2 + ns;

  if (tid == 0) {
    for (int i = 0; i < SX_NRAW; ++i) { mbar_init(&raw_full[i], 1); mbar_init(&raw_empty[i], 3); }
    for (int i = 0; i < SX_QN; ++i) { mbar_init(&item_full[i], 1); mbar_init(&item_empty[i], 1); }
    for (int i = 0; i < SX_NBUF; ++i) { mbar_init(&acc_full[i], 8); mbar_init(&acc_empty[i], 8); }
    s_ptiles = 0xffffffffu;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == SX_SW) {  // TMEM: all 512 columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s_taddr;

  // per-warpgroup register budgets (pool 640 x 96): F2 2 x 128 x 120, F1 + S 128 x 64, E 2 x 128 x 88
  if (warp < 8) asm volatile("setmaxnreg.inc.sync.aligned.u32 120;");
  else if (warp < 12) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
  else asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");

  if (warp < 8) {
    // ================================ F2 ==================================================
    const bool unit = tid < 243;
    const int uu = t8_unit(tid);           // e_a2 = 1 units on warps 0-2 (two-row loads)
    const int ea2 = uu / 81, eS = uu - 81 * ea2;
    const uint32_t tcol = tbase + (((uint32_t)(warp & 3) * 32u) << 16) + (uint32_t)(warp >> 2) * 64u;
    uint32_t qpos = 0, tb = 0;
#ifdef HC_PHASE_PROF
    long long tk0 = clock64();
#endif
    while (true) {
      const uint32_t slot = qpos % SX_QN;
#ifdef HC_PHASE_PROF
      long long tw0 = clock64();
#endif
      mbar_wait(&item_full[slot], (qpos / SX_QN) & 1);
#ifdef HC_PHASE_PROF
      if (tid == 0) SX_PROF_ADD(5, clock64() - tw0);
      long long tp0 = clock64();
#endif
      const SXItem it = s_item[slot];
      ++qpos;
      if (it.npairs == 0xffffffffu) break;
      T acc[27];
#pragma unroll
      for (int i = 0; i < 27; ++i) acc[i] = T(0);
      bar_named(1, SX_PN);  // F1(0) is in the stage; every P thread has read the item
      for (uint32_t p = 0; p < it.npairs; ++p) {
        if (unit) t8_f2<T>(Pst + (p & 1) * PS_SZ, ea2, eS, acc);
        bar_named(1, SX_PN);
      }
      // hand the accumulators to E through TMEM buffer b
      const uint32_t b = tb % SX_NBUF;
#ifdef HC_PHASE_PROF
      long long ta0 = clock64();
      if (tid == 0) SX_PROF_ADD(6, ta0 - tp0);
#endif
      if (tb >= SX_NBUF) mbar_wait(&acc_empty[b], ((tb / SX_NBUF) + 1) & 1);
#ifdef HC_PHASE_PROF
      if (tid == 0) SX_PROF_ADD(4, clock64() - ta0);
#endif
      tc_fence_after();
      if (tid == 0) { s_tile[b].dest = it.dest; s_tile[b].j = it.j; }
      tmem_st27<T>(tcol + b * 128u, acc);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_full[b]);
      ++tb;
    }
    if (tid == 0) s_ptiles = tb;
#ifdef HC_PHASE_PROF
    if (tid == 0) SX_PROF_ADD(9, clock64() - tk0);
#endif
  } else if (warp < SX_SW) {
    // ================================ F1 ==================================================
    const int es = warp - SX_F1W;
    uint32_t qpos = 0, rdone = 0;
    while (true) {
      const uint32_t slot = qpos % SX_QN;
      mbar_wait(&item_full[slot], (qpos / SX_QN) & 1);
      const uint32_t np = s_item[slot].npairs;
      ++qpos;
      if (np == 0xffffffffu) break;
      for (uint32_t p = 0; p <= np; ++p) {
        if (p < np) {  // F1 of pair p into stage p & 1
          const uint32_t st = rdone % SX_NRAW;
#ifdef HC_PHASE_PROF
          long long tr0 = clock64();
#endif
          mbar_wait(&raw_full[st], (rdone / SX_NRAW) & 1);
#ifdef HC_PHASE_PROF
          if (es == 0 && lane == 0) SX_PROF_ADD(7, clock64() - tr0);
#endif
          t8_f1<T>(R + st * RS_SZ, Pst + (p & 1) * PS_SZ, es, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&raw_empty[st]);
          ++rdone;
        }
        bar_named(1, SX_PN);
        // the item slot is released after the tile's first barrier (every P thread has read it)
        if (p == 0 && es == 0 && lane == 0) mbar_arrive(&item_empty[slot]);
      }
    }
  } else if (warp == SX_SW) {
    // ================================ S ===================================================
    if (lane == 0) {
      const uint64_t pol_in = policy_evict_first();  // middle-axes tables are streamed
      const uint64_t stride = upow3(M) * 256;
      uint32_t qslot = 0, rseq = 0;
      uint32_t q = atomicAdd(ctr1, 1u);
      while (true) {
        const bool more = q < total1;
        uint32_t j = 0, r = 0;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (more) {
          j = q / N1;
          r = q - j * N1;
          o = args.order[j];
          // throttle: pass 2 of position j - lag has finished (its slab left L2)
          if (j >= args.lag) {
            long long t0 = clock64();
            while (ld_acquire(p2fin + (j - args.lag)) < N2) __nanosleep(128);
            SX_PROF_ADD(0, clock64() - t0);
          }
        }
        const uint32_t slot = qslot % SX_QN;
        if (qslot >= SX_QN) mbar_wait(&item_empty[slot], ((qslot / SX_QN) + 1) & 1);
        SXItem itm;
        itm.npairs = more ? (1u << __popc(o.z)) : 0xffffffffu;
        itm.dest = (uint64_t)o.x * SLAB + (uint64_t)r * 6561ull;
        itm.j = j;
        s_item[slot] = itm;
        mbar_arrive(&item_full[slot]);
        ++qslot;
        if (!more) break;
        // the item's raw slices, pairs in ascending subsets of freeb (PAPER.md 173-177)
        const T* sx0 = xu + (uint64_t)o.w * args.bstride + (uint64_t)r * 256;
        const T* sy0 = yu + (uint64_t)o.w * args.bstride + (uint64_t)r * 256;
        const uint32_t base = o.y, freeb = o.z;
        uint32_t s = 0;
        do {
          const uint32_t st = rseq % SX_NRAW;
#ifdef HC_PHASE_PROF
          long long ts0 = clock64();
#endif
          if (rseq >= SX_NRAW) mbar_wait(&raw_empty[st], ((rseq / SX_NRAW) + 1) & 1);
#ifdef HC_PHASE_PROF
          SX_PROF_ADD(8, clock64() - ts0);
#endif
          fence_proxy_async();  // the stage was last read through the generic proxy
          const uint64_t iT = base | s, jT = base | (freeb & ~s);
          const T* sx = sx0 + iT * stride;
          const T* sy = sy0 + jT * stride;
          T* dst = R + st * RS_SZ;
          uint64_t* bar = &raw_full[st];
          mbar_arrive_tx(bar, 2 * 256 * sizeof(T));
          tma_load_1d(dst, sx, 128 * sizeof(T), bar, pol_in);
          tma_load_1d(dst + RS_H2, sx + 128, 128 * sizeof(T), bar, pol_in);
          tma_load_1d(dst + RS_OP, sy, 128 * sizeof(T), bar, pol_in);
          tma_load_1d(dst + RS_OP + RS_H2, sy + 128, 128 * sizeof(T), bar, pol_in);
          ++rseq;
          s = (s - freeb) & freeb;
        } while (s != 0);
        q = atomicAdd(ctr1, 1u);
      }
    }
    __syncwarp();
  } else {
    // ================================ E ===================================================
    // Work items: tile epilogues (from the local F2 warps, through TMEM) and pass-2 items
    // (three 9-column chunks of a slab whose tiles are all stored).
    const int e = tid - SX_E0;         // 0..255
    const int we = e >> 5;             // reads the TMEM lanes of F2 warp we
    const bool task = e < 243;
    const int u = t8_unit(e);          // unit of F2 thread e (same TMEM lane)
    const uint32_t tcol = tbase + (((uint32_t)(we & 3) * 32u) << 16) + (uint32_t)(we >> 2) * 64u;
    const uint64_t pol_keep = policy_evict_last();  // pass-1 tiles wait in L2 for pass 2
    constexpr uint32_t NONE = 0xffffffffu;
    uint32_t te = 0;                    // tiles taken from P
    // leader state (thread e = 0 only; in shared memory, off the other threads' registers)
    __shared__ struct {
      uint32_t held;                    // claimed pass-2 item
      uint32_t exhausted;               // pass-2 claims exhausted
      uint32_t pend;                    // slab position of a stored, not yet published tile
    } L;
    if (e == 0) { L.held = L.pend = NONE; L.exhausted = 0; }
    auto signal = [&]() {               // leader: publish a tile (fence + count)
      if (L.pend != NONE) {
        __threadfence();
        atomicAdd(done_ctr + L.pend, 1u);
        L.pend = NONE;
      }
    };
    while (true) {
      if (e == 0) {
        long long t0 = clock64();
        (void)t0;
        uint4 dec = make_uint4(0, 0, 0, 0);  // x: 1 tile, 2 pass-2 item (y), 3 exit
        while (true) {
          if (mbar_test(&acc_full[te % SX_NBUF], (te / SX_NBUF) & 1)) { dec.x = 1; break; }
          if (L.held == NONE && !L.exhausted) {
            const uint32_t q2 = atomicAdd(ctr2, 1u);
            if (q2 < total2) L.held = q2;
            else L.exhausted = 1;
          }
          if (L.held != NONE && ld_relaxed(done_ctr + L.held / N2) >= N1) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire the slab's tiles
            dec.x = 2; dec.y = L.held; L.held = NONE; break;
          }
          if (L.held == NONE && L.exhausted && s_ptiles == te) { dec.x = 3; break; }
          signal();
          __nanosleep(32);
        }
        SX_PROF_ADD(1, clock64() - t0);
        s_edec = dec;
      }
      bar_named(2, SX_EN);
      const uint4 dec = s_edec;
      if (dec.x == 3) break;
      if (dec.x == 1) {
        // ---- tile epilogue: TMEM -> registers -> interpolation over the 8 tile axes ----
        long long t0 = clock64();
        (void)t0;
        const uint32_t b = te % SX_NBUF;
        tc_fence_after();
        const SXTile tl = s_tile[b];
        T v[27];
        tmem_ld27<T>(tcol + b * 128u, v);
        tc_fence_before();
        __syncwarp();
        if ((e & 31) == 0) mbar_arrive(&acc_empty[b]);
        ++te;
        // a4: inverse on the C register axes, then B (exchange), then A + store (a6)
        if (task) {
          inv_reg<3, T>(v);
#pragma unroll
          for (int i = 0; i < 27; ++i) Eb[u * 27 + i] = v[i];
        }
        bar_named(2, SX_EN);
        if (e == 0) signal();  // previous tile: its stores have drained by now
        if (task) {
          const int c = e / 9, a = e - 9 * c;  // e_A fastest: conflict-free (stride 729 = 9 mod 16)
#pragma unroll
          for (int i = 0; i < 27; ++i) v[i] = Eb[a * 729 + i * 27 + c];
          inv_reg<3, T>(v);
#pragma unroll
          for (int i = 0; i < 27; ++i) Eb[a * 729 + i * 27 + c] = v[i];
        }
        bar_named(2, SX_EN);
        T* zt = z + tl.dest;
#pragma unroll 1
        for (int r = 0; r < 3; ++r) {
          if (task) {
            const int col = r * 243 + e;
            T w9[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) w9[i] = Eb[i * 729 + col];
            inv_reg<2, T>(w9);
#pragma unroll
            for (int i = 0; i < 9; ++i) st_hint(zt + i * 729 + col, w9[i], pol_keep);
          }
        }
        // every E thread's stores of this tile are issued once all arrive here; the leader then
        // owns the tile's publication (the others go on to the next decision barrier).  It must
        // not wait for the next item: a pass-2 item of this slab may be what the leader waits for.
        // (warp-uniform: the leader's warp waits, the other E warps only arrive)
        if (e < 32) {
          asm volatile("bar.sync 3, %0;" ::"r"(SX_EN) : "memory");
          if (e == 0) {
            if (L.pend != NONE) signal();
            L.pend = tl.j;
            SX_PROF_ADD(2, clock64() - t0);
            SX_PROF_ADD(10, 1);
          }
        } else {
          asm volatile("bar.arrive 3, %0;" ::"r"(SX_EN) : "memory");
        }
      } else {
        // ---- pass-2 item: interpolation over the M middle axes, in place, final store ----
        long long t0 = clock64();
        (void)t0;
        const uint32_t q2 = dec.y;
        const uint32_t j2 = q2 / N2, r2 = q2 - j2 * N2;
        T* zs = z + (uint64_t)args.order[j2].x * SLAB;
#pragma unroll 1
        for (int ch = 0; ch < T8_P2CH; ++ch) {
          if (ch) bar_named(2, SX_EN);
          p2_item<T, M, 8>(zs, r2 * T8_P2CH + ch, Eb, task ? e : -1, ch == 0 ? SX_E0 : -1, signal,
                           [] { bar_named(2, SX_EN); });
        }
        // (the next decision barrier orders every thread's reads of Eb before its reuse)
        if (e == 0) {
          atomicAdd(p2fin + j2, 1u);  // throttle only (no data is published through it)
          SX_PROF_ADD(3, clock64() - t0);
          SX_PROF_ADD(11, 1);
        }
      }
    }
    if (e == 0) signal();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == SX_SW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

}  // namespace hc
