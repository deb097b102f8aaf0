// hc_ws.cuh -- warp-specialised two-level slab engine (D >= 13).
//
// Same arithmetic and data layout as slab8_kernel (hc_slab.cuh),
// different schedule.  One CTA per SM, 16 warps (128 registers each):
//   * compute group, warps 0-7: pass-1 tiles back to back -- TMA-fed pair loop (F1 / F2,
//     PAPER.md 166-177 direct split on the top axes, Karatsuba / direct on the tile axes),
//     inverse on the register axes, then the tile's 3^8 values go to the SMEM buffer S;
//   * epilogue group, warps 8-15: the rest of each tile's inverse (B axes, A axes; PAPER.md
//     187-189) and its store into the slab, and every pass-2 item (inverse over the M
//     middle axes of an L2-resident slab, final store).
// The groups meet only at S (mbarriers `full` / `empty`), so the pair loop of tile n+1
// overlaps the exchanges and stores of tile n and the pass-2 items.  Work comes from two
// counters: pass-1 tiles in slab order (slabs sorted by pair count), pass-2 items in slab
// order.  Progress: the compute group never waits on another CTA except for the throttle
// (pass 1 of slab j starts once pass 2 of slab j - lag is done -- which keeps the in-flight
// slabs L2-resident); the epilogue group never blocks while its own S holds a tile, so every
// started tile completes, and a pass-2 item waits only for pass-1 tiles, which depend on
// nothing -- hence no deadlock with one co-resident CTA per SM.
#pragma once
#include "hc_slab.cuh"

namespace hc {

constexpr int WS_NT = 512;
constexpr int WS_CLEAD = 224;  // compute-group scheduler / prefetch thread (warp 7)
constexpr int WS_ELEAD = 256;  // epilogue-group leader (warp 8)
constexpr int WS_BAR_C = 1, WS_BAR_E = 2;  // named barriers of the two groups (256 threads each)

// optional per-group phase counters (-DHC_PHASE_PROF): clock64 sums of the two leaders
#ifdef HC_PHASE_PROF
#define WS_T0 long long wst_ = clock64();
#define WS_ACC(slot) do { long long t_ = clock64(); atomicAdd(&hc_phase[slot], (unsigned long long)(t_ - wst_)); wst_ = t_; } while (0)
#else
#define WS_T0
#define WS_ACC(slot) do { } while (0)
#endif

template <class T, int M>
struct WSCfg {
  static constexpr int P_OFF = 0;
  static constexpr int R_OFF = 2 * PS_SZ;
  static constexpr int S_OFF = R_OFF + T8_NRAW * RS_SZ;
  static constexpr int Q_OFF = S_OFF + 6568;  // 6561 rounded up to 16-byte multiples
  static constexpr int END = Q_OFF + P2Cfg<M>::SIZE;
  static constexpr size_t SMEM = sizeof(T) * (size_t)END;
  static_assert(SMEM <= 227 * 1024, "one CTA per SM");
};

__device__ __forceinline__ void bar_named(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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
__device__ __forceinline__ void mbar_arrive1(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b)) : "memory");
}

// counters (device, zeroed per launch): [0] pass-1 claims, [1] pass-2 claims,
// [2 + j] pass-1 tiles done in slab position j, [2 + ns + j] pass-2 items done in slab j
template <class T, int M>
__global__ void __launch_bounds__(WS_NT, 1)
slabws_kernel(const T* __restrict__ xu, const T* __restrict__ yu, T* __restrict__ z, SlabArgs args) {
  using Cfg = WSCfg<T, M>;
  constexpr uint32_t N1 = (uint32_t)ipow3(M);
  constexpr uint32_t N2 = (uint32_t)(ipow3(8) / P2W);  // 9-column pass-2 items per slab
  constexpr uint64_t SLAB = upow3(M + 8);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* P = sm + Cfg::P_OFF;
  T* R = sm + Cfg::R_OFF;
  T* S = sm + Cfg::S_OFF;
  T* Q = sm + Cfg::Q_OFF;
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  __shared__ __align__(8) uint64_t full_bar, empty_bar;
  __shared__ Prefetch pf;
  constexpr int QN = 3;
  __shared__ uint32_t s_cq[QN];              // pass-1 claims, FIFO (position n in s_cq[n % QN])
  __shared__ uint32_t s_citem[4];            // current tile: q, base, freeb, slab offset
  __shared__ unsigned long long s_tile_dst;  // element offset of the tile handed to the epilogue
  __shared__ uint32_t s_tile_j;
  __shared__ int s_cdone;                    // compute group finished (after its last hand-off)
  __shared__ uint32_t s_ejob[4];             // epilogue job: kind, j, c, loc

  const int tid = threadIdx.x;
  const uint32_t ns = args.nslab;
  const uint32_t total1 = ns * N1, total2 = ns * N2;
  uint32_t* const c_p1 = args.ctr;
  uint32_t* const c_p2 = args.ctr + 1;
  uint32_t* const p1done = args.ctr + 2;
  uint32_t* const p2done = args.ctr + 2 + ns;
  const uint32_t lag = args.lag;

  if (tid == 0) {
    for (int i = 0; i < T8_NRAW; ++i) mbar_init(&raw_bar[i], 1);
    mbar_init(&full_bar, 1);
    mbar_init(&empty_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_cdone = 0;
  }
  __syncthreads();

  if (tid < 256) {
    // =============================== compute group ===============================
    RawRing rr{raw_bar, 0, 0};
    const uint64_t pol_in = policy_evict_first();
    const uint64_t stride = upow3(M) * 256;
    auto dec = [&](uint32_t q, uint32_t& j, uint32_t& r, uint32_t& base, uint32_t& freeb) {
      j = q / N1;
      r = q - j * N1;
      base = args.order[j].y, freeb = args.order[j].z;
    };
    // prefetch cursor over the queued claims (claim order = processing order)
    uint32_t head = 0;  // WS_CLEAD only
    auto next = [&](Prefetch& c) -> bool {
      uint32_t np = (c.pos == T8_EXH) ? head : c.pos + 1;
      if (np < head) np = head;
      if (np - head >= (uint32_t)QN) return false;
      const uint32_t q = s_cq[np % QN];
      if (q >= total1) return false;
      uint32_t j, r, base, freeb;
      dec(q, j, r, base, freeb);
      c.pos = np;
      c.sx0 = xu + (uint64_t)r * 256;
      c.sy0 = yu + (uint64_t)r * 256;
      c.stride = stride;
      c.base = base;
      c.freeb = freeb;
      c.s = 0;
      c.left = 1 << __popc(freeb);
      return true;
    };
    auto pump = [&]() { pf_pump<T>(pf, rr, R, pol_in, next); };
    if (tid == WS_CLEAD) {
      for (int i = 0; i < QN; ++i) s_cq[i] = atomicAdd(c_p1, 1u);
      pf.left = 0;
      pf.pos = T8_EXH;
    }
    const int w = tid >> 5, lane = tid & 31;
    const bool unit = tid < 243;
    const int u = t8_unit(tid);
    const int ea2 = u / 81, eS = u - 81 * ea2;
    const int f1es = t8_f1_es(w);
    uint32_t ntile = 0;
    WS_T0
    while (true) {
      if (tid == WS_CLEAD) {
        WS_ACC(3);  // hand-off and loop overhead
        const uint32_t q = s_cq[head % QN];
        s_citem[0] = q;
        if (q < total1) {
          uint32_t j, r, base, freeb;
          dec(q, j, r, base, freeb);
          s_citem[1] = base;
          s_citem[2] = freeb;
          s_citem[3] = args.order[j].x;
          // throttle: slab j's pass 1 starts once slab j - lag has been finished by pass 2
          if (j >= lag && ld_relaxed(p2done + (j - lag)) < N2) {
            pump();
            while (ld_relaxed(p2done + (j - lag)) < N2) __nanosleep(128);
          }
        }
        WS_ACC(0);  // throttle
      }
      bar_named(WS_BAR_C, 256);
      const uint32_t q = s_citem[0];
      if (q >= total1) break;
      const int npairs = 1 << __popc(s_citem[2]);
      uint32_t claim = 0;
      if (tid == WS_CLEAD) claim = atomicAdd(c_p1, 1u);  // refills position head after this tile

      // ---- pair loop (as tile8, group barrier instead of __syncthreads) ----
      auto f1 = [&](T* Pd) {
        if (f1es >= 0) t8_f1<T>(R + t8_wait(rr) * RS_SZ, Pd, f1es, lane);
        else ++rr.done;
      };
      if (tid == WS_CLEAD) pump();
      f1(P);
      bar_named(WS_BAR_C, 256);
      T acc[27];
#pragma unroll
      for (int i = 0; i < 27; ++i) acc[i] = T(0);
      for (int p = 0; p < npairs; ++p) {
        if (tid == WS_CLEAD) pump();
        if (p + 1 < npairs) f1(P + ((p + 1) & 1) * PS_SZ);
        if (unit) t8_f2<T>(P + (p & 1) * PS_SZ, ea2, eS, acc);
        bar_named(WS_BAR_C, 256);
      }
      if (tid == WS_CLEAD) {
        pump();
        WS_ACC(1);  // pair loop
      }
      // ---- inverse on the register axes, hand the tile to the epilogue group ----
      if (unit) {
        inv_reg<3, T>(acc);
      }
      if (ntile > 0) mbar_wait(&empty_bar, (ntile - 1) & 1);  // S free (tile ntile-1 consumed)
      if (tid == WS_CLEAD) WS_ACC(2);  // waiting for S
      if (unit) {
#pragma unroll
        for (int i = 0; i < 27; ++i) S[u * 27 + i] = acc[i];
      }
      if (tid == WS_CLEAD) {
        const uint32_t j = q / N1, r = q - j * N1;
        s_tile_dst = (unsigned long long)s_citem[3] * SLAB + (unsigned long long)r * 6561ull;
        s_tile_j = j;
      }
      bar_named(WS_BAR_C, 256);  // all of S written
      if (tid == WS_CLEAD) {
        mbar_arrive1(&full_bar);  // release (CTA scope): S and the tile info
        s_cq[head % QN] = claim;
        ++head;
      }
      ++ntile;
    }
    if (tid == WS_CLEAD) {
      // the epilogue learns through s_cdone that no further tile will arrive; the flag is
      // set after the last hand-off (a tile still in S is detected through full_bar first)
      atomicExch(&s_cdone, 1);
    }
  } else {
    // =============================== epilogue group ==============================
    const int et = tid - 256;
    const bool etask = et < 243;
    const uint64_t pol_keep = policy_evict_last();
    uint32_t nt = 0;          // tiles consumed
    uint32_t q2 = T8_EXH;     // leader: current pass-2 claim (T8_EXH = none yet)
    uint32_t pend[2] = {T8_EXH, T8_EXH};  // leader: finished tiles to publish (slab positions)
    auto publish_one = [&]() {  // publish the older pending tile (its stores have drained)
      if (pend[0] != T8_EXH) {
        __threadfence();
        atomicAdd(p1done + pend[0], 1u);
      }
      pend[0] = pend[1];
      pend[1] = T8_EXH;
    };
    WS_T0
    while (true) {
      if (tid == WS_ELEAD) {
        uint32_t kind = 0, j = 0, c = 0;
        while (true) {
          if (mbar_test(&full_bar, nt & 1)) { kind = 1; break; }
          if (q2 == T8_EXH) q2 = atomicAdd(c_p2, 1u);
          if (q2 < total2) {
            j = q2 / N2;
            c = q2 - j * N2;
            if (ld_relaxed(p1done + j) >= N1) { kind = 2; break; }
          } else if (*(volatile int*)&s_cdone && !mbar_test(&full_bar, nt & 1)) {
            kind = 0;  // no pass-2 work left and no tile will come
            break;
          }
          // idle: publish what is pending (the fence is cheap now), then poll again
          publish_one();
          publish_one();
          __nanosleep(64);
        }
        WS_ACC(6);  // idle / polling
        s_ejob[0] = kind;
        s_ejob[1] = j;
        s_ejob[2] = c;
        s_ejob[3] = kind == 2 ? args.order[j].x : 0;
        if (kind == 2) q2 = T8_EXH;
      }
      bar_named(WS_BAR_E, 256);
      const uint32_t kind = s_ejob[0];
      if (kind == 0) break;
      if (kind == 1) {
        // ---- tile epilogue: B axes, then A axes + store (a4, a6) ----
        const uint64_t dst = s_tile_dst;
        const uint32_t tj = s_tile_j;
        if (etask) {
          const int a = et / 27, cc = et - 27 * a;
          T v[27];
#pragma unroll
          for (int e = 0; e < 27; ++e) v[e] = S[a * 729 + e * 27 + cc];
          inv_reg<3, T>(v);
#pragma unroll
          for (int e = 0; e < 27; ++e) S[a * 729 + e * 27 + cc] = v[e];
        }
        bar_named(WS_BAR_E, 256);
        if (tid == WS_ELEAD) publish_one();  // only SMEM traffic since the last job's stores
        if (etask) {
          T* zt = z + dst;
#pragma unroll 1
          for (int r = 0; r < 3; ++r) {
            const int col = r * 243 + et;
            T v[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) v[e] = S[e * 729 + col];
            inv_reg<2, T>(v);
#pragma unroll
            for (int e = 0; e < 9; ++e) st_hint(zt + e * 729 + col, v[e], pol_keep);
          }
        }
        bar_named(WS_BAR_E, 256);  // S fully read
        if (tid == WS_ELEAD) {
          mbar_arrive1(&empty_bar);
          if (pend[0] == T8_EXH) pend[0] = tj;
          else pend[1] = tj;
          if (pend[1] != T8_EXH) publish_one();  // keep at most one pending
        }
        ++nt;
        if (tid == WS_ELEAD) WS_ACC(4);  // tile epilogue
      } else {
        // ---- pass-2 item (a5, a6): slab position j, columns [9c, 9c + 9) ----
        // the slab's tiles are complete (relaxed read of its counter saw N1, then the group
        // barrier orders these L2 (.cg) reads after it; producers fenced before counting)
        const uint32_t j = s_ejob[1], c = s_ejob[2], loc = s_ejob[3];
        p2_item<T, M, 8>(z + (uint64_t)loc * SLAB, c, Q, etask ? et : -1, WS_ELEAD, publish_one,
                         [] { bar_named(WS_BAR_E, 256); });
        if (tid == WS_ELEAD) {
          atomicAdd(p2done + j, 1u);  // progress for the throttle only
          WS_ACC(5);                  // pass-2 item
        }
      }
    }
    if (tid == WS_ELEAD) {
      publish_one();
      publish_one();
    }
  }
}

// ---- warp-specialised single-level engine (8 <= D <= 12, batched D >= 8) ---------------
// Compute group: tiles w = blockIdx.x, + gridDim.x, ... (item w: batch w / nslab, top index
// slab0 + w % nslab; prefetcher over the same sequence), pair loop + register-axes inverse,
// tile to S.  Epilogue group: B and A axes, final streaming store to z[w * 6561 ...].  The
// last hand-off carries an end marker.
struct TWSCfg {
  static constexpr int S_OFF = 2 * PS_SZ + T8_NRAW * RS_SZ;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(S_OFF + 6568);
};

template <class T>
__global__ void __launch_bounds__(WS_NT, 1)
tilews_kernel(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ z, int D, uint64_t slab0,
              uint64_t nslab, uint64_t nitems) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* P = sm;
  T* R = sm + 2 * PS_SZ;
  T* S = sm + TWSCfg::S_OFF;
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  __shared__ __align__(8) uint64_t full_bar, empty_bar;
  __shared__ Prefetch pf;
  __shared__ unsigned long long s_dst;  // element offset of the tile in S, ~0ull = end
  const int tid = threadIdx.x;
  constexpr unsigned long long END = ~0ull;
  if (tid == 0) {
    for (int i = 0; i < T8_NRAW; ++i) mbar_init(&raw_bar[i], 1);
    mbar_init(&full_bar, 1);
    mbar_init(&empty_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < 256) {
    // ------------------------------- compute group --------------------------------
    RawRing rr{raw_bar, 0, 0};
    const int k = D - 8;
    const uint64_t pol_in = policy_evict_last();
    if (tid == WS_CLEAD) {
      pf.left = 0;
      pf.pos = 0xffffffffu;
    }
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
    const int w8 = tid >> 5, lane = tid & 31;
    const bool unit = tid < 243;
    const int u = t8_unit(tid);
    const int ea2 = u / 81, eS = u - 81 * ea2;
    const int f1es = t8_f1_es(w8);
    auto f1 = [&](T* Pd) {
      if (f1es >= 0) t8_f1<T>(R + t8_wait(rr) * RS_SZ, Pd, f1es, lane);
      else ++rr.done;
    };
    uint32_t ntile = 0;
    for (uint64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
      const uint64_t b = w / nslab;
      uint32_t base, freeb;
      trit_split(slab0 + (w - b * nslab), k, base, freeb);
      const int npairs = 1 << __popc(freeb);
      if (tid == WS_CLEAD) pump();
      f1(P);
      bar_named(WS_BAR_C, 256);
      T acc[27];
#pragma unroll
      for (int i = 0; i < 27; ++i) acc[i] = T(0);
      for (int p = 0; p < npairs; ++p) {
        if (tid == WS_CLEAD) pump();
        if (p + 1 < npairs) f1(P + ((p + 1) & 1) * PS_SZ);
        if (unit) t8_f2<T>(P + (p & 1) * PS_SZ, ea2, eS, acc);
        bar_named(WS_BAR_C, 256);
      }
      if (tid == WS_CLEAD) pump();
      if (unit) inv_reg<3, T>(acc);
      if (ntile > 0) mbar_wait(&empty_bar, (ntile - 1) & 1);
      if (unit) {
#pragma unroll
        for (int i = 0; i < 27; ++i) S[u * 27 + i] = acc[i];
      }
      if (tid == WS_CLEAD) s_dst = (unsigned long long)w * 6561ull;
      bar_named(WS_BAR_C, 256);
      if (tid == WS_CLEAD) mbar_arrive1(&full_bar);
      ++ntile;
    }
    if (tid == WS_CLEAD) {  // end marker, once the epilogue has taken the last tile
      if (ntile > 0) mbar_wait(&empty_bar, (ntile - 1) & 1);
      s_dst = END;
      mbar_arrive1(&full_bar);
    }
  } else {
    // ------------------------------- epilogue group -------------------------------
    const int et = tid - 256;
    const bool etask = et < 243;
    for (uint32_t nt = 0;; ++nt) {
      mbar_wait(&full_bar, nt & 1);
      const unsigned long long dst = s_dst;
      if (dst == END) break;
      if (etask) {  // B axes
        const int a = et / 27, cc = et - 27 * a;
        T v[27];
#pragma unroll
        for (int e = 0; e < 27; ++e) v[e] = S[a * 729 + e * 27 + cc];
        inv_reg<3, T>(v);
#pragma unroll
        for (int e = 0; e < 27; ++e) S[a * 729 + e * 27 + cc] = v[e];
      }
      bar_named(WS_BAR_E, 256);
      if (etask) {  // A axes + final store
        T* zt = z + dst;
#pragma unroll 1
        for (int r = 0; r < 3; ++r) {
          const int col = r * 243 + et;
          T v[9];
#pragma unroll
          for (int e = 0; e < 9; ++e) v[e] = S[e * 729 + col];
          inv_reg<2, T>(v);
#pragma unroll
          for (int e = 0; e < 9; ++e) st_cs(zt + e * 729 + col, v[e]);
        }
      }
      bar_named(WS_BAR_E, 256);  // S fully read
      if (tid == WS_ELEAD) mbar_arrive1(&empty_bar);
    }
  }
}

}  // namespace hc
