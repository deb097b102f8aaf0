// hc_tile8n.cuh -- batched D = 8 int64 cubes computed in the 32-bit ring (BASELINE.json config 2).
//
// The whole pipeline -- forward (a0, a0 + a1, a1), pointwise product, inverse
// (c0, (c1 - c0) - c2, c2) (PAPER.md 185-192) -- is a ring homomorphism (reading R3),
// so computing it mod 2^32 gives every output exactly mod 2^32; when the true output lies in
// [-2^31, 2^31) that residue, sign-extended, IS the int64 result.  A cube is safe when
// 2^D max|x| max|y| < 2^31 (every output is a sum of at most 2^D products x[i] y[j]).  The
// kernel checks that bound per cube from the inputs it has already staged (no host round trip):
// safe cubes are computed with 32-bit words -- half the shared-memory traffic of the 64-bit
// tile (F1 stage and tile exchange), one IMAD per multiply-add instead of the five of a 64-bit
// one, 27 accumulator registers instead of 54, so four CTAs fit per SM instead of two -- and
// every unsafe cube is appended to a list that the 64-bit engine (tile8_kernel over the list)
// then computes.  For config 2 (entries in [0, 255]) every cube is safe: 2^8 255^2 < 2^31.
//
// Tile axes and roles as tile8 (hc_slab.cuh): C = {0,1,2} register axes, B = {3,4,5} and
// a1 = 6 evaluated by the F1 warps (3, 4, 6), a2 = 7 summed by the F2 threads while loading.
#pragma once
#include "hc_slab.cuh"

namespace hc {

// F1 stage of 32-bit words: op * PN_OP + b_a2 * PN_A2 + e_S * PN_ROW + b_C.  PN_ROW = 12 words:
// the F2 lanes (consecutive e_S) read 16 B at a 48-B stride, conflict-free per quarter warp;
// PN_A2 = 8, PN_OP = 16 (mod 32): the 32 F1 lanes (op, b_a2, b_C) store to 32 distinct banks.
// The CTA's three store rounds are kept in step by barriers (0.688 vs 0.700 ms at config 2,
// as for the 64-bit tile).  Measured and dropped: P and S in separate buffers with a 2-stage
// raw ring, three barriers per cube instead of five (0.706 ms with the rounds in step, 0.726
// without): the next cube's F1 then overlaps the stores, which costs more than the barriers.
#ifndef HC_T8N_INSTEP
#define HC_T8N_INSTEP 1
#endif
constexpr int PN_ROW = 12, PN_A2 = 1000, PN_OP = 2000, PN_SZ = 4000;
constexpr int T8N_S = 6561;                           // tile exchange (32-bit words), aliases P
constexpr int T8N_ALIAS = T8N_S > PN_SZ ? T8N_S : PN_SZ;
// shared memory: [ALIAS words][raw ring of T8_NRAW stages of RS_SZ 64-bit words]
constexpr size_t T8N_SMEM = (size_t)((T8N_ALIAS * 4 + 15) / 16 * 16) + (size_t)T8_NRAW * RS_SZ * 8;

__device__ __forceinline__ void lds4(const uint32_t* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void st_cs_i64(uint64_t* p, uint32_t v) {  // sign-extended residue
  const uint64_t s = (uint64_t)(int64_t)(int32_t)v;
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(s) : "memory");
}
// |v| of an int64 as uint64 (INT64_MIN -> 2^63)
__device__ __forceinline__ uint64_t abs64(uint64_t v) { return (int64_t)v < 0 ? 0ull - v : v; }

template <int D>
__global__ void __launch_bounds__(T8_NT, 4)
tile8n_kernel(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y, uint64_t* __restrict__ z,
              uint64_t nitems, uint32_t* __restrict__ fb_count, uint32_t* __restrict__ fb_list) {
  static_assert(D == 8, "one 3^8 tile per cube");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* P = reinterpret_cast<uint32_t*>(smem_raw);   // F1 stage, then the tile exchange S
  uint32_t* S = P;
  uint64_t* R = reinterpret_cast<uint64_t*>(smem_raw + (T8N_ALIAS * 4 + 15) / 16 * 16);
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  __shared__ Prefetch pf;
  __shared__ uint32_t s_mag[2];  // max |x| and max |y| of the cube (saturated at 2^31)
  ring_init(raw_bar);
  RawRing<> rr{raw_bar, 0, 0};
  const uint64_t pol_in = policy_evict_first();  // every cube's inputs are read once
  if (threadIdx.x == T8_SCHED) {
    pf.left = 0;
    pf.pos = 0xffffffffu;
  }
  auto next = [&](Prefetch& c) -> bool {
    const uint32_t np = c.pos + 1;
    const uint64_t w = blockIdx.x + (uint64_t)np * gridDim.x;
    if (w >= nitems) return false;
    c.pos = np;
    c.sx0 = x + (w << D);
    c.sy0 = y + (w << D);
    c.stride = 256;
    c.base = 0;
    c.freeb = 0;
    c.s = 0;
    c.left = 1;
    return true;
  };
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const bool unit = tid < 243;
  const int u = t8_unit(tid);
  const int ea2 = u / 81, eS = u - 81 * ea2;
  const int f1es = t8_f1_es(w);
  for (uint64_t cube = blockIdx.x; cube < nitems; cube += gridDim.x) {
    if (tid == T8_SCHED) pf_pump<uint64_t>(pf, rr, R, pol_in, next);
    // ---- F1: evaluate a1 (at e_s) and the B axes of the cube's inputs, mod 2^32 ----
    if (f1es >= 0) {
      const uint64_t* src = R + t8_wait(rr) * RS_SZ;
      const int op = lane >> 4, ba2 = (lane >> 3) & 1, bc = lane & 7;
      const uint64_t* s0 = src + op * RS_OP + ba2 * RS_H2 + bc;
      uint32_t in[8];
      if (f1es != 1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) in[j] = (uint32_t)s0[(f1es >> 1) * RS_H1 + 8 * j];
      } else {  // e_s = 1 reads both a1 rows, i.e. every input value: it takes max|x|, max|y|
        uint64_t mag = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint64_t a = s0[8 * j], b = s0[RS_H1 + 8 * j];
          mag = max(mag, max(abs64(a), abs64(b)));
          in[j] = (uint32_t)a + (uint32_t)b;
        }
        // max over the half warp of each operand (values >= 2^31 saturate: never safe)
        uint32_t m = mag >= (1ull << 31) ? 0x80000000u : (uint32_t)mag;
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((lane & 15) == 0) s_mag[op] = m;
      }
      uint32_t* dst = P + op * PN_OP + ba2 * PN_A2 + (27 * f1es) * PN_ROW + bc;
      fwd_store<3, PN_ROW, uint32_t>(in, dst);
    } else {
      ++rr.done;
    }
    __syncthreads();
    // ---- F2: 8 + 8 base values of unit (e_a2, e_S), C-axes forward fused with the product ----
    uint32_t acc[27];
    if (unit) {
      const uint32_t* px = P + eS * PN_ROW;
      uint32_t xt[8], yt[8];
      if (ea2 != 1) {
        const uint32_t* a = px + (ea2 >> 1) * PN_A2;
        lds4(a, xt[0], xt[1], xt[2], xt[3]);
        lds4(a + 4, xt[4], xt[5], xt[6], xt[7]);
        lds4(a + PN_OP, yt[0], yt[1], yt[2], yt[3]);
        lds4(a + PN_OP + 4, yt[4], yt[5], yt[6], yt[7]);
      } else {
        uint32_t u0, u1, u2, u3;
#pragma unroll
        for (int j = 0; j < 8; j += 4) {
          lds4(px + j, xt[j], xt[j + 1], xt[j + 2], xt[j + 3]);
          lds4(px + PN_A2 + j, u0, u1, u2, u3);
          xt[j] += u0; xt[j + 1] += u1; xt[j + 2] += u2; xt[j + 3] += u3;
          lds4(px + PN_OP + j, yt[j], yt[j + 1], yt[j + 2], yt[j + 3]);
          lds4(px + PN_OP + PN_A2 + j, u0, u1, u2, u3);
          yt[j] += u0; yt[j + 1] += u1; yt[j + 2] += u2; yt[j + 3] += u3;
        }
      }
#pragma unroll
      for (int i = 0; i < 27; ++i) acc[i] = 0u;
      fwd_mul_acc<3, uint32_t>(xt, yt, acc);
    }
    // safe when 2^8 max|x| max|y| < 2^31 (every output sums at most 2^8 products)
    const bool safe = (uint64_t)s_mag[0] * s_mag[1] < (1ull << (31 - D));
    __syncthreads();  // P is read; S (aliasing it) may be written
    // ---- a4: inverse on C (registers), B (exchange), A (exchange) + store (a6) ----
    if (unit) {
      inv_reg<3, uint32_t>(acc);
#pragma unroll
      for (int i = 0; i < 27; ++i) S[u * 27 + i] = acc[i];
    }
    __syncthreads();
    if (unit) {
      const int c = tid / 9, a = tid - 9 * c;  // e_A fastest (stride 729 = 25 mod 32)
      uint32_t v[27];
#pragma unroll
      for (int e = 0; e < 27; ++e) v[e] = S[a * 729 + e * 27 + c];
      inv_reg<3, uint32_t>(v);
#pragma unroll
      for (int e = 0; e < 27; ++e) S[a * 729 + e * 27 + c] = v[e];
    }
    __syncthreads();
    if (safe) {
      uint64_t* zt = z + cube * 6561ull;
#pragma unroll 1
      for (int r = 0; r < 3; ++r) {
        if (unit) {
          const int col = r * 243 + tid;
          uint32_t v[9];
#pragma unroll
          for (int e = 0; e < 9; ++e) v[e] = S[e * 729 + col];
          inv_reg<2, uint32_t>(v);
#pragma unroll
          for (int e = 0; e < 9; ++e) st_cs_i64(zt + e * 729 + col, v[e]);
        }
#if HC_T8N_INSTEP
        if (r < 2) __syncthreads();  // the CTA's store rounds in step
#endif
      }
    } else if (tid == 0) {
      const uint32_t slot = atomicAdd(fb_count, 1u);
      HC_ASSERT(slot < nitems);
      fb_list[slot] = (uint32_t)cube;  // the 64-bit engine redoes this cube
    }
    __syncthreads();  // S is read before the next cube's F1 overwrites P
  }
}

// The 64-bit engine over the cubes listed by tile8n_kernel (count read on the device): the
// same tile8 pipeline, one cube per item (D = 8: one pair).
__global__ void __launch_bounds__(T8_NT, 2)
tile8_list_kernel(const uint64_t* __restrict__ x, const uint64_t* __restrict__ y, uint64_t* __restrict__ z,
                  const uint32_t* __restrict__ fb_count, const uint32_t* __restrict__ fb_list) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smem_raw);
  __shared__ __align__(8) uint64_t raw_bar[T8_NRAW];
  __shared__ Prefetch pf;
  ring_init(raw_bar);
  RawRing<> rr{raw_bar, 0, 0};
  const uint32_t n = *fb_count;
  const uint64_t pol_in = policy_evict_first();
  if (threadIdx.x == T8_SCHED) {
    pf.left = 0;
    pf.pos = 0xffffffffu;
  }
  uint64_t* R = sm + T8Cfg<uint64_t>::ALIAS;
  auto next = [&](Prefetch& c) -> bool {
    const uint32_t np = c.pos + 1;
    const uint64_t i = blockIdx.x + (uint64_t)np * gridDim.x;
    if (i >= n) return false;
    const uint64_t b = fb_list[i];
    c.pos = np;
    c.sx0 = x + (b << 8);
    c.sy0 = y + (b << 8);
    c.stride = 256;
    c.base = 0;
    c.freeb = 0;
    c.s = 0;
    c.left = 1;
    return true;
  };
  auto pump = [&]() { pf_pump<uint64_t>(pf, rr, R, pol_in, next); };
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    tile8<uint64_t, true>(1, z + (uint64_t)fb_list[i] * 6561ull, sm, rr, 0, pump, [] {});
    __syncthreads();
  }
}

}  // namespace hc
