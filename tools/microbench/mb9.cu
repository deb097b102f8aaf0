// Compile-only probe (ptxas -v): can the pair loop live in its own non-inlined function with
// a plain interface (pointers and scalars only), so that ptxas allocates it separately from a
// register-heavy pass-2 function in the same kernel?  Reports registers / spills per function.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -I../../paper_1608_00206_b200/csrc -c mb9.cu
#include "hc_slab.cuh"

using namespace hc;

// pair loop over SMEM-resident stages (no TMA), accumulators interpolated (C axes) and
// stored to S: everything the phase needs comes in as pointers / scalars
__device__ __noinline__ void pairs_phase(int npairs, double* sm, const double* R, int ea2, int eS, int f1es,
                                         int lane, bool unit, int u) {
  double* P = sm;
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0;
  for (int p = 0; p < npairs; ++p) {
    if (f1es >= 0) t8_f1<double>(R + (p % T8_NRAW) * RS_SZ, P + ((p + 1) & 1) * PS_SZ, f1es, lane);
    if (unit) t8_f2<double>(P + (p & 1) * PS_SZ, ea2, eS, acc);
    __syncthreads();
  }
  if (unit) {
    inv_reg<3, double>(acc);
#pragma unroll
    for (int i = 0; i < 27; ++i) sm[u * 27 + i] = acc[i];
  }
}

// pass 2 with the next chunk's loads in flight during the current chunk's round 2
__device__ __noinline__ void p2_phase(double* zs, uint32_t c0, double* sm, int task) {
  using Q = P2Cfg<6>;
  constexpr int NLO = Q::NLO, NHI = Q::NHI, P2S = Q::P2S;
  constexpr uint64_t ROW = 6561;
  const bool act = task >= 0 && task < 243;
  const int eh = task / P2W, pos1 = task - eh * P2W;
  const double* src = zs + (uint64_t)eh * NLO * ROW + (uint64_t)c0 * P2W + pos1;
  double* dst = zs + (uint64_t)eh * ROW + (uint64_t)c0 * P2W + pos1;
  double v[NLO];
  if (act)
    for (int e = 0; e < NLO; ++e) v[e] = ld_cg(src + e * ROW);
#pragma unroll 1
  for (int ch = 0; ch < 3; ++ch) {
    if (act) {
      inv_reg<3, double>(v);
#pragma unroll
      for (int e = 0; e < NLO; ++e) sm[eh * P2S + e * P2W + pos1] = v[e];
    }
    __syncthreads();
    if (act && ch + 1 < 3) {
#pragma unroll
      for (int e = 0; e < NLO; ++e) v[e] = ld_cg(src + (ch + 1) * P2W + e * ROW);
    }
    if (act) {
      double w[NHI];
#pragma unroll
      for (int e = 0; e < NHI; ++e) w[e] = sm[e * P2S + eh * P2W + pos1];
      inv_reg<3, double>(w);
#pragma unroll
      for (int e = 0; e < NHI; ++e) st_cs(dst + ch * P2W + (uint64_t)e * NLO * ROW, w[e]);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(T8_NT, 2) k_split(double* z, int items, int npairs) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int u = t8_unit(tid);
  const int ea2 = u / 81, eS = u - 81 * ea2;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    if (it & 1) p2_phase(z + (uint64_t)it * 4782969ull, 0, sm, tid < 243 ? tid : -1);
    else pairs_phase(npairs, sm, sm + T8Cfg<double>::ALIAS, ea2, eS, t8_f1_es(w), lane, tid < 243, u);
    __syncthreads();
  }
}
