// hc_api.cu -- the C ABI of include/hc.h: plans, dispatch, sharding, host entry point,
// instrumentation.  See include/hc.h for the contract of every entry point.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/hc.h"
#include "hc_common.cuh"
#include "hc_tile.cuh"
#include "hc_slab.cuh"
#include "hc_slabx.cuh"
#include "hc_tile8n.cuh"

using namespace hc;

// ---------------------------------------------------------------------------------------
// instrumentation
namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_prof{0};
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_recs;

struct LaunchScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(const char* n, cudaStream_t s) : name(n), st(s) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (g_prof.load(std::memory_order_relaxed)) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~LaunchScope() {
    if (a) {
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_prof_mu);
      g_prof_recs.push_back({name, a, b});
    }
  }
};
}  // namespace

extern "C" uint64_t hc_launch_count(void) { return g_launches.load(); }
extern "C" void hc_prof_enable(int on) { g_prof.store(on ? 1 : 0); }
extern "C" void hc_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof_recs.clear();
}
extern "C" hc_status hc_prof_read(const char* name, double* total_ms, uint64_t* launches) {
  if (!name || !total_ms || !launches) return HC_ERR_NULL;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double t = 0;
  uint64_t n = 0;
  for (auto& r : g_prof_recs) {
    if (r.name != name) continue;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return HC_ERR_CUDA;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return HC_ERR_CUDA;
    t += ms;
    ++n;
  }
  *total_ms = t;
  *launches = n;
  return HC_OK;
}

// ---------------------------------------------------------------------------------------
extern "C" const char* hc_status_str(hc_status s) {
  switch (s) {
    case HC_OK: return "ok";
    case HC_ERR_INVALID_DIM: return "invalid dimension (need 1 <= D <= HC_MAX_D, B >= 1)";
    case HC_ERR_DTYPE: return "unknown dtype";
    case HC_ERR_NULL: return "null pointer";
    case HC_ERR_ALIGN: return "x / y not 16-byte aligned, or z not 8-byte aligned";
    case HC_ERR_DEVICE: return "no usable CUDA device (needs sm_100)";
    case HC_ERR_CAPACITY: return "insufficient device memory";
    case HC_ERR_CUDA: return "CUDA error";
    case HC_ERR_SHARD: return "rank/ngpu inconsistent with plan";
  }
  return "unknown status";
}

extern "C" uint64_t hc_in_len(int D) { return (D >= 1 && D <= HC_MAX_D) ? (1ull << D) : 0ull; }
extern "C" uint64_t hc_out_len(int D) { return (D >= 1 && D <= HC_MAX_D) ? upow3(D) : 0ull; }

namespace {

constexpr int kTileL = 8;  // low axes handled inside one CTA (3^8 = 6561 outputs)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

// Device capability check, cached per device (cudaGetDeviceProperties is slow).
hc_status check_device() {
  static std::atomic<int> ok_dev[64];  // 0 = unknown, 1 = ok, 2 = unusable
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) { cudaGetLastError(); return HC_ERR_DEVICE; }
  if (dev < 64) {
    const int v = ok_dev[dev].load(std::memory_order_relaxed);
    if (v) return v == 1 ? HC_OK : HC_ERR_DEVICE;
  }
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) {
    cudaGetLastError();
    return HC_ERR_DEVICE;
  }
  const bool ok = major == 10;
  if (dev < 64) ok_dev[dev].store(ok ? 1 : 2, std::memory_order_relaxed);
  return ok ? HC_OK : HC_ERR_DEVICE;
}

// Per-device launch caches: kernel attributes (dynamic shared memory size) and occupancy are
// set / queried once per device, so one process may drive several GPUs.
constexpr int kMaxDev = 64;
inline int& dev_slot(int* cache, int& scratch) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) {
    scratch = 0;
    return scratch;  // no caching: recomputed on every call
  }
  return cache[d];
}

// ---- 8-axis tiles: single level (tile8_kernel) and two levels (prep + slab8_kernel) ----
// persistent grid size for a T8 kernel: SMs x resident CTAs per SM
template <class K>
cudaError_t t8_grid(K kern, int& grid_max, size_t smem = T8Cfg<double>::SMEM) {
  if (grid_max) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0, dev = 0, sms = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T8_NT, smem);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (occ < 1) return cudaErrorInvalidConfiguration;
  grid_max = occ * sms;
  return cudaSuccess;
}

template <class T>
cudaError_t launch_tile8(const T* x, const T* y, T* z, int D, uint64_t slab0, uint64_t nslab, uint64_t nitems,
                         cudaStream_t st) {
  auto kern = tile8_kernel<T>;
  static int gm_cache[kMaxDev] = {};
  int gm_scratch = 0;
  int& grid_max = dev_slot(gm_cache, gm_scratch);
  cudaError_t e = t8_grid(kern, grid_max);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)(nitems < (uint64_t)grid_max ? nitems : (uint64_t)grid_max);
  LaunchScope ls("tile", st);
  kern<<<grid, T8_NT, T8Cfg<T>::SMEM, st>>>(x, y, z, D, slab0, nslab, nitems);
  return cudaGetLastError();
}

// batched D = 8 int64 in the 32-bit ring (hc_tile8n.cuh) + the 64-bit engine over the cubes
// whose bound check failed.  The fallback list lives in stream-ordered scratch (B + 1 words),
// so concurrent calls on different streams never share it.  HC_NARROW=0 disables the path.
static bool use_narrow() {
  static const bool on = [] {
    const char* s = getenv("HC_NARROW");
    return !(s && s[0] == '0');
  }();
  return on;
}

// the library's own stream-ordered pool on the current device: it keeps what it has mapped
// (release threshold = max) so per-call scratch costs no remapping after the first call, and
// it is separate from the process's default pool
static cudaError_t scratch_pool(cudaMemPool_t& pool) {
  static std::mutex mu;
  static cudaMemPool_t pools[kMaxDev] = {};
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return e;
  if (d < 0 || d >= kMaxDev) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> g(mu);
  if (!pools[d]) {
    cudaMemPoolProps pr = {};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = d;
    cudaMemPool_t np = nullptr;
    e = cudaMemPoolCreate(&np, &pr);
    if (e != cudaSuccess) return e;
    uint64_t keep = ~0ull;
    e = cudaMemPoolSetAttribute(np, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e != cudaSuccess) {
      cudaMemPoolDestroy(np);
      return e;
    }
    pools[d] = np;
  }
  pool = pools[d];
  return cudaSuccess;
}

static cudaError_t launch_tile8n(const uint64_t* x, const uint64_t* y, uint64_t* z, uint64_t B, cudaStream_t st) {
  if (B >= (1ull << 32)) return cudaErrorInvalidValue;  // list entries are 32-bit cube indices
  static int gn_cache[kMaxDev] = {}, gl_cache[kMaxDev] = {};
  int gn_scratch = 0, gl_scratch = 0;
  int& gn = dev_slot(gn_cache, gn_scratch);
  int& gl = dev_slot(gl_cache, gl_scratch);
  cudaError_t e;
  auto kn = tile8n_kernel<8>;
  const size_t smem = T8N_SMEM;
  if (!gn) {
    e = cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0, dev = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kn, T8_NT, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gn = occ * sms;
  }
  e = t8_grid(tile8_list_kernel, gl);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  e = scratch_pool(pool);
  if (e != cudaSuccess) return e;
  uint32_t* ws = nullptr;
  e = cudaMallocFromPoolAsync((void**)&ws, sizeof(uint32_t) * (size_t)(B + 1), pool, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ws, 0, sizeof(uint32_t), st);
  if (e == cudaSuccess) {
    const unsigned grid = (unsigned)(B < (uint64_t)gn ? B : (uint64_t)gn);
    LaunchScope ls("tile", st);
    kn<<<grid, T8_NT, smem, st>>>(x, y, z, B, ws, ws + 1);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {  // exits at once when every cube was safe
    const unsigned grid = (unsigned)(B < (uint64_t)gl ? B : (uint64_t)gl);
    LaunchScope ls("tile_fb", st);
    tile8_list_kernel<<<grid, T8_NT, T8Cfg<uint64_t>::SMEM, st>>>(x, y, z, ws, ws + 1);
    e = cudaGetLastError();
  }
  cudaError_t ef = cudaFreeAsync(ws, st);
  return e != cudaSuccess ? e : ef;
}

template <class T, int M>
cudaError_t launch_prep(const T* x, const T* y, T* xu, T* yu, int k, cudaStream_t st, unsigned batch = 1) {
  // a batch of same-D problems stored back to back is one problem with batch * 2^k input slices
  LaunchScope lp("prep", st);
  dim3 pg((unsigned)upow3(M), batch << k, 2);
  prep_kernel<T, M><<<pg, 256, 0, st>>>(x, y, xu, yu);
  return cudaGetLastError();
}

template <class T, int M, int EPI = 0, int P2CH = T8_P2CH>
cudaError_t launch_slab8_m(const T* x, const T* y, T* z, T* xu, T* yu, const SlabArgs& a, cudaStream_t st,
                           bool prep) {
  auto kern = slab8_kernel<T, M, EPI, P2CH>;
  constexpr size_t smem = T8Cfg<T, slab_nraw<M, EPI>()>::SMEM;
  static int gm_cache[kMaxDev] = {};
  int gm_scratch = 0;
  int& grid_max = dev_slot(gm_cache, gm_scratch);
  cudaError_t e = t8_grid(kern, grid_max, smem);
  if (e != cudaSuccess) return e;
  const uint64_t items = (uint64_t)a.nslab * (upow3(M) + upow3(8) / (P2W * P2CH));
  const unsigned grid = (unsigned)(items < (uint64_t)grid_max ? items : (uint64_t)grid_max);
  e = cudaMemsetAsync(a.ctr, 0, sizeof(uint32_t) * (1 + 2 * (size_t)a.nslab), st);
  if (e != cudaSuccess) return e;
  if (prep) {
    e = launch_prep<T, M>(x, y, xu, yu, a.k, st);
    if (e != cudaSuccess) return e;
  }
  LaunchScope ls("slab", st);
  kern<<<grid, T8_NT, smem, st>>>(xu, yu, z, a);
  return cudaGetLastError();
}

// warp-specialised engine (hc_slabx.cuh): one CTA of 640 threads per SM
template <class T, int M>
cudaError_t launch_slabx_m(const T* x, const T* y, T* z, T* xu, T* yu, const SlabArgs& a, cudaStream_t st,
                           bool prep) {
  auto kern = slabx_kernel<T, M>;
  static int sms_cache[kMaxDev] = {};
  int sms_scratch = 0;
  int& sms = dev_slot(sms_cache, sms_scratch);
  if (!sms) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SXCfg<T, M>::SMEM);
    if (e != cudaSuccess) return e;
    int occ = 0, dev = 0, n = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SX_NT, SXCfg<T, M>::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms = n;
  }
  const uint64_t tiles = (uint64_t)a.nslab * upow3(M);
  const unsigned grid = (unsigned)(tiles < (uint64_t)sms ? tiles : (uint64_t)sms);
  cudaError_t e = cudaMemsetAsync(a.ctr, 0, sizeof(uint32_t) * (2 + 2 * (size_t)a.nslab), st);
  if (e != cudaSuccess) return e;
  if (prep) {
    e = launch_prep<T, M>(x, y, xu, yu, a.k, st);
    if (e != cudaSuccess) return e;
  }
  static const int lag_env = getenv("HC_SLABX_LAG") ? atoi(getenv("HC_SLABX_LAG")) : 3;
  SlabxArgs sa{a.nslab, (uint32_t)(lag_env < 1 ? 1 : lag_env), a.ctr, a.order, a.bstride};
  LaunchScope ls("slab", st);
  kern<<<grid, SX_NT, SXCfg<T, M>::SMEM, st>>>(xu, yu, z, sa);
  return cudaGetLastError();
}

// engine for the plain two-level convolution: the fork-join "slab8" (default, faster on B200:
// DESIGN.md §4) or the warp-specialised "slabx" (HC_ENGINE=slabx); the fused-carry
// applications always use slab8
inline bool use_slabx() {
  static const int v = [] {
    const char* s = getenv("HC_ENGINE");
    return (s && std::string(s) == "slabx") ? 1 : 0;
  }();
  return v != 0;
}

template <class T>
cudaError_t launch_slab8(const T* x, const T* y, T* z, T* xu, T* yu, int M, const SlabArgs& a, cudaStream_t st,
                         bool prep) {
  if constexpr (std::is_same<T, uint64_t>::value) {
    if (a.cout) {  // f1: carries fused into pass 2; tiles in z (2) or in the slab ring (3)
      switch (M * 2 + (a.ring != nullptr)) {
        case 10: return launch_slab8_m<T, 5, 2>(x, y, z, xu, yu, a, st, prep);
        case 11: return launch_slab8_m<T, 5, 3>(x, y, z, xu, yu, a, st, prep);
        case 12: return launch_slab8_m<T, 6, 2>(x, y, z, xu, yu, a, st, prep);
        case 13: return launch_slab8_m<T, 6, 3>(x, y, z, xu, yu, a, st, prep);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  if (use_slabx() && !a.debug_skip) {
    switch (M) {
      case 5: return launch_slabx_m<T, 5>(x, y, z, xu, yu, a, st, prep);
      case 6: return launch_slabx_m<T, 6>(x, y, z, xu, yu, a, st, prep);
      default: return cudaErrorInvalidValue;
    }
  }
  if (a.nslab <= 3 && a.p2_head == 0xffffffffu) {  // few slabs: single-chunk pass-2 items
    switch (M) {
      case 5: return launch_slab8_m<T, 5, 0, 1>(x, y, z, xu, yu, a, st, prep);
      case 6: return launch_slab8_m<T, 6, 0, 1>(x, y, z, xu, yu, a, st, prep);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (M) {
    case 5: return launch_slab8_m<T, 5>(x, y, z, xu, yu, a, st, prep);
    case 6: return launch_slab8_m<T, 6>(x, y, z, xu, yu, a, st, prep);
    default: return cudaErrorInvalidValue;
  }
}

// ---- launch of the tile engine for L = min(D, 8) --------------------------------------
template <class T, int C, int B, int A>
cudaError_t launch_tile_cfg(const T* x, const T* y, T* z, int D, uint64_t slab0, uint64_t nslab,
                            uint64_t nitems, cudaStream_t st) {
  using Cfg = TileCfg<T, C, B, A>;
  auto kern = tile_kernel<T, C, B, A>;
  static int attr_cache[kMaxDev] = {};  // per instantiation and device
  int attr_scratch = 0;
  int& attr_set = dev_slot(attr_cache, attr_scratch);
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = 1;
  }
  // items [off, off + n) per launch (gridDim.x <= 2^31 - 1): the kernel gets the item offset,
  // so batch and slab indices stay exact across chunks
  const uint64_t maxgrid = 0x7fffffffull;
  for (uint64_t off = 0; off < nitems; off += maxgrid) {
    const uint64_t n = nitems - off < maxgrid ? nitems - off : maxgrid;
    LaunchScope ls("tile", st);
    kern<<<(unsigned)n, Cfg::NT, Cfg::SMEM, st>>>(x, y, z, D, slab0, nslab, off);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <class T>
cudaError_t launch_tile(const T* x, const T* y, T* z, int D, uint64_t slab0, uint64_t nslab,
                        uint64_t nitems, cudaStream_t st) {
  const int L = D < kTileL ? D : kTileL;
  switch (L) {
    case 1: return launch_tile_cfg<T, 0, 1, 0>(x, y, z, D, slab0, nslab, nitems, st);
    case 2: return launch_tile_cfg<T, 1, 1, 0>(x, y, z, D, slab0, nslab, nitems, st);
    case 3: return launch_tile_cfg<T, 2, 1, 0>(x, y, z, D, slab0, nslab, nitems, st);
    case 4: return launch_tile_cfg<T, 3, 1, 0>(x, y, z, D, slab0, nslab, nitems, st);
    case 5: return launch_tile_cfg<T, 3, 2, 0>(x, y, z, D, slab0, nslab, nitems, st);
    case 6: return launch_tile_cfg<T, 3, 3, 0>(x, y, z, D, slab0, nslab, nitems, st);
    case 7: return launch_tile_cfg<T, 3, 3, 1>(x, y, z, D, slab0, nslab, nitems, st);
    default: return launch_tile8<T>(x, y, z, D, slab0, nslab, nitems, st);
  }
}

// single pair, 9 <= D <= 12: the 3^8-tile engine gives only 3^(D-8) CTAs (9 at D = 10, BASELINE
// config 1).  Optionally (HC_SMALL_L = 5..7) the work is cut into smaller tiles of L' < 8 axes,
// one CTA each (tile_kernel); unit u of 3^8 outputs = sub-tiles [u 3^(8-L'), (u+1) 3^(8-L')).
// Measured on B200 (L2 flushed, int64, us for D = 9/10/11/12): L' = 5: 18/31/49/88, 6: 12/16/25/43,
// 7: 10/14/21/37, 8: 10/12/16/25 -- more, smaller CTAs lose to the TMA-fed 3^8 tiles, so the
// default stays L' = 8 (profiles/r02_small_d_tiles.txt).
template <class T>
cudaError_t launch_tile_small(const T* x, const T* y, T* z, int D, int L, uint64_t u0, uint64_t nu, cudaStream_t st) {
  const uint64_t f = upow3(8 - L);
  const uint64_t nslab = upow3(D - L);
  switch (L) {
    case 5: return launch_tile_cfg<T, 3, 2, 0>(x, y, z, D, u0 * f, nslab, nu * f, st);
    case 6: return launch_tile_cfg<T, 3, 3, 0>(x, y, z, D, u0 * f, nslab, nu * f, st);
    case 7: return launch_tile_cfg<T, 3, 3, 1>(x, y, z, D, u0 * f, nslab, nu * f, st);
    default: return launch_tile8<T>(x, y, z, D, u0, upow3(D - 8), nu, st);
  }
}

// tile axes L' for a single-pair D in 9..12 (HC_SMALL_L overrides; 8 = the 3^8-tile engine)
int small_tile_axes(int D) {
  static const int env = getenv("HC_SMALL_L") ? atoi(getenv("HC_SMALL_L")) : 0;
  if (env >= 5 && env <= 8) return env;
  (void)D;
  return 8;
}

cudaError_t launch_any(hc_dtype dt, const void* x, const void* y, void* z, int D, uint64_t slab0,
                       uint64_t nslab, uint64_t nitems, cudaStream_t st) {
  if (dt == HC_INT64)
    return launch_tile<uint64_t>((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)z, D, slab0, nslab,
                                 nitems, st);
  return launch_tile<double>((const double*)x, (const double*)y, (double*)z, D, slab0, nslab, nitems, st);
}

}  // namespace

// ---------------------------------------------------------------------------------------
// Geometry: how the D axes are split.
//   D <= 12 : single level -- tile of L = min(D, 8) low axes, k = D - L top axes direct.
//   D >= 13 : two levels   -- slab of s = min(D, 14) axes (tile 8 + M = s - 8 middle axes,
//             interpolated in L2), k = D - s top axes direct.
// The unit of work distribution and sharding is one output slab (3^(L+M) entries).
struct Geometry {
  bool two_level;
  int L, M, k;
  uint64_t unit, nunits;
};
static Geometry geometry(int D) {
  Geometry g;
  g.two_level = D >= 13;
  g.L = D < kTileL ? D : kTileL;
  // slab axes s = min(D, 14) (38 MB fp64 slabs fit twice in the 126 MB L2); HC_SLAB_AXES
  // overrides it for experiments (13 or 14)
  static const int s_env = getenv("HC_SLAB_AXES") ? atoi(getenv("HC_SLAB_AXES")) : 14;
  const int smax = (s_env == 13 || s_env == 14) ? s_env : 14;
  g.M = g.two_level ? (D < smax ? D : smax) - kTileL : 0;
  g.k = D - g.L - g.M;
  g.unit = upow3(g.L + g.M);
  g.nunits = upow3(g.k);
  return g;
}

struct hc_plan_s {
  int D;
  hc_dtype dtype;
  int ngpu, rank;
  Geometry g;
  std::vector<uint64_t> cuts;     // ngpu+1 unit (slab) boundaries (equal cost)
  uint32_t* ctr[3] = {nullptr, nullptr, nullptr};  // slab-engine counters (device, per stream slot)
  void* ring = nullptr;  // hc_conv1d (fused carries): T8_RING slab buffers for pass-1 tiles
  void* xu = nullptr;             // two-level: middle-axes-evaluated input slices (prep kernel)
  void* yu = nullptr;
  std::mutex order_mu;
  std::map<std::pair<uint64_t, uint64_t>, uint4*> orders;  // [u0,u1) -> device processing order
  std::map<std::pair<uint64_t, uint64_t>, std::pair<uint2*, uint32_t>> pair_items;  // [u0,u1) -> (tile, pair) items
  // host entry point workspace
  void* dx = nullptr;
  void* dy = nullptr;
  void* dz[2] = {nullptr, nullptr};
  uint64_t chunk_units = 0;
  cudaStream_t hs[2] = {nullptr, nullptr};
  // application scratch (hc_convolve_difference, hc_maxconv_pnorm): 2 x 2^D elements + maxima
  void* app_a = nullptr;
  void* app_b = nullptr;
  unsigned long long* app_mx = nullptr;
};

// Equal-cost contiguous split of the 3^k output slabs over ngpu ranks.  Cost of slab
// t_T ~ alpha + 2^{#1(t_T)}: one unit per direct-split pair (PAPER.md 166-177) plus alpha
// for the slab's interpolation and store, in units of one pair.  alpha is fitted from shards
// timed alone on a B200 (tools/shard_times.py, profiles/r02_shard_balance.txt);
// HC_SHARD_ALPHA overrides it (calibration runs).
static double shard_alpha() {
  static const double a = getenv("HC_SHARD_ALPHA") ? atof(getenv("HC_SHARD_ALPHA")) : 11.0;
  return a;
}
static std::vector<uint64_t> compute_cuts(int k, int ngpu) {
  const double alpha = shard_alpha();
  const uint64_t n = upow3(k);
  std::vector<double> pref(n + 1, 0.0);
  for (uint64_t t = 0; t < n; ++t) {
    uint64_t v = t;
    int ones = 0;
    for (int a = 0; a < k; ++a) {
      if (v % 3 == 1) ++ones;
      v /= 3;
    }
    pref[t + 1] = pref[t] + alpha + (double)(1ull << ones);
  }
  std::vector<uint64_t> cuts(ngpu + 1, 0);
  cuts[ngpu] = n;
  uint64_t j = 0;
  for (int r = 1; r < ngpu; ++r) {
    const double target = pref[n] * r / ngpu;
    while (j < n && pref[j] < target) ++j;
    // nearest boundary to the target, then keep every rank non-empty
    uint64_t c = (j > 0 && target - pref[j - 1] < pref[j] - target) ? j - 1 : j;
    const uint64_t lo = cuts[r - 1] + 1, hi = n - (uint64_t)(ngpu - r);
    c = c < lo ? lo : (c > hi ? hi : c);
    cuts[r] = c;
  }
  return cuts;
}

extern "C" hc_status hc_shard_range(int D, int ngpu, int rank, uint64_t* zb, uint64_t* ze) {
  if (!zb || !ze) return HC_ERR_NULL;
  if (D < 1 || D > HC_MAX_D) return HC_ERR_INVALID_DIM;
  const Geometry g = geometry(D);
  if (ngpu < 1 || rank < 0 || rank >= ngpu || (uint64_t)ngpu > g.nunits) return HC_ERR_SHARD;
  std::vector<uint64_t> cuts = compute_cuts(g.k, ngpu);
  *zb = cuts[rank] * g.unit;
  *ze = cuts[rank + 1] * g.unit;
  return HC_OK;
}

static const uint4* slab_order(hc_plan_t p, uint64_t u0, uint64_t u1);
static std::pair<uint2*, uint32_t> pair_items(hc_plan_t p, uint64_t u0, uint64_t u1);

// single-level int64 plans with fewer tiles than CTA slots run one item per (tile, pair) and
// accumulate with atomics (tile8_pairs_kernel); HC_PAIR_SPLIT=0 turns it off.  Measured with the
// L2 flushed (tools/r02/t25.py, per call incl. the zeroing): D = 10 / 11 / 12 11.1 / 11.3 / 15.3 us
// against 12.3 / 16.4 / 24.4 us per tile; D = 9 (4 pairs) 11.2 against 10.2 us.  In a stream of
// back-to-back calls the separate zeroing launch costs more than D = 10 gains (bench.py C1:
// 18.9 against 17.9 us per step, kernel 10.1 against 12.8 us), so D >= 11 only
static bool use_pair_split(const hc_plan_s* p) {
  static const bool on = [] {
    const char* s = getenv("HC_PAIR_SPLIT");
    return !(s && s[0] == '0');
  }();
  return on && p->dtype == HC_INT64 && !p->g.two_level && p->D >= 11 && p->D <= 12;
}

extern "C" hc_status hc_plan_create(hc_plan_t* out, int D, hc_dtype dtype, int ngpu, int rank) {
  if (!out) return HC_ERR_NULL;
  *out = nullptr;
  if (D < 1 || D > HC_MAX_D) return HC_ERR_INVALID_DIM;
  if (dtype != HC_INT64 && dtype != HC_FP64) return HC_ERR_DTYPE;
  if (ngpu < 1 || rank < 0 || rank >= ngpu) return HC_ERR_SHARD;
  hc_status ds = check_device();
  if (ds != HC_OK) return ds;
  const Geometry g = geometry(D);
  if ((uint64_t)ngpu > g.nunits) return HC_ERR_SHARD;
  auto* p = new hc_plan_s();
  p->D = D;
  p->dtype = dtype;
  p->ngpu = ngpu;
  p->rank = rank;
  p->g = g;
  p->cuts = compute_cuts(g.k, ngpu);
  {
    for (auto& c : p->ctr) {
      if (cudaMalloc(&c, sizeof(uint32_t) * (2 + 2 * g.nunits)) != cudaSuccess) {
        cudaGetLastError();
        for (auto& c2 : p->ctr) cudaFree(c2);
        delete p;
        return HC_ERR_CAPACITY;
      }
    }
  }
  if (g.two_level) {
    const size_t bytes = sizeof(double) * (size_t)(1ull << g.k) * upow3(g.M) * 256;
    if (cudaMalloc(&p->xu, bytes) != cudaSuccess || cudaMalloc(&p->yu, bytes) != cudaSuccess) {
      cudaGetLastError();
      hc_plan_destroy(p);
      return HC_ERR_CAPACITY;
    }
    // the slab processing order of the plan's own range is uploaded here, so hc_convolve /
    // hc_convolve_sharded do no synchronous work (stream-ordered, graph-capturable)
    if (!slab_order(p, p->cuts[rank], p->cuts[rank + 1])) {
      hc_plan_destroy(p);
      return HC_ERR_CAPACITY;
    }
  }
  if (use_pair_split(p) && !pair_items(p, p->cuts[rank], p->cuts[rank + 1]).first) {
    hc_plan_destroy(p);
    return HC_ERR_CAPACITY;
  }
  *out = p;
  return HC_OK;
}

extern "C" hc_status hc_plan_destroy(hc_plan_t p) {
  if (!p) return HC_ERR_NULL;
  cudaFree(p->dx);
  cudaFree(p->dy);
  cudaFree(p->dz[0]);
  cudaFree(p->dz[1]);
  for (auto& c : p->ctr) cudaFree(c);
  cudaFree(p->xu);
  cudaFree(p->yu);
  cudaFree(p->ring);
  cudaFree(p->app_a);
  cudaFree(p->app_b);
  cudaFree(p->app_mx);
  for (auto& kv : p->orders) cudaFree(kv.second);
  for (auto& kv : p->pair_items) cudaFree(kv.second.first);
  for (auto& s : p->hs)
    if (s) cudaStreamDestroy(s);
  delete p;
  return HC_OK;
}

extern "C" hc_status hc_shard_info(hc_plan_t p, int rank, uint64_t* zb, uint64_t* ze) {
  if (!p || !zb || !ze) return HC_ERR_NULL;
  if (rank < 0 || rank >= p->ngpu) return HC_ERR_SHARD;
  *zb = p->cuts[rank] * p->g.unit;
  *ze = p->cuts[rank + 1] * p->g.unit;
  return HC_OK;
}

// Processing order of the slabs [u0, u1) for the slab engine: sorted by the number of
// direct-split pairs 2^{#1(t_T)} so that consecutive slabs cost the same and a pass-2 item
// rarely waits for a slow pass-1 item of its slab.  Cached per range on the plan; the plan's
// own range is built at plan creation, other ranges (the host entry point's chunks) on their
// first use inside hc_convolve_host, which synchronises anyway.
static const uint4* slab_order(hc_plan_t p, uint64_t u0, uint64_t u1) {
  std::lock_guard<std::mutex> lk(p->order_mu);
  auto key = std::make_pair(u0, u1);
  auto it = p->orders.find(key);
  if (it != p->orders.end()) return it->second;
  const uint64_t n = u1 - u0;
  std::vector<std::pair<int, uint32_t>> v(n);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t t = u0 + i;
    int ones = 0;
    for (int a = 0; a < p->g.k; ++a) {
      ones += (t % 3 == 1);
      t /= 3;
    }
    v[i] = {ones, (uint32_t)i};
  }
  std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<uint4> h(n);
  for (uint64_t i = 0; i < n; ++i) {
    // trit split of the top index (PAPER.md 173-177): digit 2 -> base bit, digit 1 -> free bit
    uint64_t t = u0 + v[i].second;
    uint32_t base = 0, freeb = 0;
    for (int a = 0; a < p->g.k; ++a, t /= 3) {
      if (t % 3 == 2) base |= 1u << a;
      else if (t % 3 == 1) freeb |= 1u << a;
    }
    h[i] = make_uint4(v[i].second, base, freeb, 0);
  }
  uint4* d = nullptr;
  if (cudaMalloc(&d, sizeof(uint4) * n) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  if (cudaMemcpy(d, h.data(), sizeof(uint4) * n, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  p->orders[key] = d;
  return d;
}

// (tile, pair) items of the tiles [u0, u1) for tile8_pairs_kernel: tile t - u0 and every subset
// s of its free top bits (digit 1), in the prefetcher's ascending-subset order; cached per range
static std::pair<uint2*, uint32_t> pair_items(hc_plan_t p, uint64_t u0, uint64_t u1) {
  std::lock_guard<std::mutex> lk(p->order_mu);
  auto key = std::make_pair(u0, u1);
  auto it = p->pair_items.find(key);
  if (it != p->pair_items.end()) return it->second;
  std::vector<uint2> h;
  for (uint64_t t = u0; t < u1; ++t) {
    uint32_t freeb = 0;
    uint64_t v = t;
    for (int a = 0; a < p->g.k; ++a, v /= 3)
      if (v % 3 == 1) freeb |= 1u << a;
    uint32_t s = 0;
    do {
      h.push_back(make_uint2((uint32_t)(t - u0), s));
      s = (s - freeb) & freeb;
    } while (s != 0);
  }
  uint2* d = nullptr;
  if (cudaMalloc(&d, sizeof(uint2) * h.size()) != cudaSuccess) {
    cudaGetLastError();
    return {nullptr, 0};
  }
  if (cudaMemcpy(d, h.data(), sizeof(uint2) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return {nullptr, 0};
  }
  return p->pair_items[key] = {d, (uint32_t)h.size()};
}

static cudaError_t launch_tile8_pairs(const uint64_t* x, const uint64_t* y, uint64_t* z, int D, uint64_t u0,
                                      uint64_t nu, const uint2* items, uint32_t nitems, cudaStream_t st) {
  static int gm_cache[kMaxDev] = {};
  int gm_scratch = 0;
  int& grid_max = dev_slot(gm_cache, gm_scratch);
  cudaError_t e = t8_grid(tile8_pairs_kernel, grid_max);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(z, 0, sizeof(uint64_t) * nu * 6561ull, st);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)(nitems < (uint32_t)grid_max ? nitems : (uint32_t)grid_max);
  LaunchScope ls("tile", st);
  tile8_pairs_kernel<<<grid, T8_NT, T8Cfg<uint64_t>::SMEM, st>>>(x, y, z, D, u0, items, nitems);
  return cudaGetLastError();
}

// units [u0, u1) of the plan's geometry into z (z points at unit u0)
static hc_status run_range(hc_plan_t p, const void* x, const void* y, void* z, uint64_t u0, uint64_t u1,
                           cudaStream_t st, int slot, unsigned long long* cout = nullptr, void* ring = nullptr,
                           bool prep = true) {
  if (u1 <= u0) return HC_OK;
  const Geometry& g = p->g;
  cudaError_t e;
  if (!g.two_level) {
    const int Ls = (p->D >= 9 && p->D <= 12) ? small_tile_axes(p->D) : 8;
    if (use_pair_split(p) && Ls == 8) {
      const auto pi = pair_items(p, u0, u1);
      if (!pi.first) return HC_ERR_CAPACITY;
      e = launch_tile8_pairs((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)z, p->D, u0, u1 - u0, pi.first,
                             pi.second, st);
    } else if (Ls < 8) {
      if (p->dtype == HC_INT64)
        e = launch_tile_small<uint64_t>((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)z, p->D, Ls, u0, u1 - u0, st);
      else
        e = launch_tile_small<double>((const double*)x, (const double*)y, (double*)z, p->D, Ls, u0, u1 - u0, st);
    } else {
      e = launch_any(p->dtype, x, y, z, p->D, u0, g.nunits, u1 - u0, st);
    }
  } else {
    const uint4* order = slab_order(p, u0, u1);
    if (!order) return HC_ERR_CAPACITY;
    static const int dbg = getenv("HC_DEBUG_SKIP") ? atoi(getenv("HC_DEBUG_SKIP")) : 0;
    static const int lag = getenv("HC_SLAB_LAG") ? atoi(getenv("HC_SLAB_LAG")) : 1;
    // lag >= 1; with the slab ring (fused carries) a pass-1 item of position j waits for the
    // pass-2 items of j - T8_RING, which must be claimed earlier: lag <= T8_RING - 1
    uint32_t lg = (uint32_t)(lag < 1 ? 1 : lag);
    if (ring && lg > T8_RING - 1) lg = T8_RING - 1;
    static const int keep = getenv("HC_KEEP_POLICY") ? atoi(getenv("HC_KEEP_POLICY")) : 0;
    static const int persist_mb = [] {
      const int mb = getenv("HC_L2_PERSIST_MB") ? atoi(getenv("HC_L2_PERSIST_MB")) : 0;
      if (mb > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mb << 20);
      return mb;
    }();
    (void)persist_mb;
    static const int p2pf = getenv("HC_P2_PREFETCH") ? atoi(getenv("HC_P2_PREFETCH")) : 0;
    // pass-2 interleave: H pass-1 items of slab j + lag, then the rest mixed with slab j's
    // pass-2 items; H must leave a multiple of the N2 = 243 pass-2 items (3^M - H = 243 m)
    static const long head_env = getenv("HC_P2_HEAD") ? atol(getenv("HC_P2_HEAD")) : -1;
    uint32_t head = 0xffffffffu;
    if (head_env >= 0 && !ring) {
      const long n1 = (long)upow3(g.M), n2 = (long)(upow3(8) / (P2W * T8_P2CH));
      if (head_env < n1 && (n1 - head_env) % n2 == 0) head = (uint32_t)head_env;
    }
    SlabArgs a{u0, (uint32_t)(u1 - u0), g.k, p->ctr[slot], order, dbg, lg, cout, ring, keep, p2pf, head};
#ifdef HC_PHASE_PROF
    {
      unsigned long long zero[16] = {0};
      cudaMemcpyToSymbolAsync(hc_phase, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
    }
#endif
    if (p->dtype == HC_INT64)
      e = launch_slab8<uint64_t>((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)z, (uint64_t*)p->xu,
                                 (uint64_t*)p->yu, g.M, a, st, prep);
    else
      e = launch_slab8<double>((const double*)x, (const double*)y, (double*)z, (double*)p->xu, (double*)p->yu,
                               g.M, a, st, prep);
#ifdef HC_PHASE_PROF
    {
      unsigned long long h[16];
      cudaMemcpyFromSymbolAsync(h, hc_phase, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      double tot = 0;
      for (int i : {0, 1, 4, 5, 6}) tot += (double)h[i];
      if (use_slabx()) {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const double c = 1e3 * nsm;  // kclk per CTA
        fprintf(stderr, "slabx phase (kclk per CTA): F2 total %.0f pairloop %.0f item-wait %.0f acc-empty-wait %.0f | "
                "F1 raw-wait %.0f | S throttle %.0f ring-full %.0f | E idle %.0f tiles %.0f (%llu) p2 %.0f (%llu)\n",
                h[9] / c, h[6] / c, h[5] / c, h[4] / c, h[7] / c, h[0] / c, h[8] / c, h[1] / c, h[2] / c, h[10], h[3] / c,
                h[11]);
      } else
      fprintf(stderr, "phase(Mclk/CTA-sum): select+wait %.0f pairloop %.0f inv+store %.0f p2 %.0f end %.0f "
              "(tot %.0f) | F1 mbar wait %.0f | t224 select %.0f end %.0f\n", h[0] / 1e6, h[1] / 1e6, h[6] / 1e6,
              h[4] / 1e6, h[5] / 1e6, tot / 1e6, h[7] / 1e6, h[2] / 1e6, h[3] / 1e6);
    }
#endif
  }
  return e == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

// middle-axes tables of the two-level engine for inputs x, y (prep_kernel) on stream st
static hc_status run_prep(hc_plan_t p, const void* x, const void* y, cudaStream_t st) {
  const Geometry& g = p->g;
  cudaError_t e = cudaErrorInvalidValue;
  if (p->dtype == HC_INT64) {
    if (g.M == 5) e = launch_prep<uint64_t, 5>((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)p->xu, (uint64_t*)p->yu, g.k, st);
    if (g.M == 6) e = launch_prep<uint64_t, 6>((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)p->xu, (uint64_t*)p->yu, g.k, st);
  } else {
    if (g.M == 5) e = launch_prep<double, 5>((const double*)x, (const double*)y, (double*)p->xu, (double*)p->yu, g.k, st);
    if (g.M == 6) e = launch_prep<double, 6>((const double*)x, (const double*)y, (double*)p->xu, (double*)p->yu, g.k, st);
  }
  return e == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

extern "C" hc_status hc_convolve(hc_plan_t p, const void* x, const void* y, void* z, void* stream) {
  if (!p || !x || !y || !z) return HC_ERR_NULL;
  if (!aligned16(x) || !aligned16(y) || !aligned8(z)) return HC_ERR_ALIGN;
  return run_range(p, x, y, z, 0, p->g.nunits, (cudaStream_t)stream, 0);
}

extern "C" hc_status hc_convolve_sharded(hc_plan_t p, const void* x, const void* y, void* zs, void* stream) {
  if (!p || !x || !y || !zs) return HC_ERR_NULL;
  if (!aligned16(x) || !aligned16(y) || !aligned8(zs)) return HC_ERR_ALIGN;
  return run_range(p, x, y, zs, p->cuts[p->rank], p->cuts[p->rank + 1], (cudaStream_t)stream, 0);
}

extern "C" hc_status hc_convolve_batched(int B, int D, hc_dtype dtype, const void* x, const void* y, void* z,
                                         void* stream) {
  if (B < 1 || D < 1 || D > HC_MAX_D) return HC_ERR_INVALID_DIM;
  if (dtype != HC_INT64 && dtype != HC_FP64) return HC_ERR_DTYPE;
  if (!x || !y || !z) return HC_ERR_NULL;
  if (!aligned16(x) || !aligned16(y) || !aligned8(z)) return HC_ERR_ALIGN;
  hc_status ds = check_device();
  if (ds != HC_OK) return ds;
  const int L = D < kTileL ? D : kTileL;
  const uint64_t nslab = upow3(D - L);
  const uint64_t nitems = (uint64_t)B * nslab;
  cudaError_t e;
  if (dtype == HC_INT64 && D == 8 && use_narrow())
    e = launch_tile8n((const uint64_t*)x, (const uint64_t*)y, (uint64_t*)z, (uint64_t)B, (cudaStream_t)stream);
  else
    e = launch_any(dtype, x, y, z, D, 0, nslab, nitems, (cudaStream_t)stream);
  return e == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

static void host_ws_free(hc_plan_t p) {
  cudaFree(p->dx);
  cudaFree(p->dy);
  cudaFree(p->dz[0]);
  cudaFree(p->dz[1]);
  p->dx = p->dy = p->dz[0] = p->dz[1] = nullptr;
  for (auto& s : p->hs) {
    if (s) cudaStreamDestroy(s);
    s = nullptr;
  }
  p->chunk_units = 0;
}

// host-entry workspace: inputs, two chunk buffers of ~1 GiB of output, two streams; on any
// failure everything is released (no half-initialised state survives to the next call)
static hc_status host_ws_alloc(hc_plan_t p) {
  if (p->dx && p->dy && p->dz[0] && p->dz[1] && p->hs[0] && p->hs[1]) return HC_OK;
  host_ws_free(p);
  const size_t esz = 8;
  const uint64_t nin = 1ull << p->D, tile = p->g.unit;
  const uint64_t s0 = p->cuts[p->rank], s1 = p->cuts[p->rank + 1];
  uint64_t cs = ((1ull << 30) / esz) / tile;
  if (cs > s1 - s0) cs = s1 - s0;
  if (cs < 1) cs = 1;
  bool ok = cudaMalloc(&p->dx, nin * esz) == cudaSuccess && cudaMalloc(&p->dy, nin * esz) == cudaSuccess &&
            cudaMalloc(&p->dz[0], cs * tile * esz) == cudaSuccess &&
            cudaMalloc(&p->dz[1], cs * tile * esz) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    host_ws_free(p);
    return HC_ERR_CAPACITY;
  }
  for (auto& s : p->hs) {
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      s = nullptr;
      host_ws_free(p);
      return HC_ERR_CUDA;
    }
  }
  p->chunk_units = cs;
  return HC_OK;
}

extern "C" hc_status hc_convolve_host(hc_plan_t p, const void* xh, const void* yh, void* zh, void* stream) {
  if (!p || !xh || !yh || !zh) return HC_ERR_NULL;
  const size_t esz = 8;
  const uint64_t nin = 1ull << p->D;
  const uint64_t tile = p->g.unit;
  const uint64_t s0 = p->cuts[p->rank], s1 = p->cuts[p->rank + 1];
  cudaStream_t st = (cudaStream_t)stream;
  hc_status hs = host_ws_alloc(p);
  if (hs != HC_OK) return hs;
  // every chunk's slab order exists before the first launch (built once per range)
  if (p->g.two_level)
    for (uint64_t c = s0; c < s1; c += p->chunk_units)
      if (!slab_order(p, c, c + p->chunk_units < s1 ? c + p->chunk_units : s1)) return HC_ERR_CAPACITY;
  if (cudaMemcpyAsync(p->dx, xh, nin * esz, cudaMemcpyHostToDevice, st) != cudaSuccess) return HC_ERR_CUDA;
  if (cudaMemcpyAsync(p->dy, yh, nin * esz, cudaMemcpyHostToDevice, st) != cudaSuccess) return HC_ERR_CUDA;
  // the middle-axes tables of the two-level engine depend only on x, y: built once on the
  // input stream, before the chunks (which then skip it)
  if (p->g.two_level) {
    hc_status r = run_prep(p, p->dx, p->dy, st);
    if (r != HC_OK) return r;
  }
  cudaEvent_t ready;
  if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) return HC_ERR_CUDA;
  hc_status r = HC_OK;
  if (cudaEventRecord(ready, st) != cudaSuccess) r = HC_ERR_CUDA;
  int i = 0;
  for (uint64_t c = s0; c < s1 && r == HC_OK; c += p->chunk_units, i ^= 1) {
    const uint64_t ce = c + p->chunk_units < s1 ? c + p->chunk_units : s1;
    cudaStream_t hs2 = p->hs[i];
    if (cudaStreamWaitEvent(hs2, ready, 0) != cudaSuccess) { r = HC_ERR_CUDA; break; }
    r = run_range(p, p->dx, p->dy, p->dz[i], c, ce, hs2, 1 + i, nullptr, nullptr, /*prep=*/false);
    if (r != HC_OK) break;
    if (cudaMemcpyAsync((char*)zh + (c - s0) * tile * esz, p->dz[i], (ce - c) * tile * esz,
                        cudaMemcpyDeviceToHost, hs2) != cudaSuccess)
      r = HC_ERR_CUDA;
  }
  cudaError_t e1 = cudaStreamSynchronize(p->hs[0]);
  cudaError_t e2 = cudaStreamSynchronize(p->hs[1]);
  cudaEventDestroy(ready);
  if (r != HC_OK) return r;
  return (e1 == cudaSuccess && e2 == cudaSuccess) ? HC_OK : HC_ERR_CUDA;
}

// ---------------------------------------------------------------------------------------
// Evaluation-point variant (include/hc.h, hc_ep_*; kernels in hc_ep.cuh).
#include "hc_ep.cuh"

struct hc_ep_s {
  int D, k, ngpu, rank;
  hc_dtype dtype;
  uint64_t e0, e1, c0, c1;   // owned evaluation points and columns
  hc_plan_t low = nullptr;   // plan of the (D-k)-dimensional convolution (geometry; non-batched path)
  void* xh = nullptr;        // forward-evaluated operands of the owned points ([point][2^(D-k)])
  void* yh = nullptr;
  // batched two-level engine over all owned points (D - k >= 13): middle-axes tables of every
  // point, the slab order of points x slabs, and the engine's counters
  void* xu = nullptr;
  void* yu = nullptr;
  uint4* order = nullptr;
  uint32_t* ctr = nullptr;
};

extern "C" hc_status hc_ep_range(int D, int k, int ngpu, int rank, uint64_t* e_begin, uint64_t* e_end,
                                 uint64_t* col_begin, uint64_t* col_end) {
  if (!e_begin || !e_end || !col_begin || !col_end) return HC_ERR_NULL;
  if (D < 2 || D > HC_MAX_D || k < 1 || k > EP_MAX_K || k >= D) return HC_ERR_INVALID_DIM;
  const uint64_t np = upow3(k), nc = upow3(D - k);
  if (ngpu < 1 || rank < 0 || rank >= ngpu || (uint64_t)ngpu > np) return HC_ERR_SHARD;
  *e_begin = np * (uint64_t)rank / (uint64_t)ngpu;
  *e_end = np * (uint64_t)(rank + 1) / (uint64_t)ngpu;
  *col_begin = nc * (uint64_t)rank / (uint64_t)ngpu;
  *col_end = nc * (uint64_t)(rank + 1) / (uint64_t)ngpu;
  return HC_OK;
}

extern "C" hc_status hc_ep_create(hc_ep_t* out, int D, int k, hc_dtype dtype, int ngpu, int rank) {
  if (!out) return HC_ERR_NULL;
  *out = nullptr;
  if (dtype != HC_INT64 && dtype != HC_FP64) return HC_ERR_DTYPE;
  auto* p = new hc_ep_s();
  p->D = D; p->k = k; p->ngpu = ngpu; p->rank = rank; p->dtype = dtype;
  hc_status s = hc_ep_range(D, k, ngpu, rank, &p->e0, &p->e1, &p->c0, &p->c1);
  if (s == HC_OK) s = hc_plan_create(&p->low, D - k, dtype, 1, 0);
  const uint64_t P = p->e1 - p->e0;
  if (s == HC_OK && P > 0) {
    const size_t bytes = sizeof(double) * (1ull << (D - k)) * P;
    if (cudaMalloc(&p->xh, bytes) != cudaSuccess || cudaMalloc(&p->yh, bytes) != cudaSuccess) {
      cudaGetLastError();
      s = HC_ERR_CAPACITY;
    }
  }
  if (s == HC_OK && P > 0 && p->low->g.two_level) {
    const Geometry& g = p->low->g;
    const size_t tbl = sizeof(double) * (size_t)(1ull << g.k) * upow3(g.M) * 256 * P;
    const uint64_t ns = P * g.nunits;  // slabs of all owned points
    if (cudaMalloc(&p->xu, tbl) != cudaSuccess || cudaMalloc(&p->yu, tbl) != cudaSuccess ||
        cudaMalloc(&p->ctr, sizeof(uint32_t) * (1 + 2 * ns)) != cudaSuccess ||
        cudaMalloc(&p->order, sizeof(uint4) * ns) != cudaSuccess) {
      cudaGetLastError();
      s = HC_ERR_CAPACITY;
    } else {
      // processing order: every point's slabs, cost-sorted together (as slab_order), slab
      // (point b, top index t) at output offset b * 3^k + t, problem index b in .w
      std::vector<std::pair<int, uint64_t>> v(ns);
      for (uint64_t i = 0; i < ns; ++i) {
        uint64_t t = i % g.nunits;
        int ones = 0;
        for (int a = 0; a < g.k; ++a, t /= 3) ones += (t % 3 == 1);
        v[i] = {ones, i};
      }
      std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      std::vector<uint4> h(ns);
      for (uint64_t i = 0; i < ns; ++i) {
        const uint64_t slab = v[i].second, b = slab / g.nunits;
        uint64_t t = slab % g.nunits;
        uint32_t base = 0, freeb = 0;
        for (int a = 0; a < g.k; ++a, t /= 3) {
          if (t % 3 == 2) base |= 1u << a;
          else if (t % 3 == 1) freeb |= 1u << a;
        }
        h[i] = make_uint4((uint32_t)slab, base, freeb, (uint32_t)b);
      }
      if (cudaMemcpy(p->order, h.data(), sizeof(uint4) * ns, cudaMemcpyHostToDevice) != cudaSuccess)
        s = HC_ERR_CUDA;
    }
  }
  if (s != HC_OK) {
    hc_ep_destroy(p);
    return s;
  }
  *out = p;
  return HC_OK;
}

extern "C" hc_status hc_ep_destroy(hc_ep_t p) {
  if (!p) return HC_ERR_NULL;
  if (p->low) hc_plan_destroy(p->low);
  cudaFree(p->xh);
  cudaFree(p->yh);
  cudaFree(p->xu);
  cudaFree(p->yu);
  cudaFree(p->order);
  cudaFree(p->ctr);
  delete p;
  return HC_OK;
}

namespace {
// all owned points in one pass: one evaluation launch for every point, then ONE batched
// (D-k)-dimensional convolution over the points (the tile engine's batch for D - k <= 12, the
// two-level engine over points x slabs otherwise), w = [point][3^(D-k)]
template <class T>
cudaError_t ep_local_t(hc_ep_t p, const T* x, const T* y, T* w, cudaStream_t st) {
  const int L = p->D - p->k;
  const uint64_t P = p->e1 - p->e0;
  if (P == 0) return cudaSuccess;
  {
    LaunchScope ls("ep_eval", st);
    dim3 g((unsigned)(((1ull << L) + 255) / 256), 2, (unsigned)P);
    ep_eval_kernel<T><<<g, 256, 0, st>>>(x, y, (T*)p->xh, (T*)p->yh, L, p->k, p->e0);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  const Geometry& g = p->low->g;
  if (!g.two_level)
    return launch_any(p->dtype, p->xh, p->yh, w, L, 0, g.nunits, P * g.nunits, st);
  const uint64_t ns = P * g.nunits;
  cudaError_t e = cudaErrorInvalidValue;
  if (g.M == 5) e = launch_prep<T, 5>((const T*)p->xh, (const T*)p->yh, (T*)p->xu, (T*)p->yu, g.k, st, (unsigned)P);
  if (g.M == 6) e = launch_prep<T, 6>((const T*)p->xh, (const T*)p->yh, (T*)p->xu, (T*)p->yu, g.k, st, (unsigned)P);
  if (e != cudaSuccess) return e;
  static const int lag = getenv("HC_SLAB_LAG") ? atoi(getenv("HC_SLAB_LAG")) : 1;
  SlabArgs a{0, (uint32_t)ns, g.k, p->ctr, p->order, 0, (uint32_t)(lag < 1 ? 1 : lag), nullptr, nullptr, 0, 0,
             0xffffffffu, (uint64_t)(1ull << g.k) * upow3(g.M) * 256};
  return launch_slab8<T>((const T*)p->xh, (const T*)p->yh, w, (T*)p->xu, (T*)p->yu, g.M, a, st, /*prep=*/false);
}
template <class T>
cudaError_t ep_finish_t(hc_ep_t p, const T* wt, T* z, cudaStream_t st) {
  const uint64_t ncols = p->c1 - p->c0;
  if (ncols == 0) return cudaSuccess;
  const unsigned g = (unsigned)((ncols + 127) / 128);
  if (p->k == 5) {
    cudaError_t e = cudaFuncSetAttribute(ep_top_inverse5<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)EP5_SMEM);
    if (e != cudaSuccess) return e;
  }
  LaunchScope ls("ep_inverse", st);
  switch (p->k) {
    case 1: ep_top_inverse<T, 1><<<g, 128, 0, st>>>(wt, z, ncols); break;
    case 2: ep_top_inverse<T, 2><<<g, 128, 0, st>>>(wt, z, ncols); break;
    case 3: ep_top_inverse<T, 3><<<g, 128, 0, st>>>(wt, z, ncols); break;
    case 4: ep_top_inverse<T, 4><<<g, 128, 0, st>>>(wt, z, ncols); break;
    default:
      ep_top_inverse5<T, false><<<(unsigned)((ncols + EP5_CW - 1) / EP5_CW), 256, EP5_SMEM, st>>>(
          wt, EPPeer{}, z, ncols, ncols, 0);
      break;
  }
  return cudaGetLastError();
}
}  // namespace

extern "C" hc_status hc_ep_local(hc_ep_t p, const void* x, const void* y, void* w, void* stream) {
  if (!p || !x || !y || !w) return HC_ERR_NULL;
  if (!aligned16(x) || !aligned16(y) || !aligned8(w)) return HC_ERR_ALIGN;
  cudaError_t e = p->dtype == HC_INT64
                      ? ep_local_t<uint64_t>(p, (const uint64_t*)x, (const uint64_t*)y, (uint64_t*)w, (cudaStream_t)stream)
                      : ep_local_t<double>(p, (const double*)x, (const double*)y, (double*)w, (cudaStream_t)stream);
  return e == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

extern "C" hc_status hc_ep_finish_peer(hc_ep_t p, const void* const* w_ranks, void* z, void* stream) {
  if (!p || !w_ranks || !z) return HC_ERR_NULL;
  if (p->ngpu > 8) return HC_ERR_SHARD;
  EPPeer pe{};
  const uint64_t np = upow3(p->k);
  for (int r = 0; r < p->ngpu; ++r) {
    if (!w_ranks[r]) return HC_ERR_NULL;
    pe.w[r] = w_ranks[r];
    uint64_t e0, e1, c0, c1;
    hc_ep_range(p->D, p->k, p->ngpu, r, &e0, &e1, &c0, &c1);
    for (uint64_t e = e0; e < e1; ++e) {
      pe.own[e] = (uint8_t)r;
      pe.base[e] = (uint32_t)(e - e0);
    }
  }
  (void)np;
  const uint64_t ncols = p->c1 - p->c0, nct = upow3(p->D - p->k);
  if (ncols == 0) return HC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = (unsigned)((ncols + 127) / 128);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    if (p->k == 5 && cudaFuncSetAttribute(ep_top_inverse5<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)EP5_SMEM) != cudaSuccess)
      return;
    LaunchScope ls("ep_inverse_peer", st);
    switch (p->k) {
      case 1: ep_top_inverse_peer<T, 1><<<g, 128, 0, st>>>(pe, (T*)z, ncols, nct, p->c0); break;
      case 2: ep_top_inverse_peer<T, 2><<<g, 128, 0, st>>>(pe, (T*)z, ncols, nct, p->c0); break;
      case 3: ep_top_inverse_peer<T, 3><<<g, 128, 0, st>>>(pe, (T*)z, ncols, nct, p->c0); break;
      case 4: ep_top_inverse_peer<T, 4><<<g, 128, 0, st>>>(pe, (T*)z, ncols, nct, p->c0); break;
      default:
        ep_top_inverse5<T, true><<<(unsigned)((ncols + EP5_CW - 1) / EP5_CW), 256, EP5_SMEM, st>>>(
            nullptr, pe, (T*)z, ncols, nct, p->c0);
        break;
    }
  };
  if (p->dtype == HC_INT64) go(uint64_t{});
  else go(double{});
  return cudaGetLastError() == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

extern "C" hc_status hc_ep_finish(hc_ep_t p, const void* wt, void* z, void* stream) {
  if (!p || !wt || !z) return HC_ERR_NULL;
  cudaError_t e = p->dtype == HC_INT64
                      ? ep_finish_t<uint64_t>(p, (const uint64_t*)wt, (uint64_t*)z, (cudaStream_t)stream)
                      : ep_finish_t<double>(p, (const double*)wt, (double*)z, (cudaStream_t)stream);
  return e == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

// ---------------------------------------------------------------------------------------
// Applications (include/hc.h; kernels in hc_apps.cuh)
#include "hc_apps.cuh"

namespace {
hc_status app_scratch(hc_plan_t p) {
  if (p->app_a) return HC_OK;
  const size_t bytes = sizeof(double) << p->D;
  if (cudaMalloc(&p->app_a, bytes) != cudaSuccess || cudaMalloc(&p->app_b, bytes) != cudaSuccess ||
      cudaMalloc(&p->app_mx, 2 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p->app_a);
    cudaFree(p->app_b);
    cudaFree(p->app_mx);
    p->app_a = p->app_b = nullptr;
    p->app_mx = nullptr;
    return HC_ERR_CAPACITY;
  }
  return HC_OK;
}
unsigned ew_grid(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}
template <class T, int L>
cudaError_t carry_tile(const T* z, T* part, uint64_t ntiles, cudaStream_t st) {
  if constexpr (L == 8) {
    const size_t sm = sizeof(T) * (size_t)(6561 + 243 * 15 + 81 * 31);
    auto k = carry_tile8_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t grid = ntiles < 2ull * nsm ? ntiles : 2ull * nsm;
    LaunchScope ls("carry", st);
    k<<<(unsigned)grid, 256, sm, st>>>(z, part, ntiles);
    return cudaGetLastError();
  } else {
    const size_t sm = 2 * sizeof(T) * (size_t)ipow3(L);
    auto k = carry_tile_kernel<T, L>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    LaunchScope ls("carry", st);
    k<<<(unsigned)ntiles, 256, sm, st>>>(z, part);
    return cudaGetLastError();
  }
}
// one global combining step for axis c (compile-time c, 32-bit indices when they fit)
template <class T, int C>
cudaError_t carry_step_c(const T* A, T* B, uint64_t nr2, uint64_t n2, cudaStream_t st) {
  if (n2 < (1ull << 32)) carry_step_kernel<T, uint32_t, C><<<ew_grid(n2), 256, 0, st>>>(A, B, nr2);
  else carry_step_kernel<T, uint64_t, C><<<ew_grid(n2), 256, 0, st>>>(A, B, nr2);
  return cudaGetLastError();
}
template <class T, int C = 8>
cudaError_t carry_step(const T* A, T* B, uint64_t nr2, uint64_t n2, int c, cudaStream_t st) {
  if constexpr (C < HC_MAX_D) {
    if (c == C) return carry_step_c<T, C>(A, B, nr2, n2, st);
    return carry_step<T, C + 1>(A, B, nr2, n2, c, st);
  }
  return cudaErrorInvalidValue;
}
template <class T>
cudaError_t apply_carries_t(int D, const T* z, T* out, T* work, cudaStream_t st) {
  const int L = D < 8 ? D : 8;
  const uint64_t ntiles = upow3(D - L);
  T* part = D == L ? out : work;
  cudaError_t e;
  switch (L) {
    case 1: e = carry_tile<T, 1>(z, part, ntiles, st); break;
    case 2: e = carry_tile<T, 2>(z, part, ntiles, st); break;
    case 3: e = carry_tile<T, 3>(z, part, ntiles, st); break;
    case 4: e = carry_tile<T, 4>(z, part, ntiles, st); break;
    case 5: e = carry_tile<T, 5>(z, part, ntiles, st); break;
    case 6: e = carry_tile<T, 6>(z, part, ntiles, st); break;
    case 7: e = carry_tile<T, 7>(z, part, ntiles, st); break;
    default: e = carry_tile<T, 8>(z, part, ntiles, st); break;
  }
  if (e != cudaSuccess) return e;
  // remaining axes c = L .. D-1 in global memory, ping-pong in `work`
  const uint64_t half = D > 8 ? upow3(D - 8) * 511 : 0;
  T* A = part;
  uint64_t nr = ntiles;
  for (int c = L; c < D; ++c) {
    const uint64_t nr2 = nr / 3;
    T* B = (c + 1 == D) ? out : (A == work ? work + half : work);
    const uint64_t n2 = nr2 * ((4ull << c) - 1);
    LaunchScope ls("carry", st);
    e = carry_step<T>(A, B, nr2, n2, c, st);
    if (e != cudaSuccess) return e;
    A = B;
    nr = nr2;
  }
  return cudaSuccess;
}
}  // namespace

extern "C" uint64_t hc_carries_work_len(int D) {
  if (D < 1 || D > HC_MAX_D) return 0;
  return D <= 8 ? 0 : 2 * upow3(D - 8) * 511;
}

extern "C" hc_status hc_apply_carries(int D, hc_dtype dtype, const void* z, void* out, void* work, void* stream) {
  if (D < 1 || D > HC_MAX_D) return HC_ERR_INVALID_DIM;
  if (dtype != HC_INT64 && dtype != HC_FP64) return HC_ERR_DTYPE;
  if (!z || !out || (D > 8 && !work)) return HC_ERR_NULL;
  hc_status ds = check_device();
  if (ds != HC_OK) return ds;
  cudaError_t e = dtype == HC_INT64
                      ? apply_carries_t<uint64_t>(D, (const uint64_t*)z, (uint64_t*)out, (uint64_t*)work, (cudaStream_t)stream)
                      : apply_carries_t<double>(D, (const double*)z, (double*)out, (double*)work, (cudaStream_t)stream);
  return e == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

extern "C" hc_status hc_conv1d(hc_plan_t p, const void* x, const void* y, void* z_work, void* out, void* work,
                               void* stream) {
  if (!p || !x || !y || !out) return HC_ERR_NULL;
  if (!aligned16(x) || !aligned16(y) || !aligned8(out)) return HC_ERR_ALIGN;
  if (p->ngpu != 1) return HC_ERR_SHARD;
  const int D = p->D;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->dtype == HC_INT64 && p->g.two_level) {
    // the slab engine adds every final z[k] into out[val(k)] (uint64, exact in any order);
    // pass-1 tiles live in z_work when given (3^D), else in the plan's ring of slab buffers
    if (cudaMemsetAsync(out, 0, sizeof(uint64_t) * ((2ull << D) - 1), st) != cudaSuccess) return HC_ERR_CUDA;
    if (z_work) {
      if (!aligned8(z_work)) return HC_ERR_ALIGN;
      return run_range(p, x, y, z_work, 0, p->g.nunits, st, 0, (unsigned long long*)out, nullptr);
    }
    if (!p->ring) {
      if (cudaMalloc(&p->ring, sizeof(uint64_t) * (size_t)p->g.unit * T8_RING) != cudaSuccess) {
        cudaGetLastError();
        p->ring = nullptr;
        return HC_ERR_CAPACITY;
      }
    }
    return run_range(p, x, y, nullptr, 0, p->g.nunits, st, 0, (unsigned long long*)out, p->ring);
  }
  if (!z_work) return HC_ERR_NULL;
  if (!aligned8(z_work)) return HC_ERR_ALIGN;
  if (D > 8 && !work) return HC_ERR_NULL;
  hc_status s = run_range(p, x, y, z_work, 0, p->g.nunits, st, 0);
  if (s != HC_OK) return s;
  return hc_apply_carries(D, p->dtype, z_work, out, work, stream);
}

extern "C" hc_status hc_convolve_difference(hc_plan_t p, const void* x, const void* y, void* z, void* stream) {
  if (!p || !x || !y || !z) return HC_ERR_NULL;
  if (!aligned16(x) || !aligned16(y) || !aligned8(z)) return HC_ERR_ALIGN;
  hc_status s = app_scratch(p);
  if (s != HC_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  {
    LaunchScope ls("flip", st);
    if (p->dtype == HC_INT64) flip_kernel<uint64_t><<<ew_grid(1ull << p->D), 256, 0, st>>>((const uint64_t*)y, (uint64_t*)p->app_a, p->D);
    else flip_kernel<double><<<ew_grid(1ull << p->D), 256, 0, st>>>((const double*)y, (double*)p->app_a, p->D);
    if (cudaGetLastError() != cudaSuccess) return HC_ERR_CUDA;
  }
  return run_range(p, x, p->app_a, z, 0, p->g.nunits, st, 0);
}

extern "C" hc_status hc_maxconv_pnorm(hc_plan_t p, const void* x, const void* y, void* z, double pw, int round_to_int,
                                      void* stream) {
  if (!p || !x || !y || !z) return HC_ERR_NULL;
  if (p->dtype != HC_FP64) return HC_ERR_DTYPE;
  if (!(pw >= 1.0)) return HC_ERR_INVALID_DIM;
  if (!aligned16(x) || !aligned16(y) || !aligned8(z)) return HC_ERR_ALIGN;
  hc_status s = app_scratch(p);
  if (s != HC_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t n = 1ull << p->D;
  int sq = -1;  // p = 2^sq: powers by squaring and roots by square roots (exact shape of the paper's p)
  for (int k = 0; k < 11; ++k)
    if (pw == (double)(1 << k)) sq = k;
  if (cudaMemsetAsync(p->app_mx, 0, 2 * sizeof(unsigned long long), st) != cudaSuccess) return HC_ERR_CUDA;
  {
    LaunchScope ls("pnorm_pre", st);
    max_nonneg_kernel<<<ew_grid(n), 256, 0, st>>>((const double*)x, n, p->app_mx);
    max_nonneg_kernel<<<ew_grid(n), 256, 0, st>>>((const double*)y, n, p->app_mx + 1);
    pnorm_pre_kernel<<<ew_grid(n), 256, 0, st>>>((const double*)x, (double*)p->app_a, n, pw, sq, p->app_mx);
    pnorm_pre_kernel<<<ew_grid(n), 256, 0, st>>>((const double*)y, (double*)p->app_b, n, pw, sq, p->app_mx + 1);
    if (cudaGetLastError() != cudaSuccess) return HC_ERR_CUDA;
  }
  s = run_range(p, p->app_a, p->app_b, z, 0, p->g.nunits, st, 0);
  if (s != HC_OK) return s;
  LaunchScope ls("pnorm_post", st);
  pnorm_post_kernel<<<ew_grid(upow3(p->D)), 256, 0, st>>>((double*)z, upow3(p->D), pw, sq, p->app_mx, round_to_int);
  return cudaGetLastError() == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}
