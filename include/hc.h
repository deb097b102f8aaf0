/*
 * hc.h -- C ABI of the B200-native hypercube-convolution library (libhc.so).
 *
 * Operation (Introduction):
 *     z[k] = sum_{i,j : k = i + j} x[i] * y[j],   i, j in {0,1}^D,  k in {0,1,2}^D,
 * computed with the paper's Karatsuba-style per-axis split (PAPER.md lines 185-192,
 * Methods): forward (a0, a1) -> (a0, a0 + a1, a1), pointwise product, inverse
 * (c0, c1, c2) -> (c0, (c1 - c0) - c2, c2) (the two subtraction loops of Algorithm 2,
 * PAPER.md lines 248-251), combined with the paper's 4-sub-convolution split
 * on the top axes.  The result is identical (int64) or equal
 * up to rounding (fp64) to the naive Algorithm 1.
 *
 * Layout (all entry points):
 *   x, y : 2^D elements, flat index i = sum_b i_b 2^b  (bit b = axis b; PAPER.md 109-112)
 *   z    : 3^D elements, flat index k = sum_b k_b 3^b  (trit b = axis b)
 *   batched: row-major [B][2^D] -> [B][3^D].
 * Element types: HC_INT64 (computed as wrapping uint64: exact whenever the true z[k]
 *   fits in int64; PAPER.md 191-192 "exact when the dynamic range allows (a+b)-a=b"),
 *   HC_FP64 (IEEE double; deterministic, bit-identical run to run).
 * Ownership: the caller owns x, y, z.  x and y are never modified (unlike Algorithm 2,
 *   PAPER.md 225, which destroys its inputs).  z must not alias x or y.  A plan owns
 *   only small tables, its own device buffers for the host-pointer entry point, and
 *   counters.  x and y must be 16-byte aligned (their slices are staged by TMA bulk copies),
 *   z 8-byte aligned (one element); torch allocations are 256-B aligned.
 * Streams: all device work is enqueued on `stream` (a cudaStream_t passed as void*;
 *   NULL = legacy default stream).  Calls return after enqueueing; launch errors are
 *   reported immediately (HC_ERR_CUDA); execution errors surface at the caller's sync.
 * Errors: every function returns hc_status; nothing throws across the ABI.  D must be in
 *   [1, HC_MAX_D] (D = 0 is rejected; the paper's recursion bottoms out at D = 1,
 *   PAPER.md 255-263).
 * Thread safety / concurrency: a plan holds device state that its calls reuse -- the slab
 *   engine's work and completion counters (D >= 13), the scratch of the application entry
 *   points and the host-buffer entry point's workspace.  Calls on ONE plan must therefore be
 *   ordered (one stream, or streams ordered by events); to run convolutions concurrently on
 *   several streams or threads, create one plan per stream.  Plans of different devices are
 *   independent (create each with its device current).
 */
#ifndef HC_H
#define HC_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_MAX_D 24

typedef enum {
    HC_OK = 0,
    HC_ERR_INVALID_DIM = 1,  /* D outside [1, HC_MAX_D], or B < 1 */
    HC_ERR_DTYPE = 2,        /* unknown hc_dtype */
    HC_ERR_NULL = 3,         /* a required pointer is NULL */
    HC_ERR_ALIGN = 4,        /* x or y not 16-byte aligned, or z not 8-byte aligned */
    HC_ERR_DEVICE = 5,       /* no CUDA device / wrong architecture (needs sm_100) */
    HC_ERR_CAPACITY = 6,     /* device memory cannot hold the requested buffers */
    HC_ERR_CUDA = 7,         /* a CUDA runtime call or kernel launch failed */
    HC_ERR_SHARD = 9         /* rank / ngpu inconsistent with the plan */
} hc_status;

typedef enum { HC_INT64 = 0, HC_FP64 = 1 } hc_dtype;

typedef struct hc_plan_s* hc_plan_t;

/* Status text (static string). */
const char* hc_status_str(hc_status s);

/* 2^D and 3^D (0 if D is out of range, i.e. outside [1, HC_MAX_D]): the lengths of the
 * inputs x, y in {0,1}^D and of the output z in {0,1,2}^D of the convolution
 * z[k] = sum_{i+j=k} x[i] y[j] (PAPER.md 30-34, Introduction; reading R2 for D >= 1). */
uint64_t hc_in_len(int D);
uint64_t hc_out_len(int D);

/* Create a plan for one D-dimensional convolution on the current CUDA device.
 * ngpu >= 1 ranks share the output: rank r owns the contiguous flat range of z returned
 * by hc_shard_info (the zero-communication split of the output by its top trits, using
 * the paper's 4-way split, PAPER.md 166-177).  ngpu == 1, rank == 0 for a single GPU. */
hc_status hc_plan_create(hc_plan_t* out, int D, hc_dtype dtype, int ngpu, int rank);
hc_status hc_plan_destroy(hc_plan_t plan);

/* Flat range [z_begin, z_end) of z owned by `rank` under the plan's ngpu-way split: whole
 * output slabs (fixed top trits t_T), which the paper's 4-way split computes independently
 * of each other (PAPER.md 166-177, Methods), cut at equal estimated cost (hc_shard_range).
 * Errors: HC_ERR_NULL (null pointer), HC_ERR_SHARD (rank outside [0, ngpu)). */
hc_status hc_shard_info(hc_plan_t plan, int rank, uint64_t* z_begin, uint64_t* z_end);

/* Pure host function (no device needed): the flat range [z_begin, z_end) of z that rank
 * `rank` of `ngpu` owns for dimension D -- the same split hc_plan_create uses.  Ranges
 * are contiguous, disjoint, cover [0, 3^D) in rank order, and are cut at output-slab
 * boundaries so that the per-rank cost (one unit per direct-split pair plus a fixed cost
 * per slab) is balanced. */
hc_status hc_shard_range(int D, int ngpu, int rank, uint64_t* z_begin, uint64_t* z_end);

/* Whole convolution: x, y device pointers (2^D elements), z device pointer (3^D).
 * Stream-ordered, no host synchronisation (the plan's processing order is uploaded at plan
 * creation).  Results are deterministic: fp64 sums in a fixed order; int64 is exact mod 2^64
 * (reading R3) -- at D = 11, 12 the engine zeroes z on the stream and adds each direct-split
 * pair's contribution with 64-bit atomics, which commute exactly.  One call at a time per plan
 * and stream slot (the plan's counters are reused). */
hc_status hc_convolve(hc_plan_t plan, const void* x, const void* y, void* z, void* stream);

/* This rank's share: x, y replicated (2^D each, device); z_shard has
 * z_end - z_begin elements (device) and receives z[z_begin : z_end]. */
hc_status hc_convolve_sharded(hc_plan_t plan, const void* x, const void* y, void* z_shard,
                              void* stream);

/* B independent convolutions of dimension D (PAPER.md 30-34 for each pair; BASELINE.json
 * config 2 / north_star (5): many small cubes).  Layout (reading R8): x, y are [B][2^D]
 * row-major, z is [B][3^D] row-major; device pointers owned by the caller; x, y 16-byte
 * aligned, z 8-byte aligned; z must not alias x or y.  Stream-ordered; int64 is exact mod
 * 2^64 (reading R3).  int64 at D = 8 computes every cube with 2^8 max|x| max|y| < 2^31 in
 * 32-bit words (exact: reading R14) and the others in 64-bit words; the list of the latter
 * lives in stream-ordered scratch (B + 1 words from a library-owned memory pool, freed on
 * the stream), so concurrent calls on different streams are independent (HC_NARROW=0 in
 * the environment forces 64-bit words).  Errors: HC_ERR_INVALID_DIM (B < 1 or D outside
 * [1, HC_MAX_D]), HC_ERR_DTYPE, HC_ERR_NULL, HC_ERR_ALIGN, HC_ERR_DEVICE, HC_ERR_CUDA
 * (launch or scratch-allocation failure). */
hc_status hc_convolve_batched(int B, int D, hc_dtype dtype, const void* x, const void* y,
                              void* z, void* stream);

/* End-to-end entry point with HOST buffers: copies x, y (2^D each) to the device,
 * computes this rank's share of z and copies it back into z_host (z_end - z_begin
 * elements).  Host buffers should be pinned for full PCIe/C2C bandwidth.  Device
 * output is produced and drained in chunks so the copy overlaps the computation.
 * Synchronous: returns after z_host is complete. */
hc_status hc_convolve_host(hc_plan_t plan, const void* x_host, const void* y_host,
                           void* z_host, void* stream);

/* ---- Evaluation-point variant of the multi-GPU split (BASELINE.json north_star (4);
 * SURVEY.md §8(e) "K5b").  The top k axes (1 <= k <= 5, k < D) use the paper's Karatsuba
 * split (PAPER.md 185-192) ACROSS ranks: rank r owns the evaluation points
 * e_T in [e_begin, e_end) of {0,1,2}^k (flat base-3 index, trit b = axis D-k+b) and computes
 *     w[e_T][.] = conv_{D-k}( xh[e_T], yh[e_T] ),   xh[e_T][i_L] = sum_{i_T ~ e_T} x[i_T][i_L]
 * (the forward over the top axes -- a0, a0 + a1, a1 per axis -- then the whole
 * (D-k)-dimensional convolution with this library's engine).  An all-to-all, done by the
 * caller (NCCL send/recv or peer copies), gives rank h the columns [col_begin, col_end) of
 * w for all 3^k points; hc_ep_finish then interpolates over the top k axes,
 *     z[k_T][col] = sum_{e_T} Inv[k_T][e_T] w[e_T][col],  per axis (c0, (c1-c0)-c2, c2),
 * PAPER.md 187-189 / 248-251.  Rank h's output is the 3^k strided chunks
 * z[k_T * 3^(D-k) + col], col in its column range, delivered dense as [3^k][ncols]. */
typedef struct hc_ep_s* hc_ep_t;

/* Pure host: the evaluation points [e_begin, e_end) and columns [col_begin, col_end) of
 * `rank` (contiguous, disjoint, in rank order, sizes differing by at most one).
 * Requires ngpu <= 3^k; HC_ERR_SHARD otherwise. */
hc_status hc_ep_range(int D, int k, int ngpu, int rank, uint64_t* e_begin, uint64_t* e_end,
                      uint64_t* col_begin, uint64_t* col_end);
/* Plan for one rank: the (D-k)-dimensional geometry, the evaluated operands of every owned
 * point (2 x P x 2^(D-k) elements, P = e_end - e_begin) and, when D - k >= 13, the
 * two-level engine's middle-axes tables, slab order and counters for all P points.
 * HC_ERR_CAPACITY when device memory runs out (nothing is left allocated). */
hc_status hc_ep_create(hc_ep_t* out, int D, int k, hc_dtype dtype, int ngpu, int rank);
hc_status hc_ep_destroy(hc_ep_t p);
/* Local step: x, y (2^D each, device, replicated); w (device) receives
 * (e_end - e_begin) x 3^(D-k) elements, row e_T - e_begin.  All owned points run as one
 * batch: one evaluation launch, then one batched (D-k)-dimensional convolution (tile engine
 * for D - k <= 12, two-level engine over points x slabs otherwise).  Stream-ordered; the
 * plan's scratch is reused, so calls on one plan must not overlap (one stream at a time). */
hc_status hc_ep_local(hc_ep_t p, const void* x, const void* y, void* w, void* stream);
/* Final step: wt = [3^k][ncols] gathered columns of w (device), z = [3^k][ncols] (device),
 * ncols = col_end - col_begin; z must not alias wt. */
hc_status hc_ep_finish(hc_ep_t p, const void* wt, void* z, void* stream);

/* f3: the exchange fused into the final step.  w_ranks[r] is rank r's
 * hc_ep_local output (device pointers; on a multi-GPU node peer-mapped buffers of the other
 * ranks, e.g. CUDA IPC / symmetric memory, read over NVLink), ngpu entries; z = [3^k][ncols]
 * as in hc_ep_finish.  No gathered copy of w is made: each thread reads its column's 3^k
 * values straight from their owners' buffers. */
hc_status hc_ep_finish_peer(hc_ep_t p, const void* const* w_ranks, void* z, void* stream);

/* ---- Applications built on the hot path ------------------------------ */

/* f4: PMF of the difference X - Y of independent random vectors with Bernoulli axes
 * (PAPER.md 35-38, 147-149).  x[i] = P(X = i), y[j] = P(Y = j) (2^D each); z (3^D) receives
 * z[k] = P(X - Y = d) with d_b = k_b - 1 in {-1, 0, 1}, k = sum_b k_b 3^b.  Computed as
 * conv(x, flip(y)), flip(y)[j] = y[~j] (per-axis complement: X - Y + 1 = X + (1 - Y)); the
 * plan keeps flip(y) in its own scratch (2^D elements).  Whole output (like hc_convolve). */
hc_status hc_convolve_difference(hc_plan_t plan, const void* x, const void* y, void* z, void* stream);

/* f1: carries -- turns the carry-free convolution (the hot path on two length-2^D vectors,
 * bit b of an index = axis b; PAPER.md 354-373) into the ordinary 1-D convolution:
 *     out[m] = sum_{k : sum_b k_b 2^b = m} z[k],   m in [0, 2^(D+1) - 1).
 * z: 3^D elements (device), out: 2^(D+1) - 1 elements (device), work: hc_carries_work_len(D)
 * elements of the same type (device; may be NULL when that is 0).  Stream-ordered. */
uint64_t hc_carries_work_len(int D);
hc_status hc_apply_carries(int D, hc_dtype dtype, const void* z, void* out, void* work, void* stream);

/* Ordinary 1-D convolution out[m] = sum_i x[i] y[m - i], m < 2^(D+1) - 1, of two length-2^D
 * vectors: the carry-free (hypercube) convolution of their bit-axis embeddings followed by the
 * carries (PAPER.md 354-373).  plan: single-GPU plan of dimension D and the vectors' dtype.
 * out: 2^(D+1) - 1 elements (device, overwritten).  For int64 plans with D >= 13 the carries
 * are fused into the slab engine's pass 2 (every final z[k] is added into out[sum_b k_b 2^b]
 * with exact wrapping uint64 atomics) and z is never formed; pass-1 tiles live in z_work
 * (3^D elements) when it is given, else in a plan-owned ring of 4 slab buffers
 * (4 x 3^min(D,14) elements, allocated on first use; ~4% slower at D = 20) -- work may be
 * NULL.  Otherwise (fp64, D < 13) z_work (3^D elements, device) and work
 * (hc_carries_work_len(D) elements) are required: hc_convolve, then hc_apply_carries.
 * Errors: HC_ERR_SHARD for a multi-rank plan; otherwise as hc_convolve. */
hc_status hc_conv1d(hc_plan_t plan, const void* x, const void* y, void* z_work, void* out, void* work,
                    void* stream);

/* f2: p-norm max-convolution (PAPER.md 341-352), fp64 plans only.  x, y >= 0 (2^D each):
 *     z[k] = mx * my * ( sum_{i+j=k} (x[i]/mx)^p (y[j]/my)^p )^(1/p),   mx = max x, my = max y,
 * which lies in [M, n_k^(1/p) M] for the max-convolution M = max_{i+j=k} x[i] y[j] and the
 * n_k = 2^{#1(k)} terms of cell k (relative error <= 1 - n_k^(-1/p)).  round_to_int != 0
 * rounds z to the nearest integer: exact for integer inputs whenever M (2^D)^(1/p) - M < 0.5
 * over all cells (the paper's bounded-range criterion) and no nonzero term underflows.
 * p >= 1.  The plan keeps the scaled powers in its scratch (2 x 2^D elements). */
hc_status hc_maxconv_pnorm(hc_plan_t plan, const void* x, const void* y, void* z, double p, int round_to_int,
                           void* stream);

/* Instrumentation (for bench.py / tests): cumulative number of kernels this library has
 * launched in this process, and per-kernel device time when profiling is enabled
 * (events recorded around each launch on the launching stream). */
uint64_t hc_launch_count(void);
void hc_prof_enable(int on);
/* name: "small", "tile", "slab_p1", "slab_p2", "prep" ...; returns HC_OK and fills
 * total milliseconds and launch count (0 if never launched).  Synchronizes the events. */
hc_status hc_prof_read(const char* name, double* total_ms, uint64_t* launches);
void hc_prof_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* HC_H */
