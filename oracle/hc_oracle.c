/*
 * hc_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU
 * oracle for hypercube convolution (Serang, arXiv:1608.00206).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * this library.  It shares no code, header, table or helper with the CUDA path in
 * paper_1608_00206_b200/csrc/ and neither side includes the other.
 *
 * What it computes (PAPER.md, Introduction, lines 30-34):
 *     (x * y)[k] = sum_{i,j : k = i + j} x[i] * y[j]
 * with i, j in {0,1}^D and k = i + j taken digit-wise, so k in {0,1,2}^D.
 * The oracle is the paper's Algorithm 1 "Naive multidimensional convolution"
 * (PAPER.md lines 40-60): z <- 0; for i: for j: z[i+j] += x[i]*y[j].
 *
 * Layout (reading R1; "boolean indices ... embedded
 * into a single machine precision integer"): bit b of the flat input index is axis b;
 * the flat output index is k = sum_b k_b * 3^b.  Because every digit sum i_b + j_b <= 2
 * there is never a carry, so flat(i + j) = T(i) + T(j) with T(i) = sum_b bit_b(i) 3^b.
 *
 * Arithmetic: fp64 as C `double`; int64 as uint64_t (wrap-around mod 2^64, then
 * reinterpreted as int64 -- DESIGN.md reading R3).  Build with -O2 -ffp-contract=off and
 * without -ffast-math so no multiply-add is contracted into an FMA (the accumulation is
 * exactly Algorithm 1's "z[i+j] += x[i]*y[j]": one rounded product, one rounded add).
 *
 * Functions:
 *   orc_ternary_of_binary   T(i) above.
 *   orc_conv_scatter_*      Algorithm 1 literally (i-major, j-minor).  Single thread.
 *   orc_conv_gather_*       The same sums, cell by cell: for cell k the pairs (i,j) with
 *                           i + j = k are enumerated in ascending i, i.e. in the order
 *                           Algorithm 1 adds them into z[k], so the result is bitwise
 *                           identical to the scatter form (each i has at most one partner
 *                           j for a fixed k).  Parallel over cells with OpenMP.
 *   orc_conv_cells_*        the gather form for a caller-chosen list of cells (sampled
 *                           parity at sizes where 4^D pairs is too many).
 *   orc_conv_batched_*      the gather form over B independent pairs (row-major batches,
 *                           DESIGN.md reading R8).
 * No function here is the method under test: none uses the Karatsuba split.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* T(i) = sum_b bit_b(i) * 3^b  (PAPER.md 109-112; R1). */
uint64_t orc_ternary_of_binary(uint64_t i) {
    uint64_t t = 0, p = 1;
    while (i) {
        if (i & 1u) t += p;
        p *= 3u;
        i >>= 1;
    }
    return t;
}

uint64_t orc_pow3(int D) {
    uint64_t p = 1;
    for (int b = 0; b < D; ++b) p *= 3u;
    return p;
}

/* ---- Algorithm 1, literal (PAPER.md 40-60) --------------------------------------- */
void orc_conv_scatter_f64(int D, const double* x, const double* y, double* z) {
    const uint64_t n = (uint64_t)1 << D, m = orc_pow3(D);
    memset(z, 0, m * sizeof(double));                 /* "Initialize with zeros" */
    for (uint64_t i = 0; i < n; ++i) {                /* for i */
        const uint64_t ti = orc_ternary_of_binary(i);
        for (uint64_t j = 0; j < n; ++j) {            /* for j */
            z[ti + orc_ternary_of_binary(j)] += x[i] * y[j];   /* z[i+j] += x[i]*y[j] */
        }
    }
}

void orc_conv_scatter_i64(int D, const int64_t* x, const int64_t* y, int64_t* z) {
    const uint64_t n = (uint64_t)1 << D, m = orc_pow3(D);
    uint64_t* zu = (uint64_t*)z;
    const uint64_t* xu = (const uint64_t*)x;
    const uint64_t* yu = (const uint64_t*)y;
    memset(z, 0, m * sizeof(int64_t));
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t ti = orc_ternary_of_binary(i);
        for (uint64_t j = 0; j < n; ++j)
            zu[ti + orc_ternary_of_binary(j)] += xu[i] * yu[j];
    }
}

/* ---- one output cell, pairs in ascending i ----------------------------------------
 * Digits of k: k_b = 0 -> i_b = j_b = 0; k_b = 2 -> i_b = j_b = 1;
 * k_b = 1 -> (i_b, j_b) in {(0,1), (1,0)} (PAPER.md 166-171, the three cases for k_1).
 * base = bits with k_b = 2, free = bits with k_b = 1; i = base | s for every subset s of
 * free, j = base | (free & ~s).  Subsets are visited in ascending order of s, which is
 * ascending i. */
static inline int cell_split(int D, uint64_t k, uint64_t* base, uint64_t* freeb) {
    uint64_t b2 = 0, b1 = 0;
    for (int b = 0; b < D; ++b) {
        const uint64_t d = k % 3u;
        k /= 3u;
        if (d == 2u) b2 |= (uint64_t)1 << b;
        else if (d == 1u) b1 |= (uint64_t)1 << b;
    }
    *base = b2;
    *freeb = b1;
    return k == 0;   /* 0 if k >= 3^D */
}

static inline double cell_f64(int D, const double* x, const double* y, uint64_t k) {
    uint64_t base, fr;
    if (!cell_split(D, k, &base, &fr)) return 0.0;
    double acc = 0.0;
    uint64_t s = 0;
    do {
        acc += x[base | s] * y[base | (fr & ~s)];
        s = (s - fr) & fr;           /* next subset of fr in ascending order */
    } while (s != 0);
    return acc;
}

static inline uint64_t cell_u64(int D, const uint64_t* x, const uint64_t* y, uint64_t k) {
    uint64_t base, fr;
    if (!cell_split(D, k, &base, &fr)) return 0;
    uint64_t acc = 0;
    uint64_t s = 0;
    do {
        acc += x[base | s] * y[base | (fr & ~s)];
        s = (s - fr) & fr;
    } while (s != 0);
    return acc;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_conv_gather_f64(int D, const double* x, const double* y, double* z, int nthreads) {
    const int64_t m = (int64_t)orc_pow3(D);
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t k = 0; k < m; ++k) z[k] = cell_f64(D, x, y, (uint64_t)k);
}

void orc_conv_gather_i64(int D, const int64_t* x, const int64_t* y, int64_t* z, int nthreads) {
    const int64_t m = (int64_t)orc_pow3(D);
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t k = 0; k < m; ++k)
        ((uint64_t*)z)[k] = cell_u64(D, (const uint64_t*)x, (const uint64_t*)y, (uint64_t)k);
}

void orc_conv_cells_f64(int D, const double* x, const double* y, const uint64_t* ks, int64_t n,
                        double* out, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < n; ++c) out[c] = cell_f64(D, x, y, ks[c]);
}

void orc_conv_cells_i64(int D, const int64_t* x, const int64_t* y, const uint64_t* ks, int64_t n,
                        int64_t* out, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < n; ++c)
        ((uint64_t*)out)[c] = cell_u64(D, (const uint64_t*)x, (const uint64_t*)y, ks[c]);
}

/* B independent pairs, row-major: x[b*2^D + i], z[b*3^D + k]  (R8). */
void orc_conv_batched_f64(int B, int D, const double* x, const double* y, double* z, int nthreads) {
    const uint64_t n = (uint64_t)1 << D, m = orc_pow3(D);
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b)
        for (uint64_t k = 0; k < m; ++k)
            z[(uint64_t)b * m + k] = cell_f64(D, x + (uint64_t)b * n, y + (uint64_t)b * n, k);
}

void orc_conv_batched_i64(int B, int D, const int64_t* x, const int64_t* y, int64_t* z, int nthreads) {
    const uint64_t n = (uint64_t)1 << D, m = orc_pow3(D);
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b)
        for (uint64_t k = 0; k < m; ++k)
            ((uint64_t*)z)[(uint64_t)b * m + k] =
                cell_u64(D, (const uint64_t*)x + (uint64_t)b * n, (const uint64_t*)y + (uint64_t)b * n, k);
}

/* sampled cells of a batched problem: (batch index, cell index) pairs */
void orc_conv_batched_cells_i64(int D, const int64_t* x, const int64_t* y, const uint64_t* bs,
                                const uint64_t* ks, int64_t n, int64_t* out, int nthreads) {
    const uint64_t nn = (uint64_t)1 << D;
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < n; ++c)
        ((uint64_t*)out)[c] = cell_u64(D, (const uint64_t*)x + bs[c] * nn, (const uint64_t*)y + bs[c] * nn, ks[c]);
}
