/* Minimal C user of the boundary (include/hc.h): one D = 10 int64 convolution through the
 * host-buffer entry point, checked against the definition z[k] = sum_{i+j=k} x[i] y[j]
 * (digit-wise index addition, PAPER.md 30-34) computed here by brute force.
 *
 * Build (from the repository root, after `python paper_1608_00206_b200/build.py`):
 *   gcc -O2 -Iinclude examples/hc_example.c -Lpaper_1608_00206_b200 -lhc \
 *       -Wl,-rpath,$PWD/paper_1608_00206_b200 -o examples/hc_example
 * Run on a machine with a B200: ./examples/hc_example  (exit status 0 = match) */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hc.h"

enum { D = 10 };

/* ternary value of the bits of i: sum_b bit_b(i) 3^b */
static uint64_t ternary_of_bits(uint64_t i) {
  uint64_t t = 0, p = 1;
  for (int b = 0; b < D; ++b, p *= 3) t += ((i >> b) & 1u) * p;
  return t;
}

int main(void) {
  const uint64_t n = hc_in_len(D), m = hc_out_len(D);
  int64_t* x = malloc(n * sizeof *x);
  int64_t* y = malloc(n * sizeof *y);
  int64_t* z = malloc(m * sizeof *z);
  int64_t* want = calloc(m, sizeof *want);
  if (!x || !y || !z || !want) return 2;
  uint64_t s = 12345;
  for (uint64_t i = 0; i < n; ++i) {  /* small pseudo-random entries in [0, 9] */
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    x[i] = (int64_t)((s >> 33) % 10);
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    y[i] = (int64_t)((s >> 33) % 10);
  }
  hc_plan_t plan = NULL;
  hc_status st = hc_plan_create(&plan, D, HC_INT64, 1, 0);
  if (st != HC_OK) {
    fprintf(stderr, "hc_plan_create: %s\n", hc_status_str(st));
    return 1;
  }
  st = hc_convolve_host(plan, x, y, z, NULL);
  hc_plan_destroy(plan);
  if (st != HC_OK) {
    fprintf(stderr, "hc_convolve_host: %s\n", hc_status_str(st));
    return 1;
  }
  for (uint64_t i = 0; i < n; ++i)  /* the definition: every pair (i, j) lands on T(i) + T(j) */
    for (uint64_t j = 0; j < n; ++j) want[ternary_of_bits(i) + ternary_of_bits(j)] += x[i] * y[j];
  uint64_t bad = 0;
  for (uint64_t k = 0; k < m; ++k) bad += z[k] != want[k];
  printf("D=%d: %llu of %llu output entries differ\n", D, (unsigned long long)bad, (unsigned long long)m);
  free(x);
  free(y);
  free(z);
  free(want);
  return bad != 0;
}
