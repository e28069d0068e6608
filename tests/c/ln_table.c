/* Test helper (not product): ln of consecutive integers correctly rounded to fp64, through
 * binary128 logq (~2^-112) and one rounding -- the definition R31 gives P:193's log.
 * Compiled by tests/test_gpu_boundary.py with gcc -O2 -ffp-contract=off -fopenmp. */
#include <quadmath.h>
#include <stdint.h>

void host_ln_table(uint64_t n0, uint64_t count, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)count; i++) out[i] = (double)logq((__float128)(n0 + (uint64_t)i));
}
