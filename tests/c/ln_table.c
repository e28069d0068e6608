/* Test helper (not product, not oracle): the host C library's natural log of consecutive
 * integers, the function oracle/riki_oracle.c applies to the label-class counts.
 * Compiled by tests/test_gpu_parity.py with gcc -O2 -ffp-contract=off -fopenmp. */
#include <math.h>
#include <stdint.h>

void host_ln_table(uint64_t n0, uint64_t count, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)count; i++) out[i] = log((double)(n0 + (uint64_t)i));
}
