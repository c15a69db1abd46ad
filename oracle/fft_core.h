/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * fp64 CPU complex DFT used by (a) the FFTW3 API stand-in that lets the
 * reference's own proj/core/src/dft.cpp compile unmodified into oracle/_ref,
 * and (b) the plain-C restatement oracle/grf_oracle.c. Only tests/, bench.py's
 * cpu_baseline leg and __graft_entry__.smoke() may execute it, as a checker.
 *
 * Conventions follow FFTW's unnormalised transform:
 *   out[K] = sum_J in[J] * exp(sign * 2 pi i * sum_a k_a j_a / N_a)
 * with sign = -1 (FFTW_FORWARD) or +1 (FFTW_BACKWARD). The reference maps its
 * own "forward" (exp(+)) onto FFTW_BACKWARD and "inverse" onto FFTW_FORWARD
 * then x 1/P (/root/reference/proj/core/src/dft.cpp:95-108).
 */
#ifndef GRF_ORACLE_FFT_CORE_H
#define GRF_ORACLE_FFT_CORE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fc_plan_s fc_plan;

/* rank-d plan over row-major dims (last index fastest); any N >= 1. */
fc_plan* fc_plan_create(int rank, const int64_t* dims, int sign);
void fc_plan_destroy(fc_plan* p);
/* Out-of-place or in-place; interleaved (re, im) doubles. Thread-safe for
 * concurrent calls on the same plan (all scratch is per call). */
void fc_execute(const fc_plan* p, const double* in, double* out);

#ifdef __cplusplus
}
#endif

#endif
