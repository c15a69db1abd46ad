/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Minimal stand-in for the FFTW3 C API, exposing exactly the symbols the
 * reference's /root/reference/proj/core/src/dft.cpp uses (dft.cpp:3,50-85,91,
 * 98-99,105). FFTW itself is absent from this image, so the
 * reference's own dft.cpp is compiled unmodified against this header and the
 * transforms are executed by oracle/fft_core.c. Declared semantics follow the
 * public FFTW3 manual: fftw_plan_dft computes the unnormalised rank-d DFT
 * with exponent sign `sign` (FFTW_FORWARD = -1, FFTW_BACKWARD = +1).
 */
#ifndef GRF_ORACLE_FFTW3_STANDIN_H
#define GRF_ORACLE_FFTW3_STANDIN_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);
int fftw_alignment_of(double* p);
fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
