/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE. Implements standin/fftw3.h on top of
 * fft_core.c so that the reference's dft.cpp links (SURVEY.md §8c recipe).
 */
#include "standin/fftw3.h"

#include <stdint.h>
#include <stdlib.h>

#include "fft_core.h"

struct fftw_plan_s {
  fc_plan* core;
};

fftw_complex* fftw_alloc_complex(size_t n) {
  void* p = NULL;
  if (posix_memalign(&p, 64, (n ? n : 1) * sizeof(fftw_complex)) != 0) return NULL;
  return (fftw_complex*)p;
}

void fftw_free(void* p) { free(p); }

/* FFTW reports the alignment class of a pointer modulo its SIMD width; the
 * reference only compares these values for equality (dft.cpp:76-78). */
int fftw_alignment_of(double* p) { return (int)((uintptr_t)p % 64); }

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags) {
  (void)in;
  (void)out;
  (void)flags;
  int64_t dims[16];
  if (rank < 1 || rank > 16) return NULL;
  for (int a = 0; a < rank; ++a) dims[a] = n[a];
  fc_plan* core = fc_plan_create(rank, dims, sign);
  if (!core) return NULL;
  fftw_plan p = (fftw_plan)malloc(sizeof(struct fftw_plan_s));
  p->core = core;
  return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  fc_execute(p->core, (const double*)in, (double*)out);
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  fc_plan_destroy(p->core);
  free(p);
}
