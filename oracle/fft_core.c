/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE. See fft_core.h.
 *
 * Row-column rank-d complex DFT in fp64: each axis is a batch of strided 1D
 * transforms, each 1D transform a mixed-radix Stockham autosort pass sequence
 * (radix 4, 2, 3, 5, then any remaining prime by a direct O(p^2) butterfly).
 * Twiddles come from one exact-angle table per axis length, so the result is
 * accurate to a few ulps times log2(N) — well inside the 1e-11 agreement the
 * reference demands between its FFTW and naive backends
 * (/root/reference/proj/tests/test_synth.cpp:21-48).
 */
#include "fft_core.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FC_MAX_RANK 16
#define FC_MAX_FACTORS 64
#define FC_BLOCK 8 /* adjacent lines gathered together on strided axes */

typedef struct {
  int64_t n;
  int nf;
  int64_t fac[FC_MAX_FACTORS];
  double* tw; /* 2n doubles: exp(sign * 2 pi i m / n), m in [0, n) */
} fc_line;

struct fc_plan_s {
  int rank;
  int sign;
  int64_t dims[FC_MAX_RANK];
  int64_t total;
  fc_line line[FC_MAX_RANK];
};

static void line_init(fc_line* L, int64_t n, int sign) {
  L->n = n;
  L->nf = 0;
  int64_t m = n;
  while (m % 4 == 0) { L->fac[L->nf++] = 4; m /= 4; }
  while (m % 2 == 0) { L->fac[L->nf++] = 2; m /= 2; }
  for (int64_t p = 3; m > 1; p += 2) {
    while (m % p == 0) { L->fac[L->nf++] = p; m /= p; }
    if (p * p > m && m > 1) { L->fac[L->nf++] = m; m = 1; }
  }
  L->tw = (double*)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
  for (int64_t t = 0; t < n; ++t) {
    /* Angle reduced to [0, pi/4]-ish symmetric form is unnecessary at fp64:
     * 2 pi t / n is formed once, with one rounding. */
    const double a = 2.0 * M_PI * (double)t / (double)n;
    L->tw[2 * t] = cos(a);
    L->tw[2 * t + 1] = (double)sign * sin(a);
  }
}

/* One Stockham pass: radix R, Ns = product of the radices already applied. */
static void stockham_pass(const fc_line* L, int64_t R, int64_t Ns, int sign, const double* src,
                          double* dst, double* v) {
  const int64_t n = L->n, m = n / R, tstep = n / (Ns * R);
  const double* tw = L->tw;
  for (int64_t j = 0; j < m; ++j) {
    const int64_t k = j % Ns;
    for (int64_t i = 0; i < R; ++i) {
      double re = src[2 * (j + i * m)], im = src[2 * (j + i * m) + 1];
      if (i > 0 && k > 0) {
        const int64_t t = (i * k * tstep) % n;
        const double wr = tw[2 * t], wi = tw[2 * t + 1];
        const double r2 = re * wr - im * wi;
        im = re * wi + im * wr;
        re = r2;
      }
      v[2 * i] = re;
      v[2 * i + 1] = im;
    }
    const int64_t out0 = (j / Ns) * Ns * R + k;
    if (R == 2) {
      const double ar = v[0], ai = v[1], br = v[2], bi = v[3];
      dst[2 * out0] = ar + br;
      dst[2 * out0 + 1] = ai + bi;
      dst[2 * (out0 + Ns)] = ar - br;
      dst[2 * (out0 + Ns) + 1] = ai - bi;
    } else if (R == 4) {
      const double t0r = v[0] + v[4], t0i = v[1] + v[5];
      const double t1r = v[0] - v[4], t1i = v[1] - v[5];
      const double t2r = v[2] + v[6], t2i = v[3] + v[7];
      const double dr = v[2] - v[6], di = v[3] - v[7];
      /* (v1 - v3) * exp(sign * i pi / 2) = (v1 - v3) * (sign * i) */
      const double t3r = -(double)sign * di, t3i = (double)sign * dr;
      dst[2 * out0] = t0r + t2r;
      dst[2 * out0 + 1] = t0i + t2i;
      dst[2 * (out0 + Ns)] = t1r + t3r;
      dst[2 * (out0 + Ns) + 1] = t1i + t3i;
      dst[2 * (out0 + 2 * Ns)] = t0r - t2r;
      dst[2 * (out0 + 2 * Ns) + 1] = t0i - t2i;
      dst[2 * (out0 + 3 * Ns)] = t1r - t3r;
      dst[2 * (out0 + 3 * Ns) + 1] = t1i - t3i;
    } else {
      const int64_t step = n / R; /* exp(sign 2 pi i q i / R) = tw[(q i step) mod n] */
      for (int64_t q = 0; q < R; ++q) {
        double ar = 0.0, ai = 0.0;
        for (int64_t i = 0; i < R; ++i) {
          const int64_t t = ((q * i) % R) * step;
          const double wr = tw[2 * t], wi = tw[2 * t + 1];
          ar += v[2 * i] * wr - v[2 * i + 1] * wi;
          ai += v[2 * i] * wi + v[2 * i + 1] * wr;
        }
        dst[2 * (out0 + q * Ns)] = ar;
        dst[2 * (out0 + q * Ns) + 1] = ai;
      }
    }
  }
}

/* In-place 1D transform of x (n complex) using scratch y (n complex). */
static void line_exec(const fc_line* L, int sign, double* x, double* y, double* v) {
  double* src = x;
  double* dst = y;
  int64_t Ns = 1;
  for (int f = 0; f < L->nf; ++f) {
    stockham_pass(L, L->fac[f], Ns, sign, src, dst, v);
    Ns *= L->fac[f];
    double* t = src;
    src = dst;
    dst = t;
  }
  if (src != x) memcpy(x, src, sizeof(double) * 2 * (size_t)L->n);
}

fc_plan* fc_plan_create(int rank, const int64_t* dims, int sign) {
  if (rank < 1 || rank > FC_MAX_RANK) return NULL;
  fc_plan* p = (fc_plan*)calloc(1, sizeof(fc_plan));
  p->rank = rank;
  p->sign = sign >= 0 ? 1 : -1;
  p->total = 1;
  for (int a = 0; a < rank; ++a) {
    if (dims[a] < 1) { free(p); return NULL; }
    p->dims[a] = dims[a];
    p->total *= dims[a];
    line_init(&p->line[a], dims[a], p->sign);
  }
  return p;
}

void fc_plan_destroy(fc_plan* p) {
  if (!p) return;
  for (int a = 0; a < p->rank; ++a) free(p->line[a].tw);
  free(p);
}

void fc_execute(const fc_plan* p, const double* in, double* out) {
  if (in != out) memmove(out, in, sizeof(double) * 2 * (size_t)p->total);
  int64_t maxn = 1, maxr = 1;
  for (int a = 0; a < p->rank; ++a) {
    if (p->dims[a] > maxn) maxn = p->dims[a];
    for (int f = 0; f < p->line[a].nf; ++f)
      if (p->line[a].fac[f] > maxr) maxr = p->line[a].fac[f];
  }
  double* buf = (double*)malloc(sizeof(double) * 2 * (size_t)(maxn * (FC_BLOCK + 1) + maxr));
  double* scratch = buf + 2 * maxn * FC_BLOCK;
  double* v = scratch + 2 * maxn;
  for (int a = 0; a < p->rank; ++a) {
    const int64_t n = p->dims[a];
    if (n == 1) continue;
    int64_t inner = 1, outer = 1;
    for (int b = a + 1; b < p->rank; ++b) inner *= p->dims[b];
    for (int b = 0; b < a; ++b) outer *= p->dims[b];
    const fc_line* L = &p->line[a];
    for (int64_t o = 0; o < outer; ++o) {
      double* base = out + 2 * o * n * inner;
      if (inner == 1) {
        line_exec(L, p->sign, base, scratch, v);
        continue;
      }
      for (int64_t s0 = 0; s0 < inner; s0 += FC_BLOCK) {
        const int64_t bl = (inner - s0) < FC_BLOCK ? (inner - s0) : FC_BLOCK;
        for (int64_t t = 0; t < n; ++t)
          for (int64_t b = 0; b < bl; ++b) {
            buf[2 * (b * n + t)] = base[2 * (t * inner + s0 + b)];
            buf[2 * (b * n + t) + 1] = base[2 * (t * inner + s0 + b) + 1];
          }
        for (int64_t b = 0; b < bl; ++b) line_exec(L, p->sign, buf + 2 * b * n, scratch, v);
        for (int64_t t = 0; t < n; ++t)
          for (int64_t b = 0; b < bl; ++b) {
            base[2 * (t * inner + s0 + b)] = buf[2 * (b * n + t)];
            base[2 * (t * inner + s0 + b) + 1] = buf[2 * (b * n + t) + 1];
          }
      }
    }
  }
  free(buf);
}
