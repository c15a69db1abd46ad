/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE. See grf_oracle.h.
 *
 * Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj/core).
 */
#include "grf_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fft_core.h"

#define GRO_MAX_D 16

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* gro_last_error(void) { return g_err; }

/* GridSpec validation — src/grid.cpp:10-30. */
int gro_validate_grid(int d, const int64_t* n, const double* l) {
  if (d < 1 || d > GRO_MAX_D) return fail(GRO_EINVAL, "GridSpec: dimension must be >= 1");
  int64_t p = 1;
  for (int i = 0; i < d; ++i) {
    if (n[i] < 2 || n[i] % 2 != 0)
      return fail(GRO_EINVAL, "GridSpec: point counts must be even and >= 2");
    if (l && (!(l[i] > 0.0) || !isfinite(l[i])))
      return fail(GRO_EINVAL, "GridSpec: edge lengths must be positive and finite");
    if (p > INT64_MAX / n[i]) return fail(GRO_EINVAL, "GridSpec: total point count overflows");
    p *= n[i];
  }
  return GRO_OK;
}

static int64_t point_count(int d, const int64_t* n) {
  int64_t p = 1;
  for (int i = 0; i < d; ++i) p *= n[i];
  return p;
}

/* count_draws — src/synth.cpp:211-218; spectrum_draw_count — src/hermitian.cpp:228-236. */
uint64_t gro_count_draws(int d, const int64_t* n, int alg) {
  const uint64_t p = (uint64_t)point_count(d, n);
  if (alg == GRO_TWO_FFT || alg == GRO_ONE_FFT_RECURSIVE) return p;
  uint64_t cells = (uint64_t)(n[d - 1] / 2 + 1);
  for (int i = 0; i + 1 < d; ++i) cells *= (uint64_t)n[i];
  return 2 * cells - ((uint64_t)1 << d);
}

/* ipow — src/spectral.cpp:16-24. */
static double ipow(double x, int e) {
  double r = 1.0;
  while (e > 0) {
    if (e & 1) r *= x;
    x *= x;
    e >>= 1;
  }
  return r;
}

/* Density families:
 *  0 poly   (m=r0, k=i0, l=i1, n=i2)          — src/spectral.cpp:42-55
 *  1 aniso  (m=r0, n=i0, k_a=i[1+a])          — src/spectral.cpp:65-78
 *  2 test1d                                   — src/spectral.cpp:88-93
 *  3 gaussian covariance (ell=r0): (ell/sqrt(2pi))^d exp(-ell^2|w|^2/2)
 *  4 matern (nu=r0, ell=r1): c (1+ell^2|w|^2)^-(nu+d/2),
 *           c = ell^d Gamma(nu+d/2) / (pi^{d/2} Gamma(nu))
 *  5 constant (c=r0)                          — tests/test_support.hpp:13-27
 * 3 and 4 are the SURVEY.md §A.5 additions; ref_harness.cpp defines the same
 * formulas as SpectralDensity subclasses for the reference build. */
double gro_density_eval(const gro_density* g, const double* w) {
  const int d = g->dim;
  double s2 = 0.0;
  switch (g->family) {
    case 0: {
      const double mkl = pow(g->r[0], (double)g->i[0] * (double)g->i[1]);
      double s = 0.0;
      for (int a = 0; a < d; ++a) s += ipow(w[a] * w[a], g->i[0]);
      return 1.0 / ipow(mkl + ipow(s, g->i[1]), g->i[2]);
    }
    case 1: {
      double s = g->r[0];
      for (int a = 0; a < d; ++a) s += ipow(w[a] * w[a], g->i[1 + a]);
      return 1.0 / ipow(s, g->i[0]);
    }
    case 2: {
      const double q = 100.0 + w[0] * w[0];
      const double q2 = q * q;
      return (32.0e6 / M_PI) / (q2 * q2);
    }
    case 3: {
      const double ell = g->r[0];
      for (int a = 0; a < d; ++a) s2 += w[a] * w[a];
      return pow(ell / sqrt(2.0 * M_PI), d) * exp(-0.5 * ell * ell * s2);
    }
    case 4: {
      const double nu = g->r[0], ell = g->r[1], alpha = nu + 0.5 * d;
      for (int a = 0; a < d; ++a) s2 += w[a] * w[a];
      const double c = pow(ell, d) * tgamma(alpha) / (pow(M_PI, 0.5 * d) * tgamma(nu));
      return c * pow(1.0 + ell * ell * s2, -alpha);
    }
    case 5: return g->r[0];
  }
  return NAN;
}

/* Row-major walk over a Cartesian product of per-axis value lists, last axis
 * fastest; skipped when any list is empty — src/hermitian.cpp:13-35. */
typedef struct {
  int64_t* vals[GRO_MAX_D];
  int64_t len[GRO_MAX_D];
} axis_lists;

typedef void (*cell_fn)(const int64_t* k, int self, void* ctx);

static void walk_product(int d, const axis_lists* L, int self, cell_fn fn, void* ctx) {
  for (int a = 0; a < d; ++a)
    if (L->len[a] == 0) return;
  int64_t pos[GRO_MAX_D] = {0}, k[GRO_MAX_D];
  for (int a = 0; a < d; ++a) k[a] = L->vals[a][0];
  for (;;) {
    fn(k, self, ctx);
    int a = d - 1;
    while (a >= 0) {
      if (++pos[a] < L->len[a]) {
        k[a] = L->vals[a][pos[a]];
        break;
      }
      pos[a] = 0;
      k[a] = L->vals[a][0];
      --a;
    }
    if (a < 0) return;
  }
}

/* Representative-set enumeration (paper Appendix): L0 = {0, M}^d row-major,
 * then blocks n = 1..d over lexicographic axis subsets; first chosen axis in
 * [1, M-1], further chosen axes in [1, M-1] u [M+1, N-1], unchosen in {0, M}
 * — src/hermitian.cpp:39-84. */
static void walk_conjugate_reps(int d, const int64_t* n, cell_fn fn, void* ctx) {
  axis_lists L;
  int64_t maxn = 2;
  for (int a = 0; a < d; ++a) maxn = n[a] > maxn ? n[a] : maxn;
  int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(d * maxn));
  for (int a = 0; a < d; ++a) {
    L.vals[a] = buf + a * maxn;
    L.vals[a][0] = 0;
    L.vals[a][1] = n[a] / 2;
    L.len[a] = 2;
  }
  walk_product(d, &L, 1, fn, ctx);

  int chosen[GRO_MAX_D];
  for (int m = 1; m <= d; ++m) {
    for (int i = 0; i < m; ++i) chosen[i] = i;
    for (;;) {
      for (int a = 0, c = 0; a < d; ++a) {
        const int64_t half = n[a] / 2;
        L.len[a] = 0;
        if (c < m && chosen[c] == a) {
          for (int64_t x = 1; x < half; ++x) L.vals[a][L.len[a]++] = x;
          if (c > 0)
            for (int64_t x = half + 1; x < n[a]; ++x) L.vals[a][L.len[a]++] = x;
          ++c;
        } else {
          L.vals[a][L.len[a]++] = 0;
          L.vals[a][L.len[a]++] = half;
        }
      }
      walk_product(d, &L, 0, fn, ctx);
      int i = m - 1;
      while (i >= 0 && chosen[i] == d - m + i) --i;
      if (i < 0) break;
      ++chosen[i];
      for (int j = i + 1; j < m; ++j) chosen[j] = chosen[j - 1] + 1;
    }
  }
  free(buf);
}

typedef struct {
  int d;
  const int64_t* n;
  int64_t* lin;
  uint8_t* self;
  int64_t cap, count;
} reps_ctx;

static int64_t linear_of(int d, const int64_t* n, const int64_t* k) {
  int64_t idx = 0;
  for (int a = 0; a < d; ++a) idx = idx * n[a] + k[a];
  return idx;
}

static void reps_cb(const int64_t* k, int self, void* vctx) {
  reps_ctx* c = (reps_ctx*)vctx;
  if (c->count < c->cap) {
    c->lin[c->count] = linear_of(c->d, c->n, k);
    c->self[c->count] = (uint8_t)self;
  }
  c->count++;
}

/* for_each_conjugate_rep — include/grf/hermitian.hpp:36-42. */
int64_t gro_conjugate_reps(int d, const int64_t* n, int64_t* lin, uint8_t* self, int64_t cap) {
  if (gro_validate_grid(d, n, NULL) != GRO_OK) return -1;
  reps_ctx c = {d, n, lin, self, cap, 0};
  walk_conjugate_reps(d, n, reps_cb, &c);
  return c.count;
}

/* ---- spectrum assembly — src/hermitian.cpp:105-203 ---- */
typedef struct {
  int d;
  const int64_t* n;
  const gro_density* g;
  double* omega[GRO_MAX_D]; /* FrequencyTables, hermitian.cpp:105-124 */
  int64_t stride[GRO_MAX_D];
  const double* draws;
  uint64_t ndraws, pos;
  double* out;
  int err;
} spec_ctx;

static double next_draw(spec_ctx* c) {
  if (c->pos >= c->ndraws) {
    c->err = fail(GRO_ERUNTIME, "FixedStream: stream exhausted");
    return 0.0;
  }
  return c->draws[c->pos++];
}

static double gamma_sqrt(spec_ctx* c, const int64_t* k) {
  double w[GRO_MAX_D];
  for (int a = 0; a < c->d; ++a) w[a] = c->omega[a][k[a]];
  const double g = gro_density_eval(c->g, w);
  if (!(g >= 0.0) || isnan(g))
    c->err = fail(GRO_ERUNTIME, "synthesize_spectrum: density evaluated to NaN or negative");
  return sqrt(g);
}

static void spec_cb(const int64_t* k, int self, void* vctx) {
  spec_ctx* c = (spec_ctx*)vctx;
  if (c->err) return;
  const double inv_sqrt2 = 1.0 / sqrt(2.0);
  int64_t lin = 0;
  for (int a = 0; a < c->d; ++a) lin += c->stride[a] * k[a];
  const double gs = gamma_sqrt(c, k);
  if (c->err) return;
  if (self) { /* set_self, hermitian.cpp:167-171 */
    const double z = next_draw(c);
    c->out[2 * lin] = gs * z;
    c->out[2 * lin + 1] = 0.0;
    return;
  }
  /* set_pair, hermitian.cpp:157-166 */
  const double re = gs * inv_sqrt2 * next_draw(c);
  const double im = gs * inv_sqrt2 * next_draw(c);
  int64_t neg = 0;
  for (int a = 0; a < c->d; ++a) neg += c->stride[a] * (k[a] == 0 ? 0 : c->n[a] - k[a]);
  c->out[2 * lin] = re;
  c->out[2 * lin + 1] = im;
  c->out[2 * neg] = re;
  c->out[2 * neg + 1] = -im;
}

static void overwrite_cb(const int64_t* k, int self_unused, void* vctx) {
  (void)self_unused;
  spec_ctx* c = (spec_ctx*)vctx;
  int self = 1; /* hermitian.cpp:182-201 */
  for (int a = 0; a < c->d; ++a)
    if (k[a] != 0 && k[a] != c->n[a] / 2) {
      self = 0;
      break;
    }
  spec_cb(k, self, vctx);
}

int gro_spectrum(int d, const int64_t* n, const double* l, const gro_density* g, int mode,
                 const double* draws, uint64_t ndraws, double* out) {
  int rc = gro_validate_grid(d, n, l);
  if (rc) return rc;
  if (g->dim != d) return fail(GRO_EINVAL, "synthesize_spectrum: density dimension mismatch");
  spec_ctx c;
  memset(&c, 0, sizeof c);
  c.d = d;
  c.n = n;
  c.g = g;
  c.draws = draws;
  c.ndraws = ndraws;
  c.out = out;
  for (int a = 0; a < d; ++a) {
    c.omega[a] = (double*)malloc(sizeof(double) * (size_t)n[a]);
    for (int64_t kk = 0; kk < n[a]; ++kk) {
      const int64_t w = (kk <= n[a] / 2) ? kk : kk - n[a];
      c.omega[a][kk] = 2.0 * M_PI * (double)w / l[a];
    }
  }
  c.stride[d - 1] = 1;
  for (int a = d - 2; a >= 0; --a) c.stride[a] = c.stride[a + 1] * n[a + 1];

  if (mode == GRO_EXACT_SET) {
    walk_conjugate_reps(d, n, spec_cb, &c);
  } else {
    axis_lists L;
    int64_t maxn = 1;
    for (int a = 0; a < d; ++a) maxn = n[a] > maxn ? n[a] : maxn;
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(d * maxn));
    for (int a = 0; a < d; ++a) {
      L.vals[a] = buf + a * maxn;
      L.len[a] = (a == d - 1) ? n[a] / 2 + 1 : n[a];
      for (int64_t x = 0; x < L.len[a]; ++x) L.vals[a][x] = x;
    }
    walk_product(d, &L, 0, overwrite_cb, &c);
    free(buf);
  }
  for (int a = 0; a < d; ++a) free(c.omega[a]);
  return c.err;
}

/* DftBackend conventions — include/grf/dft.hpp:11-14, src/dft.cpp:95-108. */
void gro_dft(int d, const int64_t* n, const double* in, double* out, int sign) {
  fc_plan* p = fc_plan_create(d, n, sign > 0 ? +1 : -1);
  fc_execute(p, in, out);
  fc_plan_destroy(p);
  if (sign < 0) {
    const int64_t P = point_count(d, n);
    const double s = 1.0 / (double)P;
    for (int64_t i = 0; i < 2 * P; ++i) out[i] *= s;
  }
}

static double two_pi_pow(int d) { /* src/synth.cpp:13-17 */
  double v = 1.0;
  for (int i = 0; i < d; ++i) v *= 2.0 * M_PI;
  return v;
}

static double domain_volume(int d, const double* l) { /* src/grid.cpp:38-42 */
  double v = 1.0;
  for (int i = 0; i < d; ++i) v *= l[i];
  return v;
}

/* extract_real — src/synth.cpp:20-33. */
static int extract_real(const double* buf, int64_t P, double scale, double* field, double* residue) {
  double max_re = 0.0, max_im = 0.0;
  for (int64_t i = 0; i < P; ++i) {
    const double re = fabs(buf[2 * i]), im = fabs(buf[2 * i + 1]);
    if (re > max_re) max_re = re;
    if (im > max_im) max_im = im;
    field[i] = buf[2 * i] * scale;
  }
  const double r = (max_re > 0.0) ? max_im / max_re : max_im;
  if (residue) *residue = r;
  if (r > 1e-10) return fail(GRO_ERUNTIME, "synthesize: imaginary residue exceeds 1e-10");
  return GRO_OK;
}

/* synthesize(grid, density, stream, algorithm) — src/synth.cpp:68-127, with
 * the stream a FixedStream over `draws` (include/grf/random.hpp:50-62). */
int gro_synthesize(int d, const int64_t* n, const double* l, const gro_density* g, int alg,
                   const double* draws, uint64_t ndraws, double* field, double* residue) {
  int rc = gro_validate_grid(d, n, l);
  if (rc) return rc;
  if (g->dim != d) return fail(GRO_EINVAL, "synthesize: density dimension mismatch");
  const int64_t P = point_count(d, n);
  double* a = (double*)malloc(sizeof(double) * 2 * (size_t)P);
  double* b = (double*)malloc(sizeof(double) * 2 * (size_t)P);
  if (alg == GRO_TWO_FFT) { /* synth.cpp:81-116 */
    if ((uint64_t)P > ndraws) {
      free(a);
      free(b);
      return fail(GRO_ERUNTIME, "FixedStream: stream exhausted");
    }
    for (int64_t i = 0; i < P; ++i) {
      a[2 * i] = draws[i];
      a[2 * i + 1] = 0.0;
    }
    gro_dft(d, n, a, b, +1);
    const double scale = sqrt(two_pi_pow(d) * (double)P / domain_volume(d, l));
    int64_t k[GRO_MAX_D] = {0};
    double w[GRO_MAX_D];
    for (int64_t i = 0; i < P; ++i) {
      for (int ax = 0; ax < d; ++ax) {
        const int64_t kk = k[ax] <= n[ax] / 2 ? k[ax] : k[ax] - n[ax];
        w[ax] = 2.0 * M_PI * (double)kk / l[ax];
      }
      const double gv = gro_density_eval(g, w);
      if (!(gv >= 0.0) || isnan(gv)) {
        free(a);
        free(b);
        return fail(GRO_ERUNTIME, "synthesize: density evaluated to NaN or negative");
      }
      const double m = sqrt(gv) * scale;
      b[2 * i] *= m;
      b[2 * i + 1] *= m;
      for (int ax = d - 1; ax >= 0; --ax) {
        if (++k[ax] < n[ax]) break;
        k[ax] = 0;
      }
    }
    gro_dft(d, n, b, a, -1);
    rc = extract_real(a, P, 1.0, field, residue);
  } else { /* synth.cpp:118-126 */
    rc = gro_spectrum(d, n, l, g, alg == GRO_ONE_FFT_OVERWRITE ? GRO_OVERWRITE : GRO_EXACT_SET,
                      draws, ndraws, a);
    if (rc == GRO_OK) {
      gro_dft(d, n, a, b, -1);
      const double scale = sqrt(two_pi_pow(d) / domain_volume(d, l)) * (double)P;
      rc = extract_real(b, P, scale, field, residue);
    }
  }
  free(a);
  free(b);
  return rc;
}

/* exact_discrete_covariance_all — src/synth.cpp:188-209. */
int gro_exact_cov_all(int d, const int64_t* n, const double* l, const gro_density* g, double* out) {
  int rc = gro_validate_grid(d, n, l);
  if (rc) return rc;
  const int64_t P = point_count(d, n);
  double* a = (double*)malloc(sizeof(double) * 2 * (size_t)P);
  double* b = (double*)malloc(sizeof(double) * 2 * (size_t)P);
  int64_t k[GRO_MAX_D] = {0};
  double w[GRO_MAX_D];
  for (int64_t i = 0; i < P; ++i) {
    for (int ax = 0; ax < d; ++ax) {
      const int64_t kk = k[ax] <= n[ax] / 2 ? k[ax] : k[ax] - n[ax];
      w[ax] = 2.0 * M_PI * (double)kk / l[ax];
    }
    a[2 * i] = gro_density_eval(g, w);
    a[2 * i + 1] = 0.0;
    for (int ax = d - 1; ax >= 0; --ax) {
      if (++k[ax] < n[ax]) break;
      k[ax] = 0;
    }
  }
  gro_dft(d, n, a, b, -1);
  const double scale = two_pi_pow(d) / domain_volume(d, l) * (double)P;
  for (int64_t i = 0; i < P; ++i) out[i] = b[2 * i] * scale;
  free(a);
  free(b);
  return GRO_OK;
}
