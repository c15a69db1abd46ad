// grfc C-ABI: plans, dispatch, the host<->device boundary and error mapping.
// See include/grfc.h for the contract and the reference interfaces replaced.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/grfc.h"
#include "fast2d.h"
#include "fast3d.h"
#include "grfc_internal.cuh"
#include "host_lattice.h"
#include "kernels.h"

namespace grfc {

static thread_local std::string t_err;
static thread_local uint64_t t_launches = 0;
void count_launch(uint64_t n) { t_launches += n; }

// ---- per-kernel timing (benchmarks)
struct TimedLaunch {
  const char* name;
  cudaEvent_t start, stop;
};
static thread_local bool t_timing = false;
static thread_local std::vector<TimedLaunch> t_timed;
struct TimingRow {
  std::string name;
  double ms = 0;
  uint64_t launches = 0;
};
static thread_local std::vector<TimingRow> t_rows;

LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s) {
  if (t_timing) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    start = (void*)e;
  }
}

LaunchScope::~LaunchScope() {
  count_launch();
  if (start) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    t_timed.push_back({name, (cudaEvent_t)start, e});
  }
}

static grfc_status fail(grfc_status s, const std::string& msg) {
  t_err = msg;
  return s;
}

grfc_status set_error(grfc_status s, const std::string& msg) { return fail(s, msg); }

#define GRFC_CUDA(expr)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return fail(GRFC_ECUDA, std::string("CUDA: ") + #expr + ": " + \
                                                       cudaGetErrorString(e_));          \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

Factors factorize(int64_t n) {
  Factors F{};
  int64_t m = n;
  while (m % 8 == 0 && F.nf < 40) F.r[F.nf++] = 8, m /= 8;
  while (m % 4 == 0) F.r[F.nf++] = 4, m /= 4;
  while (m % 2 == 0) F.r[F.nf++] = 2, m /= 2;
  for (int64_t p = 3; m > 1; p += 2) {
    while (m % p == 0) F.r[F.nf++] = (int)p, m /= p;
    if (p * p > m && m > 1) F.r[F.nf++] = (int)m, m = 1;
  }
  return F;
}

// exp(+2 pi i m / n), m < n, from long-double angles (one rounding to T).
template <typename T>
static std::vector<C_t<T>> twiddle_table(int64_t n) {
  std::vector<C_t<T>> t((size_t)n);
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int64_t m = 0; m < n; ++m) {
    const long double a = two_pi * (long double)m / (long double)n;
    t[(size_t)m].x = (T)cosl(a);
    t[(size_t)m].y = (T)sinl(a);
  }
  return t;
}

static double two_pi_pow(int d) {  // src/synth.cpp:13-17
  double v = 1.0;
  for (int i = 0; i < d; ++i) v *= 2.0 * M_PI;
  return v;
}

}  // namespace grfc

using namespace grfc;

struct grfc_plan_s {
  int d = 0;
  int64_t n[GRFC_MAX_DIM] = {};
  double l[GRFC_MAX_DIM] = {};
  int dtype = GRFC_F32, alg = 1, device = 0;
  grfc_density dens{};
  GridDesc g{};
  DensityDesc D{};
  uint64_t cells = 0, points = 0;
  size_t csize = 8;  // bytes per complex element
  void* d_tw = nullptr;
  size_t tw_off[GRFC_MAX_DIM] = {};  // element offsets per axis
  Factors F[GRFC_MAX_DIM]{};
  Factors FM{};  // last axis: factors of n_d / 2
  double* d_table = nullptr;
  bool table_set = false;
  double s_one = 1.0;  // Alg 2/3: sqrt((2 pi)^d / |A|)         (synth.cpp:123)
  double s_two = 1.0;  // Alg 1:   sqrt((2 pi)^d P / |A|) / P   (synth.cpp:89-90 + dft.cpp:106)
  bool fast = false;
  Fast2D fast2d{};
  bool fast3 = false;
  Fast3D fast3d{};
  std::string path = "generic";

  const void* tw(int a) const { return (const char*)d_tw + tw_off[a] * csize; }
};

namespace grfc {

static grfc_status validate_density(const grfc_density* dn, int d) {
  if (!dn) return fail(GRFC_EINVAL, "grfc: density is null");
  if (dn->dim != d) return fail(GRFC_EINVAL, "synthesize: density dimension mismatch");
  switch (dn->family) {
    case GRFC_DENSITY_POLY:
      if (!(dn->r[0] > 0.0) || !std::isfinite(dn->r[0]))
        return fail(GRFC_EINVAL, "PolyDecayDensity: m must be positive");
      if (dn->i[0] < 1 || dn->i[1] < 1 || dn->i[2] < 1)
        return fail(GRFC_EINVAL, "PolyDecayDensity: k, l, n must be >= 1");
      return GRFC_OK;
    case GRFC_DENSITY_ANISO:
      if (!(dn->r[0] > 0.0) || !std::isfinite(dn->r[0]))
        return fail(GRFC_EINVAL, "AnisoPolyDensity: m must be positive");
      if (dn->i[0] < 1) return fail(GRFC_EINVAL, "AnisoPolyDensity: n must be >= 1");
      for (int a = 0; a < d; ++a)
        if (dn->i[1 + a] < 1) return fail(GRFC_EINVAL, "AnisoPolyDensity: exponents must be >= 1");
      return GRFC_OK;
    case GRFC_DENSITY_TEST1D:
      if (d != 1) return fail(GRFC_EINVAL, "density spec: test1d is one-dimensional");
      return GRFC_OK;
    case GRFC_DENSITY_GAUSSIAN_COV:
      if (!(dn->r[0] > 0.0) || !std::isfinite(dn->r[0])) return fail(GRFC_EINVAL, "gaussian-cov: ell must be > 0");
      return GRFC_OK;
    case GRFC_DENSITY_MATERN:
      if (!(dn->r[0] > 0.0) || !std::isfinite(dn->r[0])) return fail(GRFC_EINVAL, "matern: nu must be > 0");
      if (!(dn->r[1] > 0.0) || !std::isfinite(dn->r[1])) return fail(GRFC_EINVAL, "matern: ell must be > 0");
      return GRFC_OK;
    case GRFC_DENSITY_CONSTANT:
      if (!(dn->r[0] >= 0.0) || std::isnan(dn->r[0]))
        return fail(GRFC_ERUNTIME, "synthesize_spectrum: density evaluated to NaN or negative");
      return GRFC_OK;
    case GRFC_DENSITY_TABLE: return GRFC_OK;
  }
  return fail(GRFC_EINVAL, "grfc: unknown density family");
}

template <typename T>
static grfc_status run_fields(grfc_plan p, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                              int64_t stride, const double2* inj_half, const double* inj_points, cudaStream_t s) {
  const int d = p->d;
  const int nd = (int)p->n[d - 1];
  const int64_t rows_pf = (int64_t)(p->points / (uint64_t)nd);
  const int64_t rows = rows_pf * nf;
  if (p->fast && !inj_half && !inj_points && stride % 2 == 0) {
    GRFC_CUDA(launch_fast2d(p->fast2d, p->alg, seed, field0, nf, W, out, stride, s));
    return GRFC_OK;
  }
  auto axes = [&](int sign) -> grfc_status {
    for (int a = 0; a < d - 1; ++a) {
      int64_t inner = p->n[d - 1] / 2 + 1, outer = nf;
      for (int b = a + 1; b < d - 1; ++b) inner *= p->n[b];
      for (int b = 0; b < a; ++b) outer *= p->n[b];
      // longer than one CTA's shared memory, or a long prime factor: four-step /
      // Bluestein through global memory
      cudaError_t e = needs_long_line(p->n[a], sizeof(C_t<T>))
                          ? long_c2c<T>(W, p->n[a], inner, outer, sign, s)
                          : launch_line_c2c<T>(W, (int)p->n[a], inner, outer, sign, p->F[a], p->tw(a), s);
      if (e == cudaErrorInvalidValue) e = long_c2c<T>(W, p->n[a], inner, outer, sign, s);
      GRFC_CUDA(e);
    }
    return GRFC_OK;
  };
  grfc_status st;
  if (p->alg == GRFC_TWO_FFT) {
    const bool long_last = needs_long_line(nd / 2, sizeof(C_t<T>));
    cudaError_t e = long_last ? cudaErrorInvalidValue
                              : launch_r2c_last_noise<T>(W, nd, rows, rows_pf, seed, field0, inj_points, p->FM,
                                                         p->tw(d - 1), s);
    if (e == cudaErrorInvalidValue) e = long_r2c_last_noise<T>(W, nd, rows, rows_pf, seed, field0, inj_points, s);
    GRFC_CUDA(e);
    if ((st = axes(+1)) != GRFC_OK) return st;
    GRFC_CUDA(launch_scale_half<T>(p->g, p->D, p->s_two, W, nf, s));
    if ((st = axes(-1)) != GRFC_OK) return st;
    e = long_last ? cudaErrorInvalidValue
                  : launch_c2r_last<T>(W, out, nd, rows, rows_pf, stride, 1, p->FM, p->tw(d - 1), s);
    if (e == cudaErrorInvalidValue) e = long_c2r_last<T>(W, out, nd, rows, rows_pf, stride, 1, s);
    GRFC_CUDA(e);
  } else {
    GRFC_CUDA(launch_gen_half<T>(p->g, p->D, p->alg, p->s_one, seed, field0, inj_half, W, nf, s));
    if ((st = axes(+1)) != GRFC_OK) return st;
    cudaError_t e = needs_long_line(nd / 2, sizeof(C_t<T>))
                        ? cudaErrorInvalidValue
                        : launch_c2r_last<T>(W, out, nd, rows, rows_pf, stride, 0, p->FM, p->tw(d - 1), s);
    if (e == cudaErrorInvalidValue) e = long_c2r_last<T>(W, out, nd, rows, rows_pf, stride, 0, s);
    GRFC_CUDA(e);
  }
  return GRFC_OK;
}

static grfc_status run_fields_any(grfc_plan p, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                                  int64_t stride, const double2* inj_half, const double* inj_points,
                                  cudaStream_t s) {
  if (p->dtype == GRFC_F64) return run_fields<double>(p, seed, field0, nf, W, out, stride, inj_half, inj_points, s);
  return run_fields<float>(p, seed, field0, nf, W, out, stride, inj_half, inj_points, s);
}

// Fields per workspace chunk: keep the half-spectrum intermediate L2-resident.
static int64_t chunk_fields(grfc_plan p, uint64_t nfields) {
  const double wbytes = (double)p->cells * (double)p->csize;
  int64_t c = (int64_t)std::floor((p->fast ? p->fast2d.l2_budget : 48.0 * 1024 * 1024) / wbytes);
  c = std::max<int64_t>(1, std::min<int64_t>(c, (int64_t)nfields));
  return c;
}

static size_t dsize(grfc_plan p) { return p->dtype == GRFC_F64 ? 8 : 4; }

}  // namespace grfc

extern "C" {

const char* grfc_last_error(void) { return t_err.c_str(); }
uint64_t grfc_last_launch_count(void) { return t_launches; }

void grfc_kernel_timing_enable(int on) {
  for (auto& t : t_timed) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  t_timed.clear();
  t_rows.clear();
  t_timing = on != 0;
}

grfc_status grfc_kernel_timing_read(int index, const char** name, double* total_ms, uint64_t* launches) {
  for (auto& t : t_timed) {
    cudaEventSynchronize(t.stop);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.start, t.stop);
    auto it = std::find_if(t_rows.begin(), t_rows.end(), [&](const TimingRow& r) { return r.name == t.name; });
    if (it == t_rows.end()) {
      t_rows.push_back({t.name, 0.0, 0});
      it = t_rows.end() - 1;
    }
    it->ms += ms;
    it->launches += 1;
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  t_timed.clear();
  if (index < 0 || index >= (int)t_rows.size()) return fail(GRFC_EINVAL, "grfc: no such timing row");
  if (name) *name = t_rows[(size_t)index].name.c_str();
  if (total_ms) *total_ms = t_rows[(size_t)index].ms;
  if (launches) *launches = t_rows[(size_t)index].launches;
  return GRFC_OK;
}

grfc_status grfc_count_draws(int dim, const int64_t* counts, int algorithm, uint64_t* out) {
  std::string err;
  if (!counts || !out) return fail(GRFC_EINVAL, "grfc: null argument");
  if (!validate_grid(dim, counts, nullptr, err)) return fail(GRFC_EINVAL, err);
  if (algorithm < 0 || algorithm > 2) return fail(GRFC_EINVAL, "count_draws: unknown algorithm");
  *out = grfc::count_draws(dim, counts, algorithm);
  return GRFC_OK;
}

grfc_status grfc_half_lattice_cells(int dim, const int64_t* counts, uint64_t* out) {
  std::string err;
  if (!counts || !out) return fail(GRFC_EINVAL, "grfc: null argument");
  if (!validate_grid(dim, counts, nullptr, err)) return fail(GRFC_EINVAL, err);
  *out = half_cells(dim, counts);
  return GRFC_OK;
}

grfc_status grfc_conjugate_reps(int dim, const int64_t* counts, int64_t* lin, uint8_t* self_flag, uint64_t cap,
                                uint64_t* count) {
  std::string err;
  if (!counts || !count || (cap && (!lin || !self_flag))) return fail(GRFC_EINVAL, "grfc: null argument");
  if (!validate_grid(dim, counts, nullptr, err)) return fail(GRFC_EINVAL, err);
  uint64_t i = 0;
  for_each_rep(dim, counts, [&](const int64_t* k, bool self) {
    if (i < cap) {
      int64_t l = 0;
      for (int a = 0; a < dim; ++a) l = l * counts[a] + k[a];
      lin[i] = l;
      self_flag[i] = self ? 1 : 0;
    }
    ++i;
  });
  *count = i;
  return GRFC_OK;
}

grfc_status grfc_half_noise_from_draws(int dim, const int64_t* counts, int algorithm, const double* draws,
                                       uint64_t ndraws, double* w_half) {
  std::string err;
  if (!counts || !w_half || (!draws && ndraws)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (!validate_grid(dim, counts, nullptr, err)) return fail(GRFC_EINVAL, err);
  if (algorithm != GRFC_ONE_FFT_OVERWRITE && algorithm != GRFC_ONE_FFT_RECURSIVE)
    return fail(GRFC_EINVAL, "grfc: half-lattice noise exists for the one-FFT algorithms only");
  std::vector<double> w;
  if (!arrange_half_noise(dim, counts, algorithm, draws, ndraws, w, err)) return fail(GRFC_ERUNTIME, err);
  std::memcpy(w_half, w.data(), w.size() * sizeof(double));
  return GRFC_OK;
}

grfc_status grfc_grid_check(int dim, const int64_t* counts, const double* lengths, int64_t* points) {
  if (dim > 0 && !counts) return fail(GRFC_EINVAL, "grfc: null argument");
  std::string err;
  if (!check_grid_spec(dim, counts, lengths, points, err)) return fail(GRFC_EINVAL, err);
  return GRFC_OK;
}

grfc_status grfc_plan_create(grfc_plan* out, int dim, const int64_t* counts, const double* lengths, int dtype,
                             int algorithm, const grfc_density* density, int device) {
  if (!out || !counts || !lengths) return fail(GRFC_EINVAL, "grfc: null argument");
  *out = nullptr;
  std::string err;
  if (!validate_grid(dim, counts, lengths, err)) return fail(GRFC_EINVAL, err);
  if (dtype != GRFC_F32 && dtype != GRFC_F64) return fail(GRFC_EINVAL, "grfc: dtype must be F32 or F64");
  if (algorithm < 0 || algorithm > 2) return fail(GRFC_EINVAL, "synthesize: unknown algorithm");
  grfc_status st = validate_density(density, dim);
  if (st != GRFC_OK) return st;
  int ndev = 0;
  GRFC_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(GRFC_EINVAL, "grfc: bad device ordinal");
  {
    // Stream-ordered scratch (ring, workspaces) comes from the device's default
    // pool; keep freed blocks mapped so repeated calls reuse them instead of
    // re-mapping tens of MB per call.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  DeviceGuard guard(device);

  std::unique_ptr<grfc_plan_s> p(new grfc_plan_s());
  p->d = dim;
  p->dtype = dtype;
  p->alg = algorithm;
  p->device = device;
  p->dens = *density;
  p->csize = dtype == GRFC_F64 ? 16 : 8;
  p->points = 1;
  double vol = 1.0;
  for (int a = 0; a < dim; ++a) {
    p->n[a] = counts[a];
    p->l[a] = lengths[a];
    p->points *= (uint64_t)counts[a];
    vol *= lengths[a];
  }
  p->cells = half_cells(dim, counts);
  // GridDesc
  p->g.d = dim;
  for (int a = 0; a < dim; ++a) {
    p->g.n[a] = counts[a];
    p->g.l[a] = lengths[a];
    p->g.w_of_k[a] = 2.0 * M_PI / lengths[a];
  }
  p->g.hd = counts[dim - 1] / 2 + 1;
  p->g.cells = (int64_t)p->cells;
  p->g.points = (int64_t)p->points;
  // DensityDesc
  DensityDesc& D = p->D;
  D.family = density->family;
  D.d = dim;
  std::memcpy(D.r, density->r, sizeof D.r);
  std::memcpy(D.i, density->i, sizeof D.i);
  if (D.family == GRFC_DENSITY_GAUSSIAN_COV) {
    D.sqrt_c = std::sqrt(std::pow(D.r[0] / std::sqrt(2.0 * M_PI), dim));
  } else if (D.family == GRFC_DENSITY_MATERN) {
    const double nu = D.r[0], ell = D.r[1];
    D.alpha = nu + 0.5 * dim;
    D.sqrt_c = std::sqrt(std::pow(ell, dim) * std::tgamma(D.alpha) / (std::pow(M_PI, 0.5 * dim) * std::tgamma(nu)));
  } else if (D.family == GRFC_DENSITY_POLY) {
    D.mkl = std::pow(D.r[0], (double)D.i[0] * (double)D.i[1]);
  }
  p->s_one = std::sqrt(two_pi_pow(dim) / vol);
  p->s_two = std::sqrt(two_pi_pow(dim) * (double)p->points / vol) / (double)p->points;

  // Twiddle tables: one per axis length.
  size_t total = 0;
  for (int a = 0; a < dim; ++a) {
    p->tw_off[a] = total;
    total += (size_t)counts[a];
    p->F[a] = factorize(counts[a]);
  }
  p->FM = factorize(counts[dim - 1] / 2);
  GRFC_CUDA(cudaMalloc(&p->d_tw, total * p->csize));
  for (int a = 0; a < dim; ++a) {
    if (dtype == GRFC_F64) {
      auto t = twiddle_table<double>(counts[a]);
      GRFC_CUDA(cudaMemcpy((char*)p->d_tw + p->tw_off[a] * p->csize, t.data(), t.size() * p->csize,
                           cudaMemcpyHostToDevice));
    } else {
      auto t = twiddle_table<float>(counts[a]);
      GRFC_CUDA(cudaMemcpy((char*)p->d_tw + p->tw_off[a] * p->csize, t.data(), t.size() * p->csize,
                           cudaMemcpyHostToDevice));
    }
  }
  if (density->family == GRFC_DENSITY_TABLE) {
    GRFC_CUDA(cudaMalloc(&p->d_table, p->cells * sizeof(double)));
    GRFC_CUDA(cudaMemset(p->d_table, 0, p->cells * sizeof(double)));
  }
  // Fused fast path for power-of-two 2D shapes (pow2_2d.cu).
  // GRFC_DISABLE_FAST=1 forces the generic kernels (A/B parity testing).
  const char* nofast = std::getenv("GRFC_DISABLE_FAST");
  const bool allow_fast = !(nofast && nofast[0] == '1');
  if (allow_fast && fast2d_supported(dim, counts, dtype, algorithm, density->family)) {
    cudaError_t e = fast2d_init(p->fast2d, p->g, p->D, dtype, algorithm, p->s_one, p->s_two);
    if (e == cudaErrorNotSupported) {  // no fused kernel for this shape: the generic path
      fast2d_free(p->fast2d);
      p->fast2d = Fast2D{};
    } else if (e != cudaSuccess) {
      return fail(GRFC_ECUDA, std::string("CUDA: fast2d_init (") + p->fast2d.fail_what + "): " + cudaGetErrorString(e));
    } else {
      p->fast = true;
      p->path = fast2d_name(p->fast2d);
    }
  }
  if (allow_fast && fast3d_supported(dim, counts, algorithm)) {
    cudaError_t e = fast3d_init(p->fast3d, p->g, p->D, dtype, algorithm, p->s_one);
    if (e != cudaSuccess) return fail(GRFC_ECUDA, std::string("CUDA: fast3d_init: ") + cudaGetErrorString(e));
    p->fast3 = true;
    p->path = dtype == GRFC_F64 ? "pow2-3d-f64" : "pow2-3d-f32";
  }
  *out = p.release();
  return GRFC_OK;
}

grfc_status grfc_plan_set_sqrt_gamma_table(grfc_plan p, const double* sg) {
  if (!p || !sg) return fail(GRFC_EINVAL, "grfc: null argument");
  if (p->dens.family != GRFC_DENSITY_TABLE) return fail(GRFC_EINVAL, "grfc: plan density is not a table");
  for (uint64_t h = 0; h < p->cells; ++h)
    if (!(sg[h] >= 0.0) || std::isnan(sg[h]))
      return fail(GRFC_ERUNTIME, "synthesize_spectrum: density evaluated to NaN or negative");
  DeviceGuard guard(p->device);
  GRFC_CUDA(cudaMemcpy(p->d_table, sg, p->cells * sizeof(double), cudaMemcpyHostToDevice));
  p->D.table = p->d_table;
  if (p->fast) {
    const cudaError_t e = fast2d_set_table(p->fast2d, p->d_table);
    if (e != cudaSuccess) return fail(GRFC_ECUDA, std::string("CUDA: density table: ") + cudaGetErrorString(e));
  }
  if (p->fast3) p->fast3d.D.table = p->d_table;
  p->table_set = true;
  return GRFC_OK;
}

void grfc_plan_destroy(grfc_plan p) {
  if (!p) return;
  DeviceGuard guard(p->device);
  if (p->fast) fast2d_free(p->fast2d);
  if (p->fast3) fast3d_free(p->fast3d);
  cudaFree(p->d_tw);
  cudaFree(p->d_table);
  delete p;
}

grfc_status grfc_plan_info(grfc_plan p, uint64_t* cells, uint64_t* points, const char** path) {
  if (!p) return fail(GRFC_EINVAL, "grfc: null plan");
  if (cells) *cells = p->cells;
  if (points) *points = p->points;
  if (path) *path = p->path.c_str();
  return GRFC_OK;
}

grfc_status grfc_generate(grfc_plan p, uint64_t seed, uint64_t first_field, uint64_t nfields, void* d_out,
                          uint64_t field_stride, void* stream) {
  t_launches = 0;
  if (!p || (!d_out && nfields)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (p->dens.family == GRFC_DENSITY_TABLE && !p->table_set)
    return fail(GRFC_EINVAL, "grfc: sqrt-gamma table not set");
  if (field_stride < p->points && nfields > 1) return fail(GRFC_EINVAL, "grfc: field_stride < point count");
  if (nfields == 0) return GRFC_OK;
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (p->fast3 && field_stride % 2 == 0) {  // fused pow2 3D path (pow2_3d.cu)
    cudaError_t e = fast3d_generate(p->fast3d, seed, first_field, (int64_t)nfields, d_out, (int64_t)field_stride, s);
    if (e != cudaSuccess) return fail(GRFC_ECUDA, std::string("CUDA: fused3d: ") + cudaGetErrorString(e));
    return GRFC_OK;
  }
  // Fused pow2 2D path: whole batch, pipelined internally (pow2_2d.cu).
  if (p->fast && field_stride % 2 == 0) {
    cudaError_t e = fast2d_generate(p->fast2d, p->alg, seed, first_field, (int64_t)nfields, d_out,
                                    (int64_t)field_stride, s);
    if (e != cudaSuccess) return fail(GRFC_ECUDA, std::string("CUDA: fused2d: ") + cudaGetErrorString(e));
    return GRFC_OK;
  }
  const int64_t chunk = chunk_fields(p, nfields);
  void* W = nullptr;
  GRFC_CUDA(cudaMallocAsync(&W, (size_t)chunk * p->cells * p->csize, s));
  grfc_status st = GRFC_OK;
  for (uint64_t f = 0; f < nfields && st == GRFC_OK; f += (uint64_t)chunk) {
    const int64_t nf = (int64_t)std::min<uint64_t>((uint64_t)chunk, nfields - f);
    st = run_fields_any(p, seed, first_field + f, nf, W, (char*)d_out + f * field_stride * dsize(p),
                        (int64_t)field_stride, nullptr, nullptr, s);
  }
  cudaFreeAsync(W, s);
  return st;
}

grfc_status grfc_generate_host(grfc_plan p, uint64_t seed, uint64_t first_field, uint64_t nfields, void* h_out,
                               void* stream) {
  t_launches = 0;
  if (!p || (!h_out && nfields)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (nfields == 0) return GRFC_OK;
  DeviceGuard guard(p->device);
  cudaStream_t sg = (cudaStream_t)stream;
  const size_t fbytes = p->points * dsize(p);
  // Output chunks of ~64 MiB, double-buffered against the D2H copies.
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>((int64_t)nfields, (int64_t)((64u << 20) / fbytes)));
  cudaStream_t sc;
  GRFC_CUDA(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  cudaEvent_t gen[2], cp[2];
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&gen[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&cp[i], cudaEventDisableTiming);
  }
  void* buf[2] = {nullptr, nullptr};
  grfc_status st = GRFC_OK;
  cudaError_t e = cudaMallocAsync(&buf[0], (size_t)chunk * fbytes, sg);
  if (e == cudaSuccess) e = cudaMallocAsync(&buf[1], (size_t)chunk * fbytes, sg);
  if (e != cudaSuccess) st = fail(GRFC_ECUDA, std::string("CUDA: cudaMallocAsync: ") + cudaGetErrorString(e));
  uint64_t launches = 0;
  int i = 0;
  for (uint64_t f = 0; f < nfields && st == GRFC_OK; f += (uint64_t)chunk, ++i) {
    const int b = i & 1;
    const int64_t nf = (int64_t)std::min<uint64_t>((uint64_t)chunk, nfields - f);
    if (i >= 2) cudaStreamWaitEvent(sg, cp[b], 0);
    st = grfc_generate(p, seed, first_field + f, (uint64_t)nf, buf[b], p->points, sg);
    launches += t_launches;
    if (st != GRFC_OK) break;
    cudaEventRecord(gen[b], sg);
    cudaStreamWaitEvent(sc, gen[b], 0);
    e = cudaMemcpyAsync((char*)h_out + f * fbytes, buf[b], (size_t)nf * fbytes, cudaMemcpyDeviceToHost, sc);
    if (e != cudaSuccess) st = fail(GRFC_ECUDA, std::string("CUDA: D2H: ") + cudaGetErrorString(e));
    cudaEventRecord(cp[b], sc);
  }
  cudaStreamSynchronize(sc);
  cudaStreamWaitEvent(sg, cp[0], 0);
  cudaStreamWaitEvent(sg, cp[1], 0);
  if (buf[0]) cudaFreeAsync(buf[0], sg);
  if (buf[1]) cudaFreeAsync(buf[1], sg);
  e = cudaStreamSynchronize(sg);
  if (e != cudaSuccess && st == GRFC_OK) st = fail(GRFC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  for (int j = 0; j < 2; ++j) {
    cudaEventDestroy(gen[j]);
    cudaEventDestroy(cp[j]);
  }
  cudaStreamDestroy(sc);
  t_launches = launches;
  return st;
}

grfc_status grfc_generate_injected(grfc_plan p, const double* draws, uint64_t ndraws, void* d_out, void* stream) {
  t_launches = 0;
  if (!p || !d_out || (!draws && ndraws)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (p->dens.family == GRFC_DENSITY_TABLE && !p->table_set)
    return fail(GRFC_EINVAL, "grfc: sqrt-gamma table not set");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double> host;
  const double* src = nullptr;
  size_t nbytes = 0;
  if (p->alg == GRFC_TWO_FFT) {
    if (ndraws < p->points) return fail(GRFC_ERUNTIME, "FixedStream: stream exhausted");
    src = draws;
    nbytes = p->points * sizeof(double);
  } else {
    std::string err;
    if (!arrange_half_noise(p->d, p->n, p->alg, draws, ndraws, host, err)) return fail(GRFC_ERUNTIME, err);
    src = host.data();
    nbytes = host.size() * sizeof(double);
  }
  void* dnoise = nullptr;
  void* W = nullptr;
  GRFC_CUDA(cudaMallocAsync(&dnoise, nbytes, s));
  GRFC_CUDA(cudaMallocAsync(&W, p->cells * p->csize, s));
  GRFC_CUDA(cudaMemcpyAsync(dnoise, src, nbytes, cudaMemcpyHostToDevice, s));
  grfc_status st = run_fields_any(p, 0, 0, 1, W, d_out, (int64_t)p->points,
                                  p->alg == GRFC_TWO_FFT ? nullptr : (const double2*)dnoise,
                                  p->alg == GRFC_TWO_FFT ? (const double*)dnoise : nullptr, s);
  cudaFreeAsync(W, s);
  cudaFreeAsync(dnoise, s);
  // `host` is pageable: cudaMemcpyAsync from it completed before returning.
  if (st == GRFC_OK) GRFC_CUDA(cudaStreamSynchronize(s));
  return st;
}

grfc_status grfc_dump_noise(grfc_plan p, uint64_t seed, uint64_t field, double* draws, uint64_t ndraws) {
  t_launches = 0;
  if (!p || !draws) return fail(GRFC_EINVAL, "grfc: null argument");
  const uint64_t need = grfc::count_draws(p->d, p->n, p->alg);
  if (ndraws < need) return fail(GRFC_EINVAL, "grfc: draws buffer shorter than count_draws");
  DeviceGuard guard(p->device);
  std::vector<uint64_t> ctr;
  std::vector<uint8_t> nd;
  reference_order_counters(p->d, p->n, p->alg, ctr, nd);
  uint64_t* dctr = nullptr;
  double* dpairs = nullptr;
  GRFC_CUDA(cudaMalloc(&dctr, ctr.size() * sizeof(uint64_t)));
  GRFC_CUDA(cudaMalloc(&dpairs, ctr.size() * 2 * sizeof(double)));
  GRFC_CUDA(cudaMemcpy(dctr, ctr.data(), ctr.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  // Unit count per algorithm: Alg 1 point pairs, Alg 2 H cells, Alg 3 lattice points.
  const uint64_t U = p->alg == GRFC_TWO_FFT ? p->points / 2 : p->alg == GRFC_ONE_FFT_OVERWRITE ? p->cells : p->points;
  const uint64_t Uh = (U + 1) / 2;
  cudaError_t e = p->dtype == GRFC_F64
                      ? launch_philox_pairs<double>(dctr, (int64_t)ctr.size(), Uh, seed, field, dpairs, 0)
                      : launch_philox_pairs<float>(dctr, (int64_t)ctr.size(), Uh, seed, field, dpairs, 0);
  std::vector<double> pairs(ctr.size() * 2);
  if (e == cudaSuccess) e = cudaMemcpy(pairs.data(), dpairs, pairs.size() * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(dctr);
  cudaFree(dpairs);
  if (e != cudaSuccess) return fail(GRFC_ECUDA, std::string("CUDA: dump: ") + cudaGetErrorString(e));
  uint64_t pos = 0;
  for (size_t i = 0; i < ctr.size(); ++i) {
    draws[pos++] = pairs[2 * i];
    if (nd[i] == 2) draws[pos++] = pairs[2 * i + 1];
  }
  return GRFC_OK;
}

grfc_status grfc_dft_c2c(int dim, const int64_t* counts, const double* d_in, double* d_out, int sign, void* stream) {
  t_launches = 0;
  if (!counts || !d_in || !d_out) return fail(GRFC_EINVAL, "grfc: null argument");
  if (d_in == d_out) return fail(GRFC_EINVAL, "DftBackend: in-place transform not supported");
  if (dim < 1 || dim > GRFC_MAX_DIM) return fail(GRFC_EINVAL, "grfc: bad dimension");
  int64_t P = 1;
  for (int a = 0; a < dim; ++a) {
    if (counts[a] < 1) return fail(GRFC_EINVAL, "grfc: bad extent");
    P *= counts[a];
  }
  cudaStream_t s = (cudaStream_t)stream;
  // Per-length twiddle tables, cached per device for the process lifetime.
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, void*> cache;
  int dev = 0;
  GRFC_CUDA(cudaGetDevice(&dev));
  GRFC_CUDA(cudaMemcpyAsync(d_out, d_in, (size_t)P * 16, cudaMemcpyDeviceToDevice, s));
  for (int a = 0; a < dim; ++a) {
    const int64_t n = counts[a];
    if (n == 1) continue;
    void* tw = nullptr;
    {
      std::lock_guard<std::mutex> lock(mu);
      auto it = cache.find({dev, n});
      if (it == cache.end()) {
        auto t = twiddle_table<double>(n);
        GRFC_CUDA(cudaMalloc(&tw, t.size() * 16));
        GRFC_CUDA(cudaMemcpy(tw, t.data(), t.size() * 16, cudaMemcpyHostToDevice));
        cache[{dev, n}] = tw;
      } else {
        tw = it->second;
      }
    }
    int64_t inner = 1, outer = 1;
    for (int b = a + 1; b < dim; ++b) inner *= counts[b];
    for (int b = 0; b < a; ++b) outer *= counts[b];
    cudaError_t e = needs_long_line(n, 16) ? cudaErrorInvalidValue
                                           : launch_line_c2c<double>(d_out, (int)n, inner, outer, sign > 0 ? +1 : -1,
                                                                     factorize(n), tw, s);
    if (e == cudaErrorInvalidValue) e = long_c2c<double>(d_out, n, inner, outer, sign > 0 ? +1 : -1, s);
    GRFC_CUDA(e);
  }
  if (sign < 0) GRFC_CUDA(launch_scale_all<double>(d_out, P, 1.0 / (double)P, s));
  return GRFC_OK;
}

}  // extern "C"

extern "C" {

grfc_status grfc_generate_injected_host(grfc_plan p, const double* draws, uint64_t ndraws, void* h_out) {
  if (!p || !h_out) return fail(GRFC_EINVAL, "grfc: null argument");
  DeviceGuard guard(p->device);
  void* d = nullptr;
  GRFC_CUDA(cudaMalloc(&d, p->points * dsize(p)));
  grfc_status st = grfc_generate_injected(p, draws, ndraws, d, nullptr);
  if (st == GRFC_OK) {
    cudaError_t e = cudaMemcpy(h_out, d, p->points * dsize(p), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(GRFC_ECUDA, std::string("CUDA: D2H: ") + cudaGetErrorString(e));
  }
  cudaFree(d);
  return st;
}

grfc_status grfc_dft_c2c_host(int dim, const int64_t* counts, const double* h_in, double* h_out, int sign,
                              int device) {
  if (!counts || !h_in || !h_out) return fail(GRFC_EINVAL, "grfc: null argument");
  if (h_in == h_out) return fail(GRFC_EINVAL, "DftBackend: in-place transform not supported");
  if (dim < 1 || dim > GRFC_MAX_DIM) return fail(GRFC_EINVAL, "grfc: bad dimension");
  int64_t P = 1;
  for (int a = 0; a < dim; ++a) P *= counts[a];
  DeviceGuard guard(device);
  double *din = nullptr, *dout = nullptr;
  GRFC_CUDA(cudaMalloc(&din, (size_t)P * 16));
  cudaError_t e = cudaMalloc(&dout, (size_t)P * 16);
  if (e == cudaSuccess) e = cudaMemcpy(din, h_in, (size_t)P * 16, cudaMemcpyHostToDevice);
  grfc_status st = GRFC_OK;
  if (e != cudaSuccess) st = fail(GRFC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  if (st == GRFC_OK) st = grfc_dft_c2c(dim, counts, din, dout, sign, nullptr);
  if (st == GRFC_OK) {
    e = cudaMemcpy(h_out, dout, (size_t)P * 16, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(GRFC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  }
  cudaFree(din);
  cudaFree(dout);
  return st;
}

}  // extern "C"

extern "C" {

grfc_status grfc_slab_sizes(grfc_plan p, int world, uint64_t* buf_elems, uint64_t* block_elems,
                            uint64_t* slab_points) {
  if (!p) return fail(GRFC_EINVAL, "grfc: null plan");
  if (!p->fast3) return fail(GRFC_EINVAL, "grfc: slab decomposition needs a pow2 3D plan");
  SlabGeom g;
  if (!slab_geometry(p->fast3d, world, g)) return fail(GRFC_EINVAL, "grfc: world must divide N0 and N1");
  if (buf_elems) *buf_elems = g.buf_elems;
  if (block_elems) *block_elems = g.block_elems;
  if (slab_points) *slab_points = (uint64_t)g.n0p * p->n[1] * p->n[2];
  return GRFC_OK;
}

grfc_status grfc_slab_pass_a(grfc_plan p, int world, int rank, uint64_t seed, uint64_t field, void* d_send,
                             void* stream) {
  t_launches = 0;
  if (!p || !d_send) return fail(GRFC_EINVAL, "grfc: null argument");
  if (!p->fast3) return fail(GRFC_EINVAL, "grfc: slab decomposition needs a pow2 3D plan");
  SlabGeom g;
  if (!slab_geometry(p->fast3d, world, g) || rank < 0 || rank >= world)
    return fail(GRFC_EINVAL, "grfc: bad world/rank for this grid");
  DeviceGuard guard(p->device);
  GRFC_CUDA(fast3d_pass_a(p->fast3d, world, rank, seed, field, d_send, (cudaStream_t)stream));
  return GRFC_OK;
}

grfc_status grfc_slab_pass_b(grfc_plan p, int world, const void* d_recv, void* d_out, void* stream) {
  t_launches = 0;
  if (!p || !d_recv || !d_out) return fail(GRFC_EINVAL, "grfc: null argument");
  if (!p->fast3) return fail(GRFC_EINVAL, "grfc: slab decomposition needs a pow2 3D plan");
  SlabGeom g;
  if (!slab_geometry(p->fast3d, world, g)) return fail(GRFC_EINVAL, "grfc: world must divide N0 and N1");
  DeviceGuard guard(p->device);
  GRFC_CUDA(fast3d_pass_b(p->fast3d, world, d_recv, d_out, (cudaStream_t)stream));
  return GRFC_OK;
}

grfc_status grfc_plan_grid(grfc_plan p, int* dim, int64_t* counts, double* lengths, int* dtype, int* device) {
  if (!p) return fail(GRFC_EINVAL, "grfc: null argument");
  if (dim) *dim = p->d;
  for (int a = 0; a < p->d; ++a) {
    if (counts) counts[a] = p->n[a];
    if (lengths) lengths[a] = p->l[a];
  }
  if (dtype) *dtype = p->dtype;
  if (device) *device = p->device;
  return GRFC_OK;
}

// ---- Monte-Carlo covariance (stats.cu; reference src/stats.cpp:39-97) --------------------

static grfc_status cov_check(grfc_plan p, uint64_t samples, int64_t ref) {
  if (!p) return fail(GRFC_EINVAL, "grfc: null argument");
  if (samples < 1) return fail(GRFC_EINVAL, "estimate_covariance: need at least one sample");
  if (ref < 0 || (uint64_t)ref >= p->points)
    return fail(GRFC_EINVAL, "estimate_covariance: reference index out of range");
  if (p->dens.family == GRFC_DENSITY_TABLE && !p->table_set)
    return fail(GRFC_EINVAL, "grfc: sqrt-gamma table not set");
  return GRFC_OK;
}

// Fields generated per accumulate launch: <= GRFC_COV_CHUNK and ~1 GiB of
// scratch (GRFC_COV_BATCH overrides; results do not depend on it).
static uint64_t cov_batch(grfc_plan p) {
  const char* e = std::getenv("GRFC_COV_BATCH");
  uint64_t b = e ? (uint64_t)std::strtoull(e, nullptr, 10) : 0;
  if (!b) b = std::max<uint64_t>(1, (1ull << 30) / (p->points * dsize(p)));
  return std::min<uint64_t>(b, GRFC_COV_CHUNK);
}

// Chunks [c0, c0 + nc): partial sums into part + (c - c0) * P, or, when
// est != nullptr, merged into (est, comp) in chunk order through `acc`.
static grfc_status cov_chunks(grfc_plan p, uint64_t seed, uint64_t samples, uint64_t c0, uint64_t nc, int64_t ref,
                              double* part, double* acc, double* est, double* comp, cudaStream_t s,
                              uint64_t* launches) {
  const uint64_t P = p->points, B = cov_batch(p);
  void* buf = nullptr;
  grfc_status st = GRFC_OK;
  // Small grids: whole groups of chunks per generate / accumulate / merge launch
  // (k_cov_accumulate_chunks keeps every chunk's own ascending-j sum, and the
  // grouped merge performs the same Kahan steps in chunk order: bit-identical).
  const uint64_t chunk_bytes = (uint64_t)GRFC_COV_CHUNK * P * dsize(p);
  const uint64_t G = std::getenv("GRFC_COV_BATCH") ? 1 : std::min<uint64_t>(nc, (1ull << 30) / chunk_bytes);
  if (G >= 2) {
    double* gpart = nullptr;
    GRFC_CUDA(cudaMallocAsync(&buf, (size_t)(G * chunk_bytes), s));
    cudaError_t e = est ? cudaMallocAsync(&gpart, (size_t)G * P * sizeof(double), s) : cudaSuccess;
    for (uint64_t c = c0; c < c0 + nc && e == cudaSuccess && st == GRFC_OK; c += G) {
      const uint64_t g = std::min<uint64_t>(G, c0 + nc - c);
      const uint64_t begin = c * GRFC_COV_CHUNK, end = std::min<uint64_t>((c + g) * GRFC_COV_CHUNK, samples);
      st = grfc_generate(p, seed, begin, end - begin, buf, P, s);
      *launches += t_launches;
      if (st != GRFC_OK) break;
      double* out = est ? gpart : part + (c - c0) * P;
      e = launch_cov_accumulate_chunks(p->dtype, buf, end - begin, P, (uint64_t)ref, GRFC_COV_CHUNK, out, s);
      ++*launches;
      if (e == cudaSuccess && est) e = launch_cov_merge_chunks(gpart, g, est, comp, P, s), ++*launches;
    }
    if (e != cudaSuccess && st == GRFC_OK) st = fail(GRFC_ECUDA, std::string("CUDA: covariance: ") + cudaGetErrorString(e));
    if (gpart) cudaFreeAsync(gpart, s);
    cudaFreeAsync(buf, s);
    return st;
  }
  GRFC_CUDA(cudaMallocAsync(&buf, (size_t)B * P * dsize(p), s));
  for (uint64_t c = c0; c < c0 + nc && st == GRFC_OK; ++c) {
    const uint64_t begin = c * GRFC_COV_CHUNK, end = std::min<uint64_t>(begin + GRFC_COV_CHUNK, samples);
    double* a = est ? acc : part + (c - c0) * P;
    cudaError_t e = cudaMemsetAsync(a, 0, P * sizeof(double), s);
    for (uint64_t j = begin; j < end && e == cudaSuccess && st == GRFC_OK; j += B) {
      const uint64_t n = std::min<uint64_t>(B, end - j);
      st = grfc_generate(p, seed, j, n, buf, P, s);
      *launches += t_launches;
      if (st == GRFC_OK) e = launch_cov_accumulate(p->dtype, buf, n, P, P, (uint64_t)ref, a, s), ++*launches;
    }
    if (e == cudaSuccess && st == GRFC_OK && est) e = launch_cov_merge(a, est, comp, P, s), ++*launches;
    if (e != cudaSuccess && st == GRFC_OK) st = fail(GRFC_ECUDA, std::string("CUDA: covariance: ") + cudaGetErrorString(e));
  }
  cudaFreeAsync(buf, s);
  return st;
}

grfc_status grfc_covariance_accumulate(grfc_plan p, const void* d_fields, uint64_t nfields, uint64_t field_stride,
                                       int64_t ref, double* d_acc, void* stream) {
  t_launches = 0;
  if (!p || !d_acc || (!d_fields && nfields)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (ref < 0 || (uint64_t)ref >= p->points)
    return fail(GRFC_EINVAL, "estimate_covariance: reference index out of range");
  if (field_stride < p->points && nfields > 1) return fail(GRFC_EINVAL, "grfc: field_stride < point count");
  DeviceGuard guard(p->device);
  GRFC_CUDA(launch_cov_accumulate(p->dtype, d_fields, nfields, field_stride, p->points, (uint64_t)ref, d_acc,
                                  (cudaStream_t)stream));
  return GRFC_OK;
}

grfc_status grfc_covariance_partials(grfc_plan p, uint64_t seed, uint64_t samples, uint64_t chunk0, uint64_t nchunks,
                                     int64_t ref, double* d_partials, void* stream) {
  grfc_status st = cov_check(p, samples, ref);
  if (st != GRFC_OK) return st;
  const uint64_t total = (samples + GRFC_COV_CHUNK - 1) / GRFC_COV_CHUNK;
  if (chunk0 > total || nchunks > total - chunk0) return fail(GRFC_EINVAL, "grfc: chunk range out of range");
  if (!d_partials && nchunks) return fail(GRFC_EINVAL, "grfc: null argument");
  DeviceGuard guard(p->device);
  uint64_t launches = 0;
  st = cov_chunks(p, seed, samples, chunk0, nchunks, ref, d_partials, nullptr, nullptr, nullptr,
                  (cudaStream_t)stream, &launches);
  t_launches = launches;
  return st;
}

grfc_status grfc_covariance_merge(grfc_plan p, const double* d_partials, uint64_t nchunks, uint64_t samples,
                                  double* d_out, void* stream) {
  t_launches = 0;
  if (!p || !d_out || (!d_partials && nchunks)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (samples < 1) return fail(GRFC_EINVAL, "estimate_covariance: need at least one sample");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t P = p->points;
  double* comp = nullptr;
  GRFC_CUDA(cudaMallocAsync(&comp, P * sizeof(double), s));
  cudaError_t e = cudaMemsetAsync(comp, 0, P * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_out, 0, P * sizeof(double), s);
  uint64_t launches = 0;
  for (uint64_t c = 0; c < nchunks && e == cudaSuccess; ++c, ++launches)
    e = launch_cov_merge(d_partials + c * P, d_out, comp, P, s);
  if (e == cudaSuccess) e = launch_cov_scale(d_out, P, 1.0 / (double)samples, s), ++launches;
  cudaFreeAsync(comp, s);
  t_launches = launches;
  GRFC_CUDA(e);
  return GRFC_OK;
}

grfc_status grfc_estimate_covariance(grfc_plan p, uint64_t seed, uint64_t samples, int64_t ref, double* d_out,
                                     void* stream) {
  grfc_status st = cov_check(p, samples, ref);
  if (st != GRFC_OK) return st;
  if (!d_out) return fail(GRFC_EINVAL, "grfc: null argument");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t P = p->points;
  double* scratch = nullptr;  // acc | comp
  GRFC_CUDA(cudaMallocAsync(&scratch, 2 * P * sizeof(double), s));
  cudaError_t e = cudaMemsetAsync(scratch + P, 0, P * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_out, 0, P * sizeof(double), s);
  uint64_t launches = 0;
  if (e == cudaSuccess)
    st = cov_chunks(p, seed, samples, 0, (samples + GRFC_COV_CHUNK - 1) / GRFC_COV_CHUNK, ref, nullptr, scratch,
                    d_out, scratch + P, s, &launches);
  if (e == cudaSuccess && st == GRFC_OK) e = launch_cov_scale(d_out, P, 1.0 / (double)samples, s), ++launches;
  cudaFreeAsync(scratch, s);
  t_launches = launches;
  if (st != GRFC_OK) return st;
  GRFC_CUDA(e);
  return GRFC_OK;
}

grfc_status grfc_estimate_covariance_host(grfc_plan p, uint64_t seed, uint64_t samples, int64_t ref,
                                          double* h_out) {
  grfc_status st = cov_check(p, samples, ref);
  if (st != GRFC_OK) return st;
  if (!h_out) return fail(GRFC_EINVAL, "grfc: null argument");
  DeviceGuard guard(p->device);
  cudaStream_t s;
  GRFC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, p->points * sizeof(double), s);
  if (e == cudaSuccess) {
    st = grfc_estimate_covariance(p, seed, samples, ref, d, s);
    const uint64_t launches = t_launches;
    if (st == GRFC_OK) e = cudaMemcpyAsync(h_out, d, p->points * sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    t_launches = launches;
  }
  const cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (st != GRFC_OK) return st;
  GRFC_CUDA(e);
  GRFC_CUDA(e2);
  return GRFC_OK;
}

grfc_status grfc_covariance_chunk_injected_host(grfc_plan p, const double* draws, uint64_t nsamples,
                                                uint64_t ndraws, int64_t ref, double* h_partial) {
  if (!p || !h_partial || (!draws && nsamples)) return fail(GRFC_EINVAL, "grfc: null argument");
  if (ref < 0 || (uint64_t)ref >= p->points)
    return fail(GRFC_EINVAL, "estimate_covariance: reference index out of range");
  DeviceGuard guard(p->device);
  cudaStream_t s;
  GRFC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const uint64_t P = p->points, B = cov_batch(p);
  void* buf = nullptr;
  double* acc = nullptr;
  grfc_status st = GRFC_OK;
  cudaError_t e = cudaMallocAsync(&buf, (size_t)B * P * dsize(p), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&acc, P * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(acc, 0, P * sizeof(double), s);
  uint64_t launches = 0;
  for (uint64_t j = 0; j < nsamples && e == cudaSuccess && st == GRFC_OK; j += B) {
    const uint64_t n = std::min<uint64_t>(B, nsamples - j);
    for (uint64_t i = 0; i < n && st == GRFC_OK; ++i) {
      st = grfc_generate_injected(p, draws + (j + i) * ndraws, ndraws, (char*)buf + i * P * dsize(p), s);
      launches += t_launches;
    }
    if (st == GRFC_OK) e = launch_cov_accumulate(p->dtype, buf, n, P, P, (uint64_t)ref, acc, s), ++launches;
  }
  if (e == cudaSuccess && st == GRFC_OK)
    e = cudaMemcpyAsync(h_partial, acc, P * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (buf) cudaFreeAsync(buf, s);
  if (acc) cudaFreeAsync(acc, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  t_launches = launches;
  if (st != GRFC_OK) return st;
  GRFC_CUDA(e);
  GRFC_CUDA(e2);
  return GRFC_OK;
}

}  // extern "C"
