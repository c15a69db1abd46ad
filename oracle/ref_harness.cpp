// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" harness around the REFERENCE's own proj/core, compiled unmodified
// from /root/reference by oracle/Makefile into oracle/_ref/libgrf_ref.so (the
// FFT underneath FftwBackend is the standin/fftw3.h stand-in).
// It exposes, for ctypes:
//   * synthesis from an injected noise array through the reference's
//     FixedStream (random.hpp:50-62) — the parity oracle for the GPU path;
//   * the seed overload (synth.cpp:129-135) for the CPU baseline, run with the
//     reference's own batch pattern (one field per std::thread, substreams
//     (seed, j), mirroring stats.cpp:57-81);
//   * draw counts, representative-set order, spectra and exact covariance.
// The two densities the BASELINE configs need but the reference does not ship
// (Gaussian covariance, Matern) are added here as user SpectralDensity
// subclasses — the reference's own extension point (tests/test_support.hpp).
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "grf/dft.hpp"
#include "grf/field_io.hpp"
#include "grf/hermitian.hpp"
#include "grf/spectral.hpp"
#include "grf/stats.hpp"
#include "grf/synth.hpp"

namespace {

// Shared POD descriptor layout (same as oracle/grf_oracle.h gro_density).
struct ref_density {
  int family;  // 0 poly, 1 aniso, 2 test1d, 3 gaussian-cov, 4 matern, 5 constant
  int dim;
  double r[8];
  int i[8];
};

class GaussianCovDensity final : public grf::SpectralDensity {
 public:
  GaussianCovDensity(double ell, int dim) : ell_(ell), dim_(dim) {
    c_ = std::pow(ell / std::sqrt(2.0 * std::numbers::pi), dim);
  }
  int dim() const override { return dim_; }
  double eval(std::span<const double> p) const override {
    check_dim(p);
    double s = 0.0;
    for (double v : p) s += v * v;
    return c_ * std::exp(-0.5 * ell_ * ell_ * s);
  }
  std::string spec_string() const override { return "gauss-cov"; }

 private:
  double ell_, c_;
  int dim_;
};

class MaternDensity final : public grf::SpectralDensity {
 public:
  MaternDensity(double nu, double ell, int dim) : ell_(ell), dim_(dim) {
    alpha_ = nu + 0.5 * dim;
    c_ = std::pow(ell, dim) * std::tgamma(alpha_) /
         (std::pow(std::numbers::pi, 0.5 * dim) * std::tgamma(nu));
  }
  int dim() const override { return dim_; }
  double eval(std::span<const double> p) const override {
    check_dim(p);
    double s = 0.0;
    for (double v : p) s += v * v;
    return c_ * std::pow(1.0 + ell_ * ell_ * s, -alpha_);
  }
  std::string spec_string() const override { return "matern"; }

 private:
  double ell_, alpha_, c_;
  int dim_;
};

class ConstantDensity final : public grf::SpectralDensity {
 public:
  ConstantDensity(double c, int dim) : c_(c), dim_(dim) {}
  int dim() const override { return dim_; }
  double eval(std::span<const double> p) const override {
    check_dim(p);
    return c_;
  }
  std::string spec_string() const override { return "constant"; }

 private:
  double c_;
  int dim_;
};

std::unique_ptr<grf::SpectralDensity> make_density(const ref_density* d) {
  switch (d->family) {
    case 0: return std::make_unique<grf::PolyDecayDensity>(d->r[0], d->i[0], d->i[1], d->i[2], d->dim);
    case 1: {
      std::vector<int> ks(d->i + 1, d->i + 1 + d->dim);
      return std::make_unique<grf::AnisoPolyDensity>(d->r[0], ks, d->i[0]);
    }
    case 2: return std::make_unique<grf::Test1dDensity>();
    case 3: return std::make_unique<GaussianCovDensity>(d->r[0], d->dim);
    case 4: return std::make_unique<MaternDensity>(d->r[0], d->r[1], d->dim);
    case 5: return std::make_unique<ConstantDensity>(d->r[0], d->dim);
  }
  throw std::invalid_argument("ref_harness: unknown density family");
}

grf::GridSpec make_grid(int dim, const int64_t* counts, const double* lengths) {
  return grf::GridSpec(std::vector<double>(lengths, lengths + dim),
                       std::vector<std::int64_t>(counts, counts + dim));
}

grf::Algorithm to_alg(int a) {
  if (a < 0 || a > 2) throw std::invalid_argument("ref_harness: bad algorithm");
  return static_cast<grf::Algorithm>(a);
}

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

grf::DftBackend& pick_backend(int backend) {
  static grf::NaiveDftBackend naive;
  if (backend == 1) return naive;
  return grf::default_backend();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_count_draws(int dim, const int64_t* counts, int alg, uint64_t* out) {
  return guarded([&] {
    std::vector<double> ones(static_cast<std::size_t>(dim), 1.0);
    *out = grf::count_draws(make_grid(dim, counts, ones.data()), to_alg(alg));
  });
}

double ref_density_eval(const ref_density* d, const double* omega) {
  double v = NAN;
  guarded([&] {
    auto dens = make_density(d);
    v = dens->eval(std::span<const double>(omega, static_cast<std::size_t>(d->dim)));
  });
  return v;
}

// Synthesis from injected draws through FixedStream. backend: 0 = FftwBackend
// (stand-in FFT), 1 = NaiveDftBackend. consumed = draws the reference took.
int ref_synthesize_draws(int dim, const int64_t* counts, const double* lengths,
                         const ref_density* d, int alg, const double* draws, uint64_t ndraws,
                         int backend, double* out, double* residue, uint64_t* consumed) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    auto dens = make_density(d);
    grf::FixedStream rng(std::vector<double>(draws, draws + ndraws));
    const grf::RealField f = grf::synthesize(grid, *dens, rng, to_alg(alg), pick_backend(backend));
    std::memcpy(out, f.values.data(), sizeof(double) * f.values.size());
    if (residue) *residue = f.imag_residue;
    if (consumed) *consumed = rng.draws_consumed();
  });
}

// The reference seed overload (xoshiro256++ + ziggurat), for the CPU baseline.
int ref_synthesize_seed(int dim, const int64_t* counts, const double* lengths, const ref_density* d,
                        int alg, uint64_t seed, double* out) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    auto dens = make_density(d);
    const grf::RealField f = grf::synthesize(grid, *dens, seed, to_alg(alg));
    std::memcpy(out, f.values.data(), sizeof(double) * f.values.size());
  });
}

// The reference's seeded stream itself: n normals of Xoshiro256Stream(seed,
// substream) and, from a second instance, n raw next_u64 words (pins the
// drop-in's bit-identical restatement of random.cpp:56-108).
int ref_xoshiro(uint64_t seed, uint64_t substream, uint64_t n, double* normals, uint64_t* words) {
  return guarded([&] {
    grf::Xoshiro256Stream a(seed, substream), b(seed, substream);
    for (uint64_t i = 0; i < n; ++i) normals[i] = a.next();
    for (uint64_t i = 0; i < n; ++i) words[i] = b.next_u64();
  });
}

// Full-lattice spectrum (interleaved re/im) from injected draws.
int ref_spectrum(int dim, const int64_t* counts, const double* lengths, const ref_density* d,
                 int mode, const double* draws, uint64_t ndraws, double* out) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    auto dens = make_density(d);
    grf::FixedStream rng(std::vector<double>(draws, draws + ndraws));
    const auto m = mode == 0 ? grf::SpectrumMode::exact_set : grf::SpectrumMode::overwrite;
    const grf::HermitianSpectrum s = grf::synthesize_spectrum(grid, *dens, rng, m);
    std::memcpy(out, s.values.data(), sizeof(double) * 2 * s.values.size());
  });
}

// Representative set in the reference's Alg-3 draw order: row-major linear
// index and self-conjugate flag per rep. Returns the rep count or -1.
int64_t ref_conjugate_reps(int dim, const int64_t* counts, int64_t* lin, uint8_t* self,
                           int64_t cap) {
  int64_t n = -1;
  guarded([&] {
    std::vector<double> ones(static_cast<std::size_t>(dim), 1.0);
    const grf::GridSpec grid = make_grid(dim, counts, ones.data());
    int64_t i = 0;
    grf::for_each_conjugate_rep(grid, [&](const grf::MultiIndex& k, bool s) {
      if (i < cap) {
        lin[i] = grid.linear_index(k);
        self[i] = s ? 1 : 0;
      }
      ++i;
    });
    n = i;
  });
  return n;
}

int ref_exact_cov_all(int dim, const int64_t* counts, const double* lengths, const ref_density* d,
                      int backend, double* out) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    auto dens = make_density(d);
    const std::vector<double> c = grf::exact_discrete_covariance_all(grid, *dens, pick_backend(backend));
    std::memcpy(out, c.data(), sizeof(double) * c.size());
  });
}

// CPU baseline: nfields syntheses through the reference's public seed API,
// fields distributed over `threads` std::threads by an atomic counter (the
// reference's own batch pattern, stats.cpp:57-81), field j seeded
// Xoshiro256Stream(seed, j) as stats.cpp:105 does. Returns wall seconds.
int ref_bench_batch(int dim, const int64_t* counts, const double* lengths, const ref_density* d,
                    int alg, uint64_t seed, uint64_t nfields, int threads, double* seconds,
                    double* checksum) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    auto dens = make_density(d);
    const grf::Algorithm a = to_alg(alg);
    grf::DftBackend& backend = grf::default_backend();
    {  // warm-up: plans + thread_local scratch on this thread
      grf::Xoshiro256Stream rng(seed, 0);
      (void)grf::synthesize(grid, *dens, rng, a, backend);
    }
    std::atomic<uint64_t> next{0};
    std::vector<double> sums(static_cast<std::size_t>(threads > 0 ? threads : 1), 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    auto work = [&](int t) {
      for (;;) {
        const uint64_t j = next.fetch_add(1);
        if (j >= nfields) return;
        grf::Xoshiro256Stream rng(seed, j);
        const grf::RealField f = grf::synthesize(grid, *dens, rng, a, backend);
        sums[static_cast<std::size_t>(t)] += f.values[static_cast<std::size_t>(j % f.values.size())];
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    double s = 0.0;
    for (double v : sums) s += v;
    if (checksum) *checksum = s;
  });
}

// grf::estimate_covariance through the reference's StreamFactory overload
// (stats.cpp:39-97): sample j replays draws[j*ndraws ...] through a
// FixedStream. `ref` is the multi-index of the reference point.
int ref_estimate_covariance_fixed(int dim, const int64_t* counts, const double* lengths, const ref_density* d,
                                  int alg, uint64_t samples, const int64_t* ref, const double* draws,
                                  uint64_t ndraws, int threads, double* out) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    auto dens = make_density(d);
    const grf::StreamFactory streams = [&](std::uint64_t j) {
      return std::make_unique<grf::FixedStream>(
          std::vector<double>(draws + j * ndraws, draws + (j + 1) * ndraws));
    };
    const grf::CovarianceEstimate e = grf::estimate_covariance(
        grid, *dens, to_alg(alg), samples, grf::MultiIndex(ref, ref + dim), streams, threads);
    std::memcpy(out, e.estimates.data(), sizeof(double) * e.estimates.size());
  });
}

// grf::convergence_study (stats.cpp:141-174): rows (level, cells, max_err,
// mc_floor) into rows[4*i..]; *nrows rows; *slope = fitted slope or NaN.
int ref_convergence_study(int level_min, int level_max, uint64_t samples, int alg, uint64_t seed, int threads,
                          double* rows, int* nrows, double* slope) {
  return guarded([&] {
    const grf::ConvergenceReport r =
        grf::convergence_study(level_min, level_max, samples, to_alg(alg), seed, threads);
    *nrows = static_cast<int>(r.rows.size());
    for (std::size_t i = 0; i < r.rows.size(); ++i) {
      rows[4 * i] = r.rows[i].level;
      rows[4 * i + 1] = static_cast<double>(r.rows[i].cells);
      rows[4 * i + 2] = r.rows[i].max_err;
      rows[4 * i + 3] = r.rows[i].mc_floor;
    }
    *slope = r.fitted_slope ? *r.fitted_slope : std::nan("");
  });
}

// The reference's GRF1 writer / reader (src/field_io.cpp:60-107).
int ref_write_grf1(const char* path, int dim, const int64_t* counts, const double* lengths, const double* values) {
  return guarded([&] {
    const grf::GridSpec grid = make_grid(dim, counts, lengths);
    grf::RealField f{grid, std::vector<double>(values, values + grid.point_count()), {}, 0.0};
    grf::write_grf1(path, f);
  });
}

// Reads a GRF1 file: *dim, counts/lengths (up to 16), values (cap entries).
int ref_read_grf1(const char* path, int* dim, int64_t* counts, double* lengths, double* values, uint64_t cap) {
  return guarded([&] {
    const grf::RealField f = grf::read_grf1(path);
    *dim = f.grid.dim();
    for (int a = 0; a < f.grid.dim(); ++a) {
      counts[a] = f.grid.counts()[a];
      lengths[a] = f.grid.lengths()[a];
    }
    if (f.values.size() > cap) throw std::runtime_error("ref_read_grf1: buffer too small");
    std::memcpy(values, f.values.data(), sizeof(double) * f.values.size());
  });
}

}  // extern "C"
