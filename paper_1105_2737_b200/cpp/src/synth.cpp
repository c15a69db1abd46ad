// grf::synthesize on the B200 through the grfc C-ABI.
//   stream overload  -> grfc_generate_injected_host (host draw arrangement,
//                       device transforms, fp64)
//   seed overload    -> grfc_generate_host (device Philox noise, fp64)
// Reference semantics: /root/reference/proj/core/src/synth.cpp:68-218.
#include "grf/synth.hpp"

#include <algorithm>
#include <cmath>
#include <list>
#include <mutex>
#include <numbers>
#include <stdexcept>
#include <string>

#include "grfc_cpp.hpp"

namespace grf {

namespace detail {

grfc_density describe(const SpectralDensity& density) {
  grfc_density d{};
  d.dim = density.dim();
  if (auto* p = dynamic_cast<const PolyDecayDensity*>(&density)) {
    d.family = GRFC_DENSITY_POLY;
    d.r[0] = p->m();
    d.i[0] = p->k();
    d.i[1] = p->l();
    d.i[2] = p->n();
  } else if (auto* a = dynamic_cast<const AnisoPolyDensity*>(&density)) {
    d.family = GRFC_DENSITY_ANISO;
    d.r[0] = a->m();
    d.i[0] = a->n();
    for (std::size_t i = 0; i < a->ks().size() && i < 7; ++i) d.i[1 + i] = a->ks()[i];
  } else if (dynamic_cast<const Test1dDensity*>(&density)) {
    d.family = GRFC_DENSITY_TEST1D;
  } else if (auto* g = dynamic_cast<const GaussianCovDensity*>(&density)) {
    d.family = GRFC_DENSITY_GAUSSIAN_COV;
    d.r[0] = g->ell();
  } else if (auto* m = dynamic_cast<const MaternDensity*>(&density)) {
    d.family = GRFC_DENSITY_MATERN;
    d.r[0] = m->nu();
    d.r[1] = m->ell();
  } else {
    d.family = GRFC_DENSITY_TABLE;
  }
  return d;
}

std::vector<double> sqrt_gamma_table(const GridSpec& grid, const SpectralDensity& density) {
  const int d = grid.dim();
  const auto& n = grid.counts();
  std::vector<std::int64_t> ext(n.begin(), n.end());
  ext[d - 1] = n[d - 1] / 2 + 1;
  std::int64_t cells = 1;
  for (auto e : ext) cells *= e;
  std::vector<double> out(static_cast<std::size_t>(cells));
  std::vector<double> w(static_cast<std::size_t>(d));
  std::vector<std::int64_t> k(static_cast<std::size_t>(d), 0);
  for (std::int64_t h = 0; h < cells; ++h) {
    for (int a = 0; a < d; ++a) {
      const std::int64_t kw = 2 * k[a] <= n[a] ? k[a] : k[a] - n[a];
      w[a] = 2.0 * std::numbers::pi * static_cast<double>(kw) / grid.lengths()[a];
    }
    const double g = density.eval(w);
    if (!(g >= 0.0) || std::isnan(g))
      throw std::runtime_error("synthesize_spectrum: density evaluated to NaN or negative");
    out[static_cast<std::size_t>(h)] = std::sqrt(g);
    for (int a = d - 1; a >= 0; --a) {
      if (++k[a] < ext[a]) break;
      k[a] = 0;
    }
  }
  return out;
}

SharedPlan make_plan(const GridSpec& grid, const SpectralDensity& density, int algorithm, int dtype) {
  if (density.dim() != grid.dim()) throw std::invalid_argument("synthesize: density dimension mismatch");
  const grfc_density desc = describe(density);
  // Plans of in-kernel density families are immutable and safe for concurrent
  // generate calls, so they are cached (the reference caches its FFTW plans the
  // same way, dft.cpp:27-69): repeated synthesize() calls on one grid pay the
  // plan setup (twiddles, tables, kernel queries) once. Table densities depend
  // on the subclass's eval and are planned per call.
  std::string key;
  if (desc.family != GRFC_DENSITY_TABLE) {
    const auto put = [&](const void* p, std::size_t n) { key.append(static_cast<const char*>(p), n); };
    const int hdr[3] = {grid.dim(), algorithm, dtype};
    put(hdr, sizeof hdr);
    put(grid.counts().data(), grid.counts().size() * sizeof(std::int64_t));
    put(grid.lengths().data(), grid.lengths().size() * sizeof(double));
    put(&desc, sizeof desc);
    std::lock_guard<std::mutex> lock(plan_cache_mutex());
    auto& cache = plan_cache();
    for (auto it = cache.begin(); it != cache.end(); ++it)
      if (it->first == key) {
        cache.splice(cache.begin(), cache, it);  // most recently used first
        return cache.front().second;
      }
  }
  grfc_plan raw = nullptr;
  check(grfc_plan_create(&raw, grid.dim(), grid.counts().data(), grid.lengths().data(), dtype, algorithm, &desc, 0));
  SharedPlan plan(raw, PlanDeleter{});
  if (desc.family == GRFC_DENSITY_TABLE) {
    const std::vector<double> t = sqrt_gamma_table(grid, density);
    check(grfc_plan_set_sqrt_gamma_table(plan.get(), t.data()));
    return plan;
  }
  std::lock_guard<std::mutex> lock(plan_cache_mutex());
  auto& cache = plan_cache();
  cache.emplace_front(key, plan);
  constexpr std::size_t kMaxPlans = 16;
  if (cache.size() > kMaxPlans) cache.pop_back();
  return plan;
}

std::mutex& plan_cache_mutex() {
  static std::mutex mu;
  return mu;
}

std::list<std::pair<std::string, SharedPlan>>& plan_cache() {
  static auto* cache = new std::list<std::pair<std::string, SharedPlan>>();  // never destroyed: no
  return *cache;  // device frees after the CUDA runtime has shut down at exit
}

}  // namespace detail

std::string_view algorithm_name(Algorithm algorithm) {
  switch (algorithm) {
    case Algorithm::two_fft: return "two-fft";
    case Algorithm::one_fft_overwrite: return "one-fft";
    case Algorithm::one_fft_recursive: return "recursive";
  }
  return "unknown";
}

std::optional<Algorithm> parse_algorithm(std::string_view name) {
  for (Algorithm a : {Algorithm::two_fft, Algorithm::one_fft_overwrite, Algorithm::one_fft_recursive})
    if (algorithm_name(a) == name) return a;
  return std::nullopt;
}

std::uint64_t count_draws(const GridSpec& grid, Algorithm algorithm) {
  std::uint64_t n = 0;
  detail::check(grfc_count_draws(grid.dim(), grid.counts().data(), static_cast<int>(algorithm), &n));
  return n;
}

namespace {

double two_pi_pow(int d) {
  double v = 1.0;
  for (int i = 0; i < d; ++i) v *= 2.0 * std::numbers::pi;
  return v;
}

// The device kernels implement the transform of the built-in backends; any
// other DftBackend (NaiveDftBackend, user subclasses) is honoured by running
// the reference's three-step structure through it.
bool fused_backend(const DftBackend& b) { return dynamic_cast<const CudaDftBackend*>(&b) != nullptr; }

// Real part x scale, with the reference's realness guard (synth.cpp:20-33):
// residue = max|Im| / max|Re| must stay <= 1e-10.
void take_real(std::span<const std::complex<double>> buf, double scale, RealField& field) {
  field.values.resize(buf.size());
  double re_max = 0.0, im_max = 0.0;
  for (std::size_t i = 0; i < buf.size(); ++i) {
    re_max = std::max(re_max, std::abs(buf[i].real()));
    im_max = std::max(im_max, std::abs(buf[i].imag()));
    field.values[i] = buf[i].real() * scale;
  }
  field.imag_residue = re_max > 0.0 ? im_max / re_max : im_max;
  if (field.imag_residue > 1e-10)
    throw std::runtime_error("synthesize: imaginary residue " + std::to_string(field.imag_residue) +
                             " exceeds 1e-10; spectrum lost Hermitian symmetry");
}

// Algorithms 1-3 with the transforms delegated to `backend` (synth.cpp:68-127):
//   two_fft   x (rng, real) -> forward -> x sqrt(g) sqrt((2 pi)^d P/|A|) -> inverse -> Re
//   one_fft   V (synthesize_spectrum_into) -> inverse -> Re x sqrt((2 pi)^d/|A|) P
RealField synthesize_through(const GridSpec& grid, const SpectralDensity& density, GaussianStream& rng,
                             Algorithm algorithm, DftBackend& backend) {
  const auto p = static_cast<std::size_t>(grid.point_count());
  const int d = grid.dim();
  RealField field{grid, {}, {algorithm, density.spec_string(), 0}, 0.0};
  aligned_vector<std::complex<double>> a(p), b(p);
  if (algorithm == Algorithm::two_fft) {
    for (auto& v : a) v = {rng.next(), 0.0};
    backend.forward(grid, a, b);
    // sqrt(g) over the half-lattice; g is even, so a cell past N_d/2 reads its mirror's value
    const std::vector<double> sg = detail::sqrt_gamma_table(grid, density);
    const double s = std::sqrt(two_pi_pow(d) * static_cast<double>(p) / grid.domain_volume());
    const auto& n = grid.counts();
    const std::int64_t hd = n[d - 1] / 2 + 1;
    for (std::size_t i = 0; i < p; ++i) {
      MultiIndex k = grid.index_at(static_cast<std::int64_t>(i));
      if (k[d - 1] > n[d - 1] / 2) k = neg_index(k, grid);
      std::int64_t h = 0;
      for (int ax = 0; ax < d - 1; ++ax) h = h * n[ax] + k[ax];
      h = h * hd + k[d - 1];
      b[i] *= sg[static_cast<std::size_t>(h)] * s;
    }
    backend.inverse(grid, b, a);
    take_real(a, 1.0, field);
    return field;
  }
  const SpectrumMode mode =
      algorithm == Algorithm::one_fft_overwrite ? SpectrumMode::overwrite : SpectrumMode::exact_set;
  synthesize_spectrum_into(grid, density, rng, mode, a);
  backend.inverse(grid, a, b);
  take_real(b, std::sqrt(two_pi_pow(d) / grid.domain_volume()) * static_cast<double>(p), field);
  return field;
}

}  // namespace

RealField synthesize(const GridSpec& grid, const SpectralDensity& density, GaussianStream& rng, Algorithm algorithm,
                     DftBackend& backend) {
  if (density.dim() != grid.dim()) throw std::invalid_argument("synthesize: density dimension mismatch");
  if (!fused_backend(backend)) return synthesize_through(grid, density, rng, algorithm, backend);
  RealField field{grid, {}, {algorithm, density.spec_string(), 0}, 0.0};
  std::vector<double> draws(count_draws(grid, algorithm));
  for (double& v : draws) v = rng.next();  // exhaustion propagates as the reference's
  auto plan = detail::make_plan(grid, density, static_cast<int>(algorithm));
  field.values.resize(static_cast<std::size_t>(grid.point_count()));
  detail::check(grfc_generate_injected_host(plan.get(), draws.data(), draws.size(), field.values.data()));
  return field;
}

std::vector<RealField> synthesize_batch(const GridSpec& grid, const SpectralDensity& density, std::uint64_t seed,
                                        std::uint64_t first_field, std::uint64_t count, Algorithm algorithm) {
  auto plan = detail::make_plan(grid, density, static_cast<int>(algorithm));
  const auto p = static_cast<std::size_t>(grid.point_count());
  std::vector<RealField> out;
  out.reserve(count);
  if (count == 1) {  // straight into the field's own storage
    RealField f{grid, std::vector<double>(p), {algorithm, density.spec_string(), seed}, 0.0};
    detail::check(grfc_generate_host(plan.get(), seed, first_field, 1, f.values.data(), nullptr));
    out.push_back(std::move(f));
    return out;
  }
  std::vector<double> all(p * count);
  if (count) detail::check(grfc_generate_host(plan.get(), seed, first_field, count, all.data(), nullptr));
  for (std::uint64_t i = 0; i < count; ++i) {
    RealField f{grid, std::vector<double>(all.begin() + i * p, all.begin() + (i + 1) * p),
                {algorithm, density.spec_string(), seed}, 0.0};
    out.push_back(std::move(f));
  }
  return out;
}

RealField synthesize(const GridSpec& grid, const SpectralDensity& density, std::uint64_t seed, Algorithm algorithm,
                     DftBackend& backend) {
  if (!fused_backend(backend)) {
    // same noise as the fused path: the device Philox stream of (seed, field 0),
    // replayed in the reference's draw order through the caller's backend
    if (density.dim() != grid.dim()) throw std::invalid_argument("synthesize: density dimension mismatch");
    auto plan = detail::make_plan(grid, density, static_cast<int>(algorithm));
    std::vector<double> draws(count_draws(grid, algorithm));
    detail::check(grfc_dump_noise(plan.get(), seed, 0, draws.data(), draws.size()));
    FixedStream rng(std::move(draws));
    RealField field = synthesize_through(grid, density, rng, algorithm, backend);
    field.provenance.seed = seed;
    return field;
  }
  auto fields = synthesize_batch(grid, density, seed, 0, 1, algorithm);
  return std::move(fields.front());
}

double exact_discrete_covariance(const GridSpec& grid, const SpectralDensity& density, const MultiIndex& lag) {
  if (!grid.valid_index(lag)) throw std::invalid_argument("exact_discrete_covariance: invalid lag");
  if (density.dim() != grid.dim()) throw std::invalid_argument("exact_discrete_covariance: density dimension mismatch");
  const int d = grid.dim();
  const auto& n = grid.counts();
  double acc = 0.0;
  for (std::int64_t i = 0; i < grid.point_count(); ++i) {
    const MultiIndex k = grid.index_at(i);
    double t = 0.0;  // sum_a (k_a lag_a mod N_a) / N_a, exact integer reduction
    for (int a = 0; a < d; ++a) t += static_cast<double>((k[a] * lag[a]) % n[a]) / static_cast<double>(n[a]);
    acc += density.eval(angular_frequency(k, grid)) * std::cos(2.0 * std::numbers::pi * t);
  }
  return acc * two_pi_pow(d) / grid.domain_volume();
}

double exact_discrete_covariance(const GridSpec& grid, const SpectralDensity& density,
                                 std::span<const double> physical_lag) {
  if (static_cast<int>(physical_lag.size()) != grid.dim())
    throw std::invalid_argument("exact_discrete_covariance: lag dimension mismatch");
  if (density.dim() != grid.dim()) throw std::invalid_argument("exact_discrete_covariance: density dimension mismatch");
  double acc = 0.0;
  for (std::int64_t i = 0; i < grid.point_count(); ++i) {
    const std::vector<double> w = angular_frequency(grid.index_at(i), grid);
    double phase = 0.0;
    for (int a = 0; a < grid.dim(); ++a) phase += w[a] * physical_lag[a];
    acc += density.eval(w) * std::cos(phase);
  }
  return acc * two_pi_pow(grid.dim()) / grid.domain_volume();
}

std::vector<double> exact_discrete_covariance_all(const GridSpec& grid, const SpectralDensity& density,
                                                  DftBackend& backend) {
  if (density.dim() != grid.dim())
    throw std::invalid_argument("exact_discrete_covariance_all: density dimension mismatch");
  if (!fused_backend(backend)) {
    // cov = Re inverse(g) x (2 pi)^d/|A| x P through the caller's backend (synth.cpp:188-209)
    const auto p = static_cast<std::size_t>(grid.point_count());
    aligned_vector<std::complex<double>> g(p), t(p);
    for (std::size_t i = 0; i < p; ++i)
      g[i] = {density.eval(angular_frequency(grid.index_at(static_cast<std::int64_t>(i)), grid)), 0.0};
    backend.inverse(grid, g, t);
    const double s = two_pi_pow(grid.dim()) / grid.domain_volume() * static_cast<double>(p);
    std::vector<double> cov(p);
    for (std::size_t i = 0; i < p; ++i) cov[i] = t[i].real() * s;
    return cov;
  }
  // cov(J) = (2 pi)^d/|A| sum_K g(w_K) e^{+i 2 pi K.J/N}: the device C2R of g
  // on the half-lattice. Driven through the synthesis path with a table of
  // g sqrt((2 pi)^d/|A|) (one factor sqrt((2 pi)^d/|A|) is applied on device)
  // and unit noise w == 1 (one draw 1 per self-conjugate cell, (sqrt 2, 0)
  // per paired cell, in the overwrite draw order).
  std::vector<double> t = detail::sqrt_gamma_table(grid, density);
  const double s = std::sqrt(two_pi_pow(grid.dim()) / grid.domain_volume());
  for (double& v : t) v = v * v * s;
  const grfc_density desc{GRFC_DENSITY_TABLE, grid.dim(), {}, {}};
  grfc_plan raw = nullptr;
  detail::check(grfc_plan_create(&raw, grid.dim(), grid.counts().data(), grid.lengths().data(), GRFC_F64,
                                 GRFC_ONE_FFT_OVERWRITE, &desc, 0));
  detail::PlanPtr plan(raw);
  detail::check(grfc_plan_set_sqrt_gamma_table(plan.get(), t.data()));
  const int d = grid.dim();
  const auto& n = grid.counts();
  std::vector<std::int64_t> ext(n.begin(), n.end());
  ext[d - 1] = n[d - 1] / 2 + 1;
  std::vector<double> draws;
  std::vector<std::int64_t> k(static_cast<std::size_t>(d), 0);
  for (std::size_t h = 0; h < t.size(); ++h) {
    bool self = true;
    for (int a = 0; a < d; ++a) self = self && (k[a] == 0 || 2 * k[a] == n[a]);
    if (self) {
      draws.push_back(1.0);
    } else {
      draws.push_back(std::numbers::sqrt2);
      draws.push_back(0.0);
    }
    for (int a = d - 1; a >= 0; --a) {
      if (++k[a] < ext[a]) break;
      k[a] = 0;
    }
  }
  std::vector<double> cov(static_cast<std::size_t>(grid.point_count()));
  detail::check(grfc_generate_injected_host(plan.get(), draws.data(), draws.size(), cov.data()));
  return cov;
}

}  // namespace grf
