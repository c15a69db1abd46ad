// grf:: statistics of the drop-in over the grfc C-ABI. Semantics follow the
// reference's src/stats.cpp (lines cited per function); the estimator's
// arithmetic (chunks of GRFC_COV_CHUNK samples, fp64 ordered accumulation,
// chunk-ordered Kahan merge, x 1/M) runs on the device.
#include "grf/stats.hpp"

#include <cmath>
#include <cstdlib>
#include <numeric>
#include <numbers>
#include <stdexcept>
#include <thread>

#include "grf/spectral.hpp"
#include "grfc_cpp.hpp"

namespace grf {

namespace {

// Disjoint per-level seeds: splitmix64 finalizer over (seed, level) (stats.cpp:20-26).
std::uint64_t level_seed(std::uint64_t seed, int level) {
  std::uint64_t z = seed ^ (0xD1B54A32D192ED03ull * static_cast<std::uint64_t>(level + 1));
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void check_args(const GridSpec& grid, const SpectralDensity& density, std::uint64_t samples,
                const MultiIndex& reference) {
  if (samples < 1) throw std::invalid_argument("estimate_covariance: need at least one sample");
  if (!grid.valid_index(reference)) throw std::invalid_argument("estimate_covariance: reference index out of range");
  if (density.dim() != grid.dim()) throw std::invalid_argument("synthesize: density dimension mismatch");
}

}  // namespace

int resolve_threads(int requested) {  // stats.cpp:29-37
  if (requested > 0) return requested;
  if (const char* env = std::getenv("GRF_THREADS")) {
    const int v = std::atoi(env);
    if (v > 0) return v;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

CovarianceEstimate estimate_covariance(const GridSpec& grid, const SpectralDensity& density, Algorithm algorithm,
                                       std::uint64_t samples, const MultiIndex& reference, std::uint64_t seed,
                                       int /*threads*/, DftBackend& /*backend*/) {
  check_args(grid, density, samples, reference);
  auto plan = detail::make_plan(grid, density, static_cast<int>(algorithm));
  CovarianceEstimate est{grid, reference, std::vector<double>(static_cast<std::size_t>(grid.point_count())), samples,
                         seed};
  detail::check(grfc_estimate_covariance_host(plan.get(), seed, samples, grid.linear_index(reference),
                                              est.estimates.data()));
  return est;
}

CovarianceEstimate estimate_covariance(const GridSpec& grid, const SpectralDensity& density, Algorithm algorithm,
                                       std::uint64_t samples, const MultiIndex& reference,
                                       const StreamFactory& streams, int /*threads*/, DftBackend& /*backend*/) {
  check_args(grid, density, samples, reference);
  auto plan = detail::make_plan(grid, density, static_cast<int>(algorithm));
  const std::size_t p = static_cast<std::size_t>(grid.point_count());
  const std::uint64_t nd = count_draws(grid, algorithm);
  const std::int64_t ref = grid.linear_index(reference);
  CovarianceEstimate est{grid, reference, std::vector<double>(p, 0.0), samples, 0};
  std::vector<double> comp(p, 0.0), part(p), draws;
  for (std::uint64_t begin = 0; begin < samples; begin += GRFC_COV_CHUNK) {
    const std::uint64_t end = std::min<std::uint64_t>(begin + GRFC_COV_CHUNK, samples);
    draws.resize(static_cast<std::size_t>((end - begin) * nd));
    double* d = draws.data();
    for (std::uint64_t j = begin; j < end; ++j) {
      const std::unique_ptr<GaussianStream> rng = streams(j);
      for (std::uint64_t i = 0; i < nd; ++i) *d++ = rng->next();  // exhaustion propagates
    }
    detail::check(grfc_covariance_chunk_injected_host(plan.get(), draws.data(), end - begin, nd, ref, part.data()));
    for (std::size_t i = 0; i < p; ++i) {  // chunk-ordered Kahan merge (stats.cpp:84-91)
      const double y = part[i] - comp[i];
      const double t = est.estimates[i] + y;
      comp[i] = (t - est.estimates[i]) - y;
      est.estimates[i] = t;
    }
  }
  const double inv_m = 1.0 / static_cast<double>(samples);
  for (double& v : est.estimates) v *= inv_m;
  return est;
}

double max_error(const CovarianceEstimate& estimate, const std::function<double(std::span<const double>)>& oracle) {
  double err = 0.0;  // stats.cpp:111-119
  for (std::int64_t i = 0; i < estimate.grid.point_count(); ++i) {
    const std::vector<double> x = estimate.grid.point(estimate.grid.index_at(i));
    err = std::max(err, std::abs(estimate.estimates[static_cast<std::size_t>(i)] - oracle(x)));
  }
  return err;
}

std::optional<double> fit_slope(std::span<const double> x, std::span<const double> y) {
  // ordinary least squares about the means (stats.cpp:121-139 semantics)
  if (x.size() < 2 || y.size() != x.size()) return std::nullopt;
  const auto mean = [](std::span<const double> v) {
    return std::accumulate(v.begin(), v.end(), 0.0) / static_cast<double>(v.size());
  };
  const double xbar = mean(x), ybar = mean(y);
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    const double dx = x[i] - xbar;
    num += dx * (y[i] - ybar);
    den += dx * dx;
  }
  return den == 0.0 ? std::nullopt : std::optional<double>(num / den);
}

ConvergenceReport convergence_study(int level_min, int level_max, std::uint64_t samples, Algorithm algorithm,
                                    std::uint64_t seed, int threads, DftBackend& backend) {
  // stats.cpp:141-174: one device estimate per level against the closed form
  const bool ok = level_min >= 2 && level_max <= 12 && level_min <= level_max;
  if (!ok) throw std::invalid_argument("convergence_study: levels must lie within 2..12");
  const Test1dDensity test1d;
  const auto exact = [](std::span<const double> x) { return closed_form_c1d(std::abs(x[0])); };
  ConvergenceReport out;
  const double mc = 2.0 / std::sqrt(static_cast<double>(samples));
  std::vector<double> log_cells, log_err;
  for (int level = level_min; level <= level_max; ++level) {
    const std::int64_t n = std::int64_t{1} << level;
    // [-pi, pi) with n cells; the grid point n/2 sits at x = 0
    const GridSpec line({2.0 * std::numbers::pi}, {n}, {-std::numbers::pi});
    const double e = max_error(estimate_covariance(line, test1d, algorithm, samples, MultiIndex{n / 2},
                                                   level_seed(seed, level), threads, backend),
                               exact);
    out.rows.push_back(ConvergenceRow{level, n, e, mc});
    if (e > 3.0 * mc) {
      log_cells.push_back(static_cast<double>(level));  // log2(2^level)
      log_err.push_back(std::log2(e));
      out.fitted_levels.push_back(level);
    }
  }
  out.fitted_slope = fit_slope(log_cells, log_err);
  if (!out.fitted_slope) out.fitted_levels.clear();
  return out;
}

}  // namespace grf
