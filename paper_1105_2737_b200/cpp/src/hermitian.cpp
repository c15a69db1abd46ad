// Host-side Hermitian-spectrum utilities of the drop-in. The representative
// set and the noise arrangement come from the C-ABI (the same host code the
// device path's injected mode uses), so the draw order is shared.
#include "grf/hermitian.hpp"

#include <cmath>
#include <numbers>
#include <stdexcept>

#include "grfc_cpp.hpp"

namespace grf {

void for_each_conjugate_rep(const GridSpec& grid, const std::function<void(const MultiIndex&, bool)>& fn) {
  std::uint64_t n = 0;
  detail::check(grfc_conjugate_reps(grid.dim(), grid.counts().data(), nullptr, nullptr, 0, &n));
  std::vector<std::int64_t> lin(n);
  std::vector<std::uint8_t> self(n);
  detail::check(grfc_conjugate_reps(grid.dim(), grid.counts().data(), lin.data(), self.data(), n, &n));
  for (std::uint64_t i = 0; i < n; ++i) fn(grid.index_at(lin[i]), self[i] != 0);
}

ConjugateRepSet build_conjugate_reps(const GridSpec& grid) {
  ConjugateRepSet set{grid, {}, {}};
  for_each_conjugate_rep(grid, [&](const MultiIndex& k, bool self) {
    set.reps.push_back(k);
    if (self) set.self_conjugate.push_back(k);
  });
  return set;
}

std::uint64_t spectrum_draw_count(const GridSpec& grid, SpectrumMode mode) {
  std::uint64_t n = 0;
  detail::check(grfc_count_draws(grid.dim(), grid.counts().data(),
                                 mode == SpectrumMode::overwrite ? GRFC_ONE_FFT_OVERWRITE : GRFC_ONE_FFT_RECURSIVE, &n));
  return n;
}

void synthesize_spectrum_into(const GridSpec& grid, const SpectralDensity& density, GaussianStream& rng,
                              SpectrumMode mode, std::span<std::complex<double>> out) {
  if (density.dim() != grid.dim()) throw std::invalid_argument("synthesize_spectrum: density dimension mismatch");
  if (out.size() != static_cast<std::size_t>(grid.point_count()))
    throw std::invalid_argument("synthesize_spectrum: buffer size does not match grid");
  const int alg = mode == SpectrumMode::overwrite ? GRFC_ONE_FFT_OVERWRITE : GRFC_ONE_FFT_RECURSIVE;
  std::vector<double> draws(spectrum_draw_count(grid, mode));
  for (double& v : draws) v = rng.next();
  const std::vector<double> sg = detail::sqrt_gamma_table(grid, density);
  std::vector<double> w(2 * sg.size());
  detail::check(grfc_half_noise_from_draws(grid.dim(), grid.counts().data(), alg, draws.data(), draws.size(),
                                           w.data()));
  const int d = grid.dim();
  const auto& n = grid.counts();
  const std::int64_t hd = n[d - 1] / 2 + 1;
  // H cells directly; the rest by V(-K) = conj V(K).
  for (std::int64_t lin = 0; lin < grid.point_count(); ++lin) {
    MultiIndex k = grid.index_at(lin);
    bool conj = false;
    if (k[d - 1] > n[d - 1] / 2) {
      k = neg_index(k, grid);
      conj = true;
    }
    std::int64_t h = 0;
    for (int a = 0; a < d - 1; ++a) h = h * n[a] + k[a];
    h = h * hd + k[d - 1];
    const double g = sg[static_cast<std::size_t>(h)];
    const std::complex<double> v(g * w[2 * h], g * w[2 * h + 1]);
    out[static_cast<std::size_t>(lin)] = conj ? std::conj(v) : v;
  }
}

HermitianSpectrum synthesize_spectrum(const GridSpec& grid, const SpectralDensity& density, GaussianStream& rng,
                                      SpectrumMode mode) {
  HermitianSpectrum out{grid, aligned_vector<std::complex<double>>(static_cast<std::size_t>(grid.point_count()))};
  synthesize_spectrum_into(grid, density, rng, mode, out.values);
  return out;
}

bool verify_hermitian(const HermitianSpectrum& s) {
  const GridSpec& grid = s.grid;
  if (s.values.size() != static_cast<std::size_t>(grid.point_count())) return false;
  for (std::int64_t i = 0; i < grid.point_count(); ++i) {
    const std::int64_t j = grid.linear_index(neg_index(grid.index_at(i), grid));
    const auto v = s.values[static_cast<std::size_t>(i)], u = s.values[static_cast<std::size_t>(j)];
    if (u.real() != v.real() || u.imag() != -v.imag()) return false;
    if (i == j && v.imag() != 0.0) return false;
  }
  return true;
}

}  // namespace grf
