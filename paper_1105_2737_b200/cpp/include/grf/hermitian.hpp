// grf Hermitian-spectrum helpers — drop-in for the reference's
// include/grf/hermitian.hpp (host-side utilities; the generator assembles its
// spectrum on the device).
#pragma once

#include <complex>
#include <cstdint>
#include <functional>
#include <span>
#include <vector>

#include "grf/aligned.hpp"
#include "grf/grid.hpp"
#include "grf/random.hpp"
#include "grf/spectral.hpp"

namespace grf {

struct ConjugateRepSet {
  GridSpec grid;
  std::vector<MultiIndex> reps;            // L0 first, then the Appendix blocks
  std::vector<MultiIndex> self_conjugate;  // the 2^d entries of L0
};

/// Representative set in the paper-Appendix order (the Alg-3 draw order).
ConjugateRepSet build_conjugate_reps(const GridSpec& grid);
void for_each_conjugate_rep(const GridSpec& grid, const std::function<void(const MultiIndex&, bool)>& fn);

struct HermitianSpectrum {
  GridSpec grid;
  aligned_vector<std::complex<double>> values;  // P entries, row-major (hermitian.hpp:48)
};

enum class SpectrumMode { exact_set, overwrite };

/// V(K) = sqrt(g(w_K)) w(K) on the full lattice from draws pulled from rng.
HermitianSpectrum synthesize_spectrum(const GridSpec& grid, const SpectralDensity& density, GaussianStream& rng,
                                      SpectrumMode mode);
/// Allocation-free form (reference hermitian.hpp:66-70): writes all P entries
/// of out; std::invalid_argument when out.size() != P.
void synthesize_spectrum_into(const GridSpec& grid, const SpectralDensity& density, GaussianStream& rng,
                              SpectrumMode mode, std::span<std::complex<double>> out);
bool verify_hermitian(const HermitianSpectrum& spectrum);
std::uint64_t spectrum_draw_count(const GridSpec& grid, SpectrumMode mode);

}  // namespace grf
