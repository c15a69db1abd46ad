// grf::DftBackend family — drop-in for the reference's include/grf/dft.hpp:9-67.
// Contract (unchanged):
//   forward: out[K] = sum_J in[J] exp(+2 pi i K.J/N)
//   inverse: out[J] = P^{-1} sum_K in[K] exp(-2 pi i K.J/N)
// Out-of-place, P row-major entries in and out.
//
// Every backend here executes on the GPU through the grfc C-ABI:
//   FftwBackend      the fast transform (grfc_dft_c2c_host: mixed-radix Stockham
//                    kernels). The reference's FFTW-backed class name, kept so
//                    its callers compile unchanged; PlanRigor is accepted (device
//                    plans are deterministic for both rigors).
//   NaiveDftBackend  the literal O(P^2) sums (grfc_dft_naive_c2c_host), the
//                    cross-check of the fast transform on small grids.
//   CudaDftBackend   FftwBackend on a chosen device.
// grf::synthesize runs its own fused kernels when handed the default backend,
// an FftwBackend or a CudaDftBackend, and routes its transforms through the
// given backend otherwise (NaiveDftBackend, user subclasses), as the
// reference's synthesize does (synth.cpp:68-127).
#pragma once

#include <complex>
#include <span>
#include <string>

#include "grf/grid.hpp"

namespace grf {

class DftBackend {
 public:
  virtual ~DftBackend() = default;
  virtual void forward(const GridSpec& grid, std::span<const std::complex<double>> in,
                       std::span<std::complex<double>> out) = 0;
  virtual void inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
                       std::span<std::complex<double>> out) = 0;
  virtual std::string name() const = 0;
};

/// Planner effort (reference dft.hpp:27-31). Both map to the same
/// deterministic device plans.
enum class PlanRigor { estimate, measure };

/// Device fp64 complex DFT on `device` (host buffers in/out). Thread-safe.
class CudaDftBackend : public DftBackend {
 public:
  explicit CudaDftBackend(int device = 0) : device_(device) {}
  void forward(const GridSpec& grid, std::span<const std::complex<double>> in,
               std::span<std::complex<double>> out) override;
  void inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
               std::span<std::complex<double>> out) override;
  std::string name() const override { return "cuda"; }
  int device() const { return device_; }

 private:
  int device_;
};

/// The reference's fast backend class (dft.hpp:33-52), on device 0.
class FftwBackend final : public CudaDftBackend {
 public:
  explicit FftwBackend(PlanRigor rigor = PlanRigor::estimate) : CudaDftBackend(0), rigor_(rigor) {}
  FftwBackend(const FftwBackend&) = delete;
  FftwBackend& operator=(const FftwBackend&) = delete;
  std::string name() const override { return "fftw"; }
  PlanRigor rigor() const { return rigor_; }

 private:
  PlanRigor rigor_;
};

/// Literal O(P^2) sums (dft.hpp:54-64) on the device.
class NaiveDftBackend final : public DftBackend {
 public:
  void forward(const GridSpec& grid, std::span<const std::complex<double>> in,
               std::span<std::complex<double>> out) override;
  void inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
               std::span<std::complex<double>> out) override;
  std::string name() const override { return "naive"; }
};

/// Process-wide fast backend (an FftwBackend, as the reference's).
DftBackend& default_backend();

}  // namespace grf
