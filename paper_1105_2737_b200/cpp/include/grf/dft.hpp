// grf::DftBackend — drop-in for the reference's include/grf/dft.hpp contract:
//   forward: out[K] = sum_J in[J] exp(+2 pi i K.J/N)
//   inverse: out[J] = P^{-1} sum_K in[K] exp(-2 pi i K.J/N)
// CudaDftBackend executes it on the GPU (grfc_dft_c2c). grf::synthesize does
// not route through a DftBackend: its transforms are fused with generation.
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

/// Device fp64 complex DFT (host buffers in/out). Thread-safe.
class CudaDftBackend final : public DftBackend {
 public:
  explicit CudaDftBackend(int device = 0) : device_(device) {}
  void forward(const GridSpec& grid, std::span<const std::complex<double>> in,
               std::span<std::complex<double>> out) override;
  void inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
               std::span<std::complex<double>> out) override;
  std::string name() const override { return "cuda"; }
  int device() const { return device_; }

 private:
  void run(const GridSpec& grid, std::span<const std::complex<double>> in, std::span<std::complex<double>> out,
           int sign);
  int device_;
};

/// Process-wide CUDA backend (device 0).
DftBackend& default_backend();

}  // namespace grf
