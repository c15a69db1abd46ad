// The DftBackend classes of the drop-in, executed on the GPU through the C-ABI
// (fast: grfc_dft_c2c_host; naive: grfc_dft_naive_c2c_host).
#include "grf/dft.hpp"

#include <stdexcept>

#include "grfc_cpp.hpp"

namespace grf {

namespace {

using Entry = grfc_status (*)(int, const int64_t*, const double*, double*, int, int);

void run_transform(Entry fn, const GridSpec& grid, std::span<const std::complex<double>> in,
                   std::span<std::complex<double>> out, int sign, int device) {
  const auto p = static_cast<std::size_t>(grid.point_count());
  if (in.size() != p || out.size() != p) throw std::invalid_argument("DftBackend: buffer size does not match grid");
  if (in.data() == out.data()) throw std::invalid_argument("DftBackend: in-place transform not supported");
  detail::check(fn(grid.dim(), grid.counts().data(), reinterpret_cast<const double*>(in.data()),
                   reinterpret_cast<double*>(out.data()), sign, device));
}

}  // namespace

void CudaDftBackend::forward(const GridSpec& grid, std::span<const std::complex<double>> in,
                             std::span<std::complex<double>> out) {
  run_transform(grfc_dft_c2c_host, grid, in, out, +1, device_);
}

void CudaDftBackend::inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
                             std::span<std::complex<double>> out) {
  run_transform(grfc_dft_c2c_host, grid, in, out, -1, device_);
}

void NaiveDftBackend::forward(const GridSpec& grid, std::span<const std::complex<double>> in,
                              std::span<std::complex<double>> out) {
  run_transform(grfc_dft_naive_c2c_host, grid, in, out, +1, 0);
}

void NaiveDftBackend::inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
                              std::span<std::complex<double>> out) {
  run_transform(grfc_dft_naive_c2c_host, grid, in, out, -1, 0);
}

DftBackend& default_backend() {
  static FftwBackend backend;
  return backend;
}

}  // namespace grf
