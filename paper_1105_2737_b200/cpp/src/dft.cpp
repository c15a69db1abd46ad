// CudaDftBackend: the reference DftBackend contract on the device.
#include "grf/dft.hpp"

#include <stdexcept>

#include "grfc_cpp.hpp"

namespace grf {

void CudaDftBackend::run(const GridSpec& grid, std::span<const std::complex<double>> in,
                         std::span<std::complex<double>> out, int sign) {
  const auto p = static_cast<std::size_t>(grid.point_count());
  if (in.size() != p || out.size() != p) throw std::invalid_argument("DftBackend: buffer size does not match grid");
  if (in.data() == out.data()) throw std::invalid_argument("DftBackend: in-place transform not supported");
  detail::check(grfc_dft_c2c_host(grid.dim(), grid.counts().data(), reinterpret_cast<const double*>(in.data()),
                                  reinterpret_cast<double*>(out.data()), sign, device_));
}

void CudaDftBackend::forward(const GridSpec& grid, std::span<const std::complex<double>> in,
                             std::span<std::complex<double>> out) {
  run(grid, in, out, +1);
}

void CudaDftBackend::inverse(const GridSpec& grid, std::span<const std::complex<double>> in,
                             std::span<std::complex<double>> out) {
  run(grid, in, out, -1);
}

DftBackend& default_backend() {
  static CudaDftBackend backend(0);
  return backend;
}

}  // namespace grf
