// Fused power-of-two 2D fast path (placeholder until the fused kernels land:
// every shape routes to the generic kernels).
#include "fast2d.h"

namespace grfc {

bool fast2d_supported(int, const int64_t*, int, int, int) { return false; }
cudaError_t fast2d_init(Fast2D&, const GridDesc&, const DensityDesc&, int, int, double, double) {
  return cudaErrorNotSupported;
}
void fast2d_free(Fast2D&) {}
const char* fast2d_name(const Fast2D&) { return "generic"; }
cudaError_t launch_fast2d(const Fast2D&, int, uint64_t, uint64_t, int64_t, void*, void*, int64_t, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace grfc
