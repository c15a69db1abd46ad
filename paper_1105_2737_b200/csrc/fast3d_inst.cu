// Instantiation of the fused 3D kernels for one (dtype, size) pair:
// pass A for N0 = INST_N, pass B for N1 = INST_N and every supported M.
#include "fast3d_launch.cuh"

namespace grfc {
template cudaError_t launch_3d_colgen<INST_T, INST_N, GRFC_ONE_FFT_OVERWRITE>(const Fast3D&, uint64_t, uint64_t, void*,
                                                                             int, int, cudaStream_t);
template cudaError_t launch_3d_colgen<INST_T, INST_N, GRFC_ONE_FFT_RECURSIVE>(const Fast3D&, uint64_t, uint64_t, void*,
                                                                             int, int, cudaStream_t);
#define GRFC_PLANES(M)                                                                                          \
  template cudaError_t launch_3d_planes<INST_T, INST_N, M>(const Fast3D&, const void*, int, int, void*, void*, \
                                                            cudaStream_t);                                     \
  template cudaError_t planes_query<INST_T, INST_N, M>(Fast3D&);
GRFC_PLANES(64)
GRFC_PLANES(128)
GRFC_PLANES(256)
GRFC_PLANES(512)
}  // namespace grfc
