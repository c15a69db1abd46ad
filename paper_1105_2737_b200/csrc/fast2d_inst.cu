// Explicit instantiation of the fused pow2 2D kernels for one (dtype, column
// length N1) pair; the Makefile compiles this file once per pair with
// -DINST_T=<float|double> -DINST_N=<N1> so the objects build in parallel.
// Rows are instantiated for M = N1/2 (covers every supported N2 = 2M).
#include "fast2d_alg1.cuh"

namespace grfc {
template cudaError_t launch_cols<INST_T, INST_N, GRFC_ONE_FFT_OVERWRITE>(const Fast2D&, uint64_t, uint64_t, int64_t,
                                                                        void*, cudaStream_t);
template cudaError_t launch_cols<INST_T, INST_N, GRFC_ONE_FFT_RECURSIVE>(const Fast2D&, uint64_t, uint64_t, int64_t,
                                                                        void*, cudaStream_t);
template cudaError_t launch_rows<INST_T, INST_N / 2>(const Fast2D&, int64_t, const void*, void*, int64_t,
                                                    cudaStream_t);
#define GRFC_FUSED(M)                                                                                    \
  template cudaError_t launch_fused<INST_T, INST_N, M, GRFC_ONE_FFT_OVERWRITE>(                                \
      const Fast2D&, uint64_t, uint64_t, int64_t, void*, void*, int64_t, cudaStream_t, const void*);           \
  template cudaError_t fused_query<INST_T, INST_N, M, GRFC_ONE_FFT_OVERWRITE>(Fast2D&);                         \
  template cudaError_t launch_cluster<INST_T, INST_N, M>(const Fast2D&, uint64_t, uint64_t, int64_t, void*, void*,   \
                                                         int64_t, cudaStream_t);                                    \
  template cudaError_t cluster_query<INST_T, INST_N, M>(Fast2D&, int, int);
GRFC_FUSED(128)
GRFC_FUSED(256)
GRFC_FUSED(512)
GRFC_FUSED(1024)
GRFC_FUSED(2048)
// fp64: the fused kernel over a preloaded X (kPreX, small batches: c1)
#if INST_T_IS_DOUBLE
#define GRFC_FUSED_PRE(M)                                                                                      \
  template cudaError_t launch_fused<double, INST_N, M, kPreX>(const Fast2D&, uint64_t, uint64_t, int64_t, void*,  \
                                                              void*, int64_t, cudaStream_t, const void*);
GRFC_FUSED_PRE(128)
GRFC_FUSED_PRE(256)
GRFC_FUSED_PRE(512)
GRFC_FUSED_PRE(1024)
GRFC_FUSED_PRE(2048)
#endif
// Algorithm 1 (three-tile persistent kernel): every (N1, M) whose row tiles hold
// an even number of rows (alg1_valid); the others return cudaErrorNotSupported.
#define GRFC_ALG1(M)                                                                                            \
  template cudaError_t launch_fused_alg1<INST_T, INST_N, M>(const Fast2D&, uint64_t, uint64_t, int64_t, void*,   \
                                                             int64_t, cudaStream_t);                             \
  template cudaError_t alg1_check<INST_T, INST_N, M>();
GRFC_ALG1(128)
GRFC_ALG1(256)
GRFC_ALG1(512)
GRFC_ALG1(1024)
GRFC_ALG1(2048)
}  // namespace grfc
