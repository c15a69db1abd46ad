// Launcher declarations shared by the C-ABI (api.cu) and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "grfc_internal.cuh"

namespace grfc {

// Radix sequence of a line length (8s, then 4, 2, then odd primes).
struct Factors {
  int nf;
  int r[40];
};

template <typename T>
cudaError_t launch_gen_half(const GridDesc& g, const DensityDesc& D, int alg, double scale, uint64_t seed,
                            uint64_t field0, const double2* injected, void* W, int64_t nfields, cudaStream_t s);
template <typename T>
cudaError_t launch_scale_half(const GridDesc& g, const DensityDesc& D, double scale, void* W, int64_t nfields,
                              cudaStream_t s);
template <typename T>
cudaError_t launch_line_c2c(void* data, int n, int64_t inner, int64_t outer, int sign, const Factors& F,
                            const void* tw, cudaStream_t s);
template <typename T>
cudaError_t launch_c2r_last(const void* W, void* out, int n, int64_t rows, int64_t rows_per_field,
                            int64_t out_field_stride, int conj, const Factors& FM, const void* twN, cudaStream_t s);
template <typename T>
cudaError_t launch_r2c_last_noise(void* W, int n, int64_t rows, int64_t rows_per_field, uint64_t seed,
                                  uint64_t field0, const double* injected, const Factors& FM, const void* twN,
                                  cudaStream_t s);
template <typename T>
cudaError_t launch_scale_all(void* data, int64_t n, double sc, cudaStream_t s);
template <typename T>
cudaError_t launch_philox_pairs(const uint64_t* units, int64_t n, uint64_t Uh, uint64_t seed, uint64_t field,
                                double* out, cudaStream_t s);

// Lines longer than the on-chip kernels hold (long_fft.cu): four-step / Bluestein
// through global memory; same conventions as launch_line_c2c / c2r_last /
// r2c_last_noise (twiddle tables cached per length).
// true when a line of n complex (elem_bytes each) needs long_c2c: too long for one
// CTA, or a prime factor above the on-chip direct-sum limit
bool needs_long_line(int64_t n, size_t elem_bytes);
template <typename T>
cudaError_t long_c2c(void* data, int64_t n, int64_t inner, int64_t outer, int sign, cudaStream_t s);
template <typename T>
cudaError_t long_c2r_last(const void* W, void* out, int64_t n, int64_t rows, int64_t rows_per_field,
                          int64_t out_field_stride, int conj, cudaStream_t s);
template <typename T>
cudaError_t long_r2c_last_noise(void* W, int64_t n, int64_t rows, int64_t rows_per_field, uint64_t seed,
                                uint64_t field0, const double* injected, cudaStream_t s);

// Covariance estimator kernels (stats.cu).
cudaError_t launch_cov_accumulate(int dtype, const void* fields, uint64_t nf, uint64_t stride, uint64_t P,
                                  uint64_t ref, double* acc, cudaStream_t s);
cudaError_t launch_cov_merge(const double* acc, double* est, double* comp, uint64_t P, cudaStream_t s);
cudaError_t launch_cov_accumulate_chunks(int dtype, const void* fields, uint64_t nf, uint64_t P, uint64_t ref,
                                         uint64_t chunk, double* out, cudaStream_t s);
cudaError_t launch_cov_merge_chunks(const double* part, uint64_t nchunks, double* est, double* comp, uint64_t P,
                                    cudaStream_t s);
cudaError_t launch_cov_scale(double* est, uint64_t P, double inv_m, cudaStream_t s);

}  // namespace grfc
