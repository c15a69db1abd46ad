// Monte-Carlo covariance kernels: the device form of grf::estimate_covariance
// (/root/reference/proj/core/src/stats.cpp:39-97).
//
// Determinism contract (stats.cpp:17-18, 60-93): samples are grouped in fixed
// chunks of GRFC_COV_CHUNK; within a chunk every grid point K accumulates
//   acc[K] = sum_j f_j[ref] * f_j[K]
// in fp64, in ascending sample order, as a separate multiply and add (the
// reference's `acc[i] += at_ref * field.values[i]`); chunk partials are merged
// in chunk order with Kahan compensation and the sum is scaled by 1/M. The
// thread layout, the generation batch size and the number of devices never
// change a result bit.
//
// Layout: fields of the plan's dtype, field j at fields + j*stride; acc, est,
// comp: P doubles. One thread per grid point (grid-stride), so each load of
// f_j[K] is coalesced across the warp and f_j[ref] is a warp-wide broadcast.
// The accumulation is HBM-bound: nf * P * s bytes read per launch.
#include "grfc_internal.cuh"
#include "kernels.h"

namespace grfc {

template <typename T>
__global__ void __launch_bounds__(256) k_cov_accumulate(const T* __restrict__ fields, uint64_t nf, uint64_t stride,
                                                        uint64_t P, uint64_t ref, double* __restrict__ acc) {
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += step) {
    double a = acc[i];
    const T* f = fields;
#pragma unroll 8
    for (uint64_t j = 0; j < nf; ++j, f += stride) {
      const double r = (double)__ldg(f + ref);
      a = __dadd_rn(a, __dmul_rn(r, (double)__ldcs(f + i)));
    }
    acc[i] = a;
  }
}

// One Kahan step of the chunk-ordered merge (stats.cpp:84-91).
__global__ void __launch_bounds__(256) k_cov_merge(const double* __restrict__ acc, double* __restrict__ est,
                                                   double* __restrict__ comp, uint64_t P) {
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += step) {
    const double e = est[i];
    const double y = __dsub_rn(acc[i], comp[i]);
    const double t = __dadd_rn(e, y);
    comp[i] = __dsub_rn(__dsub_rn(t, e), y);
    est[i] = t;
  }
}

__global__ void __launch_bounds__(256) k_cov_scale(double* __restrict__ est, uint64_t P, double inv_m) {
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += step) est[i] = __dmul_rn(est[i], inv_m);
}

static unsigned cov_grid(uint64_t P) {
  const uint64_t b = (P + 255) / 256;
  return (unsigned)(b < 148ull * 16 ? (b ? b : 1) : 148ull * 16);
}

cudaError_t launch_cov_accumulate(int dtype, const void* fields, uint64_t nf, uint64_t stride, uint64_t P,
                                  uint64_t ref, double* acc, cudaStream_t s) {
  if (nf == 0) return cudaSuccess;
  LaunchScope ls("cov_accumulate", s);
  if (dtype == GRFC_F64)
    k_cov_accumulate<double><<<cov_grid(P), 256, 0, s>>>((const double*)fields, nf, stride, P, ref, acc);
  else
    k_cov_accumulate<float><<<cov_grid(P), 256, 0, s>>>((const float*)fields, nf, stride, P, ref, acc);
  return cudaGetLastError();
}

cudaError_t launch_cov_merge(const double* acc, double* est, double* comp, uint64_t P, cudaStream_t s) {
  LaunchScope ls("cov_merge", s);
  k_cov_merge<<<cov_grid(P), 256, 0, s>>>(acc, est, comp, P);
  return cudaGetLastError();
}

cudaError_t launch_cov_scale(double* est, uint64_t P, double inv_m, cudaStream_t s) {
  LaunchScope ls("cov_scale", s);
  k_cov_scale<<<cov_grid(P), 256, 0, s>>>(est, P, inv_m);
  return cudaGetLastError();
}

}  // namespace grfc
