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

// Grouped form for small grids: partial c (c < nchunks) of a run of samples
// that starts on a chunk boundary: out[c][K] = sum_{j in chunk c} f_j[ref] f_j[K]
// in ascending j — one thread per (chunk, point), so a whole group of chunks
// costs one launch and every partial keeps the single-chunk arithmetic.
template <typename T>
__global__ void __launch_bounds__(256) k_cov_accumulate_chunks(const T* __restrict__ fields, uint64_t nf,
                                                               uint64_t P, uint64_t ref, uint64_t chunk,
                                                               double* __restrict__ out) {
  const uint64_t nchunks = (nf + chunk - 1) / chunk, step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nchunks * P; w += step) {
    const uint64_t c = w / P, i = w - c * P;
    const uint64_t j0 = c * chunk, j1 = j0 + chunk < nf ? j0 + chunk : nf;
    double a = 0.0;
    const T* f = fields + j0 * P;
#pragma unroll 4
    for (uint64_t j = j0; j < j1; ++j, f += P) a = __dadd_rn(a, __dmul_rn((double)__ldg(f + ref), (double)f[i]));
    out[c * P + i] = a;
  }
}

// Kahan merge of `nchunks` consecutive partials into (est, comp), in chunk order
// per point — the same sequence of steps as nchunks calls of k_cov_merge.
__global__ void __launch_bounds__(256) k_cov_merge_chunks(const double* __restrict__ part, uint64_t nchunks,
                                                          double* __restrict__ est, double* __restrict__ comp,
                                                          uint64_t P) {
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += step) {
    double e = est[i], k = comp[i];
    for (uint64_t c = 0; c < nchunks; ++c) {
      const double y = __dsub_rn(part[c * P + i], k);
      const double t = __dadd_rn(e, y);
      k = __dsub_rn(__dsub_rn(t, e), y);
      e = t;
    }
    est[i] = e;
    comp[i] = k;
  }
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

cudaError_t launch_cov_accumulate_chunks(int dtype, const void* fields, uint64_t nf, uint64_t P, uint64_t ref,
                                         uint64_t chunk, double* out, cudaStream_t s) {
  if (nf == 0) return cudaSuccess;
  const uint64_t work = (nf + chunk - 1) / chunk * P;
  LaunchScope ls("cov_accumulate_chunks", s);
  if (dtype == GRFC_F64)
    k_cov_accumulate_chunks<double><<<cov_grid(work), 256, 0, s>>>((const double*)fields, nf, P, ref, chunk, out);
  else
    k_cov_accumulate_chunks<float><<<cov_grid(work), 256, 0, s>>>((const float*)fields, nf, P, ref, chunk, out);
  return cudaGetLastError();
}

cudaError_t launch_cov_merge_chunks(const double* part, uint64_t nchunks, double* est, double* comp, uint64_t P,
                                    cudaStream_t s) {
  LaunchScope ls("cov_merge_chunks", s);
  k_cov_merge_chunks<<<cov_grid(P), 256, 0, s>>>(part, nchunks, est, comp, P);
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
