// Host side of the fused pow2 2D path: plan setup and dispatch. The kernels
// live in fast2d_kernels.cuh and are instantiated per (dtype, size) by
// fast2d_inst.cu (one object per combination, compiled in parallel).
#include <cmath>
#include <vector>

#include "fast2d.h"
#include "grfc_internal.cuh"

namespace grfc {

struct F2Params;
template <typename T, int N1, int ALG>
cudaError_t launch_cols(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W, cudaStream_t s);
template <typename T, int M>
cudaError_t launch_rows(const Fast2D& f, int64_t nf, const void* W, void* out, int64_t stride, cudaStream_t s);

static bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

bool fast2d_supported(int d, const int64_t* n, int dtype, int alg, int family) {
  (void)dtype;
  (void)family;
  if (d != 2 || alg == GRFC_TWO_FFT) return false;
  if (!is_pow2(n[0]) || !is_pow2(n[1])) return false;
  return n[0] >= 256 && n[0] <= 4096 && n[1] >= 256 && n[1] <= 4096;
}

const char* fast2d_name(const Fast2D& f) { return f.dtype == GRFC_F64 ? "pow2-2d-f64" : "pow2-2d-f32"; }

template <typename T>
static std::vector<C_t<T>> host_twiddles(int64_t n) {
  std::vector<C_t<T>> t((size_t)n);
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int64_t m = 0; m < n; ++m) {
    const long double a = two_pi * (long double)m / (long double)n;
    t[(size_t)m].x = (T)cosl(a);
    t[(size_t)m].y = (T)sinl(a);
  }
  return t;
}

template <typename T, int ALG>
static cudaError_t dispatch_cols(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W,
                                 cudaStream_t s) {
  switch (f.n1) {
    case 256: return launch_cols<T, 256, ALG>(f, seed, field0, nf, W, s);
    case 512: return launch_cols<T, 512, ALG>(f, seed, field0, nf, W, s);
    case 1024: return launch_cols<T, 1024, ALG>(f, seed, field0, nf, W, s);
    case 2048: return launch_cols<T, 2048, ALG>(f, seed, field0, nf, W, s);
    case 4096: return launch_cols<T, 4096, ALG>(f, seed, field0, nf, W, s);
  }
  return cudaErrorNotSupported;
}

template <typename T>
static cudaError_t dispatch_rows(const Fast2D& f, int64_t nf, const void* W, void* out, int64_t stride,
                                 cudaStream_t s) {
  switch (f.n2 / 2) {
    case 128: return launch_rows<T, 128>(f, nf, W, out, stride, s);
    case 256: return launch_rows<T, 256>(f, nf, W, out, stride, s);
    case 512: return launch_rows<T, 512>(f, nf, W, out, stride, s);
    case 1024: return launch_rows<T, 1024>(f, nf, W, out, stride, s);
    case 2048: return launch_rows<T, 2048>(f, nf, W, out, stride, s);
  }
  return cudaErrorNotSupported;
}

template <typename T>
static cudaError_t run_fast(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                            int64_t stride, cudaStream_t s) {
  cudaError_t e = alg == GRFC_ONE_FFT_OVERWRITE ? dispatch_cols<T, GRFC_ONE_FFT_OVERWRITE>(f, seed, field0, nf, W, s)
                                                : dispatch_cols<T, GRFC_ONE_FFT_RECURSIVE>(f, seed, field0, nf, W, s);
  if (e != cudaSuccess) return e;
  return dispatch_rows<T>(f, nf, W, out, stride, s);
}

cudaError_t fast2d_init(Fast2D& f, const GridDesc& g, const DensityDesc& D, int dtype, int alg, double s_one,
                        double s_two) {
  f.n1 = (int)g.n[0];
  f.n2 = (int)g.n[1];
  f.dtype = dtype;
  f.alg = alg;
  f.g = g;
  f.D = D;
  f.s_one = s_one;
  f.s_two = s_two;
  const size_t cs = dtype == GRFC_F64 ? 16 : 8;
  cudaError_t e = cudaMalloc(&f.d_tw, (size_t)(f.n1 + f.n2) * cs);
  if (e != cudaSuccess) return e;
  if (dtype == GRFC_F64) {
    auto a = host_twiddles<double>(f.n1), b = host_twiddles<double>(f.n2);
    a.insert(a.end(), b.begin(), b.end());
    e = cudaMemcpy(f.d_tw, a.data(), a.size() * cs, cudaMemcpyHostToDevice);
  } else {
    auto a = host_twiddles<float>(f.n1), b = host_twiddles<float>(f.n2);
    a.insert(a.end(), b.begin(), b.end());
    e = cudaMemcpy(f.d_tw, a.data(), a.size() * cs, cudaMemcpyHostToDevice);
  }
  // Keep the per-chunk workspace (P*s bytes per field) well inside the 126 MB L2.
  f.l2_budget = 40.0 * 1024 * 1024;
  return e;
}

void fast2d_free(Fast2D& f) {
  cudaFree(f.d_tw);
  f.d_tw = nullptr;
}

cudaError_t launch_fast2d(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                          int64_t stride, cudaStream_t s) {
  if (f.dtype == GRFC_F64) return run_fast<double>(f, alg, seed, field0, nf, W, out, stride, s);
  return run_fast<float>(f, alg, seed, field0, nf, W, out, stride, s);
}

}  // namespace grfc
