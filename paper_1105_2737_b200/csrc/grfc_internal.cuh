// Internal device/host definitions shared by the grfc kernels and the C-ABI.
// Reference citations are relative to /root/reference/proj/core.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/grfc.h"

namespace grfc {

// ---------------------------------------------------------------- complex
template <typename T>
struct cx;
template <>
struct cx<float> {
  using type = float2;
};
template <>
struct cx<double> {
  using type = double2;
};
template <typename T>
using C_t = typename cx<T>::type;

template <typename C>
__host__ __device__ __forceinline__ C mk(decltype(C{}.x) a, decltype(C{}.x) b) {
  C r;
  r.x = a;
  r.y = b;
  return r;
}
template <typename C>
__device__ __forceinline__ C cadd(C a, C b) {
  return mk<C>(a.x + b.x, a.y + b.y);
}
template <typename C>
__device__ __forceinline__ C csub(C a, C b) {
  return mk<C>(a.x - b.x, a.y - b.y);
}
template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  return mk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename C>
__device__ __forceinline__ C cconj(C a) {
  return mk<C>(a.x, -a.y);
}
template <typename C>
__device__ __forceinline__ C cscale(C a, decltype(C{}.x) s) {
  return mk<C>(a.x * s, a.y * s);
}
// a * (SIGN * i)
template <int SIGN, typename C>
__device__ __forceinline__ C mul_si(C a) {
  return SIGN > 0 ? mk<C>(-a.y, a.x) : mk<C>(a.y, -a.x);
}

// ---------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): counter (cell_lo, cell_hi, field_lo,
// field_hi), key (seed_lo, seed_hi). Fixed key scheme, documented in
// DESIGN.md §Noise; never change it (fields must stay re-generable).
__host__ __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(M0, c.x), hi1 = __umulhi(M1, c.z);
#else
    const uint32_t hi0 = (uint32_t)(((uint64_t)M0 * c.x) >> 32);
    const uint32_t hi1 = (uint32_t)(((uint64_t)M1 * c.z) >> 32);
#endif
    const uint32_t lo0 = M0 * c.x, lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += W0;
    k.y += W1;
  }
  return c;
}

__host__ __device__ __forceinline__ uint4 philox_draw(uint64_t seed, uint64_t field, uint64_t cell) {
  return philox4x32_10(make_uint4((uint32_t)cell, (uint32_t)(cell >> 32), (uint32_t)field,
                                  (uint32_t)(field >> 32)),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// Box-Muller pair. fp32: 24-bit uniforms from x, y; u1 in (0,1], angle
// 2 pi (u2 - 1/2). fp64: 53-bit uniforms from (x,y) and (z,w), IEEE log,
// sqrt, sincospi (no fast-math).
template <typename T>
__device__ __forceinline__ void box_muller(uint4 r, T& z0, T& z1);

template <>
__device__ __forceinline__ void box_muller<float>(uint4 r, float& z0, float& z1) {
  const float u1 = (float)((r.x >> 8) + 1u) * 0x1.0p-24f;
  const float u2 = (float)(r.y >> 8) * 0x1.0p-24f;
  const float rad = sqrtf(-2.0f * __logf(u1));
  float s, c;
  __sincosf(6.2831853071795865f * (u2 - 0.5f), &s, &c);
  z0 = rad * c;
  z1 = rad * s;
}

template <>
__device__ __forceinline__ void box_muller<double>(uint4 r, double& z0, double& z1) {
  const uint64_t a = (((uint64_t)r.x << 32) | r.y) >> 11;
  const uint64_t b = (((uint64_t)r.z << 32) | r.w) >> 11;
  const double u1 = (double)(a + 1) * 0x1.0p-53;
  const double u2 = (double)b * 0x1.0p-53;
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2 - 1.0, &s, &c);
  z0 = rad * c;
  z1 = rad * s;
}

template <typename T>
__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t field, uint64_t cell, T& z0, T& z1) {
  box_muller<T>(philox_draw(seed, field, cell), z0, z1);
}

// ---------------------------------------------------------------- grid
struct GridDesc {
  int d;
  int64_t n[GRFC_MAX_DIM];
  int64_t hd;      // n[d-1]/2 + 1
  int64_t cells;   // |H|
  int64_t points;  // P
  double w_of_k[GRFC_MAX_DIM];  // 2 pi / l_a: w = (2 pi * k~) / l_a, grid.cpp:107-111
  double l[GRFC_MAX_DIM];
};

// Density descriptor for device evaluation (see grfc.h for the families).
struct DensityDesc {
  int family;
  int d;
  double r[8];
  int i[8];
  double sqrt_c;  // GAUSSIAN_COV / MATERN normalisation, sqrt'ed
  double alpha;   // MATERN nu + d/2
  double mkl;     // POLY m^{kl}
  const double* table;  // TABLE: sqrt(g) per H cell
};

__device__ __forceinline__ double ipow_d(double x, int e) {  // spectral.cpp:16-24
  double r = 1.0;
  while (e > 0) {
    if (e & 1) r *= x;
    x *= x;
    e >>= 1;
  }
  return r;
}

// sqrt(g(w)) for the cell with wrapped integer frequencies kw[] (k~, grid.cpp:96-105),
// half-lattice index h (TABLE lookups). T is the arithmetic precision.
template <typename T>
__device__ __forceinline__ T sqrt_gamma(const GridDesc& g, const DensityDesc& D, const int64_t* kw,
                                        int64_t h) {
  if (D.family == GRFC_DENSITY_TABLE) return (T)D.table[h];
  T w[GRFC_MAX_DIM];
  T s = 0;
  for (int a = 0; a < g.d; ++a) {
    // 2 pi * k~ / l, evaluated as the reference does ((2 pi k~) / l).
    w[a] = (T)((6.283185307179586 * (double)kw[a]) / g.l[a]);
    s += w[a] * w[a];
  }
  switch (D.family) {
    case GRFC_DENSITY_GAUSSIAN_COV: {
      const T ell = (T)D.r[0];
      return (T)D.sqrt_c * exp((T)(-0.25) * ell * ell * s);
    }
    case GRFC_DENSITY_MATERN: {
      const T ell = (T)D.r[1];
      const T q = (T)1 + ell * ell * s;
      if (sizeof(T) == 4) return (T)D.sqrt_c * exp2f((float)(-0.5 * D.alpha) * __log2f((float)q));
      return (T)D.sqrt_c * (T)pow((double)q, -0.5 * D.alpha);
    }
    case GRFC_DENSITY_CONSTANT: return (T)sqrt(D.r[0]);
    case GRFC_DENSITY_TEST1D: {
      const double q = 100.0 + (double)w[0] * (double)w[0];
      const double q2 = q * q;
      return (T)sqrt((32.0e6 / 3.141592653589793) / (q2 * q2));
    }
    case GRFC_DENSITY_POLY: {
      double acc = 0.0;
      for (int a = 0; a < g.d; ++a) acc += ipow_d((double)w[a] * (double)w[a], D.i[0]);
      return (T)sqrt(1.0 / ipow_d(D.mkl + ipow_d(acc, D.i[1]), D.i[2]));
    }
    case GRFC_DENSITY_ANISO: {
      double acc = D.r[0];
      for (int a = 0; a < g.d; ++a) acc += ipow_d((double)w[a] * (double)w[a], D.i[1 + a]);
      return (T)sqrt(1.0 / ipow_d(acc, D.i[0]));
    }
  }
  return (T)0;
}

// ---------------------------------------------------------------- launch accounting
void count_launch(uint64_t n = 1);

// Brackets one kernel launch: counts it, and when per-kernel timing is on for
// the calling thread (grfc_kernel_timing_enable) records CUDA events around it
// on the launching stream.
struct LaunchScope {
  const char* name;
  cudaStream_t stream;
  void* start = nullptr;
  LaunchScope(const char* n, cudaStream_t s);
  ~LaunchScope();
};

}  // namespace grfc
