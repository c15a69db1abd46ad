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

// ---- float2 specialisations on the sm_100 packed fp32x2 pipe (FADD2 / FMUL2 /
// FFMA2). ptxas folds the broadcast (.F32), swap (.LO_HI) and partial-negate
// operand forms, so a complex add is 1 instruction and a complex multiply 2.
__device__ __forceinline__ unsigned long long f2pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2upk(unsigned long long r) {
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ unsigned long long f2add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return f2upk(f2add(f2pk(a.x, a.y), f2pk(b.x, b.y))); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return f2upk(f2sub(f2pk(a.x, a.y), f2pk(b.x, b.y))); }
// a * w = w.x (a.x, a.y) + w.y (-a.y, a.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
  const unsigned long long t = f2mul(f2pk(w.x, w.x), f2pk(a.x, a.y));
  return f2upk(f2fma(f2pk(w.y, w.y), f2pk(-a.y, a.x), t));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return f2upk(f2mul(f2pk(s, s), f2pk(a.x, a.y))); }
// a * (c + i s) with c, s constants
__device__ __forceinline__ float2 cmul_cs(float2 a, float c, float s) {
  const unsigned long long t = f2mul(f2pk(c, c), f2pk(a.x, a.y));
  return f2upk(f2fma(f2pk(s, s), f2pk(-a.y, a.x), t));
}
template <typename C>
__device__ __forceinline__ C cmul_cs(C a, decltype(C{}.x) c, decltype(C{}.x) s) {
  return mk<C>(a.x * c - a.y * s, a.x * s + a.y * c);
}

// ---------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): counter (cell_lo, cell_hi, field_lo,
// field_hi), key (seed_lo, seed_hi). Fixed key scheme, documented in
// DESIGN.md §Noise; never change it (fields must stay re-generable).
// Round keys precomputed on the host (k[2r], k[2r+1]) = (seed_lo + r W0,
// seed_hi + r W1): a round is then 2 IMAD.WIDE.U32 + 2 LOP3 with the keys
// read straight from the kernel-parameter constant bank.
struct PhiloxKey {
  uint32_t k[20];
};

inline PhiloxKey philox_key(uint64_t seed) {
  PhiloxKey K;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    K.k[2 * r] = k0;
    K.k[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return K;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxKey& K) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ K.k[2 * r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ K.k[2 * r + 1],
                   (uint32_t)p0);
  }
  return c;
}

__device__ __forceinline__ uint4 philox_draw(const PhiloxKey& K, uint64_t field, uint64_t cell) {
  return philox4x32_10(make_uint4((uint32_t)cell, (uint32_t)(cell >> 32), (uint32_t)field, (uint32_t)(field >> 32)),
                       K);
}

// Box-Muller pair. fp32: 24-bit uniforms from x, y; u1 in (0,1], angle
// 2 pi (u2 - 1/2). fp64: 53-bit uniforms from (x,y) and (z,w), IEEE log,
// sqrt, sincospi (no fast-math).
template <typename T>
__device__ __forceinline__ void box_muller(uint4 r, T& z0, T& z1);

// fp32 SFU forms (MUFU.LG2 / .SQRT / .SIN / .COS): the noise definition itself,
// shared bit-for-bit by generation and grfc_dump_noise.
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sincos_approx(float x, float& s, float& c) {
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(x));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(x));
}

// fp32 Box-Muller in parts: z0 = rad c, z1 = rad s. u1 = ((x >> 8) + 1) 2^-24 in
// (0, 1], u2 = (y >> 8) 2^-24 in [0, 1), angle 2 pi u2 - pi; the 2^-24 of u2 is
// folded into the angle's FMA constant (exact: the product is the same real
// number, so the result is bit-identical to fma(u2, 2 pi, -pi)).
__device__ __forceinline__ void box_muller_parts_f32(uint32_t x, uint32_t y, float& rad, float& s, float& c) {
  const float u1 = (float)((x >> 8) + 1u) * 0x1.0p-24f;
  rad = sqrt_approx(-1.38629436111989061883f * lg2_approx(u1));  // sqrt(-2 ln u1)
  sincos_approx(__fmaf_rn((float)(y >> 8), 6.28318530717958647693f * 0x1.0p-24f, -3.14159265358979323846f), s, c);
}

template <>
__device__ __forceinline__ void box_muller<float>(uint4 r, float& z0, float& z1) {
  float rad, s, c;
  box_muller_parts_f32(r.x, r.y, rad, s, c);
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
__device__ __forceinline__ void normal_pair(const PhiloxKey& K, uint64_t field, uint64_t cell, T& z0, T& z1) {
  box_muller<T>(philox_draw(K, field, cell), z0, z1);
}

// Noise units. Every algorithm draws one N(0,1) pair (a_u, b_u) per "unit" u
// of a field: Alg 2 the half-lattice cell index, Alg 3 the full-lattice index
// of a representative, Alg 1 the point pair J/2. With
// U units and Uh = ceil(U/2):
//   fp64: Philox counter u, all 128 bits feed one pair (53-bit uniforms);
//   fp32: Philox counter u mod Uh; words (x, y) feed unit u < Uh and
//         words (z, w) feed unit u + Uh — one call serves two units.
__device__ __forceinline__ void box_muller_f32(uint32_t x, uint32_t y, float& z0, float& z1) {
  box_muller<float>(make_uint4(x, y, 0u, 0u), z0, z1);
}

template <typename T>
__device__ __forceinline__ void unit_pair(const PhiloxKey& K, uint64_t field, uint64_t u, uint64_t Uh, T& z0, T& z1) {
  if constexpr (sizeof(T) == 8) {
    normal_pair<T>(K, field, u, z0, z1);
  } else {
    const bool hi = u >= Uh;
    const uint4 r = philox_draw(K, field, hi ? u - Uh : u);
    float a, b;
    box_muller_f32(hi ? r.z : r.x, hi ? r.w : r.y, a, b);
    z0 = a;
    z1 = b;
  }
}

// fp32: both units of one Philox call, u (< Uh) and u + Uh.
__device__ __forceinline__ void unit_quad_f32(const PhiloxKey& K, uint64_t field, uint64_t u, float& a0, float& b0,
                                              float& a1, float& b1) {
  const uint4 r = philox_draw(K, field, u);
  box_muller_f32(r.x, r.y, a0, b0);
  box_muller_f32(r.z, r.w, a1, b1);
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

// ---------------------------------------------------------------- cell rules
__device__ __forceinline__ void decode_half(const GridDesc& g, int64_t h, int64_t* k) {
  k[g.d - 1] = h % g.hd;
  int64_t r = h / g.hd;
  for (int a = g.d - 2; a >= 0; --a) {
    k[a] = r % g.n[a];
    r /= g.n[a];
  }
}

__device__ __forceinline__ void wrap_freq(const GridDesc& g, const int64_t* k, int64_t* kw) {
  for (int a = 0; a < g.d; ++a) kw[a] = (k[a] <= g.n[a] / 2) ? k[a] : k[a] - g.n[a];
}

// Unit-variance Hermitian noise w(K) for a half-lattice cell with the device
// Philox stream — the closed forms of SURVEY.md §A.3, verified against
// src/hermitian.cpp:128-203:
//  overwrite (Alg 2): counter = row-major H index c; self-conjugate -> a_c;
//    otherwise, if the mirror -K lies in H (k_d in {0, N_d/2}) and is visited
//    later (c(-K) > c), the later visit's draws win: r (a_{c(-K)} - i b_{c(-K)});
//    else r (a_c + i b_c).
//  exact set (Alg 3): counter = full-lattice index of rep(K), rep(K) = K iff
//    K is self-conjugate or its lowest non-{0,N/2} component is < N/2
//    (hermitian.cpp:39-84 membership); conjugated when K != rep(K).
template <typename T>
__device__ __forceinline__ C_t<T> philox_cell_noise(const GridDesc& g, int alg, const int64_t* k, int64_t h,
                                                    const PhiloxKey& key, uint64_t field) {
  using C = C_t<T>;
  const T r = (T)0.70710678118654752440;
  bool self = true;
  for (int a = 0; a < g.d; ++a)
    if (k[a] != 0 && k[a] != g.n[a] / 2) self = false;
  uint64_t u, Uh;
  bool conj = false;
  if (alg == GRFC_ONE_FFT_OVERWRITE) {
    Uh = ((uint64_t)g.cells + 1) / 2;
    u = (uint64_t)h;
    const int64_t kd = k[g.d - 1];
    if (!self && (kd == 0 || kd == g.n[g.d - 1] / 2)) {
      int64_t hm = 0;
      for (int a = 0; a < g.d - 1; ++a) hm = hm * g.n[a] + (k[a] == 0 ? 0 : g.n[a] - k[a]);
      hm = hm * g.hd + kd;
      if (hm > h) {
        u = (uint64_t)hm;
        conj = true;
      }
    }
  } else {  // exact set
    Uh = ((uint64_t)g.points + 1) / 2;
    bool is_rep = true;
    if (!self)
      for (int a = 0; a < g.d; ++a)
        if (k[a] != 0 && k[a] != g.n[a] / 2) {
          is_rep = k[a] < g.n[a] / 2;
          break;
        }
    int64_t lin = 0;
    for (int a = 0; a < g.d; ++a) lin = lin * g.n[a] + (is_rep ? k[a] : (k[a] == 0 ? 0 : g.n[a] - k[a]));
    u = (uint64_t)lin;
    conj = !is_rep;
  }
  T z0, z1;
  unit_pair<T>(key, field, u, Uh, z0, z1);
  if (self) return mk<C>(z0, (T)0);
  return mk<C>(r * z0, conj ? -r * z1 : r * z1);
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
