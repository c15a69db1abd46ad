// Fused power-of-two 2D path (BASELINE configs c1, c2, c3, c5).
//
// Data layout. N1 x N2 grid, M = N2/2. The half-spectrum after the column
// pass is stored as W[field][j1][k], k in [0, M) — exactly P*s bytes per field
// (the size of the real field): the Nyquist column k2 = M rides in the
// imaginary part of column 0 (both columns are Hermitian in k1, so their
// column transforms are real), and the last-axis half-complex -> real
// pre-twiddle
//     Z[k] = (X[k] + conj X[M-k]) + i e^{2 pi i k/N2} (X[k] - conj X[M-k])
// is applied in the column kernel's epilogue, which owns columns k and M-k
// together. The row kernel is then a plain M-point complex FFT whose output
// z[m] = (x[2m], x[2m+1]) is the real field row.
//
// Kernels (Algorithm 2/3, the reference's synth.cpp:118-126):
//   k_cols_gen  per (field, strip of 2*CB columns): Philox noise + Hermitian
//               rule + sqrt(g) + scale for every cell, in registers; exp(+)
//               column FFT (register radix stages, one shared-memory exchange
//               per stage boundary); Z epilogue; coalesced stores of W.
//   k_rows_c2r  per row: M-point exp(+) FFT, writes the field row (float2 /
//               double2 stores, 128 B per half-warp per instruction).
#pragma once

#include <algorithm>
#include <cstring>
#include <vector>

#include "fast2d.h"
#include "fft_reg.cuh"
#include "grfc_internal.cuh"

namespace grfc {

// ---------------------------------------------------------------- radix plans
template <int... Rs>
struct Radices {};

template <typename RS>
struct RFirst;
template <int R0, int... Rs>
struct RFirst<Radices<R0, Rs...>> {
  static constexpr int value = R0;
};
template <typename RS>
struct RLast;
template <int R0>
struct RLast<Radices<R0>> {
  static constexpr int value = R0;
};
template <int R0, int R1, int... Rs>
struct RLast<Radices<R0, R1, Rs...>> {
  static constexpr int value = RLast<Radices<R1, Rs...>>::value;
};

// ColPlan<N, T>: E elements per thread, X = CB column pairs per block.
// RowPlan<N, T>: E elements per thread, X = rows per block.
template <int N, typename T>
struct ColPlan {
  static constexpr int E = 0;
};
template <int N, typename T>
struct RowPlan {
  static constexpr int E = 0;
};

#define GRFC_PLAN(Name, N, TT, E_, X_, ...) \
  template <>                              \
  struct Name<N, TT> {                     \
    static constexpr int E = E_;           \
    static constexpr int X = X_;           \
    using R = Radices<__VA_ARGS__>;        \
  };
GRFC_PLAN(ColPlan, 256, float, 16, 8, 16, 16)
GRFC_PLAN(ColPlan, 512, float, 32, 8, 32, 16)
GRFC_PLAN(ColPlan, 1024, float, 32, 8, 32, 32)
GRFC_PLAN(ColPlan, 2048, float, 16, 4, 16, 16, 8)
GRFC_PLAN(ColPlan, 4096, float, 16, 2, 16, 16, 16)
GRFC_PLAN(ColPlan, 256, double, 16, 8, 16, 16)
GRFC_PLAN(ColPlan, 512, double, 16, 8, 16, 16, 2)
GRFC_PLAN(ColPlan, 1024, double, 16, 4, 16, 16, 4)
GRFC_PLAN(ColPlan, 2048, double, 16, 2, 16, 16, 8)
GRFC_PLAN(ColPlan, 4096, double, 16, 1, 16, 16, 16)
GRFC_PLAN(RowPlan, 128, float, 16, 16, 16, 8)
GRFC_PLAN(RowPlan, 256, float, 16, 16, 16, 16)
GRFC_PLAN(RowPlan, 512, float, 32, 16, 32, 16)
GRFC_PLAN(RowPlan, 1024, float, 32, 8, 32, 32)
GRFC_PLAN(RowPlan, 2048, float, 16, 2, 16, 16, 8)
GRFC_PLAN(RowPlan, 128, double, 16, 16, 16, 8)
GRFC_PLAN(RowPlan, 256, double, 16, 16, 16, 16)
GRFC_PLAN(RowPlan, 512, double, 16, 8, 16, 16, 2)
GRFC_PLAN(RowPlan, 1024, double, 16, 4, 16, 16, 4)
GRFC_PLAN(RowPlan, 2048, double, 16, 2, 16, 16, 8)
#undef GRFC_PLAN

template <int N, typename T>
constexpr int col_threads() {
  return 2 * ColPlan<N, T>::X * (N / ColPlan<N, T>::E);
}
template <int N, typename T>
constexpr int row_threads() {
  return RowPlan<N, T>::X * (N / RowPlan<N, T>::E);
}

// ---------------------------------------------------------------- Stockham in registers
// A team of TT = N/E threads holds one line of length N, E elements each.
// Stage (radix R, NS = product of the earlier radices): thread j runs E/R
// butterflies jj = j + b*TT on inputs x[jj + i N/R], twiddled by
// w_{NS R}^{i (jj mod NS)}; outputs go to (jj/NS) NS R + jj%NS + i NS.
template <int N, int E, int R, int NS, int SIGN, typename C>
__device__ __forceinline__ void stage_compute(C* v, int j, const C* __restrict__ tw, int tws) {
  constexpr int TT = N / E;
#pragma unroll
  for (int b = 0; b < E / R; ++b) {
    if constexpr (NS > 1) {
      const int k = (j + b * TT) % NS;
#pragma unroll
      for (int i = 1; i < R; ++i) {
        C w = __ldg(&tw[(i * k * (N / (NS * R))) * tws]);
        if (SIGN < 0) w.y = -w.y;
        v[b * R + i] = cmul(v[b * R + i], w);
      }
    }
    dft<R, SIGN>(&v[b * R]);
  }
}

template <int N, int E, int R, int NS>
__device__ __forceinline__ int stage_out_index(int j, int b, int i) {
  constexpr int TT = N / E;
  const int jj = j + b * TT;
  return (jj / NS) * NS * R + (jj % NS) + i * NS;
}

template <int N, int E, int R>
__device__ __forceinline__ int stage_in_index(int j, int b, int i) {
  constexpr int TT = N / E;
  return j + b * TT + i * (N / R);
}

// Runs the stages on v (stage-0 inputs already in v, ordered b*R0 + i).
// Exchanges go through `ex`. On return v[b*RL + i] holds output element
// j + b*TT + i*N/RL (RL the last radix).
template <int N, int E, int SIGN, int NS, int R, int... Rest, typename C, typename Ex>
__device__ __forceinline__ void run_stages(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex) {
  stage_compute<N, E, R, NS, SIGN>(v, j, tw, tws);
  if constexpr (sizeof...(Rest) > 0) {
    constexpr int R2 = RFirst<Radices<Rest...>>::value;
#pragma unroll
    for (int b = 0; b < E / R; ++b)
#pragma unroll
      for (int i = 0; i < R; ++i) ex.put(stage_out_index<N, E, R, NS>(j, b, i), v[b * R + i]);
    ex.sync();
#pragma unroll
    for (int b = 0; b < E / R2; ++b)
#pragma unroll
      for (int i = 0; i < R2; ++i) v[b * R2 + i] = ex.get(stage_in_index<N, E, R2>(j, b, i));
    ex.sync();
    run_stages<N, E, SIGN, NS * R, Rest...>(v, j, tw, tws, ex);
  }
}

template <int N, int E, int SIGN, typename C, typename Ex, int... Rs>
__device__ __forceinline__ void line_fft(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex,
                                         Radices<Rs...>) {
  run_stages<N, E, SIGN, 1, Rs...>(v, j, tw, tws, ex);
}

// Column-strip exchange: smem[e * SLOTS + slot]; slots are adjacent lanes,
// so every access is a full 128 B (fp32) / 256 B (fp64) row: conflict-free.
template <typename C, int SLOTS>
struct ColEx {
  C* s;
  int slot;
  __device__ __forceinline__ void put(int e, C v) { s[e * SLOTS + slot] = v; }
  __device__ __forceinline__ C get(int e) const { return s[e * SLOTS + slot]; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};

// Row exchange: row-contiguous, one pad element per 128 B (spreads the
// stride-R writes of the first stage across banks).
template <typename C>
struct RowEx {
  C* s;
  static constexpr int PER = 128 / (int)sizeof(C);
  __device__ __forceinline__ static int pad(int e) { return e + e / PER; }
  __device__ __forceinline__ void put(int e, C v) { s[pad(e)] = v; }
  __device__ __forceinline__ C get(int e) const { return s[pad(e)]; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};

template <int N, typename C>
constexpr int row_pitch() {
  return N + N / (128 / (int)sizeof(C));
}

// ---------------------------------------------------------------- cells
struct F2Params {
  int n1, n2, m, hd;  // hd = N2/2 + 1
  double wstep1, wstep2;  // 2 pi / l
  double sqrt_c, alpha, ell, scale;
  int family;
  DensityDesc D;
  GridDesc g;
};

// sqrt(g) at the cell (k1, k2) of the half-lattice.
template <typename T>
__device__ __forceinline__ T sqrt_g2(const F2Params& p, int k1, int k2) {
  const int k1w = k1 <= p.n1 / 2 ? k1 : k1 - p.n1;
  const int k2w = k2 <= p.n2 / 2 ? k2 : k2 - p.n2;
  if (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV) {
    const T w1 = (T)k1w * (T)p.wstep1, w2 = (T)k2w * (T)p.wstep2;
    const T s = w1 * w1 + w2 * w2;
    const T ell = (T)p.ell;
    if (p.family == GRFC_DENSITY_GAUSSIAN_COV) return (T)p.sqrt_c * exp((T)(-0.25) * ell * ell * s);
    const T q = (T)1 + ell * ell * s;
    if constexpr (sizeof(T) == 4) return (T)p.sqrt_c * exp2f((float)(-0.5 * p.alpha) * __log2f(q));
    else return (T)p.sqrt_c * pow(q, -0.5 * p.alpha);
  }
  int64_t kw[2] = {k1w, k2w};
  return sqrt_gamma<T>(p.g, p.D, kw, (int64_t)k1 * p.hd + k2);
}

// X(K) = conj(w(K)) sqrt(g) scale for a half-lattice cell with the Philox
// stream: the overwrite (Alg 2) / exact-set (Alg 3) rules of
// philox_cell_noise (generic.cu) specialised to 2D.
template <typename T, int ALG>
__device__ __forceinline__ C_t<T> gen_cell(const F2Params& p, int k1, int k2, uint64_t seed, uint64_t field) {
  using C = C_t<T>;
  const T r = (T)0.70710678118654752440;
  const bool edge = (k2 == 0 || k2 == p.m);
  const bool self = edge && (k1 == 0 || k1 == p.n1 / 2);
  T z0, z1, wx, wy;
  if constexpr (ALG == GRFC_ONE_FFT_OVERWRITE) {
    const int64_t h = (int64_t)k1 * p.hd + k2;
    if (self) {
      normal_pair<T>(seed, field, (uint64_t)h, z0, z1);
      wx = z0;
      wy = (T)0;
    } else if (edge && k1 < p.n1 / 2) {  // mirror -K visited later: its draws, conjugated
      const int64_t hm = (int64_t)(p.n1 - k1) * p.hd + k2;
      normal_pair<T>(seed, field, (uint64_t)hm, z0, z1);
      wx = r * z0;
      wy = -r * z1;
    } else {
      normal_pair<T>(seed, field, (uint64_t)h, z0, z1);
      wx = r * z0;
      wy = r * z1;
    }
  } else {
    if (self) {
      normal_pair<T>(seed, field, (uint64_t)k1 * p.n2 + k2, z0, z1);
      wx = z0;
      wy = (T)0;
    } else {
      const bool k1_free = !(k1 == 0 || k1 == p.n1 / 2);
      const bool rep = k1_free ? (k1 < p.n1 / 2) : true;
      const int64_t lin = rep ? (int64_t)k1 * p.n2 + k2
                              : (int64_t)((p.n1 - k1) % p.n1) * p.n2 + ((p.n2 - k2) % p.n2);
      normal_pair<T>(seed, field, (uint64_t)lin, z0, z1);
      wx = r * z0;
      wy = rep ? r * z1 : -r * z1;
    }
  }
  const T mlt = sqrt_g2<T>(p, k1, k2) * (T)p.scale;
  return mk<C>(wx * mlt, -wy * mlt);
}

// Slot -> column. Left slots [0, CB): k = s CB + c (k = 0 is the packed
// (0, M) column); right slots: M - k, except k = 0 which takes column M/2.
__device__ __forceinline__ int slot_column(int s, int slot, int CB, int M, bool& packed, bool& mid) {
  packed = mid = false;
  if (slot < CB) {
    const int k = s * CB + slot;
    packed = (k == 0);
    return k;
  }
  const int k = s * CB + slot - CB;
  if (k == 0) {
    mid = true;
    return M / 2;
  }
  return M - k;
}

// Z epilogue for a lane owning column kk with partner value P (column M-kk):
// Z = (X + conj P) + i w_kk (X - conj P); packed column 0: Z[0] from (Y0, YN);
// column M/2: Z = 2 conj(Y).
template <typename T, typename C>
__device__ __forceinline__ C epilogue_z(C X, C P, bool packed, bool mid, C w) {
  if (packed) return mk<C>(X.x + X.y, X.x - X.y);
  if (mid) return mk<C>((T)2 * X.x, (T)-2 * X.y);
  const C s = mk<C>(X.x + P.x, X.y - P.y);
  const C d = mk<C>(X.x - P.x, X.y + P.y);
  const C t = cmul(w, d);
  return mk<C>(s.x - t.y, s.y + t.x);
}

// ---------------------------------------------------------------- kernels
template <typename T, int N1, int ALG>
__global__ void __launch_bounds__(col_threads<N1, T>())
    k_cols_gen(F2Params p, uint64_t seed, uint64_t field0, C_t<T>* __restrict__ W,
               const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2) {
  using C = C_t<T>;
  using PL = ColPlan<N1, T>;
  constexpr int E = PL::E, CB = PL::X, SLOTS = 2 * CB, TT = N1 / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, slot = tid % SLOTS, j = tid / SLOTS;
  const int strips = p.m / (2 * CB);
  const int s = (int)(blockIdx.x % (unsigned)strips);
  const uint64_t f = blockIdx.x / (unsigned)strips;
  bool packed, mid;
  const int col = slot_column(s, slot, CB, p.m, packed, mid);

  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i) {
      const int k1 = j + b * TT + i * (N1 / R0);
      C x = gen_cell<T, ALG>(p, k1, col, seed, field0 + f);
      if (packed) {  // column 0 + i * column M
        const C y = gen_cell<T, ALG>(p, k1, p.m, seed, field0 + f);
        x = mk<C>(x.x - y.y, x.y + y.x);
      }
      v[b * R0 + i] = x;
    }
  ColEx<C, SLOTS> ex{reinterpret_cast<C*>(smem_raw), slot};
  line_fft<N1, E, +1>(v, j, tw1, 1, ex, typename PL::R{});

  const C w = __ldg(&tw2[col]);  // e^{2 pi i col / N2}
  C* Wf = W + f * (uint64_t)N1 * (uint64_t)p.m;
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) {
      const int e = b * RL + i;
      C P;
      P.x = __shfl_xor_sync(0xffffffffu, v[e].x, CB);
      P.y = __shfl_xor_sync(0xffffffffu, v[e].y, CB);
      const int row = j + b * TT + i * (N1 / RL);
      Wf[(int64_t)row * p.m + col] = epilogue_z<T>(v[e], P, packed, mid, w);
    }
}

template <typename T, int M>
__global__ void __launch_bounds__(row_threads<M, T>())
    k_rows_c2r(const C_t<T>* __restrict__ W, T* __restrict__ out, int64_t rows, int rows_per_field,
               int64_t out_stride, const C_t<T>* __restrict__ tw2) {
  using C = C_t<T>;
  using PL = RowPlan<M, T>;
  constexpr int E = PL::E, RPB = PL::X, TT = M / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, rl = tid / TT, j = tid % TT;
  int64_t row = (int64_t)blockIdx.x * RPB + rl;
  const bool live = row < rows;
  if (!live) row = rows - 1;
  const C* Wr = W + row * M;
  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i) v[b * R0 + i] = Wr[j + b * TT + i * (M / R0)];
  RowEx<C> ex{reinterpret_cast<C*>(smem_raw) + rl * row_pitch<M, C>()};
  line_fft<M, E, +1>(v, j, tw2, 2, ex, typename PL::R{});
  if (!live) return;
  const int64_t f = row / rows_per_field, rr = row - f * rows_per_field;
  C* o = reinterpret_cast<C*>(out + f * out_stride + rr * (int64_t)(2 * M));
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) o[j + b * TT + i * (M / RL)] = v[b * RL + i];
}

// ---------------------------------------------------------------- launchers
inline F2Params make_params(const Fast2D& f) {
  F2Params p{};
  p.n1 = f.n1;
  p.n2 = f.n2;
  p.m = f.n2 / 2;
  p.hd = f.n2 / 2 + 1;
  p.wstep1 = 2.0 * M_PI / f.g.l[0];
  p.wstep2 = 2.0 * M_PI / f.g.l[1];
  p.family = f.D.family;
  p.sqrt_c = f.D.sqrt_c;
  p.alpha = f.D.alpha;
  p.ell = f.D.family == GRFC_DENSITY_MATERN ? f.D.r[1] : f.D.r[0];
  p.scale = f.s_one;
  p.D = f.D;
  p.g = f.g;
  return p;
}

template <typename T, int N1, int ALG>
cudaError_t launch_cols(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W,
                               cudaStream_t s) {
  using C = C_t<T>;
  constexpr int CB = ColPlan<N1, T>::X;
  const size_t smem = (size_t)N1 * 2 * CB * sizeof(C);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_cols_gen<T, N1, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int strips = (f.n2 / 2) / (2 * CB);
  const C* tw1 = (const C*)f.d_tw;
  const C* tw2 = tw1 + f.n1;
  LaunchScope ls("fused_cols_gen", s);
  k_cols_gen<T, N1, ALG><<<(unsigned)(nf * strips), col_threads<N1, T>(), smem, s>>>(make_params(f), seed, field0,
                                                                                     (C*)W, tw1, tw2);
  return cudaGetLastError();
}

template <typename T, int M>
cudaError_t launch_rows(const Fast2D& f, int64_t nf, const void* W, void* out, int64_t stride,
                               cudaStream_t s) {
  using C = C_t<T>;
  constexpr int RPB = RowPlan<M, T>::X;
  const size_t smem = (size_t)RPB * row_pitch<M, C>() * sizeof(C);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rows_c2r<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t rows = nf * f.n1;
  const C* tw2 = (const C*)f.d_tw + f.n1;
  LaunchScope ls("fused_rows_c2r", s);
  k_rows_c2r<T, M><<<(unsigned)((rows + RPB - 1) / RPB), row_threads<M, T>(), smem, s>>>(
      (const C*)W, (T*)out, rows, f.n1, stride, tw2);
  return cudaGetLastError();
}

}  // namespace grfc
