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

#include <type_traits>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fast2d.h"
#include "fft_reg.cuh"
#include "grfc_internal.cuh"

namespace grfc {

// Pseudo-algorithm of the fused 2D kernels: the column tiles read X(K) =
// conj(w) sqrt(g) scale from a buffer filled beforehand by k_gen_half (one cell
// per thread over the whole GPU) instead of generating it. For fp64 batches too
// small to fill the GPU with column tiles (c1: one field = 64 tiles), whose
// IEEE-fp64 generation is FP64-pipe-bound on the SMs that hold column tiles.
constexpr int kPreX = 8;

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
GRFC_PLAN(ColPlan, 128, float, 16, 4, 16, 8)
GRFC_PLAN(ColPlan, 256, float, 16, 8, 16, 16)
#ifndef GRFC_COL512
#define GRFC_COL512 2
#endif
#if GRFC_COL512 == 1
GRFC_PLAN(ColPlan, 512, float, 8, 4, 8, 8, 8)
#elif GRFC_COL512 == 2
GRFC_PLAN(ColPlan, 512, float, 16, 4, 16, 16, 2)
#elif GRFC_COL512 == 3
GRFC_PLAN(ColPlan, 512, float, 16, 8, 16, 16, 2)
#else
GRFC_PLAN(ColPlan, 512, float, 32, 8, 32, 16)
#endif
#ifndef GRFC_COL1024_X
#define GRFC_COL1024_X 4
#endif
GRFC_PLAN(ColPlan, 1024, float, 32, GRFC_COL1024_X, 32, 32)
GRFC_PLAN(ColPlan, 2048, float, 16, 4, 16, 16, 8)
#ifndef GRFC_COL4096_X
#define GRFC_COL4096_X 2
#endif
GRFC_PLAN(ColPlan, 4096, float, 16, GRFC_COL4096_X, 16, 16, 16)
GRFC_PLAN(ColPlan, 128, double, 16, 4, 16, 8)
GRFC_PLAN(ColPlan, 256, double, 16, 8, 16, 16)
// fp64 512-point columns: 2 column pairs per 128-thread tile (c1, one 512^2 field:
// 64 column tiles instead of 16 spread the fp64 generation over more SMs, 55 -> 36 us)
#ifndef GRFC_COL512D_X
#define GRFC_COL512D_X 2
#endif
// GRFC_COL512D_E: elements per thread of the fp64 512-point column (16: radix 16,16,2;
// 8: 8,8,8; 4: 4,4,4,4,2) — fewer elements = more threads per column, shorter
// per-thread generation chains (c1 is one field: latency-bound)
#ifndef GRFC_COL512D_E
#define GRFC_COL512D_E 16
#endif
#if GRFC_COL512D_E == 8
GRFC_PLAN(ColPlan, 512, double, 8, GRFC_COL512D_X, 8, 8, 8)
#elif GRFC_COL512D_E == 4
GRFC_PLAN(ColPlan, 512, double, 4, GRFC_COL512D_X, 4, 4, 4, 4, 2)
#else
GRFC_PLAN(ColPlan, 512, double, 16, GRFC_COL512D_X, 16, 16, 2)
#endif
GRFC_PLAN(ColPlan, 1024, double, 16, 4, 16, 16, 4)
GRFC_PLAN(ColPlan, 2048, double, 16, 2, 16, 16, 8)
GRFC_PLAN(ColPlan, 4096, double, 16, 1, 16, 16, 16)
GRFC_PLAN(RowPlan, 64, float, 8, 16, 8, 8)
GRFC_PLAN(RowPlan, 128, float, 16, 16, 16, 8)
GRFC_PLAN(RowPlan, 256, float, 16, 16, 16, 16)
GRFC_PLAN(RowPlan, 512, float, 32, 16, 32, 16)
GRFC_PLAN(RowPlan, 1024, float, 32, 8, 32, 32)
GRFC_PLAN(RowPlan, 2048, float, 16, 2, 16, 16, 8)
GRFC_PLAN(RowPlan, 64, double, 8, 16, 8, 8)
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
// fp32 stage twiddles w^i (i = 1..R-1): the power-of-two powers are loaded,
// the others formed as w^i = w^hb(i) w^(i - hb(i)) (hb = highest power of two
// <= i; at most 3 products deep for R <= 16): R-1-log2 R complex multiplies
// (2 packed instructions each) replace the loads and their address arithmetic.
#ifndef GRFC_TWREC
#define GRFC_TWREC 1
#endif
constexpr int hibit(int i) { return i >= 16 ? 16 : i >= 8 ? 8 : i >= 4 ? 4 : i >= 2 ? 2 : 1; }

template <int N, int E, int R, int NS, int SIGN, typename C>
__device__ __forceinline__ void stage_compute(C* v, int j, const C* __restrict__ tw, int tws,
                                              const C* t16 = nullptr) {
  constexpr int TT = N / E;
#pragma unroll
  for (int b = 0; b < E / R; ++b) {
    if constexpr (NS > 1) {
      const int k = (j + b * TT) % NS;
      if constexpr (NS == 16 && R == 16 && SIGN > 0 && sizeof(C) == 8) {
        if (t16) {  // per-CTA table of e^{2 pi i i k / 256}, row i-1, column k (LDS per twiddle)
#pragma unroll
          for (int i = 1; i < R; ++i) v[b * R + i] = cmul(v[b * R + i], t16[(i - 1) * 16 + k]);
          dft<R, SIGN>(&v[b * R]);
          continue;
        }
      }
      if constexpr (GRFC_TWREC && sizeof(C) == 8 && R >= 4 && R <= 32) {
        C w[R];
        Unroll<1, R>::run([&](auto ii) {
          constexpr int i = decltype(ii)::value;
          constexpr int hb = hibit(i);
          if constexpr (hb == i) {
            w[i] = __ldg(&tw[(i * k * (N / (NS * R))) * tws]);
            if (SIGN < 0) w[i].y = -w[i].y;
          } else {
            w[i] = cmul(w[hb], w[i - hb]);
          }
          v[b * R + i] = cmul(v[b * R + i], w[i]);
        });
      } else {
#pragma unroll
        for (int i = 1; i < R; ++i) {
          C w = __ldg(&tw[(i * k * (N / (NS * R))) * tws]);
          if (SIGN < 0) w.y = -w.y;
          v[b * R + i] = cmul(v[b * R + i], w);
        }
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

// Exchange addressing. An exchange type may provide put2(base, off, v) /
// get2(base, off) taking the element index split into a runtime per-butterfly
// base and a compile-time offset, so the shared-memory address is one base
// register plus an immediate (with the pow2 padding rules used here,
// pad(base + off) = pad(base) + pad(off) for every stage: see RowEx).
template <typename Ex, typename = void>
struct HasPut2 : std::false_type {};
#ifndef GRFC_TW16
#define GRFC_TW16 1
#endif
#ifndef GRFC_GEN_NOBAR
#define GRFC_GEN_NOBAR 1
#endif
#ifndef GRFC_ROW_NAMED
#define GRFC_ROW_NAMED 1
#endif
#ifndef GRFC_ROW_WARPSYNC
#define GRFC_ROW_WARPSYNC 1
#endif
#ifndef GRFC_EX2
#define GRFC_EX2 1
#endif
template <typename Ex>
struct HasPut2<Ex, std::void_t<decltype(&Ex::template put2<0>)>> : std::bool_constant<GRFC_EX2 != 0> {};

template <int OFF, typename Ex, typename C>
__device__ __forceinline__ void ex_put(Ex& ex, int base, C v) {
  if constexpr (HasPut2<Ex>::value)
    ex.template put2<OFF>(base, v);
  else
    ex.put(base + OFF, v);
}
template <int OFF, typename C, typename Ex>
__device__ __forceinline__ C ex_get(const Ex& ex, int base) {
  if constexpr (HasPut2<Ex>::value)
    return ex.template get2<OFF>(base);
  else
    return ex.get(base + OFF);
}

// Optional shared-memory twiddle table carried by an exchange (`tw16` member).
template <typename Ex, typename = void>
struct HasTw16 : std::false_type {};
template <typename Ex>
struct HasTw16<Ex, std::void_t<decltype(Ex::tw16)>> : std::true_type {};
template <typename C, typename Ex>
__device__ __forceinline__ const C* ex_tw16(const Ex& ex) {
  if constexpr (HasTw16<Ex>::value)
    return ex.tw16;
  else
    return nullptr;
}

// Runs the stages on v (stage-0 inputs already in v, ordered b*R0 + i).
// Exchanges go through `ex`. On return v[b*RL + i] holds output element
// j + b*TT + i*N/RL (RL the last radix).
template <int N, int E, int SIGN, int NS, int R, int... Rest, typename C, typename Ex>
__device__ __forceinline__ void run_stages(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex) {
  stage_compute<N, E, R, NS, SIGN>(v, j, tw, tws, ex_tw16<C>(ex));
  if constexpr (sizeof...(Rest) > 0) {
    constexpr int R2 = RFirst<Radices<Rest...>>::value;
    constexpr int TT = N / E;
#pragma unroll
    for (int b = 0; b < E / R; ++b) {
      const int jj = j + b * TT;
      const int base = (jj / NS) * NS * R + (jj % NS);
      Unroll<0, R>::run([&](auto ii) {
        constexpr int i = decltype(ii)::value;
        ex_put<i * NS>(ex, base, v[b * R + i]);
      });
    }
    ex.sync();
#pragma unroll
    for (int b = 0; b < E / R2; ++b) {
      const int base = j + b * TT;
      Unroll<0, R2>::run([&](auto ii) {
        constexpr int i = decltype(ii)::value;
        v[b * R2 + i] = ex_get<i * (N / R2), C>(ex, base);
      });
    }
    ex.sync();
    run_stages<N, E, SIGN, NS * R, Rest...>(v, j, tw, tws, ex);
  }
}

// run_stages split at the last exchange: run_head runs every stage but the last and
// ends with the puts of the last exchange (no barrier); run_tail gets the last stage's
// inputs for team position j from `ex` (possibly another thread mapping and exchange
// view than the head's) and runs it. head + barrier + tail == run_stages.
template <int N, int E, int SIGN, int NS, int R, int... Rest, typename C, typename Ex>
__device__ __forceinline__ void run_head(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex) {
  static_assert(sizeof...(Rest) > 0, "run_head needs an exchange");
  stage_compute<N, E, R, NS, SIGN>(v, j, tw, tws, ex_tw16<C>(ex));
  constexpr int TT = N / E;
#pragma unroll
  for (int b = 0; b < E / R; ++b) {
    const int jj = j + b * TT;
    const int base = (jj / NS) * NS * R + (jj % NS);
    Unroll<0, R>::run([&](auto ii) {
      constexpr int i = decltype(ii)::value;
      ex_put<i * NS>(ex, base, v[b * R + i]);
    });
  }
  if constexpr (sizeof...(Rest) > 1) {
    constexpr int R2 = RFirst<Radices<Rest...>>::value;
    ex.sync();
#pragma unroll
    for (int b = 0; b < E / R2; ++b) {
      const int base = j + b * TT;
      Unroll<0, R2>::run([&](auto ii) {
        constexpr int i = decltype(ii)::value;
        v[b * R2 + i] = ex_get<i * (N / R2), C>(ex, base);
      });
    }
    ex.sync();
    run_head<N, E, SIGN, NS * R, Rest...>(v, j, tw, tws, ex);
  }
}
template <int N, int E, int SIGN, int RL, typename C, typename Ex>
__device__ __forceinline__ void run_tail(C* v, int j, const C* __restrict__ tw, int tws, const Ex& ex) {
  constexpr int TT = N / E;
#pragma unroll
  for (int b = 0; b < E / RL; ++b) {
    const int base = j + b * TT;
    Unroll<0, RL>::run([&](auto ii) {
      constexpr int i = decltype(ii)::value;
      v[b * RL + i] = ex_get<i * (N / RL), C>(ex, base);
    });
  }
  stage_compute<N, E, RL, N / RL, SIGN>(v, j, tw, tws);
}
template <int N, int E, int SIGN, typename C, typename Ex, int... Rs>
__device__ __forceinline__ void line_fft_head(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex, Radices<Rs...>) {
  run_head<N, E, SIGN, 1, Rs...>(v, j, tw, tws, ex);
}

template <typename RS>
struct RNext;
template <int R0, int R1, int... Rs>
struct RNext<Radices<R0, R1, Rs...>> {
  static constexpr int value = R1;
};

// Stages 1.. of a plan (stage 0 already applied, v holding stage-1 inputs).
template <int N, int E, int SIGN, int NS, typename C, typename Ex, int R0, int... Rs>
__device__ __forceinline__ void run_rest(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex, Radices<R0, Rs...>) {
  run_stages<N, E, SIGN, NS, Rs...>(v, j, tw, tws, ex);
}

template <int N, int E, int SIGN, typename C, typename Ex, int... Rs>
__device__ __forceinline__ void line_fft(C* v, int j, const C* __restrict__ tw, int tws, Ex& ex,
                                         Radices<Rs...>) {
  run_stages<N, E, SIGN, 1, Rs...>(v, j, tw, tws, ex);
}

// Column-strip exchange: smem[e * SLOTS + slot]; slots are adjacent lanes,
// so every access is a full 128 B (fp32) / 256 B (fp64) row: conflict-free.
// Deferred ring-slot dependency of a column tile, checked by thread 0 at the
// exchange barriers (the tile writes W only after its last exchange): `seen`
// is the counter value thread 0 loaded when the tile started, so the common
// case costs one compare and no extra barrier.
// `skip` barriers pass before the check (the last exchange barrier checks).
struct LateDep {
  const uint32_t* ctr = nullptr;
  uint32_t target = 0, seen = 0;
  int skip = 0;
  __device__ __forceinline__ void check() {
    if (ctr && threadIdx.x == 0 && skip-- <= 0 && seen < target) {
      while ((seen = *(const volatile uint32_t*)ctr) < target) __nanosleep(128);
    }
  }
};
template <typename RS>
struct RCount;
template <int... Rs>
struct RCount<Radices<Rs...>> {
  static constexpr int value = sizeof...(Rs);
};

template <typename C, int SLOTS>
struct ColEx {
  C* s;
  int slot;
  LateDep dep{};
  __device__ __forceinline__ void put(int e, C v) { s[e * SLOTS + slot] = v; }
  __device__ __forceinline__ C get(int e) const { return s[e * SLOTS + slot]; }
  template <int OFF>
  __device__ __forceinline__ void put2(int base, C v) { (s + slot + base * SLOTS)[OFF * SLOTS] = v; }
  template <int OFF>
  __device__ __forceinline__ C get2(int base) const { return (s + slot + base * SLOTS)[OFF * SLOTS]; }
  __device__ __forceinline__ void sync() {
    dep.check();
    __syncthreads();
  }
};

// Column-strip exchange with one padding row-block every 16 rows (row e at
// e + e/16): the stage-0 puts write rows 16 apart (stride R0 = 16), which
// with SLOTS < 16 slots per row would hit the same banks 32/SLOTS times over;
// at stride 17 row-blocks they spread across all banks. Needs
// colx_rows(N) = N + N/16 rows of SLOTS elements.
template <typename C, int SLOTS>
struct ColExPad {
  C* s;
  int slot;
  LateDep dep{};
  const C* tw16 = nullptr;  // optional shared twiddle table (stage_compute)
  __device__ __forceinline__ static int row(int e) { return e + (e >> 4); }
  __device__ __forceinline__ void put(int e, C v) { s[row(e) * SLOTS + slot] = v; }
  __device__ __forceinline__ C get(int e) const { return s[row(e) * SLOTS + slot]; }
  // row(base + OFF) = row(base) + row(OFF) (see RowEx)
  template <int OFF>
  __device__ __forceinline__ void put2(int base, C v) { (s + slot + row(base) * SLOTS)[row(OFF) * SLOTS] = v; }
  template <int OFF>
  __device__ __forceinline__ C get2(int base) const { return (s + slot + row(base) * SLOTS)[row(OFF) * SLOTS]; }
  __device__ __forceinline__ void sync() {
    dep.check();
    __syncthreads();
  }
};
constexpr int colx_rows(int n) { return n + n / 16; }
// Padded column exchange: with base + immediate addressing (put2/get2) the
// padding costs no index arithmetic, so every fp32 plan uses it (SLOTS = 8:
// stage-0 puts 4-way -> 2 wavefronts per warp, the 64-bit minimum); fp64 plans
// with SLOTS > 4 keep the plain layout.
#ifndef GRFC_COLPAD
#define GRFC_COLPAD 1
#endif
template <int N1, typename T>
constexpr bool col_padded() {
  return ColPlan<N1, T>::X <= 2 || (GRFC_COLPAD && sizeof(T) == 4);
}

// Row exchange: row-contiguous, one pad element per 128 B (spreads the
// stride-R writes of the first stage across banks). For the power-of-two
// stages here pad(base + off) = pad(base) + pad(off): a stage writes element
// base + i NS with base = (jj/NS) NS R + jj%NS, and base mod PER plus
// (i NS) mod PER never reaches PER (PER | NS, or NS R | PER, or NS < PER <= NS R
// with base mod PER = jj%NS); reads take jj + i N/R2 with jj < N/R2 likewise.
// ALL: every team of the block owns a row (no predication).
// WARP: the team of a row lies inside one warp (M/E <= 32 threads), so its
// exchange needs only __syncwarp, never a CTA barrier. NAMED > 0: the team is
// NAMED whole warps and synchronises on its own hardware barrier (id `bar`),
// so the teams of a tile do not wait for each other.
template <typename C, bool ALL = false, bool WARP = false, int NAMED = 0>
struct RowEx {
  C* s;
  bool active = true;  // idle teams (beyond the tile's rows) keep to the barriers only
  int bar = 0;
  const C* tw16 = nullptr;  // optional shared twiddle table (stage_compute)
  static constexpr int PER = 128 / (int)sizeof(C);
  __host__ __device__ __forceinline__ static constexpr int pad(int e) { return e + e / PER; }
  __device__ __forceinline__ bool on() const { return ALL || active; }
  __device__ __forceinline__ void put(int e, C v) {
    if (on()) s[pad(e)] = v;
  }
  __device__ __forceinline__ C get(int e) const { return on() ? s[pad(e)] : C{}; }
  template <int OFF>
  __device__ __forceinline__ void put2(int base, C v) {
    if (on()) (s + pad(base))[pad(OFF)] = v;
  }
  template <int OFF>
  __device__ __forceinline__ C get2(int base) const { return on() ? (s + pad(base))[pad(OFF)] : C{}; }
  __device__ __forceinline__ void sync() const {
    if constexpr (WARP)
      __syncwarp();
    else if constexpr (NAMED > 0)
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NAMED) : "memory");
    else
      __syncthreads();
  }
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
  uint64_t uh;  // ceil(U/2): noise units per half Philox (grfc_internal.cuh unit_pair)
  // fp32 copies for the SFU density path
  float f_wstep1, f_wstep2, f_sqrt_c, f_ell2, f_nhalf_alpha, f_gauss_k, f_scale;
  float f_lg2K;  // log2(sqrt_c * scale / sqrt 2) for the folded Matern multiplier
  const float* sg;  // Fast2D::d_sg (fp32 Algorithm 2) or nullptr
  const void* xpre;  // kPreX: X(K) of every half-lattice cell, [field][n1][hd] (k_gen_half)
  uint64_t xfield0;  // kPreX: field index of xpre's first field
  int family;
  DensityDesc D;
  GridDesc g;
};

// sqrt(g) at the cell (k1, k2) of the half-lattice. fp32 Matern/Gaussian use
// float parameters and the SFU (ex2/lg2); everything else the generic
// device evaluation (double inside).
// Density kinds the fp32 fused kernels are specialised on: the two families
// with SFU forms get kernels without any other family's code (no fp64
// fallbacks, no per-cell family selects: c2 0.925 -> 0.894 ms); kDensAny
// evaluates every family (runtime switch), and is the only kind for fp64.
constexpr int kDensAny = 0, kDensMatern = 1, kDensGauss = 2;

template <typename T, int DK = kDensAny>
__device__ __forceinline__ T sqrt_g2(const F2Params& p, int k1, int k2) {
  const int k1w = k1 <= p.n1 / 2 ? k1 : k1 - p.n1;
  const int k2w = k2 <= p.n2 / 2 ? k2 : k2 - p.n2;
  if constexpr (sizeof(T) == 4 && DK != kDensAny) {
    const float w1 = (float)k1w * p.f_wstep1, w2 = (float)k2w * p.f_wstep2;
    const float q = w1 * w1 + w2 * w2;
    if constexpr (DK == kDensGauss) return p.f_sqrt_c * ex2_approx(p.f_gauss_k * q);
    return p.f_sqrt_c * ex2_approx(p.f_nhalf_alpha * lg2_approx(1.0f + p.f_ell2 * q));
  }
  if constexpr (sizeof(T) == 4) {
    if (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV) {
      const float w1 = (float)k1w * p.f_wstep1, w2 = (float)k2w * p.f_wstep2;
      const float s = w1 * w1 + w2 * w2;
      if (p.family == GRFC_DENSITY_GAUSSIAN_COV) return p.f_sqrt_c * ex2_approx(p.f_gauss_k * s);
      return p.f_sqrt_c * ex2_approx(p.f_nhalf_alpha * lg2_approx(1.0f + p.f_ell2 * s));
    }
  } else {
    if (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV) {
      const double w1 = (double)k1w * p.wstep1, w2 = (double)k2w * p.wstep2;
      const double s = w1 * w1 + w2 * w2;
      if (p.family == GRFC_DENSITY_GAUSSIAN_COV) return p.sqrt_c * exp(-0.25 * p.ell * p.ell * s);
      return p.sqrt_c * pow(1.0 + p.ell * p.ell * s, -0.5 * p.alpha);
    }
  }
  int64_t kw[2] = {k1w, k2w};
  return sqrt_gamma<T>(p.g, p.D, kw, (int64_t)k1 * p.hd + k2);
}

// X(K) = conj(w(K)) sqrt(g) scale for a half-lattice cell with the Philox
// stream: the overwrite (Alg 2) / exact-set (Alg 3) rules of
// philox_cell_noise (generic.cu) specialised to 2D, one Philox call per cell.
template <typename T, int ALG, int DK = kDensAny>
__device__ __forceinline__ C_t<T> gen_cell(const F2Params& p, int k1, int k2, const PhiloxKey& key, uint64_t field) {
  using C = C_t<T>;
  const T r = (T)0.70710678118654752440;
  const bool edge = (k2 == 0 || k2 == p.m);
  const bool self = edge && (k1 == 0 || k1 == p.n1 / 2);
  uint32_t u;
  bool conj = false;
  if constexpr (ALG == GRFC_ONE_FFT_OVERWRITE) {
    if (edge && !self && k1 < p.n1 / 2) {  // mirror -K visited later: its draws, conjugated
      u = (uint32_t)(p.n1 - k1) * p.hd + k2;
      conj = true;
    } else {
      u = (uint32_t)k1 * p.hd + k2;
    }
  } else {
    const bool rep = self || !(k1 != 0 && k1 != p.n1 / 2) || k1 < p.n1 / 2;
    u = rep ? (uint32_t)k1 * p.n2 + k2 : (uint32_t)((p.n1 - k1) % p.n1) * p.n2 + ((p.n2 - k2) % p.n2);
    conj = !rep;
  }
  T z0, z1;
  unit_pair<T>(key, field, u, p.uh, z0, z1);
  const T mlt = sqrt_g2<T, DK>(p, k1, k2) * (T)p.scale;
  if (self) return mk<C>(z0 * mlt, (T)0);
  const T wy = conj ? -r * z1 : r * z1;
  return mk<C>(r * z0 * mlt, -wy * mlt);
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
#ifndef GRFC_EPI2
#define GRFC_EPI2 1
#endif
  if constexpr (GRFC_EPI2 && sizeof(T) == 4) {
    // packed fp32x2: s = X + conj P, d = X - conj P, Z = s + i (w d)
    const unsigned long long x = f2pk(X.x, X.y), pc = f2pk(P.x, -P.y);
    const float2 t = cmul(w, f2upk(f2sub(x, pc)));
    return f2upk(f2add(f2add(x, pc), f2pk(-t.y, t.x)));
  }
  const C s = mk<C>(X.x + P.x, X.y - P.y);
  const C d = mk<C>(X.x - P.x, X.y + P.y);
  const C t = cmul(w, d);
  return mk<C>(s.x - t.y, s.y + t.x);
}

#ifndef GRFC_EARLY_REL
#define GRFC_EARLY_REL 1
#endif
// Experiment only (never set in a product build): GRFC_EXP_NOW=1 drops the W
// stores of column tiles and the W loads of row tiles (fields are garbage) to
// measure the fused kernel's time without its intermediate memory traffic.
#ifndef GRFC_EXP_NOW
#define GRFC_EXP_NOW 0
#endif
// ---------------------------------------------------------------- tiles
// Release-increment of a completion counter: orders this thread's (and, after
// a CTA barrier, the CTA's) prior writes before the increment. Emits
// MEMBAR.ALL.GPU + REDG — unlike __threadfence() + atomicAdd (MEMBAR.SC.GPU,
// CCTL.IVALL, ATOMG) it neither invalidates L1 nor waits for a return value.
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// SHF2 thread mapping and final stage (see col_shf2). tid -> team position j: lane =
// slot + 8 (j >> 4) + 16 (j & 1), warp = (j >> 1) & 7.
__device__ __forceinline__ int shf2_team_pos(int tid) { return (((tid >> 3) & 1) << 4) + ((tid >> 4) & 1) + ((tid >> 5) << 1); }
// After run_stages<512, 16, +1, 1, 16, 16>: v[i] = stage-2 output 256 (j >> 4) + (j & 15) + 16 i.
// Butterfly jj = (j & 15) + 16 i pairs it with position jj + 256 (lane ^ 8, same i), twiddle
// w_512^jj (the partner sits at lane ^ XOR). Lane h = j >> 4 takes the butterflies with i = 2c + h: jj = j + 32 c, outputs rows
// jj and jj + 256 — the layout line_fft returns (v[2c + i'] = row j + 32 c + 256 i').
template <typename T, int XOR = 8>
__device__ __forceinline__ void shf2_stage(C_t<T>* v, int j, const C_t<T>* __restrict__ tw1) {
  using C = C_t<T>;
  const bool h = (j >> 4) != 0;
  const C wj = __ldg(&tw1[j]);
  Unroll<0, 8>::run([&](auto cc) {
    constexpr int c = decltype(cc)::value;
    const C snd = h ? v[2 * c] : v[2 * c + 1];
    C rcv;
    rcv.x = __shfl_xor_sync(0xffffffffu, snd.x, XOR);
    rcv.y = __shfl_xor_sync(0xffffffffu, snd.y, XOR);
    const C lo = h ? rcv : v[2 * c], hi = h ? v[2 * c + 1] : rcv;
    constexpr T wc = (T)cos_2pi(c, 16), ws = (T)sin_2pi(c, 16);  // e^{2 pi i 32 c / 512}
    const C w = c == 0 ? wj : cmul_cs(wj, wc, ws);
    const C t = cmul(hi, w);
    v[2 * c] = cadd(lo, t);
    v[2 * c + 1] = csub(lo, t);
  });
}

// Column tiles that may generate in registers (col_tile REGTILE): fp32 Algorithm 2,
// one stage-0 butterfly per thread, shared-memory (not per-warp-region) exchange.
template <typename T, int N1, int ALG>
constexpr bool col_reggen_ok();

// Column tile: one (field, strip) — 2*CB column FFTs of length N1 with
// generation fused in front and the Z epilogue behind. Block = col_threads.
// generation loop unroll of the fp32 column tiles (independent Philox chains in flight)
#ifndef GRFC_REGGEN
#define GRFC_REGGEN 1
#endif
// SHF2: column plans <16, 16, 2> of 32-thread teams (fp32 512-point columns, c2): the
// final radix-2 stage pairs team positions j and j ^ 16 on the same register index, so
// with those two in one warp (lane bit 3) it runs on shuffles — each lane passes half of
// its elements and computes both outputs of the others — instead of a second trip
// through shared memory: 16 SHFL per thread for 16 STS + 16 LDS (64-bit: 64 -> 16
// wavefronts of the shared-memory data pipe per warp) and two CTA barriers less.
#ifndef GRFC_SHF2
#define GRFC_SHF2 1
#endif
// ZROW: the half-complex pre-twiddle Z[k] = (X[k] + conj X[M-k]) + i w_k (X[k] - conj X[M-k])
// moves from the column tile's epilogue to the row tile's prologue, where a row team
// (inside one warp) holds the whole row: the partner of element k = j + TT i sits in lane
// TT - j, register E-1-i (lane 0: its own register E - i). Column tiles then own 2 CB
// ADJACENT columns in natural order: W stores are one contiguous run per row and the row
// loads one full line per half-warp (strip-blocked columns pay two half lines there).
#ifndef GRFC_ZROW
#define GRFC_ZROW 1
#endif
template <int N1, int M, typename T>
constexpr bool zrow_ok();

template <typename RS>
struct IsR16_16_2 : std::false_type {};
template <>
struct IsR16_16_2<Radices<16, 16, 2>> : std::true_type {};
template <int N1, typename T>
constexpr bool col_shf2() {
  return GRFC_SHF2 && sizeof(T) == 4 && N1 == 512 && IsR16_16_2<typename ColPlan<N1, T>::R>::value &&
         ColPlan<N1, T>::E == 16 && ColPlan<N1, T>::X == 4;
}
#ifndef GRFC_REGGEN_GROUP
#define GRFC_REGGEN_GROUP 4
#endif
#ifndef GRFC_WTAIL
#define GRFC_WTAIL 1
#endif
#ifndef GRFC_REGGEN_WCOL
#define GRFC_REGGEN_WCOL 1
#endif
#ifndef GRFC_REGGEN_MAXE
#define GRFC_REGGEN_MAXE 32
#endif
#ifndef GRFC_GEN_UNROLL
#define GRFC_GEN_UNROLL 4
#endif
constexpr int kGenUnroll = GRFC_GEN_UNROLL;
// generic generation loop (fp64 and the packed column): independent cells in flight
#ifndef GRFC_GEN64_UNROLL
#define GRFC_GEN64_UNROLL 1
#endif
constexpr int kGen64Unroll = GRFC_GEN64_UNROLL;

// Group-per-column column tiles (see col_tile): fp32 plans whose column team is
// several whole warps (N1/E > 32, c3: 256 threads per 4096-point column): each
// column's FFT synchronises on its own named barrier, so the 4 columns of a tile
// (one CTA per SM) do not wait for each other; one CTA barrier hands the results to
// the epilogue. (One warp per column, N1/E = 32, measured slower on c2: 282 vs 291.)
#ifndef GRFC_COLGROUP
#define GRFC_COLGROUP 1
#endif
template <int N1, typename T>
constexpr bool col_warp_mode() {
  return GRFC_COLGROUP && sizeof(T) == 4 && N1 / ColPlan<N1, T>::E > 32 && (N1 / ColPlan<N1, T>::E) % 32 == 0 &&
         2 * ColPlan<N1, T>::X <= 15 && 2 * ColPlan<N1, T>::X * (N1 / ColPlan<N1, T>::E) == col_threads<N1, T>();
}
// strip-blocked W (wpos) for the long-column plans of the persistent kernels
#ifndef GRFC_WPERM_ALL
#define GRFC_WPERM_ALL 1
#endif
#ifndef GRFC_WPERM
#define GRFC_WPERM 1
#endif
template <int N1, typename T>
constexpr int w_perm_cb() {
  return (GRFC_WPERM && (col_warp_mode<N1, T>() || (GRFC_WPERM_ALL && sizeof(T) == 4))) ? ColPlan<N1, T>::X : 0;
}
// per-column region: N1 padded rows + 4 elements (so the regions start 8 banks apart)
constexpr int wcol_pitch(int n1) { return n1 + n1 / 16 + 4; }

template <typename T, int N1, int MC, bool PERM = false>
__device__ __forceinline__ void col_epilogue(const F2Params& p, int s, C_t<T>* __restrict__ Wf,
                                             const C_t<T>* __restrict__ tw2, C_t<T>* sm, C_t<T>* v, int slot, int j,
                                             int col, bool packed, bool mid);
template <int N1, int M, typename T>
constexpr bool zrow_ok() {
  return GRFC_ZROW && sizeof(T) == 4 && !col_warp_mode<N1, T>() &&
         RowPlan<M, T>::E == RFirst<typename RowPlan<M, T>::R>::value && M / RowPlan<M, T>::E <= 32 &&
         32 % (M / RowPlan<M, T>::E) == 0 && RowPlan<M, T>::E % 2 == 0;
}
template <typename T, int N1, int ALG>
constexpr bool col_reggen_ok() {
  return GRFC_REGGEN && (GRFC_REGGEN_WCOL || !col_warp_mode<N1, T>()) && sizeof(T) == 4 &&
         ALG == GRFC_ONE_FFT_OVERWRITE &&
         ColPlan<N1, T>::E == RFirst<typename ColPlan<N1, T>::R>::value && ColPlan<N1, T>::E <= GRFC_REGGEN_MAXE;
}

// Strip-blocked W columns (PERM, the persistent kernels' long-column plans): the
// column tile of strip s writes its 2CB columns {s CB + c} and {M - s CB - c}
// (M/2 for s = 0, c = 0) as ONE contiguous run at s 2CB + slot of each W row,
// so every W store covers whole 32-byte sectors (natural order leaves 2CB/2-
// column runs: 16 B for c3's CB = 2). wpos maps a natural column k to its
// position; the row tiles load through it (cb = 0: natural order).
__device__ __forceinline__ int wpos(int k, int M, int cb) {
  if (cb == 0) return k;
  if (2 * k < M) return (k / cb) * 2 * cb + k % cb;
  if (2 * k == M) return cb;
  const int m = M - k;
  return (m / cb) * 2 * cb + cb + m % cb;
}
template <int N1, typename T>
constexpr int w_perm_cb();  // below (needs col_warp_mode)

// Fills the per-CTA radix-16 twiddle table (fp32; see stage_compute) and returns
// it (nullptr for fp64). Ends with a CTA barrier.
// tw: the plan's table e^{2 pi i m / n}, m < n; when 256 | n the entries are
// gathered from it (e^{2 pi i m'/256} = tw[m' n/256]) instead of 240 fp64
// sincospi per CTA (1.2% of c2's executed instructions).
template <typename T>
__device__ __forceinline__ const C_t<T>* init_tw16(C_t<T>* tab, const C_t<T>* __restrict__ tw = nullptr, int n = 0) {
  if constexpr (GRFC_TW16 && sizeof(T) == 4) {
    const bool gather = tw && n >= 256 && n % 256 == 0;
    for (int e = threadIdx.x; e < 240; e += blockDim.x) {
      const int m = (e / 16 + 1) * (e % 16);
      if (gather) {
        tab[e] = __ldg(&tw[m * (n / 256)]);
      } else {
        double sn, cs;
        sincospi(2.0 * (double)m / 256.0, &sn, &cs);
        tab[e] = mk<C_t<T>>((T)cs, (T)sn);
      }
    }
    __syncthreads();
    return tab;
  } else {
    return nullptr;
  }
}

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// `hook` runs on thread 0 once per tile, mid-tile (after the generation barrier
// of a column tile, behind the W loads of a row tile): the persistent
// scheduler checks the next tile's dependency there, off the critical path.
// `pre` runs on every thread after the column FFT and before the W stores (the
// cluster scheduler waits there for the W slot to be free).
template <typename T, int N1, int ALG, int MC = 0, typename Hook = NoHook, typename Pre = NoHook, bool PERM = false,
          int DK = kDensAny, bool REGTILE = false, bool ZROW = false>
__device__ __forceinline__ void col_tile(const F2Params& p, const PhiloxKey& key, uint64_t fld, int s, C_t<T>* __restrict__ Wf,
                                         const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2,
                                         unsigned char* smem_raw, const float* __restrict__ rowq,
                                         const uint32_t* dep = nullptr, uint32_t dep_target = 0,
                                         uint32_t* sig = nullptr, Hook hook = Hook{},
                                         const C_t<T>* t16 = nullptr, Pre pre = Pre{}) {
  using C = C_t<T>;
  using PL = ColPlan<N1, T>;
  constexpr int E = PL::E, CB = PL::X, SLOTS = 2 * CB, TT = N1 / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  // WCOL: warp w owns column slot w (one column per warp, team = the warp's 32
  // lanes): the column FFT's exchanges are warp-private (__syncwarp) in a padded
  // per-warp region, and one CTA barrier hands the results to the epilogue's
  // slot-across-lanes mapping (coalesced W stores, shuffle partner pairing).
  constexpr bool WCOL = col_warp_mode<N1, T>();
  constexpr int GTT = N1 / E;  // threads per column group (one warp or several: named barrier)
  const int tid = threadIdx.x;
  constexpr bool SHF2 = col_shf2<N1, T>();
  static_assert(!SHF2 || (!col_warp_mode<N1, T>() && SLOTS == 8 && TT == 32), "SHF2 geometry");
  // SHF2: lane = slot + 8 (j >> 4) + 16 (j & 1), warp = (j >> 1) & 7 — lanes across the
  // strip's slots as before (coalesced W stores), j ^ 16 at lane ^ 8, and two even and
  // two odd team positions per warp (the padded exchange rows stay spread over the banks)
  const int slot = WCOL ? tid / GTT : tid % SLOTS;
  const int j = WCOL ? tid % GTT : SHF2 ? shf2_team_pos(tid) : tid / SLOTS;
  bool packed, mid;
  int col = slot_column(s, slot, CB, p.m, packed, mid);
  if constexpr (ZROW) {  // 2 CB adjacent columns; column 0 is the packed (0, M) column
    col = s * SLOTS + slot;
    packed = col == 0;
    mid = false;
  }

  // Generation into shared memory (rolled loop: one copy of the Philox/Box-
  // Muller/density code in the I-cache). Thread j owns rows j + t*TT.
  C* sm = reinterpret_cast<C*>(smem_raw);
  C* const rg = sm + slot * wcol_pitch(N1);  // WCOL: this warp's region
  auto gslot = [&](int k1) -> C& { return WCOL ? rg[RowEx<C>::pad(k1)] : sm[k1 * SLOTS + slot]; };
  // Thread 0 reads the slot's "previous rows consumed" counter now (relaxed);
  // it is only needed before the W stores, so its latency hides behind the tile.
  uint32_t dep_seen = 0;
  if (dep && threadIdx.x == 0) dep_seen = ld_relaxed_u32(dep);
  C v[E];
  // REGGEN (fp32 Matern/Gaussian interior columns, one stage-0 butterfly per thread):
  // the generation loop is fully unrolled and writes the stage-0 inputs straight into
  // v (row j + t TT is input t) instead of staging them through shared memory — 2E
  // shared-memory instructions per thread and one CTA barrier per tile less (the
  // shared-memory data pipe is the busiest unit of the c2 kernel: 60% of peak).
  // REGTILE is chosen per tile by the caller (col_reggen_ok; never strip 0, which holds
  // the packed and middle columns and stages through shared memory as before): two
  // copies of the tile code instead of a merge of both generation paths into one FFT
  // (the merge made ptxas spill 280 bytes).
  constexpr bool reg_tile = REGTILE;
  // GRFC_EARLY_REL: release the previous tile before generation (its consumers
  // wait on it; the fence stalls warp 0 only while the others generate)
  if (GRFC_EARLY_REL && sig && threadIdx.x == 0) red_release_add(sig, 1u);
  if constexpr (ALG == kPreX) {
    const C* __restrict__ xs = reinterpret_cast<const C*>(p.xpre) + (uint64_t)(fld - p.xfield0) * N1 * p.hd;
#pragma unroll
    for (int t = 0; t < E; ++t) {
      const int k1 = j + t * TT;
      C x = xs[(int64_t)k1 * p.hd + col];
      if (packed) {  // column 0 + i * column M
        const C y = xs[(int64_t)k1 * p.hd + p.m];
        x = mk<C>(x.x - y.y, x.y + y.x);
      }
      gslot(k1) = x;
    }
  } else if (DK == kDensAny && ALG == GRFC_ONE_FFT_OVERWRITE && sizeof(T) == 4 && !packed && p.sg) {
    // interior column: rows k1 and k1 + N1/2 are units u and u + Uh — one Philox
    // call; sqrt(g) scale / sqrt 2 from the plan's per-cell table (L2-resident)
    const float* __restrict__ sgc = p.sg + col;
#pragma unroll(kGenUnroll)
    for (int t = 0; t < E / 2; ++t) {
      const int k1 = j + t * TT;
      const float m0 = __ldg(&sgc[k1 * p.hd]), m1 = __ldg(&sgc[(k1 + N1 / 2) * p.hd]);
      const uint4 r = philox_draw(key, fld, (uint64_t)((uint32_t)k1 * p.hd + col));
      float rad0, s0, c0, rad1, s1, c1;
      box_muller_parts_f32(r.x, r.y, rad0, s0, c0);
      box_muller_parts_f32(r.z, r.w, rad1, s1, c1);
      const float g0 = rad0 * m0, g1 = rad1 * m1;  // (rad m) (c, -s) = (z0 m, -z1 m)
      gslot(k1) = mk<C>((T)(g0 * c0), (T)(-g0 * s0));
      gslot(k1 + N1 / 2) = mk<C>((T)(g1 * c1), (T)(-g1 * s1));
    }
  } else if constexpr (reg_tile) {
    const int k2w = col <= p.n2 / 2 ? col : col - p.n2;
    const float w2 = (float)k2w * p.f_wstep2;
    const float K = p.f_sqrt_c * p.f_scale * 0.70710678118654752440f;
    const bool matern = DK == kDensMatern || (DK == kDensAny && p.family == GRFC_DENSITY_MATERN);
    const float A = 1.0f + p.f_ell2 * w2 * w2, B = K * ex2_approx(p.f_gauss_k * w2 * w2);
    uint32_t u0 = (uint32_t)j * p.hd + col;
    const uint32_t ustep = (uint32_t)TT * p.hd;
#pragma unroll
    for (int t = 0; t < E / 2; ++t) {
      const int k1 = j + t * TT;
      // groups of GRFC_REGGEN_GROUP independent Philox chains: the next group's counter
      // is made to depend on every result of this one, or ptxas runs all E/2 chains
      // at once and spills
      if (t > 0 && t % GRFC_REGGEN_GROUP == 0) {
#pragma unroll
        for (int g = 1; g <= GRFC_REGGEN_GROUP; ++g)
          asm volatile("" : "+r"(u0) : "f"(v[t - g].x), "f"(v[t - g].y), "f"(v[t - g + E / 2].x), "f"(v[t - g + E / 2].y));
      }
      const uint4 r = philox_draw(key, fld, (uint64_t)(u0 + (uint32_t)t * ustep));
      float rad0, s0, c0, rad1, s1, c1;
      box_muller_parts_f32(r.x, r.y, rad0, s0, c0);
      box_muller_parts_f32(r.z, r.w, rad1, s1, c1);
      const float q0 = rowq[k1], q1 = rowq[k1 + N1 / 2];
      const float m0 = matern ? ex2_approx(__fmaf_rn(p.f_nhalf_alpha, lg2_approx(A + q0), p.f_lg2K)) : B * q0;
      const float m1 = matern ? ex2_approx(__fmaf_rn(p.f_nhalf_alpha, lg2_approx(A + q1), p.f_lg2K)) : B * q1;
      const float g0 = rad0 * m0, g1 = rad1 * m1;  // (rad m) (c, -s) = (z0 m, -z1 m)
      v[t] = mk<C>((T)(g0 * c0), (T)(-g0 * s0));
      v[t + E / 2] = mk<C>((T)(g1 * c1), (T)(-g1 * s1));
    }
  } else if (ALG == GRFC_ONE_FFT_OVERWRITE && sizeof(T) == 4 && !packed && rowq) {
    // interior column: rows k1 and k1 + N1/2 are units u and u + Uh — one
    // Philox call. sqrt(g) from the per-CTA row table rowq (fused2d_row_table):
    //   Matern   rowq = ell^2 w1^2:      m = K ex2(-alpha/2 lg2(A_col + rowq))
    //   Gaussian rowq = ex2(-ell^2 w1^2/4 log2 e):  m = B_col rowq
    const int k2w = col <= p.n2 / 2 ? col : col - p.n2;
    const float w2 = (float)k2w * p.f_wstep2;
    const float K = p.f_sqrt_c * p.f_scale * 0.70710678118654752440f;
    const bool matern = DK == kDensMatern || (DK == kDensAny && p.family == GRFC_DENSITY_MATERN);
    const float A = 1.0f + p.f_ell2 * w2 * w2, B = K * ex2_approx(p.f_gauss_k * w2 * w2);
#pragma unroll (kGenUnroll)
    for (int t = 0; t < E / 2; ++t) {
      const int k1 = j + t * TT;
      const uint4 r = philox_draw(key, fld, (uint64_t)((uint32_t)k1 * p.hd + col));
      float rad0, s0, c0, rad1, s1, c1;
      box_muller_parts_f32(r.x, r.y, rad0, s0, c0);
      box_muller_parts_f32(r.z, r.w, rad1, s1, c1);
      const float q0 = rowq[k1], q1 = rowq[k1 + N1 / 2];
      // Matern: K ex2(-alpha/2 lg2(A + q)) with K folded into the exponent (lg2 K)
      const float m0 = matern ? ex2_approx(__fmaf_rn(p.f_nhalf_alpha, lg2_approx(A + q0), p.f_lg2K)) : B * q0;
      const float m1 = matern ? ex2_approx(__fmaf_rn(p.f_nhalf_alpha, lg2_approx(A + q1), p.f_lg2K)) : B * q1;
      const float g0 = rad0 * m0, g1 = rad1 * m1;  // (rad m) (c, -s) = (z0 m, -z1 m)
      gslot(k1) = mk<C>((T)(g0 * c0), (T)(-g0 * s0));
      gslot(k1 + N1 / 2) = mk<C>((T)(g1 * c1), (T)(-g1 * s1));
    }
  } else if (DK == kDensAny && ALG == GRFC_ONE_FFT_OVERWRITE && sizeof(T) == 4 && !packed) {
    const T r = (T)0.70710678118654752440, sc = (T)p.scale;
#pragma unroll 1
    for (int t = 0; t < E / 2; ++t) {
      const int k1 = j + t * TT;
      float a0, b0, a1, b1;
      unit_quad_f32(key, fld, (uint64_t)((uint32_t)k1 * p.hd + col), a0, b0, a1, b1);
      const T m0 = sqrt_g2<T, DK>(p, k1, col) * sc * r, m1 = sqrt_g2<T, DK>(p, k1 + N1 / 2, col) * sc * r;
      gslot(k1) = mk<C>((T)a0 * m0, -(T)b0 * m0);
      gslot(k1 + N1 / 2) = mk<C>((T)a1 * m1, -(T)b1 * m1);
    }
  } else {
#pragma unroll(kGen64Unroll)
    for (int t = 0; t < E; ++t) {
      const int k1 = j + t * TT;
      C x = gen_cell<T, ALG, DK>(p, k1, col, key, fld);
      if (packed) {  // column 0 + i * column M
        const C y = gen_cell<T, ALG, DK>(p, k1, p.m, key, fld);
        x = mk<C>(x.x - y.y, x.y + y.x);
      }
      gslot(k1) = x;
    }
  }
  // Every thread reads back exactly the rows it generated (rows j + u TT, the
  // stage-0 inputs of its team position), so no CTA barrier is needed here;
  // the one below orders these reads before the first exchange's writes.
  if (!GRFC_GEN_NOBAR) __syncthreads();
  // Release of the CTA's previous tile: no global stores are in flight here,
  // so the fence in front of the increment is cheap (persistent kernel).
  if (!GRFC_EARLY_REL && sig && threadIdx.x == 0) red_release_add(sig, 1u);
  if (threadIdx.x == 0) hook();
  if (!reg_tile) {
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int i = 0; i < R0; ++i) v[b * R0 + i] = gslot(j + b * TT + i * (N1 / R0));
  }
  if constexpr (WCOL) {
    RowEx<C, true, GTT == 32, (GTT > 32 ? GTT : 0)> wex{rg, true, 1 + slot};
    if (!reg_tile) wex.sync();  // own rows read back: the group's first exchange may overwrite them
    if constexpr (GRFC_WTAIL && RCount<typename PL::R>::value > 1) {
      // Every stage but the last in the column-group mapping; the last exchange's
      // gets and the last stage run in the epilogue's slot-across-lanes mapping
      // (slot = tid % SLOTS, j = tid / SLOTS), so the results are already where the
      // W stores and the shuffle pairing want them: no transposing pass through
      // shared memory (2E shared-memory instructions per thread less). The one CTA
      // barrier between the two mappings also carries the ring-slot check.
      line_fft_head<N1, E, +1>(v, j, tw1, 1, wex, typename PL::R{});
      LateDep{dep, dep_target, dep_seen, 0}.check();
      pre();
      __syncthreads();
      const int slot2 = tid % SLOTS, j2 = tid / SLOTS;
      const RowEx<C, true> ex2{sm + slot2 * wcol_pitch(N1)};
      run_tail<N1, E, +1, RL>(v, j2, tw1, 1, ex2);
    } else {
      line_fft<N1, E, +1>(v, j, tw1, 1, wex, typename PL::R{});
      // results to the region in natural row order, then one CTA barrier (thread 0
      // first checks the ring-slot reuse dependency: every W store follows it)
#pragma unroll
      for (int b = 0; b < E / RL; ++b)
#pragma unroll
        for (int i = 0; i < RL; ++i) rg[RowEx<C>::pad(j + b * TT + i * (N1 / RL))] = v[b * RL + i];
      LateDep{dep, dep_target, dep_seen, 0}.check();
      pre();
      __syncthreads();
    }
  } else {
    // orders the read-back of staged rows before the first exchange's writes; with
    // REGGEN only strip 0 (the packed column's threads) stages anything
    if (!reg_tile) __syncthreads();
    using Ex = std::conditional_t<col_padded<N1, T>(), ColExPad<C, SLOTS>, ColEx<C, SLOTS>>;
    Ex ex{sm, slot};
    if constexpr (HasTw16<Ex>::value) ex.tw16 = t16;
    // The slot's previous field must be consumed before W is overwritten: checked
    // at the FFT's exchange barriers (all W stores follow the last one).
    constexpr bool has_ex = RFirst<typename PL::R>::value != N1;
    if constexpr (SHF2) {
      ex.dep = LateDep{dep, dep_target, dep_seen, 1};  // checked at the (only) exchange's second barrier
      run_stages<N1, E, +1, 1, 16, 16>(v, j, tw1, 1, ex);
      shf2_stage<T>(v, j, tw1);
    } else {
      if (has_ex) ex.dep = LateDep{dep, dep_target, dep_seen, 2 * (RCount<typename PL::R>::value - 1) - 1};
      line_fft<N1, E, +1>(v, j, tw1, 1, ex, typename PL::R{});
    }
    pre();
    if (dep && !has_ex) {
      if (threadIdx.x == 0 && dep_seen < dep_target)
        while (ld_relaxed_u32(dep) < dep_target) __nanosleep(256);
      __syncthreads();
    }
  }
  if constexpr (ZROW) {
    // plain stores of the column transforms X (natural order, 2 CB adjacent columns)
    static_assert(!WCOL, "ZROW: shared-exchange column plans only");
    constexpr int RLz = RLast<typename PL::R>::value;
    const int64_t mstride = MC > 0 ? (int64_t)MC : (int64_t)p.m;
    C* __restrict__ wp = Wf + (int64_t)j * mstride + col;
#pragma unroll
    for (int b = 0; b < E / RLz; ++b)
#pragma unroll
      for (int i = 0; i < RLz; ++i) __stcg(wp + (b * TT + i * (N1 / RLz)) * mstride, v[b * RLz + i]);
  } else {
    col_epilogue<T, N1, MC, PERM>(p, s, Wf, tw2, sm, v, slot, j, col, packed, mid);
  }
}

// Z epilogue + W stores of a column tile, lanes across the strip's slots
// (slot = tid % SLOTS, team position j = tid / SLOTS). In WCOL mode the FFT
// results are re-read here from the per-warp regions in that mapping.
template <typename T, int N1, int MC, bool PERM>
__device__ __forceinline__ void col_epilogue(const F2Params& p, int s, C_t<T>* __restrict__ Wf,
                                             const C_t<T>* __restrict__ tw2, C_t<T>* sm, C_t<T>* v, int slot, int j,
                                             int col, bool packed, bool mid) {
  using C = C_t<T>;
  using PL = ColPlan<N1, T>;
  constexpr int E = PL::E, CB = PL::X, SLOTS = 2 * CB, TT = N1 / E;
  constexpr int RL = RLast<typename PL::R>::value;
  if constexpr (col_warp_mode<N1, T>()) {
    slot = threadIdx.x % SLOTS;
    j = threadIdx.x / SLOTS;
    col = slot_column(s, slot, CB, p.m, packed, mid);
    if constexpr (!(GRFC_WTAIL && RCount<typename PL::R>::value > 1)) {  // else: the tail ran in this mapping
      const C* rgs = sm + slot * wcol_pitch(N1);
#pragma unroll
      for (int b = 0; b < E / RL; ++b)
#pragma unroll
        for (int i = 0; i < RL; ++i) v[b * RL + i] = rgs[RowEx<C>::pad(j + b * TT + i * (N1 / RL))];
    }
  }
  const C w = __ldg(&tw2[col]);  // e^{2 pi i col / N2}
  const bool special = packed || mid;
  // one 64-bit pointer per thread; with a compile-time M (persistent kernel) every
  // store is that pointer plus an immediate
  const int64_t mstride = MC > 0 ? (int64_t)MC : (int64_t)p.m;
  C* __restrict__ wp = Wf + (int64_t)j * mstride + (PERM ? s * SLOTS + slot : col);
  // Only the warps of strip 0 hold the packed (0, M) and middle (M/2) columns:
  // the others take a branch-free path (warp-uniform test).
  if (!__any_sync(0xffffffffu, special)) {
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int i = 0; i < RL; ++i) {
        const int e = b * RL + i;
        C P;
        P.x = __shfl_xor_sync(0xffffffffu, v[e].x, CB);
        P.y = __shfl_xor_sync(0xffffffffu, v[e].y, CB);
        const C z = epilogue_z<T>(v[e], P, false, false, w);
        if (GRFC_EXP_NOW) {
          if (z.x == (T)1.2345) __stcg(wp, z);  // keep the arithmetic live
        } else {
          __stcg(wp + (b * TT + i * (N1 / RL)) * mstride, z);
        }
      }
    return;
  }
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) {
      const int e = b * RL + i;
      C P;
      P.x = __shfl_xor_sync(0xffffffffu, v[e].x, CB);
      P.y = __shfl_xor_sync(0xffffffffu, v[e].y, CB);
      const int rr = b * TT + i * (N1 / RL);
      if (!special) __stcg(wp + rr * mstride, epilogue_z<T>(v[e], P, false, false, w));
    }
  if (special) {
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int i = 0; i < RL; ++i) {
        const int e = b * RL + i;
        const int rr = b * TT + i * (N1 / RL);
        __stcg(wp + rr * mstride, epilogue_z<T>(v[e], v[e], packed, mid, w));
      }
  }
}

// Per-CTA row table of the fp32 fused density path (see col_tile).
template <int N1>
__device__ __forceinline__ void fused2d_row_table(const F2Params& p, float* rowq) {
  for (int k1 = threadIdx.x; k1 < N1; k1 += blockDim.x) {
    const int k1w = k1 <= p.n1 / 2 ? k1 : k1 - p.n1;
    const float w1 = (float)k1w * p.f_wstep1;
    rowq[k1] = p.family == GRFC_DENSITY_MATERN ? p.f_ell2 * w1 * w1 : ex2_approx(p.f_gauss_k * w1 * w1);
  }
  __syncthreads();
}

// Row tile: RPT consecutive rows (r0..) of one field — M-point exp(+) FFTs,
// real field rows out. Block = RPT * (M/E) threads.
template <typename T, int M, int RPT, int NT = 0, typename Hook = NoHook, int WPERM = 0, bool ZROW = false>
__device__ __forceinline__ void row_tile(const C_t<T>* __restrict__ Wf, int r0, int nrows, T* __restrict__ of,
                                         const C_t<T>* __restrict__ tw2, unsigned char* smem_raw,
                                         uint32_t* sig = nullptr, Hook hook = Hook{}, const C_t<T>* t16 = nullptr) {
  using C = C_t<T>;
  using PL = RowPlan<M, T>;
  constexpr int E = PL::E, TT = M / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  const int tid = threadIdx.x, rl = tid / TT, j = tid % TT;
  int row = r0 + rl;
  const bool live = rl < RPT && row < nrows;
  if (!live) row = nrows - 1;
  const C* Wr = Wf + (int64_t)row * M;
  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i)
      v[b * R0 + i] = GRFC_EXP_NOW ? mk<C>((decltype(C{}.x))(j + b + i), (decltype(C{}.x))row)
                                   : __ldcg(&Wr[wpos(j + b * TT + i * (M / R0), M, WPERM)]);
  // Release of the CTA's previous tile; its fence overlaps the W loads' latency.
  if (sig && threadIdx.x == 0) red_release_add(sig, 1u);
  if (threadIdx.x == 0) hook();
  if constexpr (ZROW) {
    // v[i] = X[k], k = j + TT i (column transforms, natural order). Registers are
    // processed in pairs (lo = s, hi = E-1-s): lanes j >= 1 take X[M-k] from lane
    // TT - j (its hi for our lo, its lo for our hi); lane 0 (k = TT i, partner TT (E - i))
    // from its own registers E - s (the previous step's original hi) and s + 1;
    // k = 0 is the packed (0, M) column, k = M/2 pairs with itself.
    static_assert(E == R0 && WPERM == 0 && TT <= 32 && 32 % TT == 0 && E % 2 == 0, "ZROW geometry");
    const int src = (TT - j) & (TT - 1);
    const bool l0 = j == 0;
    const C wj = __ldg(&tw2[j]);  // e^{2 pi i j / N2}; w_k = w_j e^{2 pi i TT i / N2}, TT i / N2 = i / (2 E)
    C saved = v[0];
    Unroll<0, E / 2>::run([&](auto ss) {
      constexpr int st = decltype(ss)::value, lo = st, hi = E - 1 - st;
      const C A = v[lo], B = v[hi];
      C Pa, Pb;
      Pa.x = __shfl_sync(0xffffffffu, B.x, src, TT);
      Pa.y = __shfl_sync(0xffffffffu, B.y, src, TT);
      Pb.x = __shfl_sync(0xffffffffu, A.x, src, TT);
      Pb.y = __shfl_sync(0xffffffffu, A.y, src, TT);
      const C own_b = v[st + 1];  // original: st + 1 <= hi is not overwritten yet
      if (l0) {
        Pa = saved;
        Pb = own_b;
      }
      saved = B;
      constexpr T ca = (T)cos_2pi(lo, 2 * E), sa = (T)sin_2pi(lo, 2 * E);
      constexpr T cb = (T)cos_2pi(hi, 2 * E), sb = (T)sin_2pi(hi, 2 * E);
      const C wa = lo == 0 ? wj : cmul_cs(wj, ca, sa), wb = cmul_cs(wj, cb, sb);
      C Za = epilogue_z<T>(A, Pa, false, false, wa);
      const C Zb = epilogue_z<T>(B, Pb, false, false, wb);
      if (st == 0 && l0) Za = mk<C>(A.x + A.y, A.x - A.y);
      v[lo] = Za;
      v[hi] = Zb;
    });
  }
  // every team owns a row when the block holds exactly RPT teams (c2: 16 x 16 threads)
  constexpr bool ALL = NT == RPT * TT;
  constexpr bool WARP = GRFC_ROW_WARPSYNC && TT <= 32 && 32 % TT == 0;
  // teams of whole warps (c3: 128 threads per 2048-point row) use one named
  // barrier each (ids 1..teams; 0 is __syncthreads)
  constexpr int TEAMS = (NT > 0 ? NT : RPT * TT) / TT;
  constexpr int NAMED = (GRFC_ROW_NAMED && !WARP && TT % 32 == 0 && TEAMS <= 15) ? TT : 0;
  RowEx<C, ALL, WARP, NAMED> ex{reinterpret_cast<C*>(smem_raw) + (ALL ? rl : (rl < RPT ? rl : 0)) * row_pitch<M, C>(),
                                ALL || rl < RPT, 1 + rl, t16};
  line_fft<M, E, +1>(v, j, tw2, 2, ex, typename PL::R{});
  if (!live) return;
  C* o = reinterpret_cast<C*>(of + (int64_t)row * (2 * M));
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) __stcs(&o[j + b * TT + i * (M / RL)], v[b * RL + i]);
}

template <int N1, int M, typename T>
constexpr int fused_threads() {
  return col_threads<N1, T>();
}
// Rows per row tile: one team of M/E threads per row, capped so the row
// exchange buffers fit 200 KB of shared memory (surplus teams idle).
template <int N1, int M, typename T>
constexpr int rows_per_tile() {
  constexpr int teams = fused_threads<N1, M, T>() / (M / RowPlan<M, T>::E);
  constexpr int cap = (int)(200 * 1024 / (row_pitch<M, C_t<T>>() * sizeof(C_t<T>)));
  int p2 = 1;  // power of two, so tiles divide N1 exactly
  while (2 * p2 <= cap) p2 *= 2;
  return teams < p2 ? teams : p2;
}
template <int N1, int M, typename T>
constexpr size_t fused_smem() {
  using C = C_t<T>;
  constexpr size_t a = col_warp_mode<N1, T>()
                           ? (size_t)wcol_pitch(N1) * 2 * ColPlan<N1, T>::X * sizeof(C)
                           : (size_t)(col_padded<N1, T>() ? colx_rows(N1) : N1) * 2 * ColPlan<N1, T>::X * sizeof(C);
  constexpr size_t b = (size_t)rows_per_tile<N1, M, T>() * row_pitch<M, C>() * sizeof(C);
  return a > b ? a : b;
}

// ---------------------------------------------------------------- persistent fused kernel
// One launch per batch. Tiles are claimed in ticket order from
//   C(0..L-1) | C(L) R(0) | C(L+1) R(1) | ... | R(F-L..F-1)
// (C(f) = the column tiles of field f, R(f) = its row tiles), so column work
// runs L fields ahead of row work. Field f's half-spectrum lives in ring slot
// f mod S (S slots of P*s bytes: L2-resident). Per-slot counters order the
// hand-offs: R(f) waits for C(f)'s tiles, C(f) waits until the rows of the
// slot's previous field (f - S) are consumed. Every wait targets a smaller
// ticket already held by a running CTA, so the queue cannot deadlock.
struct F2Sched {
  uint32_t* ticket;
  uint32_t* col_done;  // [S]
  uint32_t* row_done;  // [S]
  uint32_t F, L, S, strips, rtiles;
  // GRFC_TILE_STATS=1: per-launch cycle counters [col, row, col-wait, row-wait, ticket, ncol, nrow]
  unsigned long long* stats;
  // f / S = umulhi(f, s_magic) when s_magic != 0 (host-checked: F * S < 2^32)
  uint32_t s_magic;
  // Scheduler groups (GRFC_GROUP): `groups` independent queues of `gsize` CTAs
  // each; group g runs fields g, g + groups, ... with its own ticket, counters
  // (ctr_stride words apart) and ring (ring_stride elements apart). F, L, S are
  // per group; F_total is the batch. groups == 1: one queue over the grid.
  uint32_t groups, gsize, ctr_stride, F_total;
  uint64_t ring_stride;
  // Deferral schedule (GRFC_DEFER): tickets interleave a field's column and row
  // tiles (C(f+L, i), R(f, i) alternating) and a CTA whose next ticket is a row
  // tile that is not ready yet parks it and runs its following ticket first
  // (see k_fused2d): waits become column work, so a short L2-resident ring
  // (small L, S) no longer stalls the queue.
  uint32_t defer;
};

// Ring-slot division of the tile decoder (thread 0, once per tile).
__device__ __forceinline__ void slot_of(const F2Sched& q, uint32_t f, uint32_t& slot, uint32_t& use) {
  use = q.s_magic ? __umulhi(f, q.s_magic) : f / q.S;
  slot = f - use * q.S;
}
inline uint32_t slot_magic(uint32_t F, uint32_t S) {
  // floor(f / S) = floor(f * (floor(2^32 / S) + 1) / 2^32) whenever f * S < 2^32
  return (uint64_t)F * S < (1ull << 32) ? (uint32_t)((1ull << 32) / S + 1) : 0u;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Dependency-counter loads of the persistent 2D scheduler. GRFC_ACQ = 1: ld.acquire.gpu
// (LDG.STRONG + CCTL.IVALL: the issuing thread blocks for the round trip, and the
// invalidate empties the SM's L1 — the twiddle tables of all four resident CTAs — once
// per tile). GRFC_ACQ = 0 (default): ld.relaxed.gpu, non-blocking until its value is
// used at the end of the tile. W is only ever read with ld.global.cg (L2, never L1), by
// threads that pass a CTA barrier after thread 0 has seen the producers' release
// increments (red.release.gpu after their W stores), so no L1 invalidation is needed.
#ifndef GRFC_ACQ
#define GRFC_ACQ 0
#endif
__device__ __forceinline__ uint32_t dep_load(const uint32_t* p) {
  return GRFC_ACQ ? ld_acquire_u32(p) : ld_relaxed_u32(p);
}

// Thread 0 polls with relaxed loads (no L1 invalidation per poll), then one
// acquire load orders the consumer's reads after the producers' releases.
__device__ __forceinline__ void wait_geq(const uint32_t* ctr, uint32_t target) {
  if (threadIdx.x == 0) {
    if (ld_relaxed_u32(ctr) < target)
      while (ld_relaxed_u32(ctr) < target) __nanosleep(256);
    (void)ld_acquire_u32(ctr);
  }
  __syncthreads();
}

__device__ __forceinline__ void signal_done(uint32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) red_release_add(ctr, 1u);
}

// Resident CTAs per SM the fused kernel is compiled for (register budget):
// tuned for the c2 shape (fp32 512 columns: 4 x 256 threads at 64 registers,
// no spills; 3 CTAs at 80 registers measured 2% slower); other shapes let
// ptxas choose.
#ifndef GRFC_DEFER_BUILD
#define GRFC_DEFER_BUILD 0
#endif
#ifndef GRFC_MID_CHECK
#define GRFC_MID_CHECK 1
#endif
#ifndef GRFC_RES1
#define GRFC_RES1 1
#endif
#ifndef GRFC_COL_LATE_WAIT
#define GRFC_COL_LATE_WAIT 1
#endif
#ifndef GRFC_TILE_STATS_BUILD
#define GRFC_TILE_STATS_BUILD 0
#endif
#ifndef GRFC_FUSED1024_MINB
#define GRFC_FUSED1024_MINB 2
#endif
#ifndef GRFC_FUSED_MINB
#define GRFC_FUSED_MINB 4
#endif
template <int N1, int M, typename T>
constexpr int fused_min_blocks() {
  return (N1 == 512 && sizeof(T) == 4) ? GRFC_FUSED_MINB
         : (N1 == 4096 && sizeof(T) == 4 && ColPlan<N1, T>::X == 1) ? 2
         : (N1 == 1024 && sizeof(T) == 4 && ColPlan<N1, T>::X == 4) ? GRFC_FUSED1024_MINB
                                                                    : 0;
}
template <typename T, int N1, int M, int ALG, int DK = kDensAny>
__global__ void __launch_bounds__(fused_threads<N1, M, T>(), fused_min_blocks<N1, M, T>())
    k_fused2d(F2Params p, F2Sched q, PhiloxKey key, uint64_t field0, C_t<T>* __restrict__ ring, T* __restrict__ out,
              int64_t out_stride, const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ float s_rowq[N1];
  constexpr int RPT = rows_per_tile<N1, M, T>();
  const bool table = sizeof(T) == 4 && (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV);
  if (table) fused2d_row_table<N1>(p, s_rowq);
  // fp32: per-CTA table of the radix-16 stage twiddles e^{2 pi i r k / 256} (r = 1..15,
  // k < 16), shared by the column and row FFTs' NS = 16 stages (LDS instead of products)
  __shared__ C_t<T> s_tw16[GRFC_TW16 && sizeof(T) == 4 ? 240 : 1];
  const C_t<T>* t16 = init_tw16<T>(s_tw16, tw2, 2 * M);
  // One CTA barrier per tile. At the end of tile i thread 0 publishes ticket
  // i+1 (its atomic was issued when tile i started, so the round trip hides
  // behind tile i) together with whether i+1's dependency — its field's
  // columns (row tile) or its ring slot's previous rows (column tile) — is
  // already met; the barrier then both closes tile i and opens tile i+1.
  // Thread 0 signals tile i's completion after that barrier; only if i+1's
  // dependency was not yet met does it spin and add a second barrier.
  const uint64_t slot_elems = (uint64_t)N1 * M;
  // scheduler group of this CTA: its own queue over fields gid, gid + groups, ...
  uint32_t fstep = 1, foff = 0;
  if (q.groups > 1) {
    const uint32_t gid = blockIdx.x / q.gsize;
    q.ticket += (size_t)gid * q.ctr_stride;
    q.col_done += (size_t)gid * q.ctr_stride;
    q.row_done += (size_t)gid * q.ctr_stride;
    ring += gid * q.ring_stride;
    q.F = (q.F_total - gid + q.groups - 1) / q.groups;
    fstep = q.groups;
    foff = gid;
  }
  // tiles per field are compile-time (strips = M / 2CB, row tiles = N1 / RPT): the
  // decoder's divisions by them are shifts; the ring-slot division is a multiply-high
  constexpr uint32_t STRIPS = M / (2 * ColPlan<N1, T>::X), RT = N1 / RPT, G = STRIPS + RT;
  const uint32_t pro = q.L * STRIPS, nfull = q.F - q.L;
  const uint32_t total = q.F * G;
  struct Tile {
    bool col;
    uint32_t f, idx, slot, use;
  };
  auto decode = [&](uint32_t t) {
    Tile x;
    if (t < pro) {
      x.col = true;
      x.f = t / STRIPS;
      x.idx = t % STRIPS;
    } else if ((t -= pro) < nfull * G) {
      const uint32_t g = t / G, r = t % G;
      if ((GRFC_DEFER_BUILD & 1) && q.defer) {
        // proportional interleave of the group's STRIPS column and RT row tiles
        const uint32_t rb = r * RT / G, ra = (r + 1) * RT / G;  // row tiles before / through position r
        x.col = ra == rb;
        x.idx = x.col ? r - rb : rb;
      } else {
        x.col = r < STRIPS;
        x.idx = x.col ? r : r - STRIPS;
      }
      x.f = x.col ? g + q.L : g;
    } else {
      t -= nfull * G;
      x.col = false;
      x.f = nfull + t / RT;
      x.idx = t % RT;
    }
    slot_of(q, x.f, x.slot, x.use);
    return x;
  };
  // dependency counter / target of a tile (target 0: none)
  // Column tiles check their ring-slot dependency late (before their W stores,
  // see col_tile), so only row tiles wait up front.
  auto dep_of = [&](const Tile& x, const uint32_t*& ctr) -> uint32_t {
    ctr = x.col ? &q.row_done[x.slot] : &q.col_done[x.slot];
    return x.col ? (GRFC_COL_LATE_WAIT ? 0u : x.use * RT) : (x.use + 1) * STRIPS;
  };
  // Deferral schedule: what must hold before the tile may START when its CTA keeps a
  // parked row tile — for a column tile also its ring-slot dependency (normally
  // checked late, inside the tile): a CTA never blocks inside a tile while it holds
  // a parked row, so every wait points to a strictly smaller ticket (no cycles).
  auto dep_start = [&](const Tile& x, const uint32_t*& ctr) -> uint32_t {
    ctr = x.col ? &q.row_done[x.slot] : &q.col_done[x.slot];
    return x.col ? x.use * RT : (x.use + 1) * STRIPS;
  };
  // Thread 0 holds two reserved tickets: tA (the next tile) and tB (the one
  // after, its atomic in flight). At the start of each tile it issues a
  // relaxed load of tA's dependency counter, consumed at the end of the tile,
  // so neither the ticket nor the readiness check costs an exposed round trip.
  // (Reserving ahead cannot deadlock: every dependency points to a smaller
  // ticket, and the smallest unfinished ticket is always a running tile.)
  // Thread 0 also decodes the tiles (integer divisions) and publishes them in
  // shared memory, so the other threads only read the message.
  struct Msg {
    uint32_t t, ready, col, f, idx, slot, use, pf;
    uint64_t pf_off;  // element offset of the W rows of the tile after next (pf: it is a row tile)
  };
  __shared__ Msg s_msg;
  const bool DEFER = GRFC_DEFER_BUILD && q.defer;
  uint32_t tA = total, tB = total, dep_v = 0;
  // early dependency check of the next (row) tile: the 16 bytes around its counter,
  // fetched asynchronously mid-tile (s_dep_idx = 1 + word index, 0: none pending)
  __shared__ __align__(16) uint32_t s_dep[4];
  __shared__ uint32_t s_dep_idx;
  if (threadIdx.x == 0) s_dep_idx = 0;
  // deferral schedule (q.defer), thread 0: tD = parked row ticket (kNone: none) with
  // dvD = 1 + its dependency counter acquired mid-tile; haveA: tA is reserved and unused
  constexpr uint32_t kNone = 0xffffffffu;
  // (kept in shared memory: touched by thread 0 only, a few times per tile, and the
  // kernel sits at its 64-register budget)
  __shared__ uint32_t s_tD, s_dvD, s_haveA;
  if (threadIdx.x == 0) s_tD = kNone, s_dvD = 0, s_haveA = 0;
  volatile uint32_t& tD = s_tD;
  volatile uint32_t& dvD = s_dvD;
  volatile uint32_t& haveA = s_haveA;
  // The ticket atomic in inline PTX: a plain atomicAdd in thread 0's branch is
  // warp-aggregated by the compiler (vote + shuffle of the returned value), and the
  // shuffle waits for the atomic's round trip right there — warp 0 lost ~1k cycles at
  // the top of every tile. The asm result is first read at the end of the tile.
  auto claim = [&]() {
    uint32_t t;
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(q.ticket) : "memory");
    return t;
  };
  // thread 0: message for ticket t (readiness from the early counter value v)
  // plus the prefetch target of ticket t2
  auto publish = [&](uint32_t t, uint32_t v, uint32_t t2) {
    Msg m{};
    m.t = t;
    m.ready = 1;
    if (t < total) {
      const Tile x = decode(t);
      m.col = x.col, m.f = x.f, m.idx = x.idx, m.slot = x.slot, m.use = x.use;
      const uint32_t* ctr;
      const uint32_t target = dep_of(x, ctr);
      if (target) {
        if (GRFC_RES1 && !x.col) {
          // v = 1 + the value acquired mid-tile (0: none); else one round trip here,
          // the acquire load both checking and ordering
          m.ready = v > target;
          if (!m.ready) m.ready = dep_load(ctr) >= target;
        } else {
          if (v < target) v = ld_relaxed_u32(ctr);
          m.ready = v >= target;
          // rows read what other CTAs wrote: acquire; a column tile's ring-slot reuse
          // (write after the rows' reads) needs no L1-invalidating acquire
          if (m.ready && !x.col) (void)ld_acquire_u32(ctr);
        }
      }
    }
    if (t2 < total) {
      const Tile y = decode(t2);
      m.pf = !y.col;
      m.pf_off = y.slot * slot_elems + (uint64_t)y.idx * RPT * M;
    }
    s_msg = m;
  };
  if (threadIdx.x == 0) {
    const uint32_t t0 = claim();
    if (GRFC_RES1) {
      publish(t0, 0, total);
    } else {
      tA = claim();
      tB = claim();
      publish(t0, 0, tA);
    }
  }
  __syncthreads();
  uint32_t* done_ctr = nullptr;  // thread 0: counter of the tile just finished
  // tile timing counters are compiled in only with -DGRFC_TILE_STATS_BUILD=1
  const bool STATS = GRFC_TILE_STATS_BUILD && q.stats;
  long long c_col = 0, c_row = 0, c_wc = 0, c_wr = 0, c_tk = 0, n_col = 0, n_row = 0;
  for (;;) {
    long long t0 = STATS ? clock64() : 0;
    const Msg m = s_msg;
    // (the exit test comes first: with the claim in front of it ptxas threaded
    // thread 0's exit out of the middle of its divergent block, and the warp then
    // reached the tile's aligned barriers unconverged: garbage fields)
    if (m.t >= total) break;
    if (threadIdx.x == 0) {
      if ((GRFC_DEFER_BUILD & 2) && DEFER) {
        if (!haveA) {
          tA = claim();
          haveA = 1u;
        }
      } else if (GRFC_RES1) {
        // GRFC_RES1: one reservation — the next tile's ticket is claimed now and
        // read at the end of this tile (its round trip hides behind the tile)
        tA = claim();
      } else if (tA < total) {  // early dependency load of the next tile
        const uint32_t* ctr;
        dep_of(decode(tA), ctr);
        dep_v = ld_relaxed_u32(ctr);
      }
    }
    if (m.pf) {
      // the tile after this one is a row tile: pull its W rows toward L2 now
      // (one 128-byte line per thread and pass); the ring is larger than L2
      const char* base = reinterpret_cast<const char*>(ring + m.pf_off);
      constexpr uint32_t lines = (uint32_t)((uint64_t)RPT * M * sizeof(C_t<T>) / 128);
      for (uint32_t l = threadIdx.x; l < lines; l += blockDim.x)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (uint64_t)l * 128));
    }
    if (!m.ready) {  // rare: close the previous tile, wait for the dependency, one extra barrier
      if (threadIdx.x == 0) {
        if (done_ctr) red_release_add(done_ctr, 1u);
        done_ctr = nullptr;
        const uint32_t* ctr;
        const uint32_t target = dep_of(decode(m.t), ctr);
        while (ld_relaxed_u32(ctr) < target) __nanosleep(256);
        if (GRFC_ACQ && !m.col) (void)ld_acquire_u32(ctr);
      }
      __syncthreads();
    }
    if (STATS) (m.col ? c_wc : c_wr) += clock64() - t0;
    long long b = STATS ? clock64() : 0;
    C_t<T>* Wf = ring + m.slot * slot_elems;
    // GRFC_RES1 mid-tile check (thread 0): the next ticket's atomic, issued at the
    // top of this tile, has returned; if it is a row tile, its dependency counter
    // is read now with acquire semantics (ordering the CTA's later W reads after
    // the producers' releases), so publish() needs no round trip when it is met.
    auto hook = [&]() {
      if ((GRFC_DEFER_BUILD & 4) && DEFER && tD != kNone) {  // the parked row tile's columns: done by now?
        const uint32_t* ctr;
        dep_of(decode(tD), ctr);
        dvD = ld_acquire_u32(ctr) + 1u;
      }
      if (GRFC_RES1 && GRFC_MID_CHECK && tA < total) {
        const Tile y = decode(tA);
        const uint32_t* ctr;
        if (!y.col && dep_of(y, ctr)) {
          if (GRFC_ACQ) {
            dep_v = ld_acquire_u32(ctr) + 1u;  // +1: "acquired" marker
          } else {
            // cp.async (L2 -> shared, no destination register): thread 0 does not wait
            // here, and nothing stays live in a register across the tile; the aligned
            // 16 bytes around the counter are copied and publish() picks the word
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s_dep);
            const uint64_t ga = (uint64_t)ctr & ~15ull;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(ga) : "memory");
            s_dep_idx = 1u + (uint32_t)(((uint64_t)ctr >> 2) & 3u);
          }
        }
        if ((GRFC_DEFER_BUILD & 4) && DEFER && y.col && tD != kNone && dep_start(y, ctr))
          dep_v = ld_relaxed_u32(ctr) + 1u;
      }
    };
    // the previous tile's completion is released inside this one (see col_tile / row_tile)
    if (m.col) {
      // (a plan with a per-cell sqrt(g) table, p.sg, keeps the table path)
      constexpr bool ZR = ALG == GRFC_ONE_FFT_OVERWRITE && zrow_ok<N1, M, T>();
      constexpr bool PM = !ZR && w_perm_cb<N1, T>() > 0;
      if (col_reggen_ok<T, N1, ALG>() && table && !p.sg && m.idx > 0)
        col_tile<T, N1, ALG, M, decltype(hook), NoHook, PM, DK, col_reggen_ok<T, N1, ALG>(), ZR>(
            p, key, field0 + foff + (uint64_t)m.f * fstep, (int)m.idx, Wf, tw1, tw2, smem_raw, s_rowq,
            GRFC_COL_LATE_WAIT && m.use ? &q.row_done[m.slot] : nullptr, m.use * RT, done_ctr, hook, t16);
      else
        col_tile<T, N1, ALG, M, decltype(hook), NoHook, PM, DK, false, ZR>(
            p, key, field0 + foff + (uint64_t)m.f * fstep, (int)m.idx, Wf, tw1, tw2, smem_raw,
            table ? s_rowq : nullptr, GRFC_COL_LATE_WAIT && m.use ? &q.row_done[m.slot] : nullptr, m.use * RT,
            done_ctr, hook, t16);
      done_ctr = &q.col_done[m.slot];
    } else {
      constexpr bool ZR = ALG == GRFC_ONE_FFT_OVERWRITE && zrow_ok<N1, M, T>();
      row_tile<T, M, RPT, fused_threads<N1, M, T>(), decltype(hook), ZR ? 0 : w_perm_cb<N1, T>(), ZR>(
          Wf, (int)m.idx * RPT, N1, out + (int64_t)(foff + (uint64_t)m.f * fstep) * out_stride, tw2, smem_raw,
          done_ctr, hook, t16);
      done_ctr = &q.row_done[m.slot];
    }
    // every tile has internal barriers, so all threads have read s_msg
    long long e = STATS ? clock64() : 0;
    if (threadIdx.x == 0) {
      if ((GRFC_DEFER_BUILD & 8) && DEFER) {
        // Next tile: the parked row if its columns are done; else the reserved ticket
        // if it can run (a column tile, or a row tile that is ready); else park the
        // reserved row and take the following ticket (interleaved order: a column
        // tile); only when two unready rows are held does the CTA wait (for the older).
        uint32_t next = total, v = 0;
        bool picked = false;
        const uint32_t* ctr;
        if (tD != kNone) {
          const uint32_t target = dep_of(decode(tD), ctr);
          if (!dvD) dvD = ld_acquire_u32(ctr) + 1u;
          if (dvD > target) {
            next = tD, v = dvD, tD = kNone, picked = true;
          }
        }
        // can ticket y start now? (vy = 1 + its counter if already loaded, else 0)
        auto can_start = [&](const Tile& y, uint32_t& vy) {
          const bool parked = tD != kNone;
          if (y.col && !parked) return true;  // slot dependency checked late, inside the tile
          const uint32_t target = dep_start(y, ctr);
          if (!target) return true;
          if (!vy) vy = (y.col ? ld_relaxed_u32(ctr) : ld_acquire_u32(ctr)) + 1u;
          return vy > target;
        };
        if (!picked && haveA && tA < total) {
          const Tile a = decode(tA);
          uint32_t va = dep_v;
          if (can_start(a, va)) {
            next = tA, v = a.col ? 0u : va, haveA = 0u, picked = true;
          } else if (tD == kNone) {  // an unready row: park it, take the following ticket
            tD = tA;
            tA = claim();
            if (tA < total) {
              const Tile b = decode(tA);
              uint32_t vb = 0;
              if (can_start(b, vb)) next = tA, v = b.col ? 0u : vb, haveA = 0u, picked = true;
            }
          }
        }
        if (!picked && tD != kNone) next = tD, v = 0, tD = kNone;  // waits in the next iteration
        publish(next, v, total);
        dep_v = 0;
        dvD = 0;
      } else if (GRFC_RES1) {
        if (!GRFC_ACQ && s_dep_idx) {
          asm volatile("cp.async.wait_all;" ::: "memory");
          dep_v = ((volatile uint32_t*)s_dep)[s_dep_idx - 1u] + 1u;
          s_dep_idx = 0;
        }
        publish(tA < total ? tA : total, dep_v, total);
        dep_v = 0;
      } else {
        publish(tA, dep_v, tB);
        tA = tB;
        tB = tB < total ? claim() : total;
      }
    }
    __syncthreads();
    if (STATS) {
      (m.col ? c_col : c_row) += e - b;
      c_tk += clock64() - e;
      ++(m.col ? n_col : n_row);
    }
  }
  if (threadIdx.x == 0 && done_ctr) red_release_add(done_ctr, 1u);  // the CTA's last tile
  if (STATS && threadIdx.x == 0) {
    atomicAdd(&q.stats[0], (unsigned long long)c_col);
    atomicAdd(&q.stats[1], (unsigned long long)c_row);
    atomicAdd(&q.stats[2], (unsigned long long)c_wc);
    atomicAdd(&q.stats[3], (unsigned long long)c_wr);
    atomicAdd(&q.stats[4], (unsigned long long)c_tk);
    atomicAdd(&q.stats[5], (unsigned long long)n_col);
    atomicAdd(&q.stats[6], (unsigned long long)n_row);
  }
}

// X(K) of every half-lattice cell of fields [field0, field0 + nf), one cell per
// thread over the whole GPU: the same gen_cell the column tiles run, so kPreX
// fields are bit-identical to generated ones (batch composition never changes
// a field). Layout [field][k1][hd].
template <typename T>
__global__ void __launch_bounds__(256) k_gen_x2d(F2Params p, PhiloxKey key, uint64_t field0, int64_t nf,
                                                 C_t<T>* __restrict__ X) {
  const int64_t per = (int64_t)p.n1 * p.hd, total = per * nf;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = e / per, h = e - f * per;
    const int k1 = (int)(h / p.hd), k2 = (int)(h - (int64_t)k1 * p.hd);
    X[e] = gen_cell<T, GRFC_ONE_FFT_OVERWRITE>(p, k1, k2, key, field0 + (uint64_t)f);
  }
}

// ---------------------------------------------------------------- cluster-scheduled fused kernel
// One launch per batch, persistent, launched as thread-block clusters of CS
// CTAs. Cluster c owns fields c, c + nclusters, ...; CTA rank r of the cluster
// runs column strips r, r + CS, ... and row tiles r, r + CS, ... of each of
// them. The field's half-spectrum W lives in the cluster's own slot(s) of the
// workspace (nclusters x NSL x P*s bytes — sized to stay L2-resident), and the
// hand-offs are cluster barriers (barrier.cluster arrive.release /
// wait.acquire: ~400 cycles, no global atomics, no polling):
//   NSL = 1: C(f) | arrive, wait | R(f) | arrive | [C(f+1) computes] wait | stores
//   NSL = 2: C(f) -> slot f%2 | arrive, wait | R(f) | C(f+1) -> slot (f+1)%2
//            (passing the barrier after C(f) implies every CTA finished R(f-1),
//             the last reader of slot (f+1)%2)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
struct ClusterWaitPre {
  bool on;
  __device__ __forceinline__ void operator()() const {
    if (on) cluster_wait();
  }
};

#ifndef GRFC_CL_MINB
#define GRFC_CL_MINB 4
#endif
template <int N1, int M, typename T>
constexpr int cl_min_blocks() {
  return (N1 == 512 && sizeof(T) == 4) ? GRFC_CL_MINB : fused_min_blocks<N1, M, T>();
}
template <typename T, int N1, int M, int NSL>
__global__ void __launch_bounds__(fused_threads<N1, M, T>(), cl_min_blocks<N1, M, T>())
    k_fused2d_cl(F2Params p, PhiloxKey key, uint64_t field0, uint32_t F, C_t<T>* __restrict__ ws, T* __restrict__ out,
                 int64_t out_stride, const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ float s_rowq[N1];
  constexpr int RPT = rows_per_tile<N1, M, T>();
  constexpr uint32_t STRIPS = M / (2 * ColPlan<N1, T>::X), RT = N1 / RPT;
  constexpr int NT = fused_threads<N1, M, T>();
  const bool table = sizeof(T) == 4 && (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV);
  if (table) fused2d_row_table<N1>(p, s_rowq);
  __shared__ C_t<T> s_tw16[GRFC_TW16 && sizeof(T) == 4 ? 240 : 1];
  const C_t<T>* t16 = init_tw16<T>(s_tw16, tw2, 2 * M);
  const uint32_t rank = cluster_ctarank(), cs = cluster_nctarank();
  const uint32_t cid = cluster_id_x(), ncl = ncluster_x();
  const uint64_t slot_elems = (uint64_t)N1 * M;
  C_t<T>* const wbase = ws + (uint64_t)cid * NSL * slot_elems;
  uint32_t it = 0;
  for (uint32_t f = cid; f < F; f += ncl, ++it) {
    C_t<T>* Wf = wbase + (NSL == 2 ? (it & 1u) : 0u) * slot_elems;
    bool first = true;
    for (uint32_t sidx = rank; sidx < STRIPS; sidx += cs) {
      // NSL = 1: the slot is free once every CTA of the cluster finished R(f-1)
      // (the arrive after its rows); the first column tile waits for that just
      // before its W stores, so the barrier's latency hides behind its FFT.
      const ClusterWaitPre pre{NSL == 1 && first && it > 0};
      col_tile<T, N1, GRFC_ONE_FFT_OVERWRITE, M, NoHook, ClusterWaitPre, (!zrow_ok<N1, M, T>() && w_perm_cb<N1, T>() > 0),
               kDensAny, false, zrow_ok<N1, M, T>()>(
          p, key, field0 + f, (int)sidx, Wf, tw1, tw2, smem_raw, table ? s_rowq : nullptr, nullptr, 0, nullptr,
          NoHook{}, t16, pre);
      first = false;
      __syncthreads();
    }
    if (NSL == 1 && first && it > 0) cluster_wait();  // no column tile on this rank
    cluster_arrive();
    cluster_wait();
    for (uint32_t r = rank; r < RT; r += cs) {
      row_tile<T, M, RPT, NT, NoHook, (zrow_ok<N1, M, T>() ? 0 : w_perm_cb<N1, T>()), zrow_ok<N1, M, T>()>(Wf, (int)r * RPT, N1, out + (int64_t)f * out_stride, tw2,
                                                           smem_raw, nullptr, NoHook{},
                              t16);
      __syncthreads();
    }
    if (NSL == 1) cluster_arrive();
  }
  if (NSL == 1 && it > 0) cluster_wait();  // pair the last arrive
}

// Two-kernel variant (A/B and fallback): all column tiles of a chunk, then
// all its row tiles.
template <typename T, int N1, int ALG>
__global__ void __launch_bounds__(col_threads<N1, T>())
    k_cols_gen(F2Params p, PhiloxKey key, uint64_t field0, C_t<T>* __restrict__ W,
               const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ float s_rowq[N1];
  const bool table = sizeof(T) == 4 && (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV);
  if (table) fused2d_row_table<N1>(p, s_rowq);
  const int strips = p.m / (2 * ColPlan<N1, T>::X);
  const int s = (int)(blockIdx.x % (unsigned)strips);
  const uint64_t f = blockIdx.x / (unsigned)strips;
  col_tile<T, N1, ALG>(p, key, field0 + f, s, W + f * (uint64_t)N1 * (uint64_t)p.m, tw1, tw2, smem_raw,
                       table ? s_rowq : nullptr);
}

template <typename T, int M>
__global__ void __launch_bounds__(row_threads<M, T>())
    k_rows_c2r(const C_t<T>* __restrict__ W, T* __restrict__ out, int64_t rows, int rows_per_field,
               int64_t out_stride, const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int RPB = RowPlan<M, T>::X;
  const int64_t r0 = (int64_t)blockIdx.x * RPB;
  const int64_t f = r0 / rows_per_field;
  row_tile<T, M, RPB, row_threads<M, T>()>(W + f * (int64_t)rows_per_field * M, (int)(r0 - f * rows_per_field), rows_per_field,
                      out + f * out_stride, tw2, smem_raw);
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
  p.uh = f.alg == GRFC_ONE_FFT_OVERWRITE ? ((uint64_t)f.n1 * (f.n2 / 2 + 1) + 1) / 2 : ((uint64_t)f.n1 * f.n2 + 1) / 2;
  p.f_wstep1 = (float)p.wstep1;
  p.f_wstep2 = (float)p.wstep2;
  p.f_sqrt_c = (float)p.sqrt_c;
  p.f_ell2 = (float)(p.ell * p.ell);
  p.f_nhalf_alpha = (float)(-0.5 * p.alpha);
  p.f_gauss_k = (float)(-0.25 * p.ell * p.ell * 1.4426950408889634);  // -ell^2/4 * log2(e)
  p.f_scale = (float)p.scale;
  p.f_lg2K = (float)std::log2(p.sqrt_c * p.scale * 0.70710678118654752440);
  p.sg = f.d_sg;
  p.D = f.D;
  p.g = f.g;
  return p;
}

template <typename T, int N1, int ALG>
cudaError_t launch_cols(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W,
                               cudaStream_t s) {
  using C = C_t<T>;
  constexpr int CB = ColPlan<N1, T>::X;
  const size_t smem = col_warp_mode<N1, T>() ? (size_t)wcol_pitch(N1) * 2 * CB * sizeof(C)
                                             : (size_t)(col_padded<N1, T>() ? colx_rows(N1) : N1) * 2 * CB * sizeof(C);
  // set on every launch: the attribute is per device (a process may use several)
  cudaFuncSetAttribute(k_cols_gen<T, N1, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int strips = (f.n2 / 2) / (2 * CB);
  const C* tw1 = (const C*)f.d_tw;
  const C* tw2 = tw1 + f.n1;
  LaunchScope ls("fused_cols_gen", s);
  k_cols_gen<T, N1, ALG><<<(unsigned)(nf * strips), col_threads<N1, T>(), smem, s>>>(make_params(f), philox_key(seed), field0,
                                                                                     (C*)W, tw1, tw2);
  return cudaGetLastError();
}

template <typename T, int M>
cudaError_t launch_rows(const Fast2D& f, int64_t nf, const void* W, void* out, int64_t stride,
                               cudaStream_t s) {
  using C = C_t<T>;
  constexpr int RPB = RowPlan<M, T>::X;
  const size_t smem = (size_t)RPB * row_pitch<M, C>() * sizeof(C);
  // set on every launch: the attribute is per device (a process may use several)
  cudaFuncSetAttribute(k_rows_c2r<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t rows = nf * f.n1;
  const C* tw2 = (const C*)f.d_tw + f.n1;
  LaunchScope ls("fused_rows_c2r", s);
  k_rows_c2r<T, M><<<(unsigned)((rows + RPB - 1) / RPB), row_threads<M, T>(), smem, s>>>(
      (const C*)W, (T*)out, rows, f.n1, stride, tw2);
  return cudaGetLastError();
}

// Fills the persistent-kernel geometry of Fast2D (called once at plan setup).
template <typename T, int N1, int M, int ALG>
cudaError_t fused_query(Fast2D& f) {
  constexpr int NT = fused_threads<N1, M, T>(), RPT = rows_per_tile<N1, M, T>();
  constexpr size_t smem = fused_smem<N1, M, T>();
  cudaError_t e = cudaFuncSetAttribute(k_fused2d<T, N1, M, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if constexpr (sizeof(T) == 4 && ALG == GRFC_ONE_FFT_OVERWRITE) {
    e = cudaFuncSetAttribute(k_fused2d<T, N1, M, ALG, kDensMatern>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_fused2d<T, N1, M, ALG, kDensGauss>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    if (e != cudaSuccess) return e;
  }
  int occ = 0, dev = 0, sms = 148;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2d<T, N1, M, ALG>, NT, smem);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  f.occ = occ < 1 ? 1 : occ;
  f.sms = sms;
  f.strips = M / (2 * ColPlan<N1, T>::X);
  f.rtiles = N1 / RPT;
  return cudaSuccess;
}

template <typename T, int N1, int M, int ALG>
cudaError_t launch_fused(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* ws, void* out,
                         int64_t stride, cudaStream_t s, const void* xpre) {
  using C = C_t<T>;
  constexpr int NT = fused_threads<N1, M, T>();
  constexpr size_t smem = fused_smem<N1, M, T>();
  F2Params prm = make_params(f);
  Fast2D geo = f;  // geometry of this instantiation
  if constexpr (ALG == kPreX) {
    cudaError_t e = cudaFuncSetAttribute(k_fused2d<T, N1, M, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2d<T, N1, M, ALG>, NT, smem);
    if (e != cudaSuccess) return e;
    geo.occ = occ < 1 ? 1 : occ;
    prm.xpre = xpre;
    prm.xfield0 = field0;
    const int64_t cells = (int64_t)N1 * (M + 1) * nf;
    LaunchScope ls("gen_x2d", s);
    k_gen_x2d<T><<<(unsigned)std::min<int64_t>((cells + 255) / 256, (int64_t)f.sms * 16), 256, 0, s>>>(
        prm, philox_key(seed), field0, nf, (C*)const_cast<void*>(xpre));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  F2Sched q{};
  uint32_t conc = 0;
  const GroupGeom gg = group_geometry(geo, nf);
  if (gg.groups > 1) {
    q.L = gg.L;
    q.S = gg.S;
    conc = gg.groups * gg.gsize;
  } else {
    fused_geometry(geo, nf, &q.L, &q.S, &conc);
  }
  q.F = gg.groups > 1 ? (uint32_t)((nf + gg.groups - 1) / gg.groups) : (uint32_t)nf;  // largest group's
  q.F_total = (uint32_t)nf;
  q.groups = gg.groups;
  q.gsize = gg.gsize;
  q.strips = (uint32_t)f.strips;
  q.rtiles = (uint32_t)f.rtiles;
  q.s_magic = slot_magic(q.F, q.S);
  q.ctr_stride = (uint32_t)(fused_ctr_bytes(q.S) / sizeof(uint32_t));
  q.ring_stride = (uint64_t)q.S * N1 * M;
  if (const char* se = std::getenv("GRFC_DEFER")) q.defer = se[0] == '1';
  uint32_t* ctr = (uint32_t*)ws;  // per group: [ticket][col_done S][row_done S] (padded) | rings
  q.ticket = ctr;
  q.col_done = ctr + 1;
  q.row_done = ctr + 1 + q.S;
  C* ring = (C*)((char*)ws + fused_ctr_bytes(q.S) * gg.groups);
  cudaError_t e = cudaMemsetAsync(ctr, 0, fused_ctr_bytes(q.S) * gg.groups, s);
  if (e != cudaSuccess) return e;
  const C* tw1 = (const C*)f.d_tw;
  const C* tw2 = tw1 + f.n1;
  const uint32_t total = q.F * (q.strips + q.rtiles);
  const uint32_t grid = gg.groups > 1 ? conc : (total < conc ? total : conc);
  const char* st = std::getenv("GRFC_TILE_STATS");
  unsigned long long* dstats = nullptr;
  if (st && st[0] == '1') {
    cudaMalloc(&dstats, 8 * sizeof(unsigned long long));
    cudaMemsetAsync(dstats, 0, 8 * sizeof(unsigned long long), s);
  }
  q.stats = dstats;
  {
    LaunchScope ls("fused2d_persistent", s);
    // fp32 Matern / Gaussian (no sqrt(g) table): the family-specialised kernel
    const int dk = (sizeof(T) == 4 && ALG == GRFC_ONE_FFT_OVERWRITE && !f.d_sg)
                       ? (f.D.family == GRFC_DENSITY_MATERN ? kDensMatern
                          : f.D.family == GRFC_DENSITY_GAUSSIAN_COV ? kDensGauss : kDensAny)
                       : kDensAny;
    if constexpr (sizeof(T) == 4 && ALG == GRFC_ONE_FFT_OVERWRITE) {
      if (dk == kDensMatern)
        k_fused2d<T, N1, M, ALG, kDensMatern><<<grid, NT, smem, s>>>(prm, q, philox_key(seed), field0, ring, (T*)out,
                                                                      stride, tw1, tw2);
      else if (dk == kDensGauss)
        k_fused2d<T, N1, M, ALG, kDensGauss><<<grid, NT, smem, s>>>(prm, q, philox_key(seed), field0, ring, (T*)out,
                                                                     stride, tw1, tw2);
      else
        k_fused2d<T, N1, M, ALG><<<grid, NT, smem, s>>>(prm, q, philox_key(seed), field0, ring, (T*)out, stride, tw1,
                                                        tw2);
    } else {
      k_fused2d<T, N1, M, ALG><<<grid, NT, smem, s>>>(prm, q, philox_key(seed), field0, ring, (T*)out, stride, tw1,
                                                      tw2);
    }
  }
  e = cudaGetLastError();
  if (dstats) {
    unsigned long long h[8] = {};
    cudaMemcpyAsync(h, dstats, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(dstats);
    const double nc = (double)(h[5] ? h[5] : 1), nr = (double)(h[6] ? h[6] : 1);
    std::fprintf(stderr,
                 "[grfc tile stats] grid=%u L=%u S=%u | col tiles %llu: %.0f cyc/tile, wait %.0f | row tiles %llu: "
                 "%.0f cyc/tile, wait %.0f | ticket %.0f cyc/tile\n",
                 grid, q.L, q.S, h[5], h[0] / nc, h[2] / nc, h[6], h[1] / nr, h[3] / nr, h[4] / (nc + nr));
  }
  return e;
}

template <typename T, int N1, int M>
cudaError_t cluster_query(Fast2D& f, int cs, int nsl) {
  constexpr int NT = fused_threads<N1, M, T>();
  constexpr size_t smem = fused_smem<N1, M, T>();
  const void* fn = nsl == 2 ? (const void*)k_fused2d_cl<T, N1, M, 2> : (const void*)k_fused2d_cl<T, N1, M, 1>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)cs, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  e = cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
  if (e != cudaSuccess) return e;
  if (ncl < 1) return cudaErrorInvalidConfiguration;
  f.cluster = cs;
  f.cslots = nsl;
  f.nclusters = ncl;
  if (std::getenv("GRFC_CL_DEBUG"))
    std::fprintf(stderr, "[grfc cluster] size %d slots %d active clusters %d (%d CTAs of %d threads, smem %zu)\n", cs,
                 nsl, ncl, ncl * cs, NT, smem);
  return cudaSuccess;
}

template <typename T, int N1, int M>
cudaError_t launch_cluster(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* ws, void* out,
                           int64_t stride, cudaStream_t s) {
  using C = C_t<T>;
  constexpr int NT = fused_threads<N1, M, T>();
  constexpr size_t smem = fused_smem<N1, M, T>();
  const uint32_t ncl = (uint32_t)std::min<int64_t>(f.nclusters, nf);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)f.cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ncl * (unsigned)f.cluster, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const C* tw1 = (const C*)f.d_tw;
  const C* tw2 = tw1 + f.n1;
  LaunchScope ls("fused2d_cluster", s);
  if (f.cslots == 2)
    return cudaLaunchKernelEx(&cfg, k_fused2d_cl<T, N1, M, 2>, make_params(f), philox_key(seed), field0, (uint32_t)nf,
                              (C*)ws, (T*)out, stride, tw1, tw2);
  return cudaLaunchKernelEx(&cfg, k_fused2d_cl<T, N1, M, 1>, make_params(f), philox_key(seed), field0, (uint32_t)nf,
                            (C*)ws, (T*)out, stride, tw1, tw2);
}

}  // namespace grfc
