// Fused power-of-two 3D path (BASELINE config c4: 512^3 fp32, Algorithm 2),
// single GPU and slab-decomposed across ranks.
//
// Formulation. With M = N2/2, the field is the plain complex FFT (exp(+), all
// axes) of the "pre-twiddled" half spectrum over (N0, N1, M):
//   Zh(k0,k1,k) = (X(k0,k1,k) + conj X(-k0,-k1,M-k))
//               + i e^{2 pi i k/N2} (X(k0,k1,k) - conj X(-k0,-k1,M-k)),
//   z = FFT+_{N0,N1,M}(Zh),  field(j0,j1,2m) + i field(j0,j1,2m+1) = z(j0,j1,m),
// (the last-axis half-complex -> real pre-twiddle, moved in front of the
// other axes' transforms: conj(FFT(y)) = FFT(conj(y(-k)))). X = conj(V) * scale
// is the reference spectrum (hermitian.cpp:128-203), evaluated cell by cell.
//
// Pass A  k_3d_colgen   tile = (k1 pair {k1, -k1}, strip of 2*CB columns k):
//         generates X for the 4*CB columns {k1,-k1} x {k, M-k} (+ the Nyquist
//         column M where k = 0), forms Zh with its fully mirrored partner via
//         shared memory, FFTs along axis 0, stores W[j0][k1 - k1_lo][k] for
//         the k1 of this rank's slab.
// (exchange) slab all-to-all: block q of rank r = W_r[j0 in slab q] — a
//         contiguous range, no packing.
// Pass B  k_3d_planes   persistent: per plane j0, column tiles (axis-1 FFT,
//         reading the received blocks) then row tiles (axis-2 FFT = row_tile,
//         writing the field rows); planes go through an L2 ring like the 2D
//         fused kernel.
#pragma once

#include "fast2d_kernels.cuh"

namespace grfc {

// Pass-A plan: E elements per thread, CB columns per side, radices.
template <int N, typename T>
struct ColPlan3 {
  static constexpr int E = 0;
};
#define GRFC_PLAN3(N, TT, E_, X_, ...) \
  template <>                          \
  struct ColPlan3<N, TT> {             \
    static constexpr int E = E_;       \
    static constexpr int X = X_;       \
    using R = Radices<__VA_ARGS__>;    \
  };
GRFC_PLAN3(128, float, 16, 4, 16, 8)
GRFC_PLAN3(256, float, 16, 4, 16, 16)
#ifndef GRFC_COL3_512_X
#define GRFC_COL3_512_X 4
#endif
GRFC_PLAN3(512, float, 16, GRFC_COL3_512_X, 16, 16, 2)
GRFC_PLAN3(1024, float, 16, 4, 16, 16, 4)
GRFC_PLAN3(128, double, 16, 2, 16, 8)
GRFC_PLAN3(256, double, 16, 2, 16, 16)
GRFC_PLAN3(512, double, 16, 2, 16, 16, 2)
GRFC_PLAN3(1024, double, 16, 2, 16, 16, 4)
#undef GRFC_PLAN3

// Strip-blocked W columns in 3D (as wpos in the 2D kernels): pass A stores the 2 CB
// columns {s CB + c}, {M - s CB - c} of a (j0, k1) row as one contiguous run at
// s 2CB + side CB + c; pass B's column tiles work on positions (the axis-1 FFT does not
// depend on which column it holds) and its row tiles load through wpos.
#ifndef GRFC_SHF2_3D
#define GRFC_SHF2_3D 1
#endif
#ifndef GRFC_WPERM3
#define GRFC_WPERM3 1
#endif
template <typename T>
constexpr int w3_perm_cb() {
  return (GRFC_WPERM3 && sizeof(T) == 4) ? 4 : 0;
}

template <int N0, typename T>
constexpr int colgen3_threads() {
  return 4 * ColPlan3<N0, T>::X * (N0 / ColPlan3<N0, T>::E);
}

struct F3Params {
  int n0, n1, n2, m, hd;  // hd = M + 1
  double wstep[3];
  float f_wstep[3], f_sqrt_c, f_ell2, f_nhalf_alpha, f_gauss_k, f_scale;
  double sqrt_c, alpha, ell, scale;
  uint64_t uh;
  int family, alg;
  DensityDesc D;
  GridDesc g;
};

template <typename T>
__device__ __forceinline__ T sqrt_g3(const F3Params& p, int k0, int k1, int k2) {
  const int w0i = k0 <= p.n0 / 2 ? k0 : k0 - p.n0, w1i = k1 <= p.n1 / 2 ? k1 : k1 - p.n1,
            w2i = k2 <= p.n2 / 2 ? k2 : k2 - p.n2;
  if (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV) {
    if constexpr (sizeof(T) == 4) {
      const float a = (float)w0i * p.f_wstep[0], b = (float)w1i * p.f_wstep[1], c = (float)w2i * p.f_wstep[2];
      const float s = a * a + b * b + c * c;
      if (p.family == GRFC_DENSITY_GAUSSIAN_COV) return p.f_sqrt_c * ex2_approx(p.f_gauss_k * s);
      return p.f_sqrt_c * ex2_approx(p.f_nhalf_alpha * lg2_approx(1.0f + p.f_ell2 * s));
    } else {
      const double a = w0i * p.wstep[0], b = w1i * p.wstep[1], c = w2i * p.wstep[2];
      const double s = a * a + b * b + c * c;
      if (p.family == GRFC_DENSITY_GAUSSIAN_COV) return p.sqrt_c * exp(-0.25 * p.ell * p.ell * s);
      return p.sqrt_c * pow(1.0 + p.ell * p.ell * s, -0.5 * p.alpha);
    }
  }
  int64_t kw[3] = {w0i, w1i, w2i};
  return sqrt_gamma<T>(p.g, p.D, kw, ((int64_t)k0 * p.n1 + k1) * p.hd + k2);
}

// X(K) = conj(w(K)) sqrt(g) scale for any half-lattice cell (generic rules).
template <typename T>
__device__ __forceinline__ C_t<T> gen_cell3(const F3Params& p, int k0, int k1, int k2, const PhiloxKey& key,
                                            uint64_t field) {
  using C = C_t<T>;
  const int64_t k[3] = {k0, k1, k2};
  const int64_t h = ((int64_t)k0 * p.n1 + k1) * p.hd + k2;
  const C w = philox_cell_noise<T>(p.g, p.alg, k, h, key, field);
  const T m = sqrt_g3<T>(p, k0, k1, k2) * (T)p.scale;
  return mk<C>(w.x * m, -w.y * m);
}

// Pass A. Slots: h in {0: k1, 1: -k1}, side in {L: k, R: M-k}, c < CB;
// slot = h*2CB + side*CB + c. Zh partner of (h, side, c) is (1-h, 1-side, c);
// strip 0 exceptions: column 0's partner is the Nyquist column M of -k1 (kept
// in an extra shared column per h), column M/2's partner is (1-h, R, 0).
// Resident pass-A / pass-B CTAs per SM the fp32 kernels are compiled for
// (register budget; fp64 lets ptxas choose). 512^3 fp32: pass A 2 CTAs of 512
// threads at 64 registers (0.599 -> 0.515 ms), pass B 4 CTAs at 64 registers
// (0.521 -> 0.432 ms), both without spills.
#ifndef GRFC_COLGEN3_MINB
#define GRFC_COLGEN3_MINB 2
#endif
#ifndef GRFC_PLANES_MINB
#define GRFC_PLANES_MINB 4
#endif
// (capped so every thread keeps >= 64 registers; plans with 32-element rows keep
// ptxas's choice)
constexpr int minb_cap(int want, int threads) {
  return want < 65536 / (threads * 64) ? want : 65536 / (threads * 64);
}
template <typename T, int N0>
constexpr int colgen3_min_blocks() {
  return sizeof(T) == 4 ? minb_cap(GRFC_COLGEN3_MINB, colgen3_threads<N0, T>()) : 1;
}
template <typename T, int N1, int M>
constexpr int planes_min_blocks() {
  return (sizeof(T) == 4 && RowPlan<M, T>::E <= 16 && ColPlan<N1, T>::E <= 16)
             ? minb_cap(GRFC_PLANES_MINB, col_threads<N1, T>())
             : 0;
}
template <typename T, int N0, int ALG>
__global__ void __launch_bounds__(colgen3_threads<N0, T>(), colgen3_min_blocks<T, N0>())
    k_3d_colgen(F3Params p, PhiloxKey key, uint64_t fld, C_t<T>* __restrict__ W, int k1_lo, int k1_cnt,
                int a_lo0, int a_n0, int a_lo1, const C_t<T>* __restrict__ tw0, const C_t<T>* __restrict__ tw2) {
  using C = C_t<T>;
  using PL = ColPlan3<N0, T>;
  constexpr int E = PL::E, CB = PL::X, SLOTS = 4 * CB, TT = N0 / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  constexpr int PITCH = SLOTS + 2;  // + Nyquist columns of k1 and -k1
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  const int strips = p.m / (2 * CB);
  // tile rows a (quad {k1 = a, k1 = -a}): only those with a row in the rank's slab
  // [k1_lo, k1_lo + k1_cnt), as at most two intervals [a_lo0, +a_n0), [a_lo1, ...)
  const int ai = (int)(blockIdx.x / (unsigned)strips), s = (int)(blockIdx.x % (unsigned)strips);
  const int a = ai < a_n0 ? a_lo0 + ai : a_lo1 + (ai - a_n0);
  // (pass A with its final radix-2 stage on shuffles, as pass B's column tiles: no change,
  // 0.398 vs 0.400 ms — it is not bound by its exchanges)
  const int tid = threadIdx.x, slot = tid % SLOTS, j = tid / SLOTS;
  const int h = slot / (2 * CB), side = (slot / CB) & 1, c = slot % CB;
  const int k1 = h == 0 ? a : (p.n1 - a) % p.n1;
  const int kk = s * CB + c;
  const int col = side == 0 ? kk : (kk == 0 ? p.m / 2 : p.m - kk);
  const bool zero_col = side == 0 && kk == 0, mid_col = side == 1 && kk == 0;

  // generation (rolled loop): X(k0, k1, col) for k0 = j + t TT
  const bool fast = ALG == GRFC_ONE_FFT_OVERWRITE && sizeof(T) == 4 && col != 0 && col != p.m;
  // per-CTA axis-0 density table (fp32 Matern / Gaussian)
  __shared__ float s_q0[sizeof(T) == 4 ? N0 : 1];
  const float* q0 = nullptr;
  if constexpr (sizeof(T) == 4) {
    if (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV) {
      for (int k = threadIdx.x; k < N0; k += blockDim.x) {
        const int w0i = k <= p.n0 / 2 ? k : k - p.n0;
        const float a0 = (float)w0i * p.f_wstep[0];
        s_q0[k] = p.family == GRFC_DENSITY_MATERN ? p.f_ell2 * a0 * a0 : ex2_approx(p.f_gauss_k * a0 * a0);
      }
      __syncthreads();
      q0 = s_q0;
    }
  }
  if (fast && q0) {
    // interior column, Matern / Gaussian: rows k0 and k0 + N0/2 are units u and
    // u + Uh (one Philox call); the (k1, col) part of |w|^2 is per-thread and the
    // k0 part comes from the per-CTA table q0 (as the 2D column tile's rowq):
    //   Matern   q0 = ell^2 w0^2:                 m = ex2(-alpha/2 lg2(A + q0) + lg2(sqrt_c K))
    //   Gaussian q0 = ex2(-ell^2 w0^2/4 log2 e):  m = B q0
    const float K = p.f_scale * 0.70710678118654752440f;  // sqrt_g3 includes sqrt(c)
    const int w1i = k1 <= p.n1 / 2 ? k1 : k1 - p.n1, w2i = col <= p.n2 / 2 ? col : col - p.n2;
    const float b = (float)w1i * p.f_wstep[1], cc = (float)w2i * p.f_wstep[2], bc2 = b * b + cc * cc;
    const bool matern = p.family == GRFC_DENSITY_MATERN;
    const float A = 1.0f + p.f_ell2 * bc2, B = p.f_sqrt_c * K * ex2_approx(p.f_gauss_k * bc2);
    const float lgK = lg2_approx(p.f_sqrt_c * K);
#pragma unroll 4
    for (int t = 0; t < E / 2; ++t) {
      const int k0 = j + t * TT;
      const uint4 r = philox_draw(key, fld, (uint64_t)(((uint32_t)k0 * p.n1 + k1) * p.hd + col));
      float rad0, s0, c0, rad1, s1, c1;
      box_muller_parts_f32(r.x, r.y, rad0, s0, c0);
      box_muller_parts_f32(r.z, r.w, rad1, s1, c1);
      const float qa = q0[k0], qb = q0[k0 + N0 / 2];
      const float m0 = matern ? ex2_approx(__fmaf_rn(p.f_nhalf_alpha, lg2_approx(A + qa), lgK)) : B * qa;
      const float m1 = matern ? ex2_approx(__fmaf_rn(p.f_nhalf_alpha, lg2_approx(A + qb), lgK)) : B * qb;
      const float g0 = rad0 * m0, g1 = rad1 * m1;
      sm[k0 * PITCH + slot] = mk<C>((T)(g0 * c0), (T)(-g0 * s0));
      sm[(k0 + N0 / 2) * PITCH + slot] = mk<C>((T)(g1 * c1), (T)(-g1 * s1));
    }
  } else if (fast) {
    // interior column, other families
    const float K = p.f_scale * 0.70710678118654752440f;  // sqrt_g3 includes sqrt(c)
#pragma unroll 2
    for (int t = 0; t < E / 2; ++t) {
      const int k0 = j + t * TT;
      float a0, b0, a1, b1;
      unit_quad_f32(key, fld, (uint64_t)(((uint32_t)k0 * p.n1 + k1) * p.hd + col), a0, b0, a1, b1);
      const float m0 = sqrt_g3<float>(p, k0, k1, col) * K, m1 = sqrt_g3<float>(p, k0 + N0 / 2, k1, col) * K;
      sm[k0 * PITCH + slot] = mk<C>((T)(a0 * m0), (T)(-b0 * m0));
      sm[(k0 + N0 / 2) * PITCH + slot] = mk<C>((T)(a1 * m1), (T)(-b1 * m1));
    }
  } else {
#pragma unroll 1
    for (int t = 0; t < E; ++t) {
      const int k0 = j + t * TT;
      sm[k0 * PITCH + slot] = gen_cell3<T>(p, k0, k1, col, key, fld);
      if (zero_col) sm[k0 * PITCH + SLOTS + h] = gen_cell3<T>(p, k0, k1, p.m, key, fld);
    }
  }
  __syncthreads();
  // stage-0 inputs: Zh(k0) from X(k0) and the mirrored partner X(-k0)
  const int pslot = mid_col ? ((1 - h) * 2 * CB + CB) : zero_col ? SLOTS + (1 - h) : ((1 - h) * 2 * CB + (1 - side) * CB + c);
  const C w = __ldg(&tw2[col]);  // e^{2 pi i col / N2}
  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i) {
      const int k0 = j + b * TT + i * (N0 / R0);
      const C X = sm[k0 * PITCH + slot], P = sm[((N0 - k0) & (N0 - 1)) * PITCH + pslot];
      const C sum = mk<C>(X.x + P.x, X.y - P.y), dif = mk<C>(X.x - P.x, X.y + P.y);
      const C t = cmul(w, dif);
      v[b * R0 + i] = mk<C>(sum.x - t.y, sum.y + t.x);
    }
  __syncthreads();
  struct Ex3 {
    C* s;
    int slot;
    __device__ __forceinline__ void put(int e, C x) { s[e * PITCH + slot] = x; }
    __device__ __forceinline__ C get(int e) const { return s[e * PITCH + slot]; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
  } ex{sm, slot};
  line_fft<N0, E, +1>(v, j, tw0, 1, ex, typename PL::R{});
  const int kl = k1 - k1_lo;
  static_assert(w3_perm_cb<T>() == 0 || w3_perm_cb<T>() == CB, "strip-blocked W needs the pass-A CB");
  const int wcol = w3_perm_cb<T>() ? s * 2 * CB + side * CB + c : col;
  const bool store = kl >= 0 && kl < k1_cnt && !(h == 1 && k1 == a);  // h = 1 duplicates k1 in {0, N1/2}
  if (store) {
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int i = 0; i < RL; ++i) {
        const int j0 = j + b * TT + i * (N0 / RL);
        W[((int64_t)j0 * k1_cnt + kl) * p.m + wcol] = v[b * RL + i];
      }
  }
}

// Plain column tile (axis-1 FFT) of one plane: SLOTS consecutive columns,
// rows fetched through the slab block layout, output to a ring slot.
template <typename T, int N1>
__device__ __forceinline__ void c2c_col_tile(const C_t<T>* __restrict__ src, int j0l, int n0_per, int n1_per, int m,
                                             int s, C_t<T>* __restrict__ dst, const C_t<T>* __restrict__ tw1,
                                             unsigned char* smem_raw, const C_t<T>* t16 = nullptr) {
  using C = C_t<T>;
  using PL = ColPlan<N1, T>;
  constexpr int E = PL::E, SLOTS = 2 * PL::X, TT = N1 / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  // SHF2 (512-point columns): the final radix-2 stage on shuffles, as in the 2D column tile
  constexpr bool SHF2 = col_shf2<N1, T>() && GRFC_SHF2_3D;
  const int tid = threadIdx.x, slot = tid % SLOTS, j = SHF2 ? shf2_team_pos(tid) : tid / SLOTS;
  const int col = s * SLOTS + slot;
  C v[E];
  if (n1_per == N1) {
    // one rank: the plane is one contiguous [k1][k] block — one pointer, and with
    // the compile-time m of the persistent kernel every load is pointer + immediate
    const C* __restrict__ b0 = src + ((int64_t)j0l * N1 + j) * m + col;
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int i = 0; i < R0; ++i) v[b * R0 + i] = __ldcs(b0 + (int64_t)(b * TT + i * (N1 / R0)) * m);
  } else {
    // slab blocks: row k1 lives in the block of rank k1 / n1_per (n1_per = N1 /
    // world is a power of two: shifts and masks, no integer division)
    // (32-bit element offsets: a rank's receive buffer holds < 2^31 elements for
    // every pow2-3d plan, N <= 1024)
    const int sh = __ffs(n1_per) - 1;
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int i = 0; i < R0; ++i) {
        const uint32_t k1 = (uint32_t)(j + b * TT + i * (N1 / R0));
        const uint32_t r = k1 >> sh, k1l = k1 & (uint32_t)(n1_per - 1);
        v[b * R0 + i] = __ldcs(&src[((r * (uint32_t)n0_per + (uint32_t)j0l) * (uint32_t)n1_per + k1l) * (uint32_t)m + col]);
      }
  }
  std::conditional_t<col_padded<N1, T>(), ColExPad<C, SLOTS>, ColEx<C, SLOTS>> ex{reinterpret_cast<C*>(smem_raw), slot};
  if constexpr (HasTw16<decltype(ex)>::value) ex.tw16 = t16;
  if constexpr (SHF2) {
    run_stages<N1, E, +1, 1, 16, 16>(v, j, tw1, 1, ex);
    shf2_stage<T>(v, j, tw1);
  } else {
    line_fft<N1, E, +1>(v, j, tw1, 1, ex, typename PL::R{});
  }
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) __stcg(&dst[(int64_t)(j + b * TT + i * (N1 / RL)) * m + col], v[b * RL + i]);
}

template <int N1, int M, typename T>
constexpr int rows3_per_tile() {
  return rows_per_tile<N1, M, T>();
}

// Pass B: persistent over this rank's planes (same ticket/ring scheme as
// k_fused2d: C(p) tiles = axis-1 strips, R(p) tiles = rows).
template <typename T, int N1, int M>
__global__ void __launch_bounds__(col_threads<N1, T>(), planes_min_blocks<T, N1, M>())
    k_3d_planes(F2Sched q, const C_t<T>* __restrict__ src, int n0_per, int n1_per, C_t<T>* __restrict__ ring,
                T* __restrict__ out, const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_ticket;
  constexpr int RPT = rows_per_tile<N1, M, T>();
  __shared__ C_t<T> s_tw16[GRFC_TW16 && sizeof(T) == 4 ? 240 : 1];
  const C_t<T>* t16 = init_tw16<T>(s_tw16, tw2, 2 * M);
  const uint64_t slot_elems = (uint64_t)N1 * M;
  const uint32_t G = q.strips + q.rtiles, pro = q.L * q.strips, nfull = q.F - q.L;
  const uint32_t total = q.F * G;
  uint32_t next_ticket = 0;
  if (threadIdx.x == 0) next_ticket = atomicAdd(q.ticket, 1u);
  for (;;) {
    if (threadIdx.x == 0) {
      s_ticket = next_ticket;
      if (next_ticket < total) next_ticket = atomicAdd(q.ticket, 1u);
    }
    __syncthreads();
    uint32_t t = s_ticket;
    if (t >= total) break;
    bool col;
    uint32_t f, idx;
    if (t < pro) {
      col = true;
      f = t / q.strips;
      idx = t % q.strips;
    } else if ((t -= pro) < nfull * G) {
      const uint32_t g = t / G, r = t % G;
      col = r < q.strips;
      f = col ? g + q.L : g;
      idx = col ? r : r - q.strips;
    } else {
      t -= nfull * G;
      col = false;
      f = nfull + t / q.rtiles;
      idx = t % q.rtiles;
    }
    const uint32_t slot = f % q.S, use = f / q.S;
    C_t<T>* Wp = ring + slot * slot_elems;
    if (col) {
      wait_geq(&q.row_done[slot], use * q.rtiles);
      c2c_col_tile<T, N1>(src, (int)f, n0_per, n1_per, M, (int)idx, Wp, tw1, smem_raw, t16);
      signal_done(&q.col_done[slot]);
    } else {
      wait_geq(&q.col_done[slot], (use + 1) * q.strips);
      row_tile<T, M, RPT, fused_threads<N1, M, T>(), NoHook, w3_perm_cb<T>()>(
          Wp, (int)idx * RPT, N1, out + (int64_t)f * N1 * (2 * M), tw2, smem_raw, nullptr, NoHook{}, t16);
      signal_done(&q.row_done[slot]);
    }
  }
}

template <int N1, int M, typename T>
constexpr size_t planes_smem() {
  using C = C_t<T>;
  constexpr size_t a = (size_t)(col_padded<N1, T>() ? colx_rows(N1) : N1) * 2 * ColPlan<N1, T>::X * sizeof(C);
  constexpr size_t b = (size_t)rows_per_tile<N1, M, T>() * row_pitch<M, C>() * sizeof(C);
  return a > b ? a : b;
}

}  // namespace grfc
