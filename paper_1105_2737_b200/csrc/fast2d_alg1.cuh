// Fused power-of-two 2D path for Algorithm 1 (two-FFT, the reference's
// synth.cpp:81-116): white noise -> exp(+) transform -> x sqrt(g) sqrt((2pi)^d P/|A|)
// -> exp(-) transform / P -> real part.
//
// Tiles (persistent, one launch per batch, per-field ring slot in L2):
//   R1  rows: noise z(j1, m) = (x(j1, 2m), x(j1, 2m+1)) from Philox units
//       u = j1 M + m (rows j1 and j1 + N1/2 share one call), exp(+) M-point
//       row FFT -> Zf(j1, k) into the slot.
//   C   column pair (k, M-k): R2C split (X = (Zf_k + conj Zf_{M-k})/2
//       - i e^{2pi i k/N2} (Zf_k - conj Zf_{M-k})/2; k = 0 packs DC + i Nyquist),
//       exp(+) column FFT, x sqrt(g)*scale (packed column unpacked through its
//       mirror row), then the C2R pre-twiddle of the exp(-) inverse written as
//       an exp(+) transform of conj(V):
//         Zh(k1,k) = (conj V(k1,k) + V(-k1,M-k)) + i e^{2pi i k/N2} (conj V(k1,k) - V(-k1,M-k)),
//       exp(+) column FFT -> Z(j1, k) in place.
//   R2  rows: row_tile (M-point exp(+) FFT -> the field rows), as Algorithm 2.
#pragma once

#include <atomic>

#include "fast2d_kernels.cuh"

namespace grfc {

struct F2Sched3 {
  uint32_t* ticket;
  uint32_t* r1_done;   // [S]
  uint32_t* col_done;  // [S]
  uint32_t* row_done;  // [S]
  uint32_t F, L, S, g1, gc, g2;
};

template <typename T>
__device__ __forceinline__ C_t<T> half_c(C_t<T> a) {
  return mk<C_t<T>>(a.x * (T)0.5, a.y * (T)0.5);
}

// Strip-blocked W columns (wpos) in the Algorithm-1 kernel: the C tile's loads and stores
// of its 2 CB columns become one contiguous run per row; R1 stores and R2 loads go
// through wpos.
#ifndef GRFC_ALG1_WPERM
#define GRFC_ALG1_WPERM 1
#endif
template <int N1, typename T>
constexpr int alg1_perm_cb() {
  return (GRFC_ALG1_WPERM && sizeof(T) == 4) ? ColPlan<N1, T>::X : 0;
}

// R1: rows r0 + p and r0 + p + N1/2 for p < RPT/2 (Philox pair sharing).
template <typename T, int N1, int M, int RPT>
__device__ __forceinline__ void r1_tile(const F2Params& p, const PhiloxKey& key, uint64_t fld, int r0,
                                        C_t<T>* __restrict__ Wf, const C_t<T>* __restrict__ tw2,
                                        unsigned char* smem_raw, uint32_t* sig = nullptr,
                                        const C_t<T>* t16 = nullptr) {
  using C = C_t<T>;
  using PL = RowPlan<M, T>;
  constexpr int E = PL::E, TT = M / E, H = RPT / 2, PITCH = row_pitch<M, C>();
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  C* sm = reinterpret_cast<C*>(smem_raw);
  const uint64_t uh = (uint64_t)(N1 / 2) * M;
  for (int it = threadIdx.x; it < H * M; it += blockDim.x) {
    const int pr = it / M, m = it - pr * M;
    const uint64_t u = (uint64_t)(r0 + pr) * M + m;
    T a0, b0, a1, b1;
    if constexpr (sizeof(T) == 4) {
      unit_quad_f32(key, fld, u, a0, b0, a1, b1);
    } else {
      unit_pair<T>(key, fld, u, uh, a0, b0);
      unit_pair<T>(key, fld, u + uh, uh, a1, b1);
    }
    sm[pr * PITCH + RowEx<C>::pad(m)] = mk<C>(a0, b0);
    sm[(pr + H) * PITCH + RowEx<C>::pad(m)] = mk<C>(a1, b1);
  }
  __syncthreads();
  if (sig && threadIdx.x == 0) red_release_add(sig, 1u);  // the CTA's previous tile
  const int tid = threadIdx.x, rl = tid / TT, j = tid % TT;
  const bool live = rl < RPT;
  const int rs = live ? rl : 0;
  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i) v[b * R0 + i] = sm[rs * PITCH + RowEx<C>::pad(j + b * TT + i * (M / R0))];
  __syncthreads();
  // the row's team is a half warp: warp-level exchange (as row_tile)
  constexpr bool WARP = GRFC_ROW_WARPSYNC && TT <= 32 && 32 % TT == 0;
  RowEx<C, false, WARP> ex{sm + rs * PITCH, live, 0, t16};
  line_fft<M, E, +1>(v, j, tw2, 2, ex, typename PL::R{});
  if (!live) return;
  const int row = rl < H ? r0 + rl : r0 + (rl - H) + N1 / 2;
  C* o = Wf + (int64_t)row * M;
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) __stcg(&o[wpos(j + b * TT + i * (M / RL), M, alg1_perm_cb<N1, T>())], v[b * RL + i]);
}

// C: forward column FFT, spectral scaling, inverse pre-twiddle, column FFT.
template <typename T, int N1>
__device__ __forceinline__ void alg1_col_tile(const F2Params& p, int s, C_t<T>* __restrict__ Wf,
                                              const C_t<T>* __restrict__ tw1, const C_t<T>* __restrict__ tw2,
                                              unsigned char* smem_raw,
                                              uint32_t* sig = nullptr, const C_t<T>* t16 = nullptr) {
  using C = C_t<T>;
  using PL = ColPlan<N1, T>;
  constexpr int E = PL::E, CB = PL::X, SLOTS = 2 * CB, TT = N1 / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  // (the shuffle final stage of the Algorithm-2 column tile, SHF2, measured slower here:
  // 153 -> 147 Gpts/s at this kernel's 80 registers / 3 CTAs per SM)
  const int tid = threadIdx.x, slot = tid % SLOTS, j = tid / SLOTS, pslot = slot ^ CB;
  bool packed, mid;
  const int col = slot_column(s, slot, CB, p.m, packed, mid);
  const int pcol = p.m - col;  // Zh partner column (for packed: M)
  // strip-blocked W (wpos): this tile's 2 CB columns are one contiguous run per row
  const int wcol = alg1_perm_cb<N1, T>() ? s * SLOTS + slot : col;
  C* sm = reinterpret_cast<C*>(smem_raw);
  const T half = (T)0.5;
  // 1. Zf columns -> smem [j1][slot]
#pragma unroll 4
  for (int t = 0; t < E; ++t) {
    const int j1 = j + t * TT;
    sm[j1 * SLOTS + slot] = __ldcg(&Wf[(int64_t)j1 * p.m + wcol]);
  }
  __syncthreads();
  if (sig && threadIdx.x == 0) red_release_add(sig, 1u);  // the CTA's previous tile
  // 2. R2C split into the stage-0 registers
  const C w = __ldg(&tw2[col]);  // e^{2 pi i col / N2}
  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i) {
      const int j1 = j + b * TT + i * (N1 / R0);
      const C A = sm[j1 * SLOTS + slot];
      C X;
      if (packed) {
        X = mk<C>(A.x + A.y, A.x - A.y);  // X(j1,0) + i X(j1,M)
      } else if (mid) {
        X = A;
      } else {
        const C B = sm[j1 * SLOTS + pslot];
        const C sum = mk<C>(A.x + B.x, A.y - B.y), dif = mk<C>(A.x - B.x, A.y + B.y);
        const C t = cmul(w, dif);
        X = mk<C>((sum.x + t.y) * half, (sum.y - t.x) * half);
      }
      v[b * R0 + i] = X;
    }
  __syncthreads();
  std::conditional_t<col_padded<N1, T>(), ColExPad<C, SLOTS>, ColEx<C, SLOTS>> ex{sm, slot};
  if constexpr (HasTw16<decltype(ex)>::value) ex.tw16 = t16;
  // Both column FFTs run through ONE copy of the transform code (a rolled
  // two-pass loop): the kernel's three tile types otherwise overflow the
  // instruction cache (ncu: "no instruction" stalls).
#pragma unroll 1
  for (int pass = 0;; ++pass) {
    line_fft<N1, E, +1>(v, j, tw1, 1, ex, typename PL::R{});
    if (pass == 1) break;
    // 3. U -> smem in natural row order
  #pragma unroll
    for (int b = 0; b < E / RL; ++b)
  #pragma unroll
      for (int i = 0; i < RL; ++i) sm[(j + b * TT + i * (N1 / RL)) * SLOTS + slot] = v[b * RL + i];
    __syncthreads();
    // 4. V = U sqrt(g) scale, then Zh with the mirrored partner V(-k1, M-col).
    const T sc = (T)p.scale;
    // fp32: sqrt(g) x scale from the plan's table (always present for fp32 Algorithm 1)
    const float* __restrict__ sgk = p.sg + (packed ? 0 : col);
    const float* __restrict__ sgm = p.sg + (packed ? p.m : (mid ? col : pcol));
    const int uslot = (packed || mid) ? slot : pslot;
  #pragma unroll
    for (int b = 0; b < E / R0; ++b)
  #pragma unroll
      for (int i = 0; i < R0; ++i) {
        const int k1 = j + b * TT + i * (N1 / R0), km = (N1 - k1) & (N1 - 1);
        C Vk, Vm;
        if constexpr (sizeof(T) == 4) {
          const float mk_ = __ldg(&sgk[k1 * p.hd]), mm_ = __ldg(&sgm[km * p.hd]);
          const C Uk = sm[k1 * SLOTS + slot], Um = sm[km * SLOTS + uslot];
          if (packed) {
            // F0(k1) = (U(k1) + conj U(-k1))/2 ; FM(-k1) = -i (U(-k1) - conj U(k1))/2
            Vk = cscale(mk<C>((Uk.x + Um.x) * half, (Uk.y - Um.y) * half), (T)mk_);
            Vm = cscale(mk<C>((Um.y + Uk.y) * half, -(Um.x - Uk.x) * half), (T)mm_);
          } else {
            Vk = cscale(Uk, (T)mk_);
            Vm = cscale(Um, (T)mm_);
          }
        } else if (packed) {
          const C Uk = sm[k1 * SLOTS + slot], Um = sm[km * SLOTS + slot];
          // F0(k1) = (U(k1) + conj U(-k1))/2 ; FM(-k1) = -i (U(-k1) - conj U(k1))/2
          const C F0k = mk<C>((Uk.x + Um.x) * half, (Uk.y - Um.y) * half);
          const C FMm = mk<C>((Um.y + Uk.y) * half, -(Um.x - Uk.x) * half);
          Vk = cscale(F0k, sqrt_g2<T>(p, k1, 0) * sc);
          Vm = cscale(FMm, sqrt_g2<T>(p, km, p.m) * sc);
        } else {
          Vk = cscale(sm[k1 * SLOTS + slot], sqrt_g2<T>(p, k1, col) * sc);
          Vm = cscale(sm[km * SLOTS + (mid ? slot : pslot)], sqrt_g2<T>(p, km, mid ? col : pcol) * sc);
        }
        const C cV = cconj(Vk);
        const C sum = cadd(cV, Vm), dif = csub(cV, Vm);
        const C t = cmul(w, dif);
        v[b * R0 + i] = mk<C>(sum.x - t.y, sum.y + t.x);
      }
    __syncthreads();
  }
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) __stcg(&Wf[(int64_t)(j + b * TT + i * (N1 / RL)) * p.m + wcol], v[b * RL + i]);
}

#ifndef GRFC_ALG1_RES1
#define GRFC_ALG1_RES1 1
#endif
#ifndef GRFC_ALG1_MINB
#define GRFC_ALG1_MINB 3
#endif
// Three resident 256-thread CTAs per SM for the fp32 shapes (80 registers, no
// spills now that the column tile reads sqrt(g) from the plan's table: 512 x 512
// Alg 1 136 Gpts/s vs 128 with four CTAs at 64 registers and spills); larger
// blocks / fp64 let ptxas choose.
template <int N1, int M, typename T>
constexpr int alg1_min_blocks() {
  return (sizeof(T) == 4 && fused_threads<N1, M, T>() <= 256) ? GRFC_ALG1_MINB : 0;
}
template <typename T, int N1, int M>
__global__ void __launch_bounds__(fused_threads<N1, M, T>(), alg1_min_blocks<N1, M, T>())
    k_fused2d_alg1(F2Params p, F2Sched3 q, PhiloxKey key, uint64_t field0, C_t<T>* __restrict__ ring,
                   T* __restrict__ out, int64_t out_stride, const C_t<T>* __restrict__ tw1,
                   const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int RPT = rows_per_tile<N1, M, T>();
  __shared__ C_t<T> s_tw16[GRFC_TW16 && sizeof(T) == 4 ? 240 : 1];
  const C_t<T>* t16 = init_tw16<T>(s_tw16, tw2, 2 * M);
  const uint64_t slot_elems = (uint64_t)N1 * M;
  const uint32_t L = q.L, F = q.F, g1 = q.g1, gc = q.gc, g2 = q.g2;
  // ticket ranges (L <= F/2): [0,L): R1 | [L,2L): R1 C | [2L,F): R1 C R2 | [F,F+L): C R2 | [F+L,F+2L): R2
  const uint32_t nA = L * g1, nB = L * (g1 + gc), nC = (F - 2 * L) * (g1 + gc + g2), nD = L * (gc + g2);
  const uint32_t total = F * (g1 + gc + g2);
  struct Tile {
    int kind;  // 0 R1, 1 C, 2 R2
    uint32_t f, idx, slot, use;
  };
  auto decode = [&](uint32_t t) {
    Tile x;
    if (t < nA) {
      x.kind = 0, x.f = t / g1, x.idx = t % g1;
    } else if ((t -= nA) < nB) {
      const uint32_t g = t / (g1 + gc), r = t % (g1 + gc);
      if (r < g1) x.kind = 0, x.f = L + g, x.idx = r;
      else x.kind = 1, x.f = g, x.idx = r - g1;
    } else if ((t -= nB) < nC) {
      const uint32_t g = t / (g1 + gc + g2), r = t % (g1 + gc + g2);
      if (r < g1) x.kind = 0, x.f = 2 * L + g, x.idx = r;
      else if (r < g1 + gc) x.kind = 1, x.f = L + g, x.idx = r - g1;
      else x.kind = 2, x.f = g, x.idx = r - g1 - gc;
    } else if ((t -= nC) < nD) {
      const uint32_t g = t / (gc + g2), r = t % (gc + g2);
      if (r < gc) x.kind = 1, x.f = F - L + g, x.idx = r;
      else x.kind = 2, x.f = F - 2 * L + g, x.idx = r - gc;
    } else {
      t -= nD;
      x.kind = 2, x.f = F - L + t / g2, x.idx = t % g2;
    }
    x.slot = x.f % q.S;
    x.use = x.f / q.S;
    return x;
  };
  // dependency of a tile: R1 reuses the slot (rows of f - S consumed), C needs
  // f's R1 tiles, R2 needs f's column tiles
  auto dep_of = [&](const Tile& x, const uint32_t*& ctr) -> uint32_t {
    if (x.kind == 0) return ctr = &q.row_done[x.slot], x.use * g2;
    if (x.kind == 1) return ctr = &q.r1_done[x.slot], (x.use + 1) * g1;
    return ctr = &q.col_done[x.slot], (x.use + 1) * gc;
  };
  // Schedule of k_fused2d: one barrier per tile, completion released inside the
  // next tile. Default (GRFC_ALG1_RES1=1): one reserved ticket, claimed at the top
  // of a tile and checked in publish() at its end with an acquire load (exposed
  // round trip; k_fused2d hides it with a mid-tile hook). GRFC_ALG1_RES1=0: two
  // reserved tickets with early relaxed dependency loads.
  uint32_t tA = total, tB = total, dep_v = 0;
  auto claim = [&]() { return atomicAdd(q.ticket, 1u); };
  // thread 0 decodes (integer divisions) and publishes the next tile
  struct Msg {
    uint32_t t, ready, kind, f, idx, slot;
  };
  __shared__ Msg s_msg;
  auto publish = [&](uint32_t t, uint32_t v) {
    Msg m{};
    m.t = t;
    m.ready = 1;
    if (t < total) {
      const Tile x = decode(t);
      m.kind = (uint32_t)x.kind, m.f = x.f, m.idx = x.idx, m.slot = x.slot;
      const uint32_t* ctr;
      const uint32_t target = dep_of(x, ctr);
      if (target) {
        if (GRFC_ALG1_RES1 && x.kind != 0) {
          m.ready = ld_acquire_u32(ctr) >= target;  // one round trip: checks and orders
        } else {
          if (v < target) v = ld_relaxed_u32(ctr);
          m.ready = v >= target;
          if (m.ready && x.kind != 0) (void)ld_acquire_u32(ctr);
        }
      }
    }
    s_msg = m;
  };
  // GRFC_ALG1_RES1: one reservation (the next ticket is claimed at the top of a
  // tile and read at its end), as k_fused2d; otherwise two reserved tickets with
  // early relaxed dependency loads.
  if (threadIdx.x == 0) {
    const uint32_t t0 = claim();
    if (!GRFC_ALG1_RES1) {
      tA = claim();
      tB = claim();
    }
    publish(t0, 0);
  }
  __syncthreads();
  uint32_t* done_ctr = nullptr;
  for (;;) {
    const Msg m = s_msg;
    if (threadIdx.x == 0) {
      if (GRFC_ALG1_RES1) {
        if (m.t < total) tA = claim();
      } else if (tA < total) {
        const uint32_t* ctr;
        dep_of(decode(tA), ctr);
        dep_v = ld_relaxed_u32(ctr);
      }
    }
    if (m.t >= total) break;
    if (!m.ready) {
      if (threadIdx.x == 0) {
        if (done_ctr) red_release_add(done_ctr, 1u);
        done_ctr = nullptr;
        const uint32_t* ctr;
        const uint32_t target = dep_of(decode(m.t), ctr);
        while (ld_relaxed_u32(ctr) < target) __nanosleep(256);
        if (m.kind != 0) (void)ld_acquire_u32(ctr);
      }
      __syncthreads();
    }
    C_t<T>* Wf = ring + m.slot * slot_elems;
    if (m.kind == 0) {
      r1_tile<T, N1, M, RPT>(p, key, field0 + m.f, (int)m.idx * (RPT / 2), Wf, tw2, smem_raw, done_ctr, t16);
      done_ctr = &q.r1_done[m.slot];
    } else if (m.kind == 1) {
      alg1_col_tile<T, N1>(p, (int)m.idx, Wf, tw1, tw2, smem_raw, done_ctr, t16);
      done_ctr = &q.col_done[m.slot];
    } else {
      row_tile<T, M, RPT, fused_threads<N1, M, T>(), NoHook, alg1_perm_cb<N1, T>()>(Wf, (int)m.idx * RPT, N1, out + (int64_t)m.f * out_stride, tw2,
                                                     smem_raw, done_ctr, NoHook{}, t16);
      done_ctr = &q.row_done[m.slot];
    }
    if (threadIdx.x == 0) {
      if (GRFC_ALG1_RES1) {
        publish(tA < total ? tA : total, 0);
      } else {
        publish(tA, dep_v);
        tA = tB;
        tB = tB < total ? claim() : total;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && done_ctr) red_release_add(done_ctr, 1u);
}

inline size_t alg1_ctr_bytes(uint32_t S) { return ((1 + 3 * (size_t)S) * 4 + 255) / 256 * 256; }

inline void alg1_geometry(int sms, int occ, int strips, int rtiles, int64_t nf, uint32_t* L, uint32_t* S,
                          uint32_t* conc) {
  // lookahead LA x (tiles all resident CTAs run at once) / (tiles per field) between
  // consecutive stages; slots = 2 lookaheads + SL x that + 2 (GRFC_ALG1_LA / _SL override)
  const char* ela = std::getenv("GRFC_ALG1_LA");
  const char* esl = std::getenv("GRFC_ALG1_SL");
  const uint32_t la = ela ? (uint32_t)std::atoi(ela) : 5u, sl = esl ? (uint32_t)std::atoi(esl) : 4u;
  const uint32_t c = (uint32_t)(sms * occ), G = (uint32_t)(strips + 2 * rtiles);
  uint32_t l = (la * c + G - 1) / G;  // + the two tickets each CTA reserves ahead
  l = l < 1 ? 1 : l;
  l = l < (uint32_t)(nf / 2) ? l : (uint32_t)(nf / 2);
  uint32_t s = 2 * l + sl * ((c + G - 1) / G) + 2;
  s = s < (uint32_t)nf ? s : (uint32_t)nf;
  *L = l;
  *S = s;
  *conc = c;
}

// (N1, M) pairs the three-tile kernel supports: R1 tiles pair rows j1 and
// j1 + N1/2, so a tile must hold an even number (>= 2) of M-point row teams.
template <typename T, int N1, int M>
constexpr bool alg1_valid() {
  return rows_per_tile<N1, M, T>() >= 2 && rows_per_tile<N1, M, T>() % 2 == 0;
}
template <typename T, int N1, int M>
cudaError_t alg1_check() {
  return alg1_valid<T, N1, M>() ? cudaSuccess : cudaErrorNotSupported;
}

template <typename T, int N1, int M>
cudaError_t launch_fused_alg1_impl(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out,
                                   int64_t stride, cudaStream_t s);

template <typename T, int N1, int M>
cudaError_t launch_fused_alg1(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out, int64_t stride,
                              cudaStream_t s) {
  if constexpr (!alg1_valid<T, N1, M>()) {
    return cudaErrorNotSupported;
  } else {
    return launch_fused_alg1_impl<T, N1, M>(f, seed, field0, nf, out, stride, s);
  }
}

template <typename T, int N1, int M>
cudaError_t launch_fused_alg1_impl(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out,
                                   int64_t stride, cudaStream_t s) {
  using C = C_t<T>;
  constexpr int NT = fused_threads<N1, M, T>(), RPT = rows_per_tile<N1, M, T>();
  constexpr size_t smem = fused_smem<N1, M, T>();
  // the smem attribute is per device: set on every launch (cheap); the occupancy
  // is cached per device ordinal
  static std::atomic<int> occ_cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  cudaFuncSetAttribute(k_fused2d_alg1<T, N1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = dev < 64 ? occ_cache[dev].load(std::memory_order_relaxed) : 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2d_alg1<T, N1, M>, NT, smem);
    if (occ < 1) occ = 1;
    if (dev < 64) occ_cache[dev].store(occ, std::memory_order_relaxed);
  }
  F2Sched3 q{};
  uint32_t conc = 0;
  alg1_geometry(f.sms, occ, M / (2 * ColPlan<N1, T>::X), N1 / RPT, nf, &q.L, &q.S, &conc);
  q.F = (uint32_t)nf;
  q.g1 = (uint32_t)(N1 / RPT);
  q.gc = (uint32_t)(M / (2 * ColPlan<N1, T>::X));
  q.g2 = (uint32_t)(N1 / RPT);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, alg1_ctr_bytes(q.S) + (size_t)q.S * N1 * M * sizeof(C), s);
  if (e != cudaSuccess) return e;
  uint32_t* ctr = (uint32_t*)ws;
  q.ticket = ctr;
  q.r1_done = ctr + 1;
  q.col_done = ctr + 1 + q.S;
  q.row_done = ctr + 1 + 2 * q.S;
  C* ring = (C*)((char*)ws + alg1_ctr_bytes(q.S));
  e = cudaMemsetAsync(ctr, 0, (1 + 3 * q.S) * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const C* tw1 = (const C*)f.d_tw;
  const C* tw2 = tw1 + f.n1;
  F2Params p = make_params(f);
  p.scale = f.s_two;
  p.f_scale = (float)f.s_two;
  const uint32_t total = q.F * (q.g1 + q.gc + q.g2);
  const uint32_t grid = total < conc ? total : conc;
  {
    LaunchScope ls("fused2d_alg1_persistent", s);
    k_fused2d_alg1<T, N1, M><<<grid, NT, smem, s>>>(p, q, philox_key(seed), field0, ring, (T*)out, stride, tw1, tw2);
  }
  e = cudaGetLastError();
  cudaFreeAsync(ws, s);
  return e;
}

}  // namespace grfc
