// Warp-synchronous fused 2D path (Algorithm 2), opt-in (GRFC_WARP=1) for N1
// in {256, 512}; measured slower than k_fused2d on c2 (1.32 vs 1.22 ms:
// CTA barrier stalls when one warp's column task is slow). Compared with
// k_fused2d (fast2d_kernels.cuh):
//
// * Column work has no CTA barrier. A warp owns the column pair (k, M-k)
//   (k in [1, M/2); task k = 0 is the pair (0, M/2)). With the last-axis
//   pre-twiddle applied at generation (fast3d_kernels.cuh formulation),
//     Zh(k1,k)    = (X(k1,k) + conj X(-k1,M-k)) + i w_k (X(k1,k) - conj X(-k1,M-k))
//     Zh(-k1,M-k) = (X(-k1,M-k) + conj X(k1,k)) + i w_{M-k} (X(-k1,M-k) - conj X(k1,k))
//   both come from the same two cells, so a lane holding rows k1 = l + 32 i
//   builds column k in natural order and column M-k in REVERSED order
//   (x'(n) = Zh(-n, M-k)); FFT(x')(j) = FFT(Zh)(-j), so the second column is
//   stored at rows -j. Rows k1 and k1 + N1/2 of both columns are Philox units
//   u, u + Uh: 2 Philox calls per 4 cells. FFT exchanges go through a
//   warp-private shared buffer with __syncwarp.
// * The intermediate is transposed, W_T[k][j1] (k < M, N1 rows): warp column
//   stores are 256 B contiguous. The row tile loads its stage-0 inputs with a
//   row-fastest lane mapping (coalesced 128 B per half warp), swaps thread
//   roles at its one shared-memory exchange, and stores the field rows
//   row-contiguous (float2/double2, 128 B per half warp).
#pragma once

#include "fast2d_kernels.cuh"

namespace grfc {

// Warp exchange: line of N elements, padded every 128 B.
template <typename C>
struct WarpEx {
  C* s;
  static constexpr int PER = 128 / (int)sizeof(C);
  __device__ __forceinline__ static int pad(int e) { return e + e / PER; }
  __device__ __forceinline__ void put(int e, C v) { s[pad(e)] = v; }
  __device__ __forceinline__ C get(int e) const { return s[pad(e)]; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
};

template <int N, typename T>
struct WarpColPlan;
template <>
struct WarpColPlan<256, float> {
  static constexpr int E = 8;
  using R = Radices<8, 8, 4>;
};
template <>
struct WarpColPlan<512, float> {
  static constexpr int E = 16;
  using R = Radices<16, 16, 2>;
};
template <>
struct WarpColPlan<256, double> {
  static constexpr int E = 8;
  using R = Radices<8, 8, 4>;
};
template <>
struct WarpColPlan<512, double> {
  static constexpr int E = 16;
  using R = Radices<16, 16, 2>;
};

constexpr int kWarpCols = 8;  // warps (column-pair tasks) per CTA
constexpr int kWarpThreads = 32 * kWarpCols;

template <int N1, typename T>
constexpr int warp_line_pitch() {
  return N1 + N1 / (128 / (int)sizeof(C_t<T>));
}

// Zh pair from the two cells XA = X(k1, k), XB = X(-k1, M-k).
template <typename C>
__device__ __forceinline__ void zh_pair(C XA, C XB, C wA, C wB, C& ZA, C& ZB) {
  {
    const C sum = mk<C>(XA.x + XB.x, XA.y - XB.y), dif = mk<C>(XA.x - XB.x, XA.y + XB.y);
    const C t = cmul(wA, dif);
    ZA = mk<C>(sum.x - t.y, sum.y + t.x);
  }
  {
    const C sum = mk<C>(XB.x + XA.x, XB.y - XA.y), dif = mk<C>(XB.x - XA.x, XB.y + XA.y);
    const C t = cmul(wB, dif);
    ZB = mk<C>(sum.x - t.y, sum.y + t.x);
  }
}

// One warp, task k (column pair). WT: this field's transposed intermediate.
template <typename T, int N1, int ALG>
__device__ __forceinline__ void warp_col_task(const F2Params& p, const PhiloxKey& key, uint64_t fld, int k,
                                              C_t<T>* __restrict__ WT, const C_t<T>* __restrict__ tw1,
                                              const C_t<T>* __restrict__ tw2, C_t<T>* wsm,
                                              const float* __restrict__ rowq) {
  using C = C_t<T>;
  using PL = WarpColPlan<N1, T>;
  constexpr int E = PL::E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  static_assert(R0 == E, "stage 0 is one butterfly per lane");
  const int l = threadIdx.x & 31;
  const int m = p.m;
  const int ca = k == 0 ? 0 : k, cb = k == 0 ? m / 2 : m - k;  // natural / reversed column
  const C wA = __ldg(&tw2[ca]), wB = __ldg(&tw2[cb]);
  // The reversed column is parked in the warp's second buffer as it is
  // generated (stage-0 layout e = i*32 + l), so only column A lives in registers.
  C* park = wsm + warp_line_pitch<N1, T>();
  C* parka = wsm;  // column A staging; reused as the FFT exchange buffer
  if (k != 0) {
    // interior pair: own draws, units (k1, col) and (k1 + N1/2, col) share a call
    if constexpr (sizeof(T) == 4) {
      const int k2a = ca, k2b = cb;  // both interior, < N2/2
      const float w2a = (float)k2a * p.f_wstep2, w2b = (float)(k2b <= p.n2 / 2 ? k2b : k2b - p.n2) * p.f_wstep2;
      const bool matern = p.family == GRFC_DENSITY_MATERN;
      const float K = p.f_sqrt_c * p.f_scale * 0.70710678118654752440f;
      const float Aa = 1.0f + p.f_ell2 * w2a * w2a, Ab = 1.0f + p.f_ell2 * w2b * w2b;
      const float Ba = K * ex2_approx(p.f_gauss_k * w2a * w2a), Bb = K * ex2_approx(p.f_gauss_k * w2b * w2b);
#pragma unroll 1
      for (int i = 0; i < E / 2; ++i) {
        const int k1 = l + 32 * i, k1h = k1 + N1 / 2;
        const int n1 = (N1 - k1) & (N1 - 1), n1h = (N1 - k1h) & (N1 - 1);  // -k1, -(k1 + N1/2)
        float a0, b0, a1, b1, c0, d0, c1, d1;
        unit_quad_f32(key, fld, (uint64_t)((uint32_t)k1 * p.hd + ca), a0, b0, a1, b1);
        // -k1 and -(k1+N1/2) = the lower of the two is the call counter
        const int lo = n1 < n1h ? n1 : n1h;
        unit_quad_f32(key, fld, (uint64_t)((uint32_t)lo * p.hd + cb), c0, d0, c1, d1);
        if (n1 != lo) {  // n1 is the upper unit: swap halves
          float t;
          t = c0, c0 = c1, c1 = t;
          t = d0, d0 = d1, d1 = t;
        }
        float ma0, ma1, mb0, mb1;  // sqrt(g) K at (k1, ca), (k1h, ca), (-k1, cb), (-k1h, cb)
        if (rowq) {
          const float q0 = rowq[k1], q1 = rowq[k1h];  // rowq is even in k1
          if (matern) {
            ma0 = K * ex2_approx(p.f_nhalf_alpha * lg2_approx(Aa + q0));
            ma1 = K * ex2_approx(p.f_nhalf_alpha * lg2_approx(Aa + q1));
            mb0 = K * ex2_approx(p.f_nhalf_alpha * lg2_approx(Ab + q0));
            mb1 = K * ex2_approx(p.f_nhalf_alpha * lg2_approx(Ab + q1));
          } else {
            ma0 = Ba * q0, ma1 = Ba * q1, mb0 = Bb * q0, mb1 = Bb * q1;
          }
        } else {
          const float r = 0.70710678118654752440f * p.f_scale;
          ma0 = (float)sqrt_g2<T>(p, k1, ca) * r, ma1 = (float)sqrt_g2<T>(p, k1h, ca) * r;
          mb0 = (float)sqrt_g2<T>(p, n1, cb) * r, mb1 = (float)sqrt_g2<T>(p, n1h, cb) * r;
        }
        const C XA0 = mk<C>(a0 * ma0, -b0 * ma0), XA1 = mk<C>(a1 * ma1, -b1 * ma1);
        const C XB0 = mk<C>(c0 * mb0, -d0 * mb0), XB1 = mk<C>(c1 * mb1, -d1 * mb1);
        C za0, za1, zb0, zb1;
        zh_pair(XA0, XB0, wA, wB, za0, zb0);
        zh_pair(XA1, XB1, wA, wB, za1, zb1);
        parka[i * 32 + l] = za0;
        parka[(i + E / 2) * 32 + l] = za1;
        park[i * 32 + l] = zb0;
        park[(i + E / 2) * 32 + l] = zb1;
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < E; ++i) {
        const int k1 = l + 32 * i, n1 = (N1 - k1) & (N1 - 1);
        const C XA = gen_cell<T, ALG>(p, k1, ca, key, fld), XB = gen_cell<T, ALG>(p, n1, cb, key, fld);
        C za, zb;
        zh_pair(XA, XB, wA, wB, za, zb);
        parka[i * 32 + l] = za;
        park[i * 32 + l] = zb;
      }
    }
  } else {
    // task 0: column 0 (partner: Nyquist column M) and column M/2 (self-partner)
#pragma unroll 1
    for (int i = 0; i < E; ++i) {
      const int k1 = l + 32 * i, n1 = (N1 - k1) & (N1 - 1);
      const C X0 = gen_cell<T, ALG>(p, k1, 0, key, fld), XM = gen_cell<T, ALG>(p, n1, m, key, fld);
      C Z0, unused;
      zh_pair(X0, XM, wA, wA, Z0, unused);
      parka[i * 32 + l] = Z0;
      const C Xh = gen_cell<T, ALG>(p, k1, m / 2, key, fld);  // Zh(-k1, M/2) = 2 conj X(k1, M/2)
      park[i * 32 + l] = mk<C>((T)2 * Xh.x, (T)-2 * Xh.y);
    }
  }
  C va[E];
#pragma unroll
  for (int i = 0; i < E; ++i) va[i] = parka[i * 32 + l];  // own lane's entries: no sync needed
  __syncwarp();
  WarpEx<C> ex{wsm};
  line_fft<N1, E, +1>(va, l, tw1, 1, ex, typename PL::R{});
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) __stcg(&WT[(int64_t)ca * N1 + l + b * 32 + i * (N1 / RL)], va[b * RL + i]);
  __syncwarp();
  C vb[E];
#pragma unroll
  for (int i = 0; i < E; ++i) vb[i] = park[i * 32 + l];
  line_fft<N1, E, +1>(vb, l, tw1, 1, ex, typename PL::R{});
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) {
      const int j1 = l + b * 32 + i * (N1 / RL);
      __stcg(&WT[(int64_t)cb * N1 + ((N1 - j1) & (N1 - 1))], vb[b * RL + i]);
    }
  __syncwarp();
}

// Row tile over the transposed intermediate: stage 0 in role A (row-fastest
// lanes, coalesced W_T loads), exchange, remaining stages in role B
// (the RowEx layout of row_tile), row-contiguous field stores.
// Row buffer pitch of the transposed row tile: one element more than the
// RowEx pitch so role-A writes (16 rows, same column) hit 16 different banks.
template <int M, typename C>
constexpr int rowT_pitch() {
  return row_pitch<M, C>() + 1;
}

template <typename T, int N1, int M, int RPT>
__device__ __forceinline__ void rowT_tile(const C_t<T>* __restrict__ WT, int r0, T* __restrict__ of,
                                          const C_t<T>* __restrict__ tw2, unsigned char* smem_raw) {
  using C = C_t<T>;
  using PL = RowPlan<M, T>;
  constexpr int E = PL::E, TT = M / E;
  constexpr int R0 = RFirst<typename PL::R>::value, RL = RLast<typename PL::R>::value;
  static_assert(RPT * TT == kWarpThreads, "row tile uses every thread");
  const int tid = threadIdx.x;
  C* sm = reinterpret_cast<C*>(smem_raw);
  // role A: row ra = tid % RPT, team index ja = tid / RPT
  const int ra = tid % RPT, ja = tid / RPT;
  C v[E];
#pragma unroll
  for (int b = 0; b < E / R0; ++b)
#pragma unroll
    for (int i = 0; i < R0; ++i)
      v[b * R0 + i] = __ldcg(&WT[(int64_t)(ja + b * TT + i * (M / R0)) * N1 + r0 + ra]);
  stage_compute<M, E, R0, 1, +1>(v, ja, tw2, 2);
  {
    RowEx<C> exa{sm + ra * rowT_pitch<M, C>()};
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int i = 0; i < R0; ++i) exa.put(stage_out_index<M, E, R0, 1>(ja, b, i), v[b * R0 + i]);
  }
  __syncthreads();
  // role B: row rb = tid / TT, j = tid % TT
  const int rb = tid / TT, j = tid % TT;
  RowEx<C> ex{sm + rb * rowT_pitch<M, C>()};
  constexpr int R1 = RNext<typename PL::R>::value;
#pragma unroll
  for (int b = 0; b < E / R1; ++b)
#pragma unroll
    for (int i = 0; i < R1; ++i) v[b * R1 + i] = ex.get(stage_in_index<M, E, R1>(j, b, i));
  __syncthreads();
  run_rest<M, E, +1, R0>(v, j, tw2, 2, ex, typename PL::R{});
  C* o = reinterpret_cast<C*>(of + (int64_t)(r0 + rb) * (2 * M));
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int i = 0; i < RL; ++i) __stcs(&o[j + b * TT + i * (M / RL)], v[b * RL + i]);
}

template <int N1, int M, typename T>
constexpr int rowsT_per_tile() {
  return kWarpThreads / (M / RowPlan<M, T>::E);
}
template <int N1, int M, typename T>
constexpr size_t fusedw_smem() {
  using C = C_t<T>;
  constexpr size_t a = (size_t)kWarpCols * 2 * warp_line_pitch<N1, T>() * sizeof(C);
  constexpr size_t b = (size_t)rowsT_per_tile<N1, M, T>() * rowT_pitch<M, C>() * sizeof(C);
  return a > b ? a : b;
}

#ifndef GRFC_WARP_MINB
#define GRFC_WARP_MINB 3
#endif
template <typename T, int N1, int M>
__global__ void __launch_bounds__(kWarpThreads, GRFC_WARP_MINB)
    k_fused2d_w(F2Params p, F2Sched q, PhiloxKey key, uint64_t field0, C_t<T>* __restrict__ ring,
                T* __restrict__ out, int64_t out_stride, const C_t<T>* __restrict__ tw1,
                const C_t<T>* __restrict__ tw2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_ticket;
  __shared__ float s_rowq[N1];
  constexpr int RPT = rowsT_per_tile<N1, M, T>();
  const uint64_t slot_elems = (uint64_t)N1 * M;
  const bool table = sizeof(T) == 4 && (p.family == GRFC_DENSITY_MATERN || p.family == GRFC_DENSITY_GAUSSIAN_COV);
  if (table) fused2d_row_table<N1>(p, s_rowq);
  const uint32_t G = q.strips + q.rtiles, pro = q.L * q.strips, nfull = q.F - q.L;
  const uint32_t total = q.F * G;
  const int warp = threadIdx.x >> 5;
  C_t<T>* wsm = reinterpret_cast<C_t<T>*>(smem_raw) + warp * 2 * warp_line_pitch<N1, T>();
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
    C_t<T>* WT = ring + slot * slot_elems;
    if (col) {
      wait_geq(&q.row_done[slot], use * q.rtiles);
      warp_col_task<T, N1, GRFC_ONE_FFT_OVERWRITE>(p, key, field0 + f, (int)idx * kWarpCols + warp, WT, tw1, tw2, wsm,
                                                   table ? s_rowq : nullptr);
      signal_done(&q.col_done[slot]);
    } else {
      wait_geq(&q.col_done[slot], (use + 1) * q.strips);
      rowT_tile<T, N1, M, RPT>(WT, (int)idx * RPT, out + (int64_t)f * out_stride, tw2, smem_raw);
      signal_done(&q.row_done[slot]);
    }
  }
}

template <typename T, int N1, int M>
cudaError_t fusedw_query(Fast2D& f) {
  constexpr size_t smem = fusedw_smem<N1, M, T>();
  cudaError_t e = cudaFuncSetAttribute(k_fused2d_w<T, N1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0, dev = 0, sms = 148;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused2d_w<T, N1, M>, kWarpThreads, smem);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  f.occ = occ < 1 ? 1 : occ;
  f.sms = sms;
  f.strips = (M / 2) / kWarpCols;
  f.rtiles = N1 / rowsT_per_tile<N1, M, T>();
  return cudaSuccess;
}

template <typename T, int N1, int M>
cudaError_t launch_fusedw(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* ws, void* out,
                          int64_t stride, cudaStream_t s) {
  using C = C_t<T>;
  constexpr size_t smem = fusedw_smem<N1, M, T>();
  F2Sched q{};
  uint32_t conc = 0;
  fused_geometry(f, nf, &q.L, &q.S, &conc);
  q.F = (uint32_t)nf;
  q.strips = (uint32_t)f.strips;
  q.rtiles = (uint32_t)f.rtiles;
  uint32_t* ctr = (uint32_t*)ws;
  q.ticket = ctr;
  q.col_done = ctr + 1;
  q.row_done = ctr + 1 + q.S;
  q.stats = nullptr;
  C* ring = (C*)((char*)ws + fused_ctr_bytes(q.S));
  cudaError_t e = cudaMemsetAsync(ctr, 0, (1 + 2 * q.S) * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const C* tw1 = (const C*)f.d_tw;
  const C* tw2 = tw1 + f.n1;
  const uint32_t total = q.F * (q.strips + q.rtiles);
  const uint32_t grid = total < conc ? total : conc;
  {
    LaunchScope ls("fused2d_warp_persistent", s);
    k_fused2d_w<T, N1, M><<<grid, kWarpThreads, smem, s>>>(make_params(f), q, philox_key(seed), field0, ring, (T*)out,
                                                           stride, tw1, tw2);
  }
  return cudaGetLastError();
}

}  // namespace grfc
