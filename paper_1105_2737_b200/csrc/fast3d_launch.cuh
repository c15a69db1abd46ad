// Launchers of the fused 3D kernels (instantiated per (dtype, size) by
// fast3d_inst.cu).
#pragma once

#include <algorithm>
#include <cstdio>
#include <utility>

#include "fast2d.h"
#include "fast3d.h"
#include "fast3d_kernels.cuh"

namespace grfc {

inline F3Params make_params3(const Fast3D& f) {
  F3Params p{};
  p.n0 = f.n0;
  p.n1 = f.n1;
  p.n2 = f.n2;
  p.m = f.n2 / 2;
  p.hd = f.n2 / 2 + 1;
  for (int a = 0; a < 3; ++a) {
    p.wstep[a] = 2.0 * M_PI / f.g.l[a];
    p.f_wstep[a] = (float)p.wstep[a];
  }
  p.family = f.D.family;
  p.alg = f.alg;
  p.sqrt_c = f.D.sqrt_c;
  p.alpha = f.D.alpha;
  p.ell = f.D.family == GRFC_DENSITY_MATERN ? f.D.r[1] : f.D.r[0];
  p.scale = f.s_one;
  p.f_sqrt_c = (float)p.sqrt_c;
  p.f_ell2 = (float)(p.ell * p.ell);
  p.f_nhalf_alpha = (float)(-0.5 * p.alpha);
  p.f_gauss_k = (float)(-0.25 * p.ell * p.ell * 1.4426950408889634);
  p.f_scale = (float)p.scale;
  const uint64_t U = f.alg == GRFC_ONE_FFT_OVERWRITE ? (uint64_t)f.n0 * f.n1 * (f.n2 / 2 + 1)
                                                     : (uint64_t)f.n0 * f.n1 * f.n2;
  p.uh = (U + 1) / 2;
  p.D = f.D;
  p.g = f.g;
  return p;
}

template <typename T, int N0, int ALG>
cudaError_t launch_3d_colgen(const Fast3D& f, uint64_t seed, uint64_t field, void* W, int k1_lo, int k1_cnt,
                             cudaStream_t s) {
  using C = C_t<T>;
  constexpr int CB = ColPlan3<N0, T>::X, SLOTS = 4 * CB;
  const size_t smem = (size_t)N0 * (SLOTS + 2) * sizeof(C);
  // set on every launch: the attribute is per device (a process may use several)
  cudaFuncSetAttribute(k_3d_colgen<T, N0, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int strips = (f.n2 / 2) / (2 * CB);
  // The tile of row a generates k1 = a and k1 = -a (the Hermitian partner its
  // pre-twiddle needs); a rank launches only the rows a for which either lies in
  // its slab: a in [lo, hi) (k1 = a) or -a in [lo, hi), i.e. a in [N1-hi+1, N1-lo]
  // (k1 = N1 - a), both clipped to [0, N1/2] — at most two intervals.
  const int half = f.n1 / 2, hi = k1_lo + k1_cnt;
  int l0 = k1_lo, h0 = std::min(hi, half + 1);              // [l0, h0)
  int l1 = std::max(f.n1 - hi + 1, 1), h1 = std::min(f.n1 - k1_lo, half) + 1;  // [l1, h1)
  if (h0 <= l0) l0 = h0 = 0;
  if (h1 <= l1) l1 = h1 = 0;
  if (h0 > l0 && h1 > l1 && l1 <= h0 && l0 <= h1) {  // overlapping or adjacent: one interval
    l0 = std::min(l0, l1);
    h0 = std::max(h0, h1);
    l1 = h1 = 0;
  } else if (h0 <= l0 || (h1 > l1 && l1 < l0)) {  // keep the lower interval first
    std::swap(l0, l1);
    std::swap(h0, h1);
  }
  const int rows = (h0 - l0) + (h1 - l1);
  if (rows == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)(rows * strips);
  const C* tw0 = (const C*)f.d_tw;
  const C* tw2 = tw0 + f.n0 + f.n1;
  LaunchScope ls("fused3d_colgen", s);
  k_3d_colgen<T, N0, ALG><<<blocks, colgen3_threads<N0, T>(), smem, s>>>(
      make_params3(f), philox_key(seed), field, (C*)W, k1_lo, k1_cnt, l0, h0 - l0, l1, tw0, tw2);
  return cudaGetLastError();
}

template <typename T, int N1, int M>
cudaError_t planes_query(Fast3D& f) {
  constexpr size_t smem = planes_smem<N1, M, T>();
  cudaError_t e =
      cudaFuncSetAttribute(k_3d_planes<T, N1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0, dev = 0, sms = 148;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_3d_planes<T, N1, M>, col_threads<N1, T>(), smem);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  f.occ = occ < 1 ? 1 : occ;
  f.sms = sms;
  f.strips = M / (2 * ColPlan<N1, T>::X);
  f.rtiles = N1 / rows_per_tile<N1, M, T>();
  return cudaSuccess;
}

// ws: counters + ring (planes_ws_bytes); src: receive buffer; out: rank slab.
template <typename T, int N1, int M>
cudaError_t launch_3d_planes(const Fast3D& f, const void* src, int n0p, int n1p, void* ws, void* out,
                             cudaStream_t s) {
  using C = C_t<T>;
  constexpr size_t smem = planes_smem<N1, M, T>();
  F2Sched q{};
  uint32_t conc = 0;
  ring_geometry(f.sms, f.occ, f.strips, f.rtiles, n0p, &q.L, &q.S, &conc, 3, 2);
  q.F = (uint32_t)n0p;
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
  const C* tw1 = (const C*)f.d_tw + f.n0;
  const C* tw2 = tw1 + f.n1;
  const uint32_t total = q.F * (q.strips + q.rtiles);
  const uint32_t grid = total < conc ? total : conc;
  LaunchScope ls("fused3d_planes", s);
  k_3d_planes<T, N1, M><<<grid, col_threads<N1, T>(), smem, s>>>(q, (const C*)src, n0p, n1p, ring, (T*)out, tw1, tw2);
  return cudaGetLastError();
}

}  // namespace grfc
