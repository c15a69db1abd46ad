// Host side of the fused pow2 3D path (kernels: fast3d_kernels.cuh; launchers
// instantiated by fast3d_inst.cu per (dtype, size)).
#include <algorithm>
#include <cmath>
#include <vector>

#include "fast2d.h"
#include "fast3d.h"
#include "grfc_internal.cuh"

namespace grfc {

template <typename T, int N0, int ALG>
cudaError_t launch_3d_colgen(const Fast3D& f, uint64_t seed, uint64_t field, void* W, int k1_lo, int k1_cnt,
                             cudaStream_t s);
template <typename T, int N1, int M>
cudaError_t launch_3d_planes(const Fast3D& f, const void* src, int n0p, int n1p, void* ws, void* out, cudaStream_t s);
template <typename T, int N1, int M>
cudaError_t planes_query(Fast3D& f);

static bool pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

bool fast3d_supported(int d, const int64_t* n, int alg) {
  if (d != 3 || alg == GRFC_TWO_FFT) return false;
  for (int a = 0; a < 3; ++a)
    if (!pow2(n[a])) return false;
  return n[0] >= 128 && n[0] <= 1024 && n[1] >= 128 && n[1] <= 1024 && n[2] >= 128 && n[2] <= 1024;
}

template <typename T>
static std::vector<C_t<T>> tw_table(int64_t n) {
  std::vector<C_t<T>> t((size_t)n);
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int64_t m = 0; m < n; ++m) {
    const long double a = two_pi * (long double)m / (long double)n;
    t[(size_t)m].x = (T)cosl(a);
    t[(size_t)m].y = (T)sinl(a);
  }
  return t;
}

#define GRFC_M_SWITCH(T, N1, CALL)                 \
  switch (f.n2 / 2) {                              \
    case 64: return CALL(T, N1, 64);               \
    case 128: return CALL(T, N1, 128);             \
    case 256: return CALL(T, N1, 256);             \
    case 512: return CALL(T, N1, 512);             \
  }                                                \
  return cudaErrorNotSupported;
#define GRFC_N1_SWITCH(T, CALL)                             \
  switch (f.n1) {                                           \
    case 128: { GRFC_M_SWITCH(T, 128, CALL) }               \
    case 256: { GRFC_M_SWITCH(T, 256, CALL) }               \
    case 512: { GRFC_M_SWITCH(T, 512, CALL) }               \
    case 1024: { GRFC_M_SWITCH(T, 1024, CALL) }             \
  }                                                         \
  return cudaErrorNotSupported;
#define GRFC_Q(T, N1, M) planes_query<T, N1, M>(f)
#define GRFC_P(T, N1, M) launch_3d_planes<T, N1, M>(f, src, n0p, n1p, ws, out, s)

template <typename T>
static cudaError_t query(Fast3D& f) {
  GRFC_N1_SWITCH(T, GRFC_Q)
}

template <typename T>
static cudaError_t planes(const Fast3D& f, const void* src, int n0p, int n1p, void* ws, void* out, cudaStream_t s) {
  GRFC_N1_SWITCH(T, GRFC_P)
}

template <typename T, int ALG>
static cudaError_t colgen(const Fast3D& f, uint64_t seed, uint64_t field, void* W, int k1_lo, int k1_cnt,
                          cudaStream_t s) {
  switch (f.n0) {
    case 128: return launch_3d_colgen<T, 128, ALG>(f, seed, field, W, k1_lo, k1_cnt, s);
    case 256: return launch_3d_colgen<T, 256, ALG>(f, seed, field, W, k1_lo, k1_cnt, s);
    case 512: return launch_3d_colgen<T, 512, ALG>(f, seed, field, W, k1_lo, k1_cnt, s);
    case 1024: return launch_3d_colgen<T, 1024, ALG>(f, seed, field, W, k1_lo, k1_cnt, s);
  }
  return cudaErrorNotSupported;
}

cudaError_t fast3d_init(Fast3D& f, const GridDesc& g, const DensityDesc& D, int dtype, int alg, double s_one) {
  f.n0 = (int)g.n[0];
  f.n1 = (int)g.n[1];
  f.n2 = (int)g.n[2];
  f.dtype = dtype;
  f.alg = alg;
  f.g = g;
  f.D = D;
  f.s_one = s_one;
  const size_t cs = dtype == GRFC_F64 ? 16 : 8;
  cudaError_t e = cudaMalloc(&f.d_tw, (size_t)(f.n0 + f.n1 + f.n2) * cs);
  if (e != cudaSuccess) return e;
  if (dtype == GRFC_F64) {
    auto a = tw_table<double>(f.n0), b = tw_table<double>(f.n1), c = tw_table<double>(f.n2);
    a.insert(a.end(), b.begin(), b.end());
    a.insert(a.end(), c.begin(), c.end());
    e = cudaMemcpy(f.d_tw, a.data(), a.size() * cs, cudaMemcpyHostToDevice);
  } else {
    auto a = tw_table<float>(f.n0), b = tw_table<float>(f.n1), c = tw_table<float>(f.n2);
    a.insert(a.end(), b.begin(), b.end());
    a.insert(a.end(), c.begin(), c.end());
    e = cudaMemcpy(f.d_tw, a.data(), a.size() * cs, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) return e;
  return dtype == GRFC_F64 ? query<double>(f) : query<float>(f);
}

void fast3d_free(Fast3D& f) {
  cudaFree(f.d_tw);
  f.d_tw = nullptr;
}

bool slab_geometry(const Fast3D& f, int world, SlabGeom& s) {
  if (world < 1 || f.n0 % world || f.n1 % world) return false;
  s.world = world;
  s.n0p = f.n0 / world;
  s.n1p = f.n1 / world;
  s.block_elems = (uint64_t)s.n0p * s.n1p * (f.n2 / 2);
  s.buf_elems = s.block_elems * (uint64_t)world;
  return true;
}

cudaError_t fast3d_pass_a(const Fast3D& f, int world, int rank, uint64_t seed, uint64_t field, void* d_send,
                          cudaStream_t s) {
  SlabGeom g;
  if (!slab_geometry(f, world, g) || rank < 0 || rank >= world) return cudaErrorInvalidValue;
  const int lo = rank * g.n1p;
  if (f.dtype == GRFC_F64)
    return f.alg == GRFC_ONE_FFT_OVERWRITE ? colgen<double, GRFC_ONE_FFT_OVERWRITE>(f, seed, field, d_send, lo, g.n1p, s)
                                           : colgen<double, GRFC_ONE_FFT_RECURSIVE>(f, seed, field, d_send, lo, g.n1p, s);
  return f.alg == GRFC_ONE_FFT_OVERWRITE ? colgen<float, GRFC_ONE_FFT_OVERWRITE>(f, seed, field, d_send, lo, g.n1p, s)
                                         : colgen<float, GRFC_ONE_FFT_RECURSIVE>(f, seed, field, d_send, lo, g.n1p, s);
}

static size_t planes_ws_bytes(const Fast3D& f, int n0p) {
  uint32_t L, S, c;
  ring_geometry(f.sms, f.occ, f.strips, f.rtiles, n0p, &L, &S, &c, 3, 2);
  return fused_ctr_bytes(S) + (size_t)S * f.n1 * (f.n2 / 2) * (f.dtype == GRFC_F64 ? 16 : 8);
}

cudaError_t fast3d_pass_b(const Fast3D& f, int world, const void* d_recv, void* d_out, cudaStream_t s) {
  SlabGeom g;
  if (!slab_geometry(f, world, g)) return cudaErrorInvalidValue;
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, planes_ws_bytes(f, g.n0p), s);
  if (e != cudaSuccess) return e;
  e = f.dtype == GRFC_F64 ? planes<double>(f, d_recv, g.n0p, g.n1p, ws, d_out, s)
                          : planes<float>(f, d_recv, g.n0p, g.n1p, ws, d_out, s);
  cudaFreeAsync(ws, s);
  return e;
}

cudaError_t fast3d_generate(const Fast3D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out, int64_t stride,
                            cudaStream_t s) {
  const size_t esz = f.dtype == GRFC_F64 ? 8 : 4;
  void* W = nullptr;
  cudaError_t e = cudaMallocAsync(&W, (size_t)f.n0 * f.n1 * (f.n2 / 2) * 2 * esz, s);
  if (e != cudaSuccess) return e;
  for (int64_t i = 0; i < nf && e == cudaSuccess; ++i) {
    e = fast3d_pass_a(f, 1, 0, seed, field0 + (uint64_t)i, W, s);
    if (e == cudaSuccess) e = fast3d_pass_b(f, 1, W, (char*)out + i * stride * (int64_t)esz, s);
  }
  cudaFreeAsync(W, s);
  return e;
}

}  // namespace grfc
