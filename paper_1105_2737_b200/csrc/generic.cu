// Generic grfc kernels: any dimension d <= GRFC_MAX_DIM, any even N per axis,
// fp32 or fp64, all three algorithms, seeded (Philox) or injected noise.
//
// Layout in HBM: one field's half-spectrum workspace W is row-major over the
// half-lattice H = N_1 x .. x N_{d-1} x (N_d/2+1) (complex T); a batch of
// fields is [field][H]. The real field is row-major over the full grid.
//
// Passes (Alg 2/3, the reference's synth.cpp:118-126):
//   gen_half    V(K) = sqrt(g) w(K) on H, stored conjugated and scaled by
//               sqrt((2pi)^d/|A|)          (hermitian.cpp:128-203 + synth.cpp:123)
//   line_c2c    exp(+) C2C along axes 0..d-2, in shared memory
//   c2r_last    last-axis half-complex -> real (N_d/2-point complex FFT +
//               post-twiddle), writes the field (dft.cpp:102-108 + synth.cpp:20-33)
// Passes (Alg 1, synth.cpp:81-116): r2c_last (+noise) -> line_c2c(+) ->
//   scale_half (sqrt(g) sqrt((2pi)^d P/|A|)/P) -> line_c2c(-) -> c2r_last(-).
//
// The 1D transforms are mixed-radix Stockham autosort passes in shared memory
// (radix 8/4/2 register butterflies, any other prime by a direct sum).
// pow2 2D shapes take the fused fast path in pow2_2d.cu instead.
#include <algorithm>

#include "grfc_internal.cuh"
#include "kernels.h"

namespace grfc {

// ---------------------------------------------------------------- small DFTs
template <int SIGN, typename C>
__device__ __forceinline__ void dft2(C& a, C& b) {
  const C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int SIGN, typename C>
__device__ __forceinline__ void dft4(C* v) {
  const C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
  const C t2 = cadd(v[1], v[3]), t3 = mul_si<SIGN>(csub(v[1], v[3]));
  v[0] = cadd(t0, t2);
  v[2] = csub(t0, t2);
  v[1] = cadd(t1, t3);
  v[3] = csub(t1, t3);
}

template <int SIGN, typename C>
__device__ __forceinline__ void dft8(C* v) {
  using R = decltype(C{}.x);
  C e[4] = {v[0], v[2], v[4], v[6]};
  C o[4] = {v[1], v[3], v[5], v[7]};
  dft4<SIGN>(e);
  dft4<SIGN>(o);
  const R h = (R)0.70710678118654752440;
  // o[q] *= exp(SIGN 2 pi i q / 8)
  o[1] = mk<C>((o[1].x - (R)SIGN * o[1].y) * h, ((R)SIGN * o[1].x + o[1].y) * h);
  o[2] = mul_si<SIGN>(o[2]);
  o[3] = mk<C>((-o[3].x - (R)SIGN * o[3].y) * h, ((R)SIGN * o[3].x - o[3].y) * h);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = cadd(e[q], o[q]);
    v[q + 4] = csub(e[q], o[q]);
  }
}

template <int SIGN, typename C>
__device__ __forceinline__ C twiddle(const C* tw, int64_t idx) {
  const C w = tw[idx];
  return SIGN > 0 ? w : cconj(w);
}

// One Stockham pass of radix R over nl lines (line l at src + l*pitch).
// tw: table exp(+2 pi i m / Ntab) read with stride tws (Ntab = n * tws).
template <int R, int SIGN, typename C>
__device__ __forceinline__ void stockham_pass_reg(const C* src, C* dst, int nl, int pitch, int n, int Ns,
                                                  const C* tw, int tws) {
  const int m = n / R, tstep = n / (Ns * R);
  const int items = nl * m;
  for (int w = threadIdx.x; w < items; w += blockDim.x) {
    const int l = w / m, j = w - l * m, k = j % Ns;
    const C* in = src + (int64_t)l * pitch;
    C* out = dst + (int64_t)l * pitch;
    C v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v[i] = in[j + i * m];
      if (i > 0 && k > 0) v[i] = cmul(v[i], twiddle<SIGN>(tw, (int64_t)((i * k * tstep) % n) * tws));
    }
    if (R == 2) dft2<SIGN>(v[0], v[1]);
    if (R == 4) dft4<SIGN>(v);
    if (R == 8) dft8<SIGN>(v);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int i = 0; i < R; ++i) out[base + i * Ns] = v[i];
  }
}

template <int SIGN, typename C>
__device__ __forceinline__ void stockham_pass_any(const C* src, C* dst, int nl, int pitch, int n, int R,
                                                  int Ns, const C* tw, int tws) {
  using T = decltype(C{}.x);
  const int m = n / R, tstep = n / (Ns * R), qstep = n / R;
  const int items = nl * n;
  for (int w = threadIdx.x; w < items; w += blockDim.x) {
    const int l = w / n, rem = w - l * n, j = rem % m, q = rem / m, k = j % Ns;
    const C* in = src + (int64_t)l * pitch;
    C acc = mk<C>((T)0, (T)0);
    for (int i = 0; i < R; ++i) {
      C v = in[j + i * m];
      if (i > 0 && k > 0) v = cmul(v, twiddle<SIGN>(tw, (int64_t)((i * k * tstep) % n) * tws));
      const int t = ((q * i) % R) * qstep;
      acc = cadd(acc, cmul(v, twiddle<SIGN>(tw, (int64_t)t * tws)));
    }
    dst[(int64_t)l * pitch + (j / Ns) * Ns * R + k + q * Ns] = acc;
  }
}

// Full in-smem transform of nl lines; returns the buffer holding the result.
template <int SIGN, typename C>
__device__ C* smem_fft(C* a, C* b, int nl, int pitch, int n, const Factors& F, const C* tw, int tws) {
  int Ns = 1;
  for (int s = 0; s < F.nf; ++s) {
    const int R = F.r[s];
    switch (R) {
      case 2: stockham_pass_reg<2, SIGN>(a, b, nl, pitch, n, Ns, tw, tws); break;
      case 4: stockham_pass_reg<4, SIGN>(a, b, nl, pitch, n, Ns, tw, tws); break;
      case 8: stockham_pass_reg<8, SIGN>(a, b, nl, pitch, n, Ns, tw, tws); break;
      default: stockham_pass_any<SIGN>(a, b, nl, pitch, n, R, Ns, tw, tws); break;
    }
    __syncthreads();
    C* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

// ---------------------------------------------------------------- kernels
// X(K) = conj(w(K)) * sqrt(g) * scale on H, for nfields fields.
template <typename T>
__global__ void k_gen_half(GridDesc g, DensityDesc D, int alg, T scale, PhiloxKey key, uint64_t field0,
                           const double2* injected, C_t<T>* W, int64_t nfields) {
  using C = C_t<T>;
  const int64_t total = g.cells * nfields;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / g.cells, h = t - f * g.cells;
    int64_t k[GRFC_MAX_DIM], kw[GRFC_MAX_DIM];
    decode_half(g, h, k);
    wrap_freq(g, k, kw);
    C w;
    if (injected) {
      const double2 v = injected[h];
      w = mk<C>((T)v.x, (T)v.y);
    } else {
      w = philox_cell_noise<T>(g, alg, k, h, key, field0 + (uint64_t)f);
    }
    const T m = sqrt_gamma<T>(g, D, kw, h) * scale;
    W[t] = mk<C>(w.x * m, -w.y * m);
  }
}

// Alg-1 spectrum scaling on H: W *= sqrt(g) * scale.
template <typename T>
__global__ void k_scale_half(GridDesc g, DensityDesc D, T scale, C_t<T>* W, int64_t nfields) {
  const int64_t total = g.cells * nfields;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = t % g.cells;
    int64_t k[GRFC_MAX_DIM], kw[GRFC_MAX_DIM];
    decode_half(g, h, k);
    wrap_freq(g, k, kw);
    W[t] = cscale(W[t], sqrt_gamma<T>(g, D, kw, h) * scale);
  }
}

// Batched in-place C2C along one axis: data viewed as [outer][n][inner].
// inner > 1: a block takes LB adjacent inner columns of one outer slab
// (coalesced rows of LB complex); inner == 1: LB consecutive contiguous lines.
template <typename T, int SIGN>
__global__ void k_line_c2c(C_t<T>* data, int n, int64_t inner, int64_t outer, int LB, Factors F,
                           const C_t<T>* tw) {
  using C = C_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int pitch = n + 1;
  C* a = reinterpret_cast<C*>(smem_raw);
  C* b = a + (int64_t)LB * pitch;
  int nl;
  if (inner > 1) {
    const int64_t nblk = (inner + LB - 1) / LB;
    const int64_t o = blockIdx.x / nblk, i0 = (blockIdx.x % nblk) * LB;
    nl = (int)min((int64_t)LB, inner - i0);
    C* base = data + o * n * inner + i0;
    for (int w = threadIdx.x; w < nl * n; w += blockDim.x) {
      const int l = w % nl, t = w / nl;
      a[l * pitch + t] = base[(int64_t)t * inner + l];
    }
    __syncthreads();
    const C* res = smem_fft<SIGN>(a, b, nl, pitch, n, F, tw, 1);
    for (int w = threadIdx.x; w < nl * n; w += blockDim.x) {
      const int l = w % nl, t = w / nl;
      base[(int64_t)t * inner + l] = res[l * pitch + t];
    }
  } else {
    const int64_t l0 = (int64_t)blockIdx.x * LB;
    nl = (int)min((int64_t)LB, outer - l0);
    C* base = data + l0 * n;
    for (int w = threadIdx.x; w < nl * n; w += blockDim.x) {
      const int l = w / n, t = w % n;
      a[l * pitch + t] = base[(int64_t)l * n + t];
    }
    __syncthreads();
    const C* res = smem_fft<SIGN>(a, b, nl, pitch, n, F, tw, 1);
    for (int w = threadIdx.x; w < nl * n; w += blockDim.x) {
      const int l = w / n, t = w % n;
      base[(int64_t)l * n + t] = res[l * pitch + t];
    }
  }
}

// Last-axis half-complex -> real. Row r of W holds X[0..M] (M = n/2); with
// Y = X (CONJ=0) or conj(X) (CONJ=1, i.e. an exp(-) transform):
//   Z[k] = (Y[k] + conj(Y[M-k])) + i e^{+2 pi i k/n} (Y[k] - conj(Y[M-k]))
//   z = IDFT+_M(Z);  x[2m] = Re z[m], x[2m+1] = Im z[m].
// twN: exp(+2 pi i m / n), m < n (the M-point FFT reads it with stride 2).
template <typename T, int CONJ>
__global__ void k_c2r_last(const C_t<T>* W, T* out, int n, int64_t rows, int64_t rows_per_field,
                           int64_t out_field_stride, int RB, Factors F, const C_t<T>* twN) {
  using C = C_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M = n / 2, hd = M + 1, pitch = M + 1;
  C* x = reinterpret_cast<C*>(smem_raw);  // RB x hd
  C* a = x + (int64_t)RB * hd;           // RB x pitch
  C* b = a + (int64_t)RB * pitch;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nl = (int)min((int64_t)RB, rows - r0);
  for (int w = threadIdx.x; w < nl * hd; w += blockDim.x) x[w] = W[r0 * hd + w];
  __syncthreads();
  for (int w = threadIdx.x; w < nl * M; w += blockDim.x) {
    const int l = w / M, k = w - l * M;
    C yk = x[l * hd + k], ym = x[l * hd + M - k];
    if (CONJ) yk = cconj(yk);
    else ym = cconj(ym);  // ym := conj(Y[M-k])
    const C s = cadd(yk, ym), d = csub(yk, ym);
    const C t = cmul(twN[k], d);
    a[l * pitch + k] = mk<C>(s.x - t.y, s.y + t.x);
  }
  __syncthreads();
  const C* res = smem_fft<+1>(a, b, nl, pitch, M, F, twN, 2);
  for (int l = 0; l < nl; ++l) {
    const int64_t r = r0 + l, f = r / rows_per_field, rr = r - f * rows_per_field;
    T* o = out + f * out_field_stride + rr * n;
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
      const C v = res[l * pitch + m];
      o[2 * m] = v.x;
      o[2 * m + 1] = v.y;
    }
  }
}

// Alg-1 first pass: white noise on the full grid -> exp(+) R2C along the
// last axis, rows of W get X[0..M]. Noise: Philox pair per 2 points
// (counter = J/2, J the row-major point index) or injected draws[J].
//   z[m] = x[2m] + i x[2m+1]; Z = DFT+_M(z);
//   X[k] = 1/2 (Z[k] + conj(Z[M-k])) - i/2 e^{+2 pi i k/n} (Z[k] - conj(Z[M-k]))
template <typename T>
__global__ void k_r2c_last_noise(C_t<T>* W, int n, int64_t rows, int64_t rows_per_field, PhiloxKey key,
                                 uint64_t field0, const double* injected, int RB, Factors F,
                                 const C_t<T>* twN) {
  using C = C_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M = n / 2, hd = M + 1, pitch = M + 1;
  C* a = reinterpret_cast<C*>(smem_raw);
  C* b = a + (int64_t)RB * pitch;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nl = (int)min((int64_t)RB, rows - r0);
  for (int w = threadIdx.x; w < nl * M; w += blockDim.x) {
    const int l = w / M, m = w - l * M;
    const int64_t r = r0 + l, f = r / rows_per_field, rr = r - f * rows_per_field;
    const int64_t pair = rr * M + m;  // J/2 within the field
    T z0, z1;
    if (injected) {
      z0 = (T)injected[2 * pair];
      z1 = (T)injected[2 * pair + 1];
    } else {
      unit_pair<T>(key, field0 + (uint64_t)f, (uint64_t)pair, (uint64_t)(rows_per_field * M + 1) / 2, z0, z1);
    }
    a[l * pitch + m] = mk<C>(z0, z1);
  }
  __syncthreads();
  const C* Z = smem_fft<+1>(a, b, nl, pitch, M, F, twN, 2);
  for (int w = threadIdx.x; w < nl * hd; w += blockDim.x) {
    const int l = w / hd, k = w - l * hd;
    const C zk = Z[l * pitch + (k % M)], zm = cconj(Z[l * pitch + ((M - k) % M)]);
    const C s = cadd(zk, zm), d = csub(zk, zm);
    const C t = cmul(twN[k % n], d);  // e^{+2pi i k/n} (Z[k] - conj Z[M-k])
    using R = T;
    // X = s/2 - i t / 2
    W[(r0 + l) * hd + k] = mk<C>((s.x + t.y) * (R)0.5, (s.y - t.x) * (R)0.5);
  }
}

// Full-array scale (inverse DFT 1/P).
template <typename T>
__global__ void k_scale_all(C_t<T>* data, int64_t n, T s) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    data[t] = cscale(data[t], s);
}

// Philox noise for a list of counters (the dump path): out[2i], out[2i+1].
template <typename T>
__global__ void k_philox_pairs(const uint64_t* units, int64_t n, uint64_t Uh, PhiloxKey key, uint64_t field,
                               double* out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    T z0, z1;
    unit_pair<T>(key, field, units[t], Uh, z0, z1);
    out[2 * t] = (double)z0;
    out[2 * t + 1] = (double)z1;
  }
}

// ---------------------------------------------------------------- launchers
static int grid_for(int64_t work, int threads) {
  const int64_t b = (work + threads - 1) / threads;
  return (int)std::min<int64_t>(b, 148 * 64);
}

template <typename T>
cudaError_t launch_gen_half(const GridDesc& g, const DensityDesc& D, int alg, double scale, uint64_t seed,
                            uint64_t field0, const double2* injected, void* W, int64_t nfields, cudaStream_t s) {
  LaunchScope ls_("gen_half", s);
  k_gen_half<T><<<grid_for(g.cells * nfields, 256), 256, 0, s>>>(g, D, alg, (T)scale, philox_key(seed), field0, injected,
                                                                 (C_t<T>*)W, nfields);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scale_half(const GridDesc& g, const DensityDesc& D, double scale, void* W, int64_t nfields,
                              cudaStream_t s) {
  LaunchScope ls_("scale_half", s);
  k_scale_half<T><<<grid_for(g.cells * nfields, 256), 256, 0, s>>>(g, D, (T)scale, (C_t<T>*)W, nfields);
  return cudaGetLastError();
}

static size_t smem_limit() { return 200 * 1024; }

template <typename T>
cudaError_t launch_line_c2c(void* data, int n, int64_t inner, int64_t outer, int sign, const Factors& F,
                            const void* tw, cudaStream_t s) {
  LaunchScope ls_("line_c2c", s);
  using C = C_t<T>;
  const size_t per_line = 2 * (size_t)(n + 1) * sizeof(C);
  if (per_line > smem_limit()) return cudaErrorInvalidValue;
  int LB;
  if (inner > 1) LB = (int)std::min<int64_t>(inner, sizeof(T) == 4 ? 16 : 8);
  else LB = std::max(1, std::min(8, (int)(4096 / n)));
  while (LB > 1 && LB * per_line > smem_limit()) LB /= 2;
  const size_t smem = LB * per_line;
  const int64_t blocks = inner > 1 ? outer * ((inner + LB - 1) / LB) : (outer + LB - 1) / LB;
  const int threads = 256;
  if (sign > 0) {
    cudaFuncSetAttribute(k_line_c2c<T, +1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_line_c2c<T, +1><<<(unsigned)blocks, threads, smem, s>>>((C*)data, n, inner, outer, LB, F, (const C*)tw);
  } else {
    cudaFuncSetAttribute(k_line_c2c<T, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_line_c2c<T, -1><<<(unsigned)blocks, threads, smem, s>>>((C*)data, n, inner, outer, LB, F, (const C*)tw);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_c2r_last(const void* W, void* out, int n, int64_t rows, int64_t rows_per_field,
                            int64_t out_field_stride, int conj, const Factors& FM, const void* twN,
                            cudaStream_t s) {
  LaunchScope ls_("c2r_last", s);
  using C = C_t<T>;
  const int M = n / 2;
  const size_t per_row = ((size_t)(M + 1) + 2 * (size_t)(M + 1)) * sizeof(C);
  if (per_row > smem_limit()) return cudaErrorInvalidValue;
  int RB = std::max(1, std::min(8, 2048 / std::max(M, 1)));
  while (RB > 1 && RB * per_row > smem_limit()) RB /= 2;
  const size_t smem = RB * per_row;
  const int64_t blocks = (rows + RB - 1) / RB;
  if (conj) {
    cudaFuncSetAttribute(k_c2r_last<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_c2r_last<T, 1><<<(unsigned)blocks, 256, smem, s>>>((const C*)W, (T*)out, n, rows, rows_per_field,
                                                        out_field_stride, RB, FM, (const C*)twN);
  } else {
    cudaFuncSetAttribute(k_c2r_last<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_c2r_last<T, 0><<<(unsigned)blocks, 256, smem, s>>>((const C*)W, (T*)out, n, rows, rows_per_field,
                                                        out_field_stride, RB, FM, (const C*)twN);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_r2c_last_noise(void* W, int n, int64_t rows, int64_t rows_per_field, uint64_t seed,
                                  uint64_t field0, const double* injected, const Factors& FM, const void* twN,
                                  cudaStream_t s) {
  LaunchScope ls_("r2c_last_noise", s);
  using C = C_t<T>;
  const int M = n / 2;
  const size_t per_row = 2 * (size_t)(M + 1) * sizeof(C);
  if (per_row > smem_limit()) return cudaErrorInvalidValue;
  int RB = std::max(1, std::min(8, 2048 / std::max(M, 1)));
  while (RB > 1 && RB * per_row > smem_limit()) RB /= 2;
  const size_t smem = RB * per_row;
  const int64_t blocks = (rows + RB - 1) / RB;
  cudaFuncSetAttribute(k_r2c_last_noise<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_r2c_last_noise<T><<<(unsigned)blocks, 256, smem, s>>>((C*)W, n, rows, rows_per_field, philox_key(seed), field0, injected,
                                                         RB, FM, (const C*)twN);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scale_all(void* data, int64_t n, double sc, cudaStream_t s) {
  LaunchScope ls_("scale_all", s);
  k_scale_all<T><<<grid_for(n, 256), 256, 0, s>>>((C_t<T>*)data, n, (T)sc);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_philox_pairs(const uint64_t* units, int64_t n, uint64_t Uh, uint64_t seed, uint64_t field,
                                double* out, cudaStream_t s) {
  LaunchScope ls_("philox_pairs", s);
  k_philox_pairs<T><<<grid_for(n, 256), 256, 0, s>>>(units, n, Uh, philox_key(seed), field, out);
  return cudaGetLastError();
}

#define GRFC_INSTANTIATE(T)                                                                                     \
  template cudaError_t launch_gen_half<T>(const GridDesc&, const DensityDesc&, int, double, uint64_t, uint64_t, \
                                          const double2*, void*, int64_t, cudaStream_t);                       \
  template cudaError_t launch_scale_half<T>(const GridDesc&, const DensityDesc&, double, void*, int64_t,        \
                                            cudaStream_t);                                                      \
  template cudaError_t launch_line_c2c<T>(void*, int, int64_t, int64_t, int, const Factors&, const void*,       \
                                          cudaStream_t);                                                        \
  template cudaError_t launch_c2r_last<T>(const void*, void*, int, int64_t, int64_t, int64_t, int,              \
                                          const Factors&, const void*, cudaStream_t);                           \
  template cudaError_t launch_r2c_last_noise<T>(void*, int, int64_t, int64_t, uint64_t, uint64_t, const double*, \
                                                const Factors&, const void*, cudaStream_t);                     \
  template cudaError_t launch_scale_all<T>(void*, int64_t, double, cudaStream_t);                               \
  template cudaError_t launch_philox_pairs<T>(const uint64_t*, int64_t, uint64_t, uint64_t, uint64_t, double*, \
                                                   cudaStream_t);

GRFC_INSTANTIATE(float)
GRFC_INSTANTIATE(double)

}  // namespace grfc
