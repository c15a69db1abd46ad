// Line transforms longer than one CTA's shared memory: the generic path's
// fallback for axes the on-chip Stockham kernels cannot hold (any even N the
// reference's GridSpec accepts, grid.cpp:10-30, runs on the device).
//
//   long_c2c   batched C2C of lines [outer][n][inner] through global memory:
//     * n fits on chip          -> k_line_c2c (generic.cu)
//     * n = n1 n2, n1 on chip   -> four-step: n1-point DFTs over t1 (stride n2),
//                                  twiddle e^{s 2 pi i t2 k1 / n} fused with the
//                                  [k1][t2] -> [t2][k1] transpose into scratch,
//                                  n2-point DFTs (recursive), copy back
//     * otherwise (a prime factor too long for the chip)
//                               -> Bluestein: x w -> zero-padded pow2 L >= 2n-1,
//                                  FFT, x FFT(conj w), inverse FFT, x w / L,
//                                  w[m] = e^{s pi i (m^2 mod 2n) / n}
//   long_c2r_last / long_r2c_last_noise: the last-axis half-complex passes of
//     generic.cu (same pre/post-twiddles, same noise keys) around long_c2c.
//
// All twiddles and chirps come from long-double angles (one rounding to T);
// tables are cached per (device, length, dtype). Scratch is stream-ordered.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "grfc_internal.cuh"
#include "kernels.h"

namespace grfc {

Factors factorize(int64_t n);  // api.cu

namespace {

constexpr size_t kSmemLine = 200 * 1024;  // launch_line_c2c's per-CTA budget
// longest prime the on-chip kernels sum directly (stockham_pass_any is O(n R) and
// its fp32 sums lose ~sqrt(R) ulps); longer prime factors go through Bluestein
constexpr int64_t kMaxDirectRadix = 61;

template <typename T>
bool line_fits(int64_t n) {
  return 2 * (size_t)(n + 1) * sizeof(C_t<T>) <= kSmemLine;
}

std::mutex g_tab_mu;
std::map<std::tuple<int, int64_t, int, int>, void*>& tab_cache() {
  static auto* m = new std::map<std::tuple<int, int64_t, int, int>, void*>();  // process lifetime
  return *m;
}

// kind 0: e^{+2 pi i m/n}, m < n;  kind 1/2: chirp e^{+/- pi i (m^2 mod 2n)/n}, m < n
template <typename T>
const C_t<T>* device_table(int64_t n, int kind) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, n, (int)sizeof(T), kind);
  std::lock_guard<std::mutex> lock(g_tab_mu);
  auto& cache = tab_cache();
  auto it = cache.find(key);
  if (it != cache.end()) return (const C_t<T>*)it->second;
  std::vector<C_t<T>> h((size_t)n);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int64_t m = 0; m < n; ++m) {
    long double a;
    if (kind == 0) {
      a = 2 * pi * (long double)m / (long double)n;
    } else {
      const uint64_t q = ((uint64_t)m * (uint64_t)m) % (2 * (uint64_t)n);
      a = (kind == 1 ? pi : -pi) * (long double)q / (long double)n;
    }
    h[(size_t)m].x = (T)cosl(a);
    h[(size_t)m].y = (T)sinl(a);
  }
  void* d = nullptr;
  if (cudaMalloc(&d, (size_t)n * sizeof(C_t<T>)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), (size_t)n * sizeof(C_t<T>), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  cache[key] = d;
  return (const C_t<T>*)d;
}

int grid_of(int64_t work) { return (int)std::min<int64_t>((work + 255) / 256, 148 * 32); }

// four-step middle: src[o][k1 n2 + t2][i] -> dst[o][t2 n1 + k1][i] x e^{s 2 pi i t2 k1 / n}.
// inner > 1: i is contiguous on both sides (coalesced); inner == 1: 32 x 32 tiles
// through shared memory so both the reads and the writes are coalesced.
template <typename T>
__global__ void k_twiddle_transpose(const C_t<T>* __restrict__ src, C_t<T>* __restrict__ dst, int64_t n1, int64_t n2,
                                    int64_t inner, int64_t outer, const C_t<T>* __restrict__ tw, int sign) {
  using C = C_t<T>;
  const int64_t n = n1 * n2;
  if (inner > 1) {
    const int64_t total = outer * n * inner;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = e % inner, r = e / inner, t = r % n, o = r / n;  // t = t2 n1 + k1 (dst order)
      const int64_t t2 = t / n1, k1 = t - t2 * n1;
      C w = tw[(t2 * k1) % n];
      if (sign < 0) w.y = -w.y;
      dst[e] = cmul(src[(o * n + k1 * n2 + t2) * inner + i], w);
    }
    return;
  }
  __shared__ C tile[32][33];
  const int64_t tiles1 = (n1 + 31) / 32, tiles2 = (n2 + 31) / 32;
  const int64_t per_line = tiles1 * tiles2;
  for (int64_t b = blockIdx.x; b < outer * per_line; b += gridDim.x) {
    const int64_t o = b / per_line, tb = b - o * per_line;
    const int64_t K1 = (tb / tiles2) * 32, T2 = (tb % tiles2) * 32;
    const C* s = src + o * n;
    C* d = dst + o * n;
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {  // read rows k1, columns t2 (contiguous)
      const int64_t k1 = K1 + r, t2 = T2 + threadIdx.x;
      if (k1 < n1 && t2 < n2) {
        C w = tw[(t2 * k1) % n];
        if (sign < 0) w.y = -w.y;
        tile[r][threadIdx.x] = cmul(s[k1 * n2 + t2], w);
      }
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {  // write rows t2, columns k1 (contiguous)
      const int64_t t2 = T2 + r, k1 = K1 + threadIdx.x;
      if (k1 < n1 && t2 < n2) d[t2 * n1 + k1] = tile[threadIdx.x][r];
    }
  }
}

// Bluestein steps. Lines [outer][n][inner] <-> buf[line = o inner + i][L].
template <typename T>
__global__ void k_blue_pre(const C_t<T>* __restrict__ x, C_t<T>* __restrict__ buf, int64_t n, int64_t L, int64_t inner,
                           int64_t lines, const C_t<T>* __restrict__ chirp) {
  const int64_t total = lines * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = e / L, t = e - line * L;
    const int64_t o = line / inner, i = line - o * inner;
    buf[e] = t < n ? cmul(x[(o * n + t) * inner + i], chirp[t]) : C_t<T>{};
  }
}

// b[m] = conj(w[|m|]) for |m| < n at m mod L, else 0
template <typename T>
__global__ void k_blue_kernel(C_t<T>* __restrict__ b, int64_t n, int64_t L, const C_t<T>* __restrict__ chirp) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < L; m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = m < n ? m : (L - m < n ? L - m : -1);
    b[m] = a >= 0 ? cconj(chirp[a]) : C_t<T>{};
  }
}

template <typename T>
__global__ void k_blue_mul(C_t<T>* __restrict__ buf, const C_t<T>* __restrict__ B, int64_t L, int64_t lines) {
  const int64_t total = lines * L;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    buf[e] = cmul(buf[e], B[e % L]);
}

template <typename T>
__global__ void k_blue_post(C_t<T>* __restrict__ x, const C_t<T>* __restrict__ buf, int64_t n, int64_t L, int64_t inner,
                            int64_t lines, const C_t<T>* __restrict__ chirp) {
  const int64_t total = lines * n;
  const T inv = (T)(1.0 / (double)L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = e / n, k = e - line * n;
    const int64_t o = line / inner, i = line - o * inner;
    x[(o * n + k) * inner + i] = cscale(cmul(buf[line * L + k], chirp[k]), inv);
  }
}

// Last-axis passes (as generic.cu's k_c2r_last / k_r2c_last_noise, in global memory).
template <typename T, int CONJ>
__global__ void k_c2r_pre(const C_t<T>* __restrict__ W, C_t<T>* __restrict__ Z, int64_t M, int64_t rows,
                          const C_t<T>* __restrict__ twN) {
  using C = C_t<T>;
  const int64_t hd = M + 1, total = rows * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / M, k = e - r * M;
    C yk = W[r * hd + k], ym = W[r * hd + M - k];
    if (CONJ) yk = cconj(yk);
    else ym = cconj(ym);
    const C s = cadd(yk, ym), d = csub(yk, ym);
    const C t = cmul(twN[k], d);
    Z[e] = mk<C>(s.x - t.y, s.y + t.x);
  }
}

template <typename T>
__global__ void k_rows_out(const C_t<T>* __restrict__ Z, T* __restrict__ out, int64_t M, int64_t rows,
                           int64_t rows_per_field, int64_t out_field_stride) {
  const int64_t total = rows * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / M, m = e - r * M, f = r / rows_per_field, rr = r - f * rows_per_field;
    T* o = out + f * out_field_stride + rr * 2 * M + 2 * m;
    o[0] = Z[e].x;
    o[1] = Z[e].y;
  }
}

template <typename T>
__global__ void k_noise_rows(C_t<T>* __restrict__ Z, int64_t M, int64_t rows, int64_t rows_per_field, PhiloxKey key,
                             uint64_t field0, const double* __restrict__ injected) {
  const int64_t total = rows * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / M, m = e - r * M, f = r / rows_per_field, rr = r - f * rows_per_field;
    const int64_t pair = rr * M + m;  // J/2 within the field
    T z0, z1;
    if (injected) {
      z0 = (T)injected[2 * pair];
      z1 = (T)injected[2 * pair + 1];
    } else {
      unit_pair<T>(key, field0 + (uint64_t)f, (uint64_t)pair, (uint64_t)(rows_per_field * M + 1) / 2, z0, z1);
    }
    Z[e] = mk<C_t<T>>(z0, z1);
  }
}

template <typename T>
__global__ void k_r2c_post(const C_t<T>* __restrict__ Zf, C_t<T>* __restrict__ W, int64_t M, int64_t rows,
                           const C_t<T>* __restrict__ twN) {
  using C = C_t<T>;
  const int64_t hd = M + 1, total = rows * hd, n = 2 * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / hd, k = e - r * hd;
    const C zk = Zf[r * M + (k % M)], zm = cconj(Zf[r * M + ((M - k) % M)]);
    const C s = cadd(zk, zm), d = csub(zk, zm);
    const C t = cmul(twN[k % n], d);
    W[e] = mk<C>((s.x + t.y) * (T)0.5, (s.y - t.x) * (T)0.5);
  }
}

int64_t largest_prime_factor(int64_t n) {
  int64_t best = 1;
  for (int64_t p = 2; p * p <= n; ++p)
    while (n % p == 0) best = p, n /= p;
  return n > 1 ? std::max(best, n) : best;
}

// largest divisor of n that fits on chip (and is < n); 1 if none >= 2
template <typename T>
int64_t chip_divisor(int64_t n) {
  int64_t best = 1;
  for (int64_t d = 2; d * d <= n; ++d) {
    if (n % d) continue;
    if (line_fits<T>(d) && d > best) best = d;
    if (line_fits<T>(n / d) && n / d < n && n / d > best) best = n / d;
  }
  return best;
}

}  // namespace

__global__ void k_widen(const float2* __restrict__ a, double2* __restrict__ b, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    b[e] = make_double2(a[e].x, a[e].y);
}
__global__ void k_narrow(const double2* __restrict__ a, float2* __restrict__ b, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    b[e] = make_float2((float)a[e].x, (float)a[e].y);
}

template <typename T>
cudaError_t long_c2c(void* data, int64_t n, int64_t inner, int64_t outer, int sign, cudaStream_t s);

// fp32 lines with a prime factor too long for the chip: the Bluestein chirp
// products lose ~sqrt(L) ulps in fp32 (1.2e-5 rel-L2 measured at n = 7001, over
// the 1e-5 bar), so the lines are widened and transformed in fp64.
cudaError_t bluestein_via_f64(void* data, int64_t n, int64_t inner, int64_t outer, int sign, cudaStream_t s) {
  const int64_t total = outer * n * inner;
  double2* wide = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&wide, (size_t)total * sizeof(double2), s);
  if (e != cudaSuccess) return e;
  {
    LaunchScope ls("long_widen", s);
    k_widen<<<grid_of(total), 256, 0, s>>>((const float2*)data, wide, total);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = long_c2c<double>(wide, n, inner, outer, sign, s);
  if (e == cudaSuccess) {
    LaunchScope ls("long_narrow", s);
    k_narrow<<<grid_of(total), 256, 0, s>>>(wide, (float2*)data, total);
    e = cudaGetLastError();
  }
  cudaFreeAsync(wide, s);
  return e;
}

bool needs_long_line(int64_t n, size_t elem_bytes) {
  return 2 * (size_t)(n + 1) * elem_bytes > kSmemLine || largest_prime_factor(n) > kMaxDirectRadix;
}

template <typename T>
cudaError_t long_c2c(void* data, int64_t n, int64_t inner, int64_t outer, int sign, cudaStream_t s) {
  using C = C_t<T>;
  if (n <= 1) return cudaSuccess;
  const int64_t big = largest_prime_factor(n);
  if (line_fits<T>(n) && big <= kMaxDirectRadix) {
    const C* tw = device_table<T>(n, 0);
    if (!tw) return cudaErrorMemoryAllocation;
    return launch_line_c2c<T>(data, (int)n, inner, outer, sign, factorize(n), tw, s);
  }
  // split n = n1 n2: the large prime factor on its own (Bluestein below), else the
  // largest factor that fits on chip
  const int64_t n1 = big > kMaxDirectRadix ? (big == n ? 1 : big) : chip_divisor<T>(n);
  if (n1 >= 2) {  // four-step
    const int64_t n2 = n / n1;
    const C* tw = device_table<T>(n, 0);
    if (!tw) return cudaErrorMemoryAllocation;
    cudaError_t e = long_c2c<T>(data, n1, inner * n2, outer, sign, s);
    if (e != cudaSuccess) return e;
    C* scratch = nullptr;
    const size_t bytes = (size_t)(outer * n * inner) * sizeof(C);
    if ((e = cudaMallocAsync((void**)&scratch, bytes, s)) != cudaSuccess) return e;
    {
      LaunchScope ls("long_twiddle_transpose", s);
      if (inner > 1)
        k_twiddle_transpose<T><<<grid_of(outer * n * inner), 256, 0, s>>>((const C*)data, scratch, n1, n2, inner, outer,
                                                                         tw, sign);
      else
        k_twiddle_transpose<T><<<(unsigned)std::min<int64_t>(outer * ((n1 + 31) / 32) * ((n2 + 31) / 32), 148 * 16),
                                 dim3(32, 8), 0, s>>>((const C*)data, scratch, n1, n2, 1, outer, tw, sign);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = long_c2c<T>(scratch, n2, inner * n1, outer, sign, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(data, scratch, bytes, cudaMemcpyDeviceToDevice, s);
    cudaFreeAsync(scratch, s);
    return e;
  }
  if (sizeof(T) == 4) return bluestein_via_f64(data, n, inner, outer, sign, s);
  // Bluestein
  int64_t L = 1;
  while (L < 2 * n - 1) L <<= 1;
  const C* chirp = device_table<T>(n, sign > 0 ? 1 : 2);
  if (!chirp) return cudaErrorMemoryAllocation;
  const int64_t lines = outer * inner;
  C *buf = nullptr, *B = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&buf, (size_t)(lines * L) * sizeof(C), s);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync((void**)&B, (size_t)L * sizeof(C), s);
  if (e == cudaSuccess) {
    LaunchScope ls("bluestein_kernel", s);
    k_blue_kernel<T><<<grid_of(L), 256, 0, s>>>(B, n, L, chirp);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = long_c2c<T>(B, L, 1, 1, +1, s);
  if (e == cudaSuccess) {
    LaunchScope ls("bluestein_pre", s);
    k_blue_pre<T><<<grid_of(lines * L), 256, 0, s>>>((const C*)data, buf, n, L, inner, lines, chirp);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = long_c2c<T>(buf, L, 1, lines, +1, s);
  if (e == cudaSuccess) {
    LaunchScope ls("bluestein_mul", s);
    k_blue_mul<T><<<grid_of(lines * L), 256, 0, s>>>(buf, B, L, lines);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = long_c2c<T>(buf, L, 1, lines, -1, s);
  if (e == cudaSuccess) {
    LaunchScope ls("bluestein_post", s);
    k_blue_post<T><<<grid_of(lines * n), 256, 0, s>>>((C*)data, buf, n, L, inner, lines, chirp);
    e = cudaGetLastError();
  }
  if (B) cudaFreeAsync(B, s);
  cudaFreeAsync(buf, s);
  return e;
}

template <typename T>
cudaError_t long_c2r_last(const void* W, void* out, int64_t n, int64_t rows, int64_t rows_per_field,
                          int64_t out_field_stride, int conj, cudaStream_t s) {
  using C = C_t<T>;
  const int64_t M = n / 2;
  const C* twN = device_table<T>(n, 0);
  if (!twN) return cudaErrorMemoryAllocation;
  C* Z = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&Z, (size_t)(rows * M) * sizeof(C), s);
  if (e != cudaSuccess) return e;
  {
    LaunchScope ls("long_c2r_pre", s);
    if (conj) k_c2r_pre<T, 1><<<grid_of(rows * M), 256, 0, s>>>((const C*)W, Z, M, rows, twN);
    else k_c2r_pre<T, 0><<<grid_of(rows * M), 256, 0, s>>>((const C*)W, Z, M, rows, twN);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = long_c2c<T>(Z, M, 1, rows, +1, s);
  if (e == cudaSuccess) {
    LaunchScope ls("long_rows_out", s);
    k_rows_out<T><<<grid_of(rows * M), 256, 0, s>>>(Z, (T*)out, M, rows, rows_per_field, out_field_stride);
    e = cudaGetLastError();
  }
  cudaFreeAsync(Z, s);
  return e;
}

template <typename T>
cudaError_t long_r2c_last_noise(void* W, int64_t n, int64_t rows, int64_t rows_per_field, uint64_t seed,
                                uint64_t field0, const double* injected, cudaStream_t s) {
  using C = C_t<T>;
  const int64_t M = n / 2;
  const C* twN = device_table<T>(n, 0);
  if (!twN) return cudaErrorMemoryAllocation;
  C* Z = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&Z, (size_t)(rows * M) * sizeof(C), s);
  if (e != cudaSuccess) return e;
  {
    LaunchScope ls("long_noise_rows", s);
    k_noise_rows<T><<<grid_of(rows * M), 256, 0, s>>>(Z, M, rows, rows_per_field, philox_key(seed), field0, injected);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = long_c2c<T>(Z, M, 1, rows, +1, s);
  if (e == cudaSuccess) {
    LaunchScope ls("long_r2c_post", s);
    k_r2c_post<T><<<grid_of(rows * (M + 1)), 256, 0, s>>>(Z, (C*)W, M, rows, twN);
    e = cudaGetLastError();
  }
  cudaFreeAsync(Z, s);
  return e;
}

#define GRFC_LONG_INST(T)                                                                                     \
  template cudaError_t long_c2c<T>(void*, int64_t, int64_t, int64_t, int, cudaStream_t);                    \
  template cudaError_t long_c2r_last<T>(const void*, void*, int64_t, int64_t, int64_t, int64_t, int,         \
                                        cudaStream_t);                                                       \
  template cudaError_t long_r2c_last_noise<T>(void*, int64_t, int64_t, int64_t, uint64_t, uint64_t,          \
                                              const double*, cudaStream_t);
GRFC_LONG_INST(float)
GRFC_LONG_INST(double)

}  // namespace grfc
