// Direct-sum d-dimensional complex DFT on the device: the drop-in's
// NaiveDftBackend (replaces /root/reference/proj/core/src/dft.cpp:113-165, the
// reference's O(P^2) cross-check backend). Same conventions as grfc_dft_c2c:
//   sign = +1: out[K] = sum_J in[J] e^{+2 pi i sum_a k_a j_a / N_a}
//   sign = -1: out[J] = P^-1 sum_K in[K] e^{-2 pi i ...}
// The phase of each term is reduced exactly per axis, (k_a j_a) mod N_a, and
// looked up in that axis's table of e^{2 pi i m / N_a} (long-double angles), so
// the sum is independent of the fast transform's factorisation — what makes it
// a cross-check.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/grfc.h"
#include "grfc_internal.cuh"

namespace grfc {

grfc_status set_error(grfc_status s, const std::string& msg);  // api.cu: thread-local grfc_last_error()

struct NaiveGeom {
  int dim;
  int64_t n[GRFC_MAX_DIM];
  int64_t tw_off[GRFC_MAX_DIM];  // axis a's table at tw + tw_off[a]
  int64_t P;
};

// One thread per output cell; the input is walked row-major with an odometer
// that keeps the per-axis phase indices (k_a j_a) mod N_a up to date.
__global__ void k_dft_direct(NaiveGeom g, const double2* __restrict__ in, double2* __restrict__ out,
                             const double2* __restrict__ tw, int conj, double scale) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < g.P; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t k[GRFC_MAX_DIM], ph[GRFC_MAX_DIM], j[GRFC_MAX_DIM];
    int64_t rem = o;
    for (int a = g.dim - 1; a >= 0; --a) {
      k[a] = rem % g.n[a];
      rem /= g.n[a];
      ph[a] = 0;
      j[a] = 0;
    }
    double re = 0.0, im = 0.0;
    for (int64_t i = 0; i < g.P; ++i) {
      double wr = 1.0, wi = 0.0;
      for (int a = 0; a < g.dim; ++a) {
        const double2 t = tw[g.tw_off[a] + ph[a]];
        const double ti = conj ? -t.y : t.y;
        const double r2 = wr * t.x - wi * ti;
        wi = wr * ti + wi * t.x;
        wr = r2;
      }
      const double2 x = in[i];
      re += x.x * wr - x.y * wi;
      im += x.x * wi + x.y * wr;
      // odometer: last axis fastest
      for (int a = g.dim - 1; a >= 0; --a) {
        ph[a] += k[a];
        if (ph[a] >= g.n[a]) ph[a] -= g.n[a];
        if (++j[a] < g.n[a]) break;
        j[a] = 0;
        ph[a] = 0;
      }
    }
    out[o] = make_double2(re * scale, im * scale);
  }
}

}  // namespace grfc

using namespace grfc;

namespace {

grfc_status naive_fail(grfc_status st, const std::string& m) { return grfc::set_error(st, m); }

grfc_status naive_check_args(int dim, const int64_t* counts, const void* in, const void* out, NaiveGeom& g) {
  if (!counts || !in || !out) return naive_fail(GRFC_EINVAL, "grfc: null argument");
  if (in == out) return naive_fail(GRFC_EINVAL, "DftBackend: in-place transform not supported");
  if (dim < 1 || dim > GRFC_MAX_DIM) return naive_fail(GRFC_EINVAL, "grfc: bad dimension");
  g.dim = dim;
  g.P = 1;
  int64_t off = 0;
  for (int a = 0; a < dim; ++a) {
    if (counts[a] < 1) return naive_fail(GRFC_EINVAL, "grfc: bad extent");
    g.n[a] = counts[a];
    g.tw_off[a] = off;
    off += counts[a];
    g.P *= counts[a];
  }
  return GRFC_OK;
}

}  // namespace

extern "C" {

grfc_status grfc_dft_naive_c2c(int dim, const int64_t* counts, const double* d_in, double* d_out, int sign,
                               void* stream) {
  NaiveGeom g{};
  grfc_status st = naive_check_args(dim, counts, d_in, d_out, g);
  if (st != GRFC_OK) return st;
  std::vector<double2> tw;
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int a = 0; a < dim; ++a)
    for (int64_t m = 0; m < counts[a]; ++m) {
      const long double ang = two_pi * (long double)m / (long double)counts[a];
      tw.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
  cudaStream_t s = (cudaStream_t)stream;
  double2* d_tw = nullptr;
  cudaError_t e = cudaMallocAsync(&d_tw, tw.size() * sizeof(double2), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    LaunchScope ls("dft_direct", s);
    const int64_t blocks = (g.P + 127) / 128;
    k_dft_direct<<<(unsigned)(blocks < 65535 ? blocks : 65535), 128, 0, s>>>(
        g, reinterpret_cast<const double2*>(d_in), reinterpret_cast<double2*>(d_out), d_tw, sign < 0 ? 1 : 0,
        sign < 0 ? 1.0 / (double)g.P : 1.0);
    e = cudaGetLastError();
  }
  if (d_tw) cudaFreeAsync(d_tw, s);
  // the host table must outlive the async copy
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return naive_fail(GRFC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  return GRFC_OK;
}

grfc_status grfc_dft_naive_c2c_host(int dim, const int64_t* counts, const double* h_in, double* h_out, int sign,
                                    int device) {
  NaiveGeom g{};
  grfc_status st = naive_check_args(dim, counts, h_in, h_out, g);
  if (st != GRFC_OK) return st;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  double *din = nullptr, *dout = nullptr;
  const size_t bytes = (size_t)g.P * 16;
  if (e == cudaSuccess) e = cudaMalloc(&din, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&dout, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(din, h_in, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) st = naive_fail(GRFC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  if (st == GRFC_OK) st = grfc_dft_naive_c2c(dim, counts, din, dout, sign, nullptr);
  if (st == GRFC_OK) {
    e = cudaMemcpy(h_out, dout, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = naive_fail(GRFC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  }
  cudaFree(din);
  cudaFree(dout);
  cudaSetDevice(prev);
  return st;
}

}  // extern "C"
