// Host side of the fused pow2 2D path: plan setup and dispatch. The kernels
// live in fast2d_kernels.cuh and are instantiated per (dtype, size) by
// fast2d_inst.cu (one object per combination, compiled in parallel).
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "fast2d.h"
#include "grfc_internal.cuh"
#include "kernels.h"

namespace grfc {

struct F2Params;
template <typename T, int N1, int ALG>
cudaError_t launch_cols(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W, cudaStream_t s);
template <typename T, int M>
cudaError_t launch_rows(const Fast2D& f, int64_t nf, const void* W, void* out, int64_t stride, cudaStream_t s);
template <typename T, int N1, int M, int ALG>
cudaError_t launch_fused(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* ws, void* out,
                         int64_t stride, cudaStream_t s, const void* xpre);
constexpr int kPreX = 8;  // fast2d_kernels.cuh
template <typename T, int N1, int M, int ALG>
cudaError_t fused_query(Fast2D& f);
template <typename T, int N1, int M>
cudaError_t launch_cluster(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* ws, void* out,
                           int64_t stride, cudaStream_t s);
template <typename T, int N1, int M>
cudaError_t cluster_query(Fast2D& f, int cs, int nsl);
template <typename T, int N1, int M>
cudaError_t launch_fused_alg1(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out, int64_t stride,
                              cudaStream_t s);
template <typename T, int N1, int M>
cudaError_t alg1_check();

static bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

bool fast2d_supported(int d, const int64_t* n, int dtype, int alg, int family) {
  (void)dtype;
  (void)family;
  if (d != 2) return false;
  if (!is_pow2(n[0]) || !is_pow2(n[1])) return false;
  return n[0] >= 256 && n[0] <= 4096 && n[1] >= 256 && n[1] <= 4096;
}

const char* fast2d_name(const Fast2D& f) { return f.dtype == GRFC_F64 ? "pow2-2d-f64" : "pow2-2d-f32"; }

template <typename T>
static std::vector<C_t<T>> host_twiddles(int64_t n) {
  std::vector<C_t<T>> t((size_t)n);
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int64_t m = 0; m < n; ++m) {
    const long double a = two_pi * (long double)m / (long double)n;
    t[(size_t)m].x = (T)cosl(a);
    t[(size_t)m].y = (T)sinl(a);
  }
  return t;
}

template <typename T, int ALG>
static cudaError_t dispatch_cols(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W,
                                 cudaStream_t s) {
  switch (f.n1) {
    case 256: return launch_cols<T, 256, ALG>(f, seed, field0, nf, W, s);
    case 512: return launch_cols<T, 512, ALG>(f, seed, field0, nf, W, s);
    case 1024: return launch_cols<T, 1024, ALG>(f, seed, field0, nf, W, s);
    case 2048: return launch_cols<T, 2048, ALG>(f, seed, field0, nf, W, s);
    case 4096: return launch_cols<T, 4096, ALG>(f, seed, field0, nf, W, s);
  }
  return cudaErrorNotSupported;
}

template <typename T>
static cudaError_t dispatch_rows(const Fast2D& f, int64_t nf, const void* W, void* out, int64_t stride,
                                 cudaStream_t s) {
  switch (f.n2 / 2) {
    case 128: return launch_rows<T, 128>(f, nf, W, out, stride, s);
    case 256: return launch_rows<T, 256>(f, nf, W, out, stride, s);
    case 512: return launch_rows<T, 512>(f, nf, W, out, stride, s);
    case 1024: return launch_rows<T, 1024>(f, nf, W, out, stride, s);
    case 2048: return launch_rows<T, 2048>(f, nf, W, out, stride, s);
  }
  return cudaErrorNotSupported;
}

// (N1, M) -> instantiation; F is a functor template taking <N1, M>.
#define GRFC_DISPATCH_M(T, N1, ALG, CALL)                   \
  switch (f.n2 / 2) {                                      \
    case 128: return CALL(T, N1, 128, ALG);                \
    case 256: return CALL(T, N1, 256, ALG);                \
    case 512: return CALL(T, N1, 512, ALG);                \
    case 1024: return CALL(T, N1, 1024, ALG);              \
    case 2048: return CALL(T, N1, 2048, ALG);              \
  }                                                        \
  return cudaErrorNotSupported;
#define GRFC_DISPATCH_N1(T, ALG, CALL)                      \
  switch (f.n1) {                                          \
    case 256: { GRFC_DISPATCH_M(T, 256, ALG, CALL) }       \
    case 512: { GRFC_DISPATCH_M(T, 512, ALG, CALL) }       \
    case 1024: { GRFC_DISPATCH_M(T, 1024, ALG, CALL) }     \
    case 2048: { GRFC_DISPATCH_M(T, 2048, ALG, CALL) }     \
    case 4096: { GRFC_DISPATCH_M(T, 4096, ALG, CALL) }     \
  }                                                        \
  return cudaErrorNotSupported;

#define GRFC_CALL_FUSED(T, N1, M, ALG) launch_fused<T, N1, M, ALG>(f, seed, field0, nf, W, out, stride, s, nullptr)
#define GRFC_CALL_FUSED_PRE(T, N1, M, ALG) launch_fused<T, N1, M, ALG>(f, seed, field0, nf, W, out, stride, s, xpre)
#define GRFC_CALL_QUERY(T, N1, M, ALG) fused_query<T, N1, M, ALG>(f)
#define GRFC_CALL_ALG1(T, N1, M, ALG) launch_fused_alg1<T, N1, M>(f, seed, field0, nf, out, stride, s)

template <typename T>
static cudaError_t dispatch_alg1(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out,
                                 int64_t stride, cudaStream_t s) {
  GRFC_DISPATCH_N1(T, 0, GRFC_CALL_ALG1)
}

#define GRFC_CALL_ALG1_CHECK(T, N1, M, ALG) alg1_check<T, N1, M>()
template <typename T>
static cudaError_t dispatch_alg1_check(const Fast2D& f) {
  GRFC_DISPATCH_N1(T, 0, GRFC_CALL_ALG1_CHECK)
}

template <typename T, int ALG>
static cudaError_t dispatch_fused(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                                  int64_t stride, cudaStream_t s) {
  GRFC_DISPATCH_N1(T, ALG, GRFC_CALL_FUSED)
}

static cudaError_t dispatch_fused_pre(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W,
                                      void* out, int64_t stride, cudaStream_t s, const void* xpre) {
  GRFC_DISPATCH_N1(double, kPreX, GRFC_CALL_FUSED_PRE)
}

template <typename T, int ALG>
static cudaError_t dispatch_query(Fast2D& f) {
  GRFC_DISPATCH_N1(T, ALG, GRFC_CALL_QUERY)
}

#define GRFC_CALL_CL(T, N1, M, ALG) launch_cluster<T, N1, M>(f, seed, field0, nf, W, out, stride, s)
#define GRFC_CALL_CLQ(T, N1, M, ALG) cluster_query<T, N1, M>(f, cs, nsl)
template <typename T>
static cudaError_t dispatch_cluster(const Fast2D& f, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                                    int64_t stride, cudaStream_t s) {
  GRFC_DISPATCH_N1(T, 0, GRFC_CALL_CL)
}
template <typename T>
static cudaError_t dispatch_clquery(Fast2D& f, int cs, int nsl) {
  GRFC_DISPATCH_N1(T, 0, GRFC_CALL_CLQ)
}

template <typename T>
static cudaError_t run_fast(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                            int64_t stride, cudaStream_t s) {
  if (f.persistent && f.cluster && alg == GRFC_ONE_FFT_OVERWRITE)
    return dispatch_cluster<T>(f, seed, field0, nf, W, out, stride, s);
  if (f.persistent && alg == GRFC_ONE_FFT_OVERWRITE)
    return dispatch_fused<T, GRFC_ONE_FFT_OVERWRITE>(f, seed, field0, nf, W, out, stride, s);
  cudaError_t e = alg == GRFC_ONE_FFT_OVERWRITE ? dispatch_cols<T, GRFC_ONE_FFT_OVERWRITE>(f, seed, field0, nf, W, s)
                                                : dispatch_cols<T, GRFC_ONE_FFT_RECURSIVE>(f, seed, field0, nf, W, s);
  if (e != cudaSuccess) return e;
  return dispatch_rows<T>(f, nf, W, out, stride, s);
}

// sqrt(g(w_K)) * mult for every half-lattice cell, fp64 evaluation (the
// generic device density, sqrt_gamma) rounded once to fp32.
__global__ void k_sg_table(GridDesc g, DensityDesc D, double mult, float* __restrict__ out) {
  const int64_t cells = g.n[0] * g.hd;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < cells; h += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k[2] = {h / g.hd, h % g.hd};
    int64_t kw[2];
    wrap_freq(g, k, kw);
    out[h] = (float)(sqrt_gamma<double>(g, D, kw, h) * mult);
  }
}

cudaError_t fast2d_set_table(Fast2D& f, const double* d_table) {
  if (d_table) f.D.table = d_table;
  if (!f.d_sg) return cudaSuccess;
  k_sg_table<<<148, 256>>>(f.g, f.D, f.sg_mult, f.d_sg);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? cudaDeviceSynchronize() : e;
}

cudaError_t fast2d_init(Fast2D& f, const GridDesc& g, const DensityDesc& D, int dtype, int alg, double s_one,
                        double s_two) {
  f.n1 = (int)g.n[0];
  f.n2 = (int)g.n[1];
  f.dtype = dtype;
  f.alg = alg;
  if (alg == GRFC_TWO_FFT) {  // (N1, M) pairs without a fused Algorithm-1 kernel: generic path
    const cudaError_t ok = dtype == GRFC_F64 ? dispatch_alg1_check<double>(f) : dispatch_alg1_check<float>(f);
    if (ok != cudaSuccess) return cudaErrorNotSupported;
  }
  f.g = g;
  f.D = D;
  f.s_one = s_one;
  f.s_two = s_two;
  const size_t cs = dtype == GRFC_F64 ? 16 : 8;
  f.fail_what = "twiddle upload";
  cudaError_t e = cudaMalloc(&f.d_tw, (size_t)(f.n1 + f.n2) * cs);
  if (e != cudaSuccess) return e;
  if (dtype == GRFC_F64) {
    auto a = host_twiddles<double>(f.n1), b = host_twiddles<double>(f.n2);
    a.insert(a.end(), b.begin(), b.end());
    e = cudaMemcpy(f.d_tw, a.data(), a.size() * cs, cudaMemcpyHostToDevice);
  } else {
    auto a = host_twiddles<float>(f.n1), b = host_twiddles<float>(f.n2);
    a.insert(a.end(), b.begin(), b.end());
    e = cudaMemcpy(f.d_tw, a.data(), a.size() * cs, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) return e;
  // Density table of the fp32 Algorithm-2 column tiles: one L2-resident load per
  // cell replaces the per-cell evaluation. Used for every family without an SFU
  // form (otherwise evaluated per cell in fp64); Matern / Gaussian keep the SFU
  // form, which measured faster (c2 292 vs 286, c5 273 vs 269 Gpts/s).
  // GRFC_SG_TABLE=0/1 forces it off/on.
  const size_t sg_bytes = (size_t)f.n1 * (size_t)(f.n2 / 2 + 1) * sizeof(float);
  const char* sge = std::getenv("GRFC_SG_TABLE");
  const bool sfu_family = D.family == GRFC_DENSITY_MATERN || D.family == GRFC_DENSITY_GAUSSIAN_COV;
  const bool want_sg = sge ? sge[0] == '1' : !sfu_family;
  // The fp32 Algorithm-1 kernel always uses the table (sqrt(g) x its scale s_two):
  // its column tile then holds no per-cell density code at all (the inlined fp64
  // fallbacks made the kernel 48k instructions long: I-cache misses).
  const bool alg1_f32 = dtype == GRFC_F32 && alg == GRFC_TWO_FFT;
  if ((dtype == GRFC_F32 && alg == GRFC_ONE_FFT_OVERWRITE && sg_bytes <= Fast2D::kSgTableMax && want_sg) ||
      alg1_f32) {
    f.fail_what = "density table";
    e = cudaMalloc(&f.d_sg, sg_bytes);
    if (e != cudaSuccess) return e;
    f.sg_mult = alg1_f32 ? s_two : s_one * 0.70710678118654752440;
    // a user table (GRFC_DENSITY_TABLE) is not uploaded yet: fast2d_set_table
    // builds d_sg when grfc_plan_set_sqrt_gamma_table supplies it
    if (D.family != GRFC_DENSITY_TABLE) {
      e = fast2d_set_table(f, nullptr);
      if (e != cudaSuccess) return e;
    }
  }
  // Pipeline chunk: ~12 MiB of half-spectrum per slot, 3 slots in flight (L2-resident).
  const double slot = (double)f.n1 * (f.n2 / 2) * cs;
  f.chunk = (int64_t)std::max(1.0, std::floor(12.0 * 1024 * 1024 / slot));
  f.l2_budget = 40.0 * 1024 * 1024;
  f.fail_what = "pipeline streams";
  e = cudaStreamCreateWithFlags(&f.sa, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&f.sb, cudaStreamNonBlocking);
  cudaEvent_t* evs[] = {&f.ev_fork, &f.ev_ja, &f.ev_jb};
  for (auto* ev : evs)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  for (int i = 0; i < Fast2D::kRing && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&f.ev_cols[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f.ev_rows[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return e;
  f.mu = new std::mutex();
  // Default: the single-launch persistent kernel; GRFC_PERSISTENT=0 selects the
  // two-stream column/row kernel pipeline (A/B testing).
  const char* pe = std::getenv("GRFC_PERSISTENT");
  f.persistent = !(pe && pe[0] == '0');
  // Persistent fused kernel: Algorithm 2; Algorithm 3 uses the column/row kernel pair.
  if (alg != GRFC_ONE_FFT_OVERWRITE) f.persistent = false;
  if (!f.persistent) return cudaSuccess;
  f.fail_what = "persistent kernel query";
  e = dtype == GRFC_F64 ? dispatch_query<double, GRFC_ONE_FFT_OVERWRITE>(f)
                        : dispatch_query<float, GRFC_ONE_FFT_OVERWRITE>(f);
  if (e != cudaSuccess) return e;
  // Scheduler groups (group_geometry): GRFC_GROUP = CTAs per group (0: one queue),
  // GRFC_GROUP_L / GRFC_GROUP_S = lookahead / ring slots per group.
  if (const char* ge = std::getenv("GRFC_GROUP")) f.group = std::atoi(ge);
  if (const char* ge = std::getenv("GRFC_GROUP_L")) f.group_L = std::max(1, std::atoi(ge));
  if (const char* ge = std::getenv("GRFC_GROUP_S")) f.group_S = std::max(1, std::atoi(ge));
  // Cluster-scheduled variant (k_fused2d_cl): GRFC_CLUSTER = CTAs per cluster,
  // GRFC_CSLOTS = W slots per cluster (1 or 2).
  const char* ce = std::getenv("GRFC_CLUSTER");
  const int ncs = ce ? std::atoi(ce) : 0;
  if (ncs > 0) {
    const char* se = std::getenv("GRFC_CSLOTS");
    const int nsl = se && se[0] == '2' ? 2 : 1;
    f.fail_what = "cluster kernel query";
    e = dtype == GRFC_F64 ? dispatch_clquery<double>(f, ncs, nsl) : dispatch_clquery<float>(f, ncs, nsl);
  }
  return e;
}

size_t fast2d_workspace_bytes(const Fast2D& f, int64_t nf) {
  const size_t slot = (size_t)f.n1 * (size_t)(f.n2 / 2) * (f.dtype == GRFC_F64 ? 16 : 8);
  if (!f.persistent) return slot * (size_t)nf;
  if (f.cluster) return slot * (size_t)f.cslots * (size_t)std::min<int64_t>(f.nclusters, nf);
  const GroupGeom gg = group_geometry(f, nf);
  if (gg.groups > 1) return (fused_ctr_bytes(gg.S) + slot * gg.S) * gg.groups;
  uint32_t L, S, c;
  fused_geometry(f, nf, &L, &S, &c);
  return fused_ctr_bytes(S) + slot * S;
}

void fast2d_free(Fast2D& f) {
  cudaFree(f.d_tw);
  f.d_tw = nullptr;
  cudaFree(f.d_sg);
  f.d_sg = nullptr;
  if (f.sa) cudaStreamDestroy(f.sa);
  if (f.sb) cudaStreamDestroy(f.sb);
  cudaEvent_t evs[] = {f.ev_fork, f.ev_ja, f.ev_jb};
  for (auto ev : evs)
    if (ev) cudaEventDestroy(ev);
  for (int i = 0; i < Fast2D::kRing; ++i) {
    if (f.ev_cols[i]) cudaEventDestroy(f.ev_cols[i]);
    if (f.ev_rows[i]) cudaEventDestroy(f.ev_rows[i]);
  }
  delete static_cast<std::mutex*>(f.mu);
  f.mu = nullptr;
}

template <typename T>
static cudaError_t launch_cols_any(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W,
                                   cudaStream_t s) {
  return alg == GRFC_ONE_FFT_OVERWRITE ? dispatch_cols<T, GRFC_ONE_FFT_OVERWRITE>(f, seed, field0, nf, W, s)
                                       : dispatch_cols<T, GRFC_ONE_FFT_RECURSIVE>(f, seed, field0, nf, W, s);
}

cudaError_t fast2d_generate(Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* out,
                            int64_t stride, cudaStream_t s) {
  const size_t esz = f.dtype == GRFC_F64 ? 8 : 4;
  void* ws = nullptr;
  if (alg == GRFC_TWO_FFT)  // Algorithm 1: always the persistent three-tile kernel
    return f.dtype == GRFC_F64 ? dispatch_alg1<double>(f, seed, field0, nf, out, stride, s)
                               : dispatch_alg1<float>(f, seed, field0, nf, out, stride, s);
  static const bool prex_on = !(std::getenv("GRFC_PREX") && std::getenv("GRFC_PREX")[0] == '0');  // A/B switch
  if (prex_on && f.persistent && f.dtype == GRFC_F64 && !f.cluster && nf * f.strips < f.sms) {
    // a batch whose column tiles cannot fill the GPU (c1: one 512^2 field = 64
    // tiles): X(K) for every cell first, one cell per thread over all SMs
    // (k_gen_x2d), then the fused kernel with column tiles that load it (kPreX)
    const size_t xbytes = (size_t)nf * f.n1 * (f.n2 / 2 + 1) * 16;
    void* xpre = nullptr;
    cudaError_t e = cudaMallocAsync(&xpre, xbytes, s);
    if (e != cudaSuccess) return e;
    e = cudaMallocAsync(&ws, fast2d_workspace_bytes(f, nf), s);
    if (e == cudaSuccess) e = dispatch_fused_pre(f, seed, field0, nf, ws, out, stride, s, xpre);
    if (ws) cudaFreeAsync(ws, s);
    cudaFreeAsync(xpre, s);
    return e;
  }
  if (f.persistent) {
    cudaError_t e = cudaMallocAsync(&ws, fast2d_workspace_bytes(f, nf), s);
    if (e != cudaSuccess) return e;
    e = launch_fast2d(f, alg, seed, field0, nf, ws, out, stride, s);
    cudaFreeAsync(ws, s);
    return e;
  }
  std::lock_guard<std::mutex> lock(*static_cast<std::mutex*>(f.mu));
  const int64_t chunk = std::min<int64_t>(f.chunk, nf);
  const size_t slot_bytes = (size_t)chunk * f.n1 * (f.n2 / 2) * 2 * esz;
  const int ring = (int)std::min<int64_t>(Fast2D::kRing, (nf + chunk - 1) / chunk);
  cudaError_t e = cudaMallocAsync(&ws, slot_bytes * ring, s);
  if (e != cudaSuccess) return e;
  cudaEventRecord(f.ev_fork, s);
  cudaStreamWaitEvent(f.sa, f.ev_fork, 0);
  cudaStreamWaitEvent(f.sb, f.ev_fork, 0);
  int i = 0;
  for (int64_t f0 = 0; f0 < nf && e == cudaSuccess; f0 += chunk, ++i) {
    const int sl = i % ring;
    const int64_t n = std::min<int64_t>(chunk, nf - f0);
    void* W = (char*)ws + sl * slot_bytes;
    if (i >= ring) cudaStreamWaitEvent(f.sa, f.ev_rows[sl], 0);  // slot consumed by rows(i - ring)
    e = f.dtype == GRFC_F64 ? launch_cols_any<double>(f, alg, seed, field0 + f0, n, W, f.sa)
                            : launch_cols_any<float>(f, alg, seed, field0 + f0, n, W, f.sa);
    if (e != cudaSuccess) break;
    cudaEventRecord(f.ev_cols[sl], f.sa);
    cudaStreamWaitEvent(f.sb, f.ev_cols[sl], 0);
    char* o = (char*)out + f0 * stride * esz;
    e = f.dtype == GRFC_F64 ? dispatch_rows<double>(f, n, W, o, stride, f.sb)
                            : dispatch_rows<float>(f, n, W, o, stride, f.sb);
    cudaEventRecord(f.ev_rows[sl], f.sb);
  }
  cudaEventRecord(f.ev_ja, f.sa);
  cudaEventRecord(f.ev_jb, f.sb);
  cudaStreamWaitEvent(s, f.ev_ja, 0);
  cudaStreamWaitEvent(s, f.ev_jb, 0);
  cudaFreeAsync(ws, s);
  return e;
}

cudaError_t launch_fast2d(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                          int64_t stride, cudaStream_t s) {
  if (f.dtype == GRFC_F64) return run_fast<double>(f, alg, seed, field0, nf, W, out, stride, s);
  return run_fast<float>(f, alg, seed, field0, nf, W, out, stride, s);
}

}  // namespace grfc
