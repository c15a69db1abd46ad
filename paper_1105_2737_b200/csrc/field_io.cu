// GRF1 batch writer: device fields -> pinned host -> one GRF1 file per field,
// the on-disk format after the generator (reference include/grf/field_io.hpp:10-14,
// src/field_io.cpp:60-80):
//   "GRF1" | u32 version = 1 | u32 dim | per axis: u64 N_i, f64 l_i | P f64, row-major,
// all little-endian. Files are bit-exact with the reference's write_grf1 for
// the same values (fp32 plans are widened exactly to f64).
//
// Pipeline per chunk of fields (~64 MiB of device output): generation on the
// caller's stream, D2H on a copy stream into one of two pinned buffers, and
// the host writes chunk i-1's files while the device generates and copies
// chunk i. Host code only (the kernels are grfc_generate's).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/grfc.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "GRF1 writer assumes a little-endian host");

namespace grfc {

grfc_status set_error(grfc_status s, const std::string& msg);  // api.cu

namespace {

std::string expand_path(const std::string& fmt, uint64_t field) {
  static const std::string key = "{field}";
  const size_t at = fmt.find(key);
  if (at == std::string::npos) return fmt;
  return fmt.substr(0, at) + std::to_string(field) + fmt.substr(at + key.size());
}

std::string header(int dim, const int64_t* counts, const double* lengths) {
  std::string h("GRF1", 4);
  const uint32_t version = 1, d = (uint32_t)dim;
  h.append((const char*)&version, 4);
  h.append((const char*)&d, 4);
  for (int a = 0; a < dim; ++a) {
    const uint64_t n = (uint64_t)counts[a];
    h.append((const char*)&n, 8);
    h.append((const char*)&lengths[a], 8);
  }
  return h;
}

grfc_status write_one(const std::string& path, const std::string& hdr, const void* values, bool f32, uint64_t P,
                      std::vector<double>& widen) {
  std::FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) return set_error(GRFC_ERUNTIME, "write_grf1: cannot open '" + path + "' for writing");
  const void* payload = values;
  if (f32) {
    widen.resize(P);
    const float* v = (const float*)values;
    for (uint64_t i = 0; i < P; ++i) widen[i] = (double)v[i];
    payload = widen.data();
  }
  bool ok = std::fwrite(hdr.data(), 1, hdr.size(), fp) == hdr.size();
  ok = ok && std::fwrite(payload, 8, P, fp) == P;
  ok = (std::fclose(fp) == 0) && ok;
  if (!ok) return set_error(GRFC_ERUNTIME, "write_grf1: write failed for '" + path + "'");
  return GRFC_OK;
}

}  // namespace
}  // namespace grfc

using namespace grfc;

extern "C" grfc_status grfc_write_grf1(grfc_plan p, uint64_t seed, uint64_t first_field, uint64_t nfields,
                                       const char* path_format) {
  if (!p || !path_format) return set_error(GRFC_EINVAL, "grfc: null argument");
  const std::string fmt(path_format);
  if (nfields > 1 && fmt.find("{field}") == std::string::npos)
    return set_error(GRFC_EINVAL, "write_grf1: a batch needs a '{field}' placeholder in the path");
  if (nfields == 0) return GRFC_OK;
  uint64_t cells = 0, P = 0;
  const char* path_name = nullptr;
  grfc_status st = grfc_plan_info(p, &cells, &P, &path_name);
  if (st != GRFC_OK) return st;
  int dim = 0, dtype = 0, device = 0;
  int64_t counts[GRFC_MAX_DIM];
  double lengths[GRFC_MAX_DIM];
  st = grfc_plan_grid(p, &dim, counts, lengths, &dtype, &device);
  if (st != GRFC_OK) return st;
  const bool f32 = dtype == GRFC_F32;
  const size_t fbytes = (size_t)P * (f32 ? 4 : 8);
  const std::string hdr = header(dim, counts, lengths);
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(nfields, (64ull << 20) / fbytes));

  int prev_dev = 0;
  cudaGetDevice(&prev_dev);
  cudaSetDevice(device);
  cudaStream_t sg = nullptr, sc = nullptr;
  cudaEvent_t gen[2] = {}, cp[2] = {};
  void* dbuf[2] = {};
  void* hbuf[2] = {};
  cudaError_t e = cudaStreamCreateWithFlags(&sg, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaEventCreateWithFlags(&gen[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cp[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&dbuf[b], chunk * fbytes);
    if (e == cudaSuccess) e = cudaMallocHost(&hbuf[b], chunk * fbytes);
  }
  if (e != cudaSuccess) st = set_error(GRFC_ECUDA, std::string("CUDA: write_grf1 setup: ") + cudaGetErrorString(e));
  std::vector<double> widen;
  // host side: write the files of chunk i once its D2H copy has landed
  auto flush = [&](uint64_t i) -> grfc_status {
    const int b = (int)(i & 1);
    const uint64_t f0 = i * chunk, n = std::min<uint64_t>(chunk, nfields - f0);
    const cudaError_t ce = cudaEventSynchronize(cp[b]);
    if (ce != cudaSuccess) return set_error(GRFC_ECUDA, std::string("CUDA: write_grf1 D2H: ") + cudaGetErrorString(ce));
    for (uint64_t k = 0; k < n; ++k) {
      const grfc_status ws = write_one(expand_path(fmt, first_field + f0 + k), hdr,
                                       (const char*)hbuf[b] + k * fbytes, f32, P, widen);
      if (ws != GRFC_OK) return ws;
    }
    return GRFC_OK;
  };
  const uint64_t nchunks = (nfields + chunk - 1) / chunk;
  for (uint64_t i = 0; i < nchunks && st == GRFC_OK; ++i) {
    const int b = (int)(i & 1);
    const uint64_t f0 = i * chunk, n = std::min<uint64_t>(chunk, nfields - f0);
    if (i >= 2) cudaStreamWaitEvent(sg, cp[b], 0);  // device buffer b drained (its files were flushed below)
    st = grfc_generate(p, seed, first_field + f0, n, dbuf[b], P, sg);
    if (st != GRFC_OK) break;
    cudaEventRecord(gen[b], sg);
    cudaStreamWaitEvent(sc, gen[b], 0);
    e = cudaMemcpyAsync(hbuf[b], dbuf[b], n * fbytes, cudaMemcpyDeviceToHost, sc);
    if (e != cudaSuccess) {
      st = set_error(GRFC_ECUDA, std::string("CUDA: write_grf1 D2H: ") + cudaGetErrorString(e));
      break;
    }
    cudaEventRecord(cp[b], sc);
    if (i >= 1) st = flush(i - 1);  // overlaps chunk i on the device
  }
  if (st == GRFC_OK) st = flush(nchunks - 1);
  if (sg) cudaStreamSynchronize(sg);
  if (sc) cudaStreamSynchronize(sc);
  for (int b = 0; b < 2; ++b) {
    if (dbuf[b]) cudaFree(dbuf[b]);
    if (hbuf[b]) cudaFreeHost(hbuf[b]);
    if (gen[b]) cudaEventDestroy(gen[b]);
    if (cp[b]) cudaEventDestroy(cp[b]);
  }
  if (sg) cudaStreamDestroy(sg);
  if (sc) cudaStreamDestroy(sc);
  cudaSetDevice(prev_dev);
  return st;
}
