// Fused fast path for power-of-two 2D grids (the BASELINE configs c1, c2, c3,
// c5): generation fused into the column pass, Nyquist column packed into the
// imaginary part of column 0, and an L2-resident half-spectrum intermediate.
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include "grfc_internal.cuh"

namespace grfc {

struct Fast2D {
  int n1 = 0, n2 = 0;  // grid N_1 x N_2
  int dtype = 0;
  int alg = 1;
  GridDesc g{};
  DensityDesc D{};
  double s_one = 1.0, s_two = 1.0;
  double l2_budget = 48.0 * 1024 * 1024;  // bytes of workspace per chunk
  void* d_tw = nullptr;                   // twiddles
  // fp32 Algorithm 2: sqrt(g) x scale / sqrt 2 per half-lattice cell (n1 x (n2/2+1)),
  // evaluated once per plan in fp64; nullptr when larger than kSgTableMax
  float* d_sg = nullptr;
  double sg_mult = 1.0;  // the factor d_sg folds in
  static constexpr size_t kSgTableMax = 8u << 20;
  int kind = 0;
  // persistent fused kernel geometry (fused_query)
  bool persistent = false;
  int occ = 1, sms = 148, strips = 0, rtiles = 0;
  // cluster-scheduled fused kernel (k_fused2d_cl): CTAs per cluster (0 = off),
  // W slots per cluster, resident clusters
  int cluster = 0, cslots = 1, nclusters = 0;
  // scheduler groups of the persistent kernel (group_geometry; read at plan setup)
  int group = 0, group_L = 1, group_S = 2;
  // two-stream pipeline: column kernels on sa, row kernels on sb, a ring of
  // kRing chunk slots ordered by events (no in-kernel waiting).
  static constexpr int kRing = 3;
  cudaStream_t sa = nullptr, sb = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_ja = nullptr, ev_jb = nullptr;
  cudaEvent_t ev_cols[kRing] = {}, ev_rows[kRing] = {};
  void* mu = nullptr;  // std::mutex*, serialises enqueue on the shared streams
  int64_t chunk = 16;  // fields per pipeline chunk
  const char* fail_what = "";
};

// Lookahead L (fields of column work ahead of row work) and ring slots S for
// a batch of nf fields; conc = resident CTAs.
inline void ring_geometry(int sms, int occ, int strips, int rtiles, int64_t nf, uint32_t* L, uint32_t* S,
                          uint32_t* conc, uint32_t la_def = 12, uint32_t sl_def = 8) {
  // lookahead = LA x (tiles all resident CTAs run at once) / (tiles per field);
  // slots = lookahead + SL x that + 2. GRFC_RING_LA / GRFC_RING_SL override (A/B).
  // Defaults: 12 / 8 for the 2D generator (its column tiles are ~2x its row tiles
  // and a deep ring absorbs the imbalance), 3 / 2 for the 3D pass B (balanced
  // plain-FFT tiles: an L2-sized plane ring wins, 0.429 -> 0.390 ms at 512^3).
  const char* ela = std::getenv("GRFC_RING_LA");
  const char* esl = std::getenv("GRFC_RING_SL");
  const int la_env = ela ? std::atoi(ela) : -1, sl_env = esl ? std::atoi(esl) : -1;
  const uint32_t la = la_env >= 0 ? (uint32_t)la_env : la_def;
  const uint32_t sl = sl_env >= 0 ? (uint32_t)sl_env : sl_def;
  const uint32_t c = (uint32_t)(sms * occ), G = (uint32_t)(strips + rtiles);
  uint32_t l = (la * c + G - 1) / G;
  l = l < 1 ? 1 : l;
  l = l < (uint32_t)nf ? l : (uint32_t)nf;
  uint32_t s = l + sl * ((c + G - 1) / G) + 2;
  s = s < (uint32_t)nf ? s : (uint32_t)nf;
  *L = l;
  *S = s;
  *conc = c;
}
// Workspace of the persistent kernel, with occupancy `occ` (may differ per instantiation).
inline void fused_geometry_occ(const Fast2D& f, int occ, int64_t nf, uint32_t* L, uint32_t* S, uint32_t* conc) {
  ring_geometry(f.sms, occ, f.strips, f.rtiles, nf, L, S, conc);
}
inline void fused_geometry(const Fast2D& f, int64_t nf, uint32_t* L, uint32_t* S, uint32_t* conc) {
  ring_geometry(f.sms, f.occ, f.strips, f.rtiles, nf, L, S, conc);
}
inline size_t fused_ctr_bytes(uint32_t S) { return ((1 + 2 * (size_t)S) * 4 + 255) / 256 * 256; }

// Scheduler groups of the persistent 2D kernel (GRFC_GROUP = CTAs per group,
// GRFC_GROUP_L / _S = lookahead and ring slots per group): each group is an
// independent queue over every groups-th field with its own W ring, so the
// rings' total (groups x S x P*s) can stay L2-resident while each queue keeps
// its tile-level load balance. groups = 1: the single whole-grid queue.
struct GroupGeom {
  uint32_t groups = 1, gsize = 0, L = 0, S = 0;
};
inline GroupGeom group_geometry(const Fast2D& f, int64_t nf) {
  GroupGeom g;
  const int gs = f.group;
  const int conc = f.sms * f.occ;
  if (gs <= 0 || gs >= conc) return g;
  const uint32_t groups = (uint32_t)(conc / gs);
  if (groups < 2 || (int64_t)groups > nf) return g;
  const uint32_t fmin = (uint32_t)(nf / groups);  // smallest group's field count
  uint32_t L = (uint32_t)f.group_L, S = (uint32_t)f.group_S;
  L = L < 1 ? 1 : L;
  S = S < L + 1 ? L + 1 : S;
  if (L > fmin) L = fmin;
  if (L < 1) return g;
  if (S > fmin) S = fmin;
  if (S < 1) S = 1;
  g.groups = groups;
  g.gsize = (uint32_t)gs;
  g.L = L;
  g.S = S;
  return g;
}
// Device workspace one persistent launch over nf fields needs.
size_t fast2d_workspace_bytes(const Fast2D& f, int64_t nf);

bool fast2d_supported(int d, const int64_t* n, int dtype, int alg, int family);
cudaError_t fast2d_init(Fast2D& f, const GridDesc& g, const DensityDesc& D, int dtype, int alg, double s_one,
                        double s_two);
void fast2d_free(Fast2D& f);
// (Re)builds the fp32 density table d_sg from the user's sqrt(g) table (GRFC_DENSITY_TABLE).
cudaError_t fast2d_set_table(Fast2D& f, const double* d_table);
const char* fast2d_name(const Fast2D& f);
// W: workspace of nf * |H| complex; out + i*stride (elements) = field i.
cudaError_t launch_fast2d(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                          int64_t stride, cudaStream_t s);
// Whole-batch generation on `s` (workspace, pipelining and ordering inside).
cudaError_t fast2d_generate(Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* out,
                            int64_t stride, cudaStream_t s);

}  // namespace grfc
