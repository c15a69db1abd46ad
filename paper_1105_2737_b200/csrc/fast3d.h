// Fused power-of-two 3D path (pow2_3d.cu, fast3d_kernels.cuh): single GPU and
// slab decomposition along axis 0 of the field (axis 1 of the spectrum).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "grfc_internal.cuh"

namespace grfc {

struct Fast3D {
  int n0 = 0, n1 = 0, n2 = 0, dtype = 0, alg = 1;
  GridDesc g{};
  DensityDesc D{};
  double s_one = 1.0;
  void* d_tw = nullptr;  // tables of N0, N1, N2 (exp(+2 pi i t / N))
  int occ = 1, sms = 148, strips = 0, rtiles = 0;  // planes kernel geometry
};

bool fast3d_supported(int d, const int64_t* n, int alg);
cudaError_t fast3d_init(Fast3D& f, const GridDesc& g, const DensityDesc& D, int dtype, int alg, double s_one);
void fast3d_free(Fast3D& f);

// Slab geometry for `world` ranks: rank r owns spectrum k1 in [r n1p, (r+1) n1p)
// in pass A and field planes j0 in [r n0p, (r+1) n0p) in pass B. The
// all-to-all moves block q of rank r's send buffer (elements
// [q*block, (q+1)*block)) to block r of rank q's receive buffer.
struct SlabGeom {
  int world, n0p, n1p;
  uint64_t block_elems;  // complex elements per (r, q) block
  uint64_t buf_elems;    // world * block_elems (send = receive size)
};
bool slab_geometry(const Fast3D& f, int world, SlabGeom& s);

// One field: pass A (rank's k1 slab) -> send buffer (complex, buf_elems).
cudaError_t fast3d_pass_a(const Fast3D& f, int world, int rank, uint64_t seed, uint64_t field, void* d_send,
                          cudaStream_t s);
// One field: pass B from the receive buffer -> the rank's field slab
// (n0p planes of N1 x N2 reals, contiguous).
cudaError_t fast3d_pass_b(const Fast3D& f, int world, const void* d_recv, void* d_out, cudaStream_t s);
// Single-GPU batch (world 1): out + i*stride = field i.
cudaError_t fast3d_generate(const Fast3D& f, uint64_t seed, uint64_t field0, int64_t nf, void* out, int64_t stride,
                            cudaStream_t s);

}  // namespace grfc
