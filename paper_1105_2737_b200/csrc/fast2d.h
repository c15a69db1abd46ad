// Fused fast path for power-of-two 2D grids (the BASELINE configs c1, c2, c3,
// c5): generation fused into the column pass, Nyquist column packed into the
// imaginary part of column 0, and an L2-resident half-spectrum intermediate.
#pragma once

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
  int kind = 0;
};

bool fast2d_supported(int d, const int64_t* n, int dtype, int alg, int family);
cudaError_t fast2d_init(Fast2D& f, const GridDesc& g, const DensityDesc& D, int dtype, int alg, double s_one,
                        double s_two);
void fast2d_free(Fast2D& f);
const char* fast2d_name(const Fast2D& f);
// W: workspace of nf * |H| complex; out + i*stride (elements) = field i.
cudaError_t launch_fast2d(const Fast2D& f, int alg, uint64_t seed, uint64_t field0, int64_t nf, void* W, void* out,
                          int64_t stride, cudaStream_t s);

}  // namespace grfc
