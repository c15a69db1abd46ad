// FP32 issue-rate probe for the compute roofline diagnostic (SURVEY.md §8d asks
// for a measured FFMA peak beside the HBM one; MEASURED_PEAKS.json has none).
// Every thread runs 8 independent chains of packed fma.rn.f32x2 (FFMA2: 4 flops
// per lane per instruction), 8 warps x all SMs x 4 resident blocks; the result
// is stored so nothing is dead code. Returns dense FP32 TFLOP/s (FMA = 2 flops).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/grfc.h"

namespace {

__global__ void __launch_bounds__(256) k_ffma2_peak(float2* out, int iters, float2 a, float2 b) {
  uint64_t acc[8], m, c;
  asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(b.x), "f"(b.y));
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float v = (float)(threadIdx.x + k);
    asm("mov.b64 %0, {%1, %1};" : "=l"(acc[k]) : "f"(v));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[k]) : "l"(m), "l"(c));
  }
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[k]));
    s.x += x;
    s.y += y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

extern "C" grfc_status grfc_measure_fp32_peak(int device, double* tflops) {
  if (!tflops) return GRFC_EINVAL;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 4, threads = 256, iters = 1 << 14;
  float2* out = nullptr;
  cudaEvent_t e0, e1;
  cudaError_t e = cudaMalloc(&out, sizeof(float2) * blocks * threads);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_ms = 1e30f;
  for (int rep = 0; rep < 5 && e == cudaSuccess; ++rep) {
    cudaEventRecord(e0);
    k_ffma2_peak<<<blocks, threads>>>(out, iters, make_float2(0.999f, 1.001f), make_float2(1e-3f, -1e-3f));
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best_ms) best_ms = ms;  // rep 0 warms up
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return GRFC_ECUDA;
  const double flops = (double)blocks * threads * iters * 8 /*chains*/ * 4 /*f32x2 fma*/;
  *tflops = flops / (best_ms * 1e-3) / 1e12;
  return GRFC_OK;
}
