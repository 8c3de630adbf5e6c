// peak.cu -- FP64 FMA-pipe peak of this device, measured (MEASURED_PEAKS.json
// records HBM and bf16 only; SURVEY.md §8(d) asks for a DFMA measurement).
// Every thread runs 8 independent DFMA chains; grid = 8 CTAs of 512 per SM.
#include "plan.hpp"

namespace ifgf_b200 {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(512) k_dfma(double* out, int iters, double a, double b) {
  double v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fma(v[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 123.456) out[0] = s;  // keep the chains alive
}

}  // namespace
}  // namespace ifgf_b200

extern "C" int ifgf_measure_fp64_peak(int device, double* tflops, double* ms) {
  using namespace ifgf_b200;
  if (cudaSetDevice(device) != cudaSuccess) return IFGF_ERUNTIME;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return IFGF_ERUNTIME;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return IFGF_ERUNTIME;
  const int blocks = prop.multiProcessorCount * 8, threads = 512, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    best = t < best ? t : best;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return IFGF_ERUNTIME;
  const double flops = 2.0 * kChains * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms) *ms = best;
  return IFGF_OK;
}
