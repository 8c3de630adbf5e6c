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

// FP64 tensor-core path: mma.sync m8n8k4 f64 (256 MACs per warp instruction).
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

}  // namespace
}  // namespace ifgf_b200

// Best of the DFMA pipe and the FP64 tensor path (B200 measures ~34 and ~37
// TFLOP/s); the larger one is the FP64 roofline denominator.
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
  double fma_tf = 2.0 * kChains * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  const int mblocks = prop.multiProcessorCount * 4, miters = 4096;
  for (int w = 0; w < 3; ++w) k_dmma<<<mblocks, 256>>>(out, miters);
  float bestm = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dmma<<<mblocks, 256>>>(out, miters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    bestm = t < bestm ? t : bestm;
  }
  const double mma_tf = (mblocks * 256 / 32.0) * miters * 8 * 256 * 2.0 / (bestm * 1e-3) / 1e12;
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return IFGF_ERUNTIME;
  *tflops = fma_tf > mma_tf ? fma_tf : mma_tf;
  if (ms) *ms = fma_tf > mma_tf ? best : bestm;
  return IFGF_OK;
}
