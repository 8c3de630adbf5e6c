// Microbenchmark: the K3 row / K4 access pattern -- every lane streams one
// 1,248-byte block with 256-bit global loads (L2-resident data, L1 misses)
// and feeds NF = 3 node chains (6 DFMA per complex coefficient) -- with
// SHARE adjacent lanes reading the same block.  Prints DFMA/clk/SM: how much
// lanes that share a block save on the L1tex path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldg_share ldg_share.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double4 ldg256(const double2* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}

template <int SHARE>
__global__ void __launch_bounds__(384) k(const double2* blocks, unsigned nblocks, double* out,
                                         int iters) {
  constexpr int NF = 3;
  const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x);
  double acc[2 * NF];
#pragma unroll
  for (int f = 0; f < 2 * NF; ++f) acc[f] = 0.0;
  double c[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) c[f] = 1.0 + f * 1e-9 + threadIdx.x * 1e-12;
  unsigned h = (gw / SHARE) * 2654435761u + 12345u;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    const double2* b = blocks + (size_t)(h % nblocks) * 78;
#pragma unroll
    for (int kk = 0; kk < 39; ++kk) {
      const double4 v = ldg256(b + 2 * kk);
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        acc[2 * f] = fma(v.x, c[f], acc[2 * f]);
        acc[2 * f + 1] = fma(v.y, c[f], acc[2 * f + 1]);
        acc[2 * f] = fma(v.z, c[f], acc[2 * f]);
        acc[2 * f + 1] = fma(v.w, c[f], acc[2 * f + 1]);
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int f = 0; f < 2 * NF; ++f) t += acc[f];
  if (t == 12345.678) out[0] = t;
}

template <int SHARE>
void run(const double2* d, unsigned nb, double* o) {
  const int blocks = 148, iters = 400;
  k<SHARE><<<blocks, 384>>>(d, nb, o, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<SHARE><<<blocks, 384>>>(d, nb, o, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double clk = 1.965e9 * ms * 1e-3;
  const double dfma = 12.0 * iters * 39 * 2 * 2 * 3 * 32;  // per SM: warps * iters * loads * ...
  printf("share %2d: %.3f ms  DFMA/clk/SM %.1f (peak 64)\n", SHARE, ms, dfma / clk);
}

int main() {
  const unsigned nb = 60000;  // 75 MB: L2-resident
  double2* d;
  double* o;
  cudaMalloc(&d, (size_t)nb * 78 * sizeof(double2));
  cudaMemset(d, 0, (size_t)nb * 78 * sizeof(double2));
  cudaMalloc(&o, 64);
  run<1>(d, nb, o);
  run<2>(d, nb, o);
  run<4>(d, nb, o);
  run<8>(d, nb, o);
  run<32>(d, nb, o);
  return 0;
}
