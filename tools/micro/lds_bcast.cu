// Microbenchmark: shared-memory 128-bit loads with few distinct addresses per
// warp (the K3 "rows of one child cone on neighbouring lanes" pattern) vs
// distinct addresses, and the DFMA rate they sustain.  Prints loads/clk/SM and
// DFMA/clk/SM per mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bcast lds_bcast.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int NF>
__global__ void __launch_bounds__(256) k(double* out, int iters) {
  __shared__ __align__(16) double2 s[2560];  // 40 KB
  for (int i = threadIdx.x; i < 2560; i += blockDim.x) s[i] = make_double2(i * 1e-3, i * 2e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int base;  // in double2 units
  if (MODE == 0) base = 0;                    // uniform
  else if (MODE == 1) base = (lane >> 3) * 81;  // 4 distinct, stride 1296 B
  else if (MODE == 2) base = (lane >> 2) * 81;  // 8 distinct, stride 1296 B
  else base = lane;                           // 32 distinct (stride 16 B -> 4 wavefronts)
  double acc[2 * NF];
#pragma unroll
  for (int f = 0; f < 2 * NF; ++f) acc[f] = 0.0;
  double c[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) c[f] = 1.0 + f * 1e-9 + threadIdx.x * 1e-12;
  unsigned sbase = (unsigned)__cvta_generic_to_shared(s + base);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 75; ++kk) {
      double x, y;
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(x), "=d"(y) : "r"(sbase + (unsigned)(MODE == 3 ? kk * 32 : kk * 16)));
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        acc[2 * f] = fma(x, c[f], acc[2 * f]);
        acc[2 * f + 1] = fma(y, c[f], acc[2 * f + 1]);
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int f = 0; f < 2 * NF; ++f) t += acc[f];
  if (t == 12345.678) out[0] = t;
}

template <int MODE, int NF>
void run(double* d, const char* name) {
  const int blocks = 148 * 4, iters = 200;
  k<MODE, NF><<<blocks, 256>>>(d, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, NF><<<blocks, 256>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double clk = 1.965e9 * ms * 1e-3;
  const double warps_per_sm = blocks * 8.0 / 148;
  const double loads = warps_per_sm * iters * 75.0;
  const double dfma = loads * 32 * 2 * NF;
  printf("%-28s NF=%d  %.3f ms  warp-LDS/clk/SM %.3f  DFMA/clk/SM %.1f (peak 64)\n", name, NF, ms,
         loads / clk, dfma / clk);
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  run<0, 1>(d, "uniform");
  run<1, 1>(d, "4 distinct (1296 B)");
  run<2, 1>(d, "8 distinct (1296 B)");
  run<3, 1>(d, "32 distinct (512 B)");
  run<0, 3>(d, "uniform");
  run<1, 3>(d, "4 distinct (1296 B)");
  run<2, 3>(d, "8 distinct (1296 B)");
  run<3, 3>(d, "32 distinct (512 B)");
  run<0, 6>(d, "uniform");
  run<1, 6>(d, "4 distinct (1296 B)");
  run<3, 6>(d, "32 distinct (512 B)");
  return 0;
}
