// direct.cu -- K7: exact O(N M) kernel sums at M targets on the device, the
// GPU form of direct_eval / error_at_indices (engine.cpp:327-376).  Sources
// are split into chunks across CTAs (so 1,000 targets still fill 148 SMs);
// per-chunk partials are reduced in a fixed order afterwards, keeping the
// result deterministic without atomics.
#include "plan.hpp"

namespace ifgf_b200 {
namespace {

constexpr int kDT = 128;  // targets per CTA (one per thread)
constexpr int kTile = 256;

template <bool LAP>
__global__ void __launch_bounds__(kDT)
    k_direct(const double* __restrict__ x, const double* __restrict__ y,
             const double* __restrict__ z, const double* __restrict__ ar,
             const double* __restrict__ ai, size_t n, double kappa,
             const uint32_t* __restrict__ targets, size_t m, size_t chunk, double* part_re,
             double* part_im) {
  __shared__ double sx[kTile], sy[kTile], sz[kTile], sr_[kTile], si_[kTile];
  const size_t t = blockIdx.x * (size_t)kDT + threadIdx.x;
  const bool active = t < m;
  const size_t ti = active ? (targets ? targets[t] : t) : 0;
  const double tx = active ? x[ti] : 0.0, ty = active ? y[ti] : 0.0, tz = active ? z[ti] : 0.0;
  const size_t s0 = blockIdx.y * chunk;
  const size_t s1 = min(n, s0 + chunk);
  double accr = 0.0, acci = 0.0;
  for (size_t base = s0; base < s1; base += kTile) {
    const int cnt = (int)min((size_t)kTile, s1 - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += kDT) {
      sx[k] = x[base + k];
      sy[k] = y[base + k];
      sz[k] = z[base + k];
      sr_[k] = ar[base + k];
      si_[k] = ai ? ai[base + k] : 0.0;
    }
    __syncthreads();
    if (!active) continue;
    for (int k = 0; k < cnt; ++k) {
      if (base + k == ti) continue;
      const double dx = tx - sx[k], dy = ty - sy[k], dz = tz - sz[k];
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double rinv = rsqrt(r2);
      const double inv = kQuarterInvPi * rinv;
      if (LAP) {
        accr = fma(sr_[k], inv, accr);
        acci = fma(si_[k], inv, acci);
      } else {
        double sn, cs;
        sincos_fast(kappa * (r2 * rinv), sn, cs);
        const double gr = cs * inv, gi = sn * inv;
        accr = fma(sr_[k], gr, fma(-si_[k], gi, accr));
        acci = fma(sr_[k], gi, fma(si_[k], gr, acci));
      }
    }
  }
  if (active) {
    part_re[blockIdx.y * m + t] = accr;
    part_im[blockIdx.y * m + t] = acci;
  }
}

__global__ void k_direct_reduce(const double* __restrict__ part_re,
                                const double* __restrict__ part_im, size_t m, int nch,
                                double* o_re, double* o_im) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= m) return;
  double r = 0.0, i = 0.0;
  for (int c = 0; c < nch; ++c) {
    r += part_re[c * m + t];
    i += part_im[c * m + t];
  }
  o_re[t] = r;
  o_im[t] = i;
}

}  // namespace

void direct_sums(const double* x, const double* y, const double* z, const double* ar,
                 const double* ai, size_t n, double kappa, const uint32_t* targets, size_t m,
                 double* o_re, double* o_im, cudaStream_t s) {
  if (!m) return;
  const size_t tblocks = (m + kDT - 1) / kDT;
  // ~8 CTAs per SM in total, each chunk at least one tile
  size_t nch = (148 * 8 + tblocks - 1) / tblocks;
  const size_t max_ch = (n + kTile - 1) / kTile;
  if (nch > max_ch) nch = max_ch;
  if (nch < 1) nch = 1;
  if (nch > 65535) nch = 65535;
  const size_t chunk = ((n + nch - 1) / nch + kTile - 1) / kTile * kTile;
  nch = (n + chunk - 1) / chunk;
  double* part = nullptr;
  IFGF_CUDA(cudaMallocAsync(&part, 2 * nch * m * sizeof(double), s));
  dim3 grid((unsigned)tblocks, (unsigned)nch);
  if (kappa == 0.0)
    k_direct<true><<<grid, kDT, 0, s>>>(x, y, z, ar, ai, n, kappa, targets, m, chunk, part,
                                        part + nch * m);
  else
    k_direct<false><<<grid, kDT, 0, s>>>(x, y, z, ar, ai, n, kappa, targets, m, chunk, part,
                                         part + nch * m);
  k_direct_reduce<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(part, part + nch * m, m, (int)nch,
                                                              o_re, o_im);
  IFGF_CUDA(cudaGetLastError());
  IFGF_CUDA(cudaFreeAsync(part, s));
}

}  // namespace ifgf_b200
