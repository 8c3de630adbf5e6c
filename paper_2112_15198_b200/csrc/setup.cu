// setup.cu -- Problem::build on the device (engine.cpp:74-94).
//
//   bounding cube      geometry.cpp:95-114   two-stage min/max reduction
//   choose_depth       engine.cpp:55-72      host (scalar)
//   Morton sort        morton.cpp:53-95      grid index + code kernel, CUB stable radix sort
//   linear octree      octree.cpp:18-150     one "first level where point i starts a box"
//                                            pass, then per level an inclusive scan gives
//                                            every point's box ordinal; boxes, parents and
//                                            child ranges follow from those ordinals;
//                                            27-stencil neighbours by binary search;
//                                            cousin CSR by count / scan / fill
//   relevant cones     cones.cpp:90-150      per level d = 3..D: mark (box, gamma) bits from
//                                            clause 1 (cousin points) and clause 2 (parent
//                                            cone nodes), popcount prefix = cone ordinals in
//                                            (box, gamma) order, compaction to the flat lists
//
// All structural arithmetic follows the reference operation order with
// explicit _rn intrinsics (ifgf_common.cuh), so the result is identical to
// the reference's Problem, which the parity tests check list by list.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "plan.hpp"

namespace ifgf_b200 {
namespace {

constexpr int kT = 256;

inline unsigned grid_for(size_t n, int t = kT) {
  size_t g = (n + t - 1) / t;
  return (unsigned)(g ? g : 1);
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
  x = (x ^ (x >> 32)) & 0x1fffffull;
  return (uint32_t)x;
}

// ---- bounding cube ---------------------------------------------------------
__global__ void k_bbox_partial(const double* __restrict__ x, const double* __restrict__ y,
                               const double* __restrict__ z, size_t n, double* part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double v[3] = {x[i], y[i], z[i]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], v[c]);
      hi[c] = fmax(hi[c], v[c]);
    }
  }
  __shared__ double s[6][kT];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    s[c][threadIdx.x] = lo[c];
    s[3 + c][threadIdx.x] = hi[c];
  }
  __syncthreads();
  for (int w = kT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s[c][threadIdx.x] = fmin(s[c][threadIdx.x], s[c][threadIdx.x + w]);
        s[3 + c][threadIdx.x] = fmax(s[3 + c][threadIdx.x], s[3 + c][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void k_bbox_final(const double* part, int nparts, double* out) {
  if (threadIdx.x >= 6) return;
  const int c = threadIdx.x;
  double v = part[c];
  for (int b = 1; b < nparts; ++b) v = c < 3 ? fmin(v, part[b * 6 + c]) : fmax(v, part[b * 6 + c]);
  out[c] = v;
}

// ---- Morton codes (morton.cpp:53-68 grid_index, :40-45 encode) --------------
__global__ void k_morton(const double* __restrict__ x, const double* __restrict__ y,
                         const double* __restrict__ z, size_t n, double ox, double oy, double oz,
                         double side, double h, uint32_t ngrid, uint64_t* codes, uint32_t* idx,
                         int* err) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double rel[3] = {__dsub_rn(x[i], ox), __dsub_rn(y[i], oy), __dsub_rn(z[i], oz)};
  uint64_t k[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (!(rel[c] >= 0.0) || rel[c] >= side) {
      raise_err(err, kErrOutside);
      k[c] = 0;
      continue;
    }
    int64_t v = (int64_t)floor(__ddiv_rn(rel[c], h));
    if (v >= (int64_t)ngrid) v = ngrid - 1;
    k[c] = (uint64_t)v;
  }
  codes[i] = spread3(k[0]) | spread3(k[1]) << 1 | spread3(k[2]) << 2;
  idx[i] = (uint32_t)i;
}

__global__ void k_gather3(const uint32_t* __restrict__ perm, const double* __restrict__ x,
                          const double* __restrict__ y, const double* __restrict__ z, size_t n,
                          double* xs, double* ys, double* zs) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  xs[i] = x[j];
  ys[i] = y[j];
  zs[i] = z[j];
}

// First (coarsest) level at which sorted point i opens a new box; level-d
// codes are code >> 3(D-d) (octree.cpp:57-76).  Also histograms it.
__global__ void k_start_level(const uint64_t* __restrict__ codes, size_t n, int D,
                              uint8_t* start, uint32_t* hist) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  __shared__ uint32_t sh[32];
  if (threadIdx.x < 32) sh[threadIdx.x] = 0;
  __syncthreads();
  if (i < n) {
    int lvl = 1;
    if (i > 0) {
      const uint64_t diff = codes[i] ^ codes[i - 1];
      if (diff == 0) {
        lvl = 31;  // never starts a box
      } else {
        const int hb = 63 - __clzll(diff);
        lvl = D - hb / 3;
      }
    }
    start[i] = (uint8_t)lvl;
    atomicAdd(&sh[lvl], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32 && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

struct StartsAt {
  const uint8_t* start;
  int d;
  __host__ __device__ uint32_t operator()(const size_t& i) const { return start[i] <= d ? 1u : 0u; }
};

// ptbox (inclusive count) -> ordinal; box heads record first point, code, centre.
__global__ void k_boxes(uint32_t* ptbox, const uint8_t* __restrict__ start,
                        const uint64_t* __restrict__ codes, size_t n, int d, int D, double ox,
                        double oy, double oz, double h, uint32_t* first, uint64_t* bcode,
                        double* cx, double* cy, double* cz) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = ptbox[i] - 1;
  ptbox[i] = b;
  if (start[i] <= d) {
    const uint64_t c = codes[i] >> (3 * (D - d));
    first[b] = (uint32_t)i;
    bcode[b] = c;
    // octree.cpp:10-14: origin + (k + 0.5) * h
    cx[b] = __dadd_rn(ox, __dmul_rn((double)compact3(c) + 0.5, h));
    cy[b] = __dadd_rn(oy, __dmul_rn((double)compact3(c >> 1) + 0.5, h));
    cz[b] = __dadd_rn(oz, __dmul_rn((double)compact3(c >> 2) + 0.5, h));
  }
}

__global__ void k_box_links(uint32_t nb, size_t n, const uint32_t* __restrict__ first,
                            uint32_t* count, const uint32_t* __restrict__ ptbox_up,
                            uint32_t* parent, const uint32_t* __restrict__ ptbox_down,
                            uint32_t* child_begin, uint32_t nb_down) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) {
    if (child_begin) child_begin[nb] = nb_down;
    return;
  }
  const uint32_t f = first[b];
  count[b] = (b + 1 < nb ? first[b + 1] : (uint32_t)n) - f;
  if (parent) parent[b] = ptbox_up ? ptbox_up[f] : 0u;
  if (child_begin) child_begin[b] = ptbox_down[f];
}

// 27-stencil neighbours incl. self, ascending ordinals (octree.cpp:97-122).
__global__ void k_neighbors(uint32_t nb, int d, const uint64_t* __restrict__ code,
                            uint32_t* nbr, uint32_t* nbr_cnt) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint64_t c = code[b];
  const int64_t k[3] = {compact3(c), compact3(c >> 1), compact3(c >> 2)};
  const int64_t side = (int64_t)1 << (d - 1);
  uint32_t found[27];
  int cnt = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t j[3] = {k[0] + dx, k[1] + dy, k[2] + dz};
        if (j[0] < 0 || j[1] < 0 || j[2] < 0 || j[0] >= side || j[1] >= side || j[2] >= side)
          continue;
        const uint64_t t = spread3(j[0]) | spread3(j[1]) << 1 | spread3(j[2]) << 2;
        uint32_t lo = 0, hi = nb;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (code[mid] < t) lo = mid + 1;
          else hi = mid;
        }
        if (lo < nb && code[lo] == t) found[cnt++] = lo;
      }
  for (int a = 1; a < cnt; ++a)
    for (int q = a; q > 0 && found[q - 1] > found[q]; --q) {
      const uint32_t tmp = found[q];
      found[q] = found[q - 1];
      found[q - 1] = tmp;
    }
  for (int a = 0; a < cnt; ++a) nbr[(size_t)b * 27 + a] = found[a];
  nbr_cnt[b] = cnt;
}

// Cousins: children of parent-neighbours at Chebyshev distance > 1, visited in
// Morton order (octree.cpp:127-147).  fill == nullptr: count only.
// K4 work items: box b -> ceil(count / R) runs of <= R points.
__global__ void k_chunk_count(const uint32_t* __restrict__ count, uint32_t nb, int R,
                              uint32_t* c) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) c[b] = (count[b] + R - 1) / R;
}

// One thread per work item: its box is the last b with off[b] <= t.
__global__ void k_chunk_fill(const uint32_t* __restrict__ first, uint32_t nb, int R,
                             const uint32_t* __restrict__ off, size_t cap, uint2* chunk) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= cap || t >= off[nb]) return;
  uint32_t lo = 0, hi = nb;  // off[lo] <= t < off[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= t) lo = mid;
    else hi = mid;
  }
  chunk[t] = make_uint2(first[lo] + (uint32_t)(t - off[lo]) * R, lo);
}

__global__ void k_cousins(const __grid_constant__ LevelDev L, const __grid_constant__ LevelDev U, uint32_t* cnt_or_off, uint32_t* fill) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= L.nb) return;
  const uint64_t c = L.code[b];
  const uint32_t k[3] = {compact3(c), compact3(c >> 1), compact3(c >> 2)};
  const uint32_t pb = L.parent[b];
  uint32_t w = fill ? cnt_or_off[b] : 0u;
  const uint32_t np = U.nbr_cnt[pb];
  for (uint32_t a = 0; a < np; ++a) {
    const uint32_t pn = U.nbr[(size_t)pb * 27 + a];
    for (uint32_t ch = U.child_begin[pn]; ch < U.child_begin[pn + 1]; ++ch) {
      const uint64_t cc = L.code[ch];
      const uint32_t j[3] = {compact3(cc), compact3(cc >> 1), compact3(cc >> 2)};
      uint32_t dist = 0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const uint32_t dd = j[q] > k[q] ? j[q] - k[q] : k[q] - j[q];
        dist = dd > dist ? dd : dist;
      }
      if (dist > 1) {
        if (fill) fill[w] = ch;
        ++w;
      }
    }
  }
  if (!fill) cnt_or_off[b] = w;
}

__device__ __forceinline__ void set_bit(uint64_t* bits, uint64_t idx) {
  const uint64_t m = 1ull << (idx & 63);
  uint64_t* w = bits + (idx >> 6);
  if (!(*w & m)) atomicOr((unsigned long long*)w, (unsigned long long)m);
}

// set_bit with the lanes of a warp that mark the same segment merged (nodes
// of one cone, and neighbouring points, mostly fall into the same segment).
__device__ __forceinline__ void set_bit_warp(uint64_t* bits, uint64_t idx) {
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, idx);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) set_bit(bits, idx);
}

// Clause 1 (cones.cpp:100-106), transposed: every sorted point marks, in each
// cousin box of its own box (the cousin relation is symmetric), the segment
// containing it.
__global__ void k_mark_points(const __grid_constant__ LevelDev L, const uint32_t* __restrict__ ptbox,
                              const double* __restrict__ xs, const double* __restrict__ ys,
                              const double* __restrict__ zs, size_t n, uint64_t* bits, int* err) {
  __shared__ double2 trig[kTrigEntries];
  stage_trig(trig, L.trig);
  __syncthreads();
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = ptbox[i];
  const double x = xs[i], y = ys[i], z = zs[i];
  for (uint32_t ci = L.cous_off[b]; ci < L.cous_off[b + 1]; ++ci) {
    const uint32_t cb = L.cous[ci];
    const double cx = L.cx[cb], cy = L.cy[cb], cz = L.cz[cb];
    uint32_t g;
    if (!cone_index_f32(L, cx, cy, cz, x, y, z, g)) {
      const int e = cone_of_point_fast(L, trig, cx, cy, cz, x, y, z, g);
      if (e) {
        raise_err(err, e);
        return;
      }
    }
    set_bit_warp(bits, (uint64_t)cb * L.G + g);
  }
}

// Clause 1 for plans that keep K4 records: the apply-side locate
// (engine.cpp:29-51) of every (point, cousin) pair in full precision, once.
// Thread = one K4 work item (<= R consecutive points of a box, Level::chunk).
// Per pair it marks the segment (clause 1) and stores what K4 needs from the
// locate: the segment, the local Chebyshev coordinates and the kernel factor
// e^{i kappa r} / (4 pi r) (LevelDev::rec).  K4 then only looks up the cone
// and evaluates; the interpolation pass of every later apply skips the locate
// (more than half of its time), and this kernel, free of the evaluation's
// registers, runs it at four times K4's occupancy.
__global__ void k_pair_count(const uint32_t* __restrict__ count,
                             const uint32_t* __restrict__ ncous, uint32_t nb, uint32_t R,
                             uint64_t* out) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) out[b] = (uint64_t)((count[b] + R - 1) / R * R) * ncous[b];
  else if (b == nb) out[b] = 0;
}

// R values of one record plane of a work item (the item's pair index is a
// multiple of R: one aligned vector store for R = 2)
template <int R, class T>
__device__ __forceinline__ void rec_store(T* __restrict__ p, uint64_t idx, const T* v) {
  if constexpr (R == 2 && sizeof(T) == 8) {
    *reinterpret_cast<double2*>(p + idx) = make_double2(v[0], v[1]);
  } else if constexpr (R == 2 && sizeof(T) == 4) {
    *reinterpret_cast<uint2*>(p + idx) = make_uint2(v[0], v[1]);
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) p[idx + j] = v[j];
  }
}

#ifndef IFGF_LOCATE_MINB
#define IFGF_LOCATE_MINB 3
#endif
// Rank plans (MARK = false: their cone set is final) keep the records of the
// boxes [b_lo, b_hi] that hold their points; rec / rec_g then point b_lo's
// pair offset before the window and L.npairs is the window's pair count.
template <bool LAP, int R, bool MARK>
__global__ void __launch_bounds__(256, IFGF_LOCATE_MINB)
    k_locate_points(const __grid_constant__ LevelDev L, const uint2* __restrict__ chunk,
                    const uint32_t* __restrict__ nchunk, const double* __restrict__ xs,
                    const double* __restrict__ ys, const double* __restrict__ zs, double kappa,
                    uint64_t* bits, uint32_t* __restrict__ rec_g, double* __restrict__ rec,
                    uint32_t b_lo, uint32_t b_hi, int* err) {
  __shared__ double2 trig[kTrigEntries];
  __shared__ double2 ptab[LAP ? 1 : kPhaseEntries];
  stage_trig(trig, L.trig);
  if (!LAP)
    for (int k = threadIdx.x; k < kPhaseEntries; k += blockDim.x) ptab[k] = L.trig[kTrigEntries + k];
  __syncthreads();
  const double ks = kappa * kPhaseScale;
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= *nchunk) return;
  const uint2 ch = chunk[t];
  const uint32_t b = ch.y;
  if (b < b_lo || b > b_hi) return;
  const uint32_t fb = L.first[b], cnt = L.count[b];
  const uint32_t cntp = (cnt + R - 1) / R * R;
  const int n = (int)min((uint32_t)R, fb + cnt - ch.x);
  double px[R], py[R], pz[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {  // slots past the box's last point repeat the item's first point
    const size_t i = (size_t)ch.x + (j < n ? j : 0);
    px[j] = xs[i];
    py[j] = ys[i];
    pz[j] = zs[i];
  }
  const uint32_t k0 = L.cous_off[b], k1 = L.cous_off[b + 1];
  uint64_t idx = L.pair_off[b] + (ch.x - fb);
  const uint64_t np = L.npairs;
  // cousin index two steps ahead, centre one step ahead
  uint32_t cb1 = k0 < k1 ? L.cous[k0] : 0;
  uint32_t cb2 = k0 + 1 < k1 ? L.cous[k0 + 1] : 0;
  double cxn = L.cx[cb1], cyn = L.cy[cb1], czn = L.cz[cb1];
  for (uint32_t k = k0; k < k1; ++k, idx += cntp) {
    const uint32_t cb = cb1;
    const double cx = cxn, cy = cyn, cz = czn;
    cb1 = cb2;
    if (k + 2 < k1) cb2 = L.cous[k + 2];
    if (k + 1 < k1) {
      cxn = L.cx[cb1];
      cyn = L.cy[cb1];
      czn = L.cz[cb1];
    }
    Loc o[R];
    int e = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int ej = locate_fast(L, trig, cx, cy, cz, px[j], py[j], pz[j], o[j]);
      e = e ? e : ej;
    }
    if (e) {
      raise_err(err, e);
      return;
    }
    // clause 1: the bitmap words are requested here and tested after the
    // factor and the stores (a set bit -- the common case -- needs no atomic)
    uint64_t bi[R], bw[R];
    uint32_t g[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      g[j] = o[j].gamma;
      bi[j] = (uint64_t)cb * L.G + g[j];
      bw[j] = MARK ? bits[bi[j] >> 6] : ~0ull;
    }
    double v[R];
    rec_store<R>(rec_g, idx, g);
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = o[j].ts;
    rec_store<R>(rec, idx, v);
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = o[j].tt;
    rec_store<R>(rec + np, idx, v);
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = o[j].tp;
    rec_store<R>(rec + 2 * np, idx, v);
    double gi[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const double inv = kQuarterInvPi * o[j].rinv;
      v[j] = inv;
      gi[j] = 0.0;
      if (!LAP) {
        double sn, cn;
        sincos_tab<true>(ptab, ks * o[j].r, sn, cn);
        v[j] = cn * inv;
        gi[j] = sn * inv;
      }
    }
    rec_store<R>(rec + 3 * np, idx, v);
    if (!LAP) rec_store<R>(rec + 4 * np, idx, gi);
    if (MARK) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const uint64_t m = 1ull << (bi[j] & 63);
        if (!(bw[j] & m) && (j == 0 || bi[j] != bi[0]))
          atomicOr((unsigned long long*)(bits + (bi[j] >> 6)), (unsigned long long)m);
      }
    }
  }
}

// K4 records, second step (after the level's cones are numbered): the stored
// segment of every pair becomes the ordinal of its cone (find_cone), so the
// apply reads the block address without touching the bitmap.
template <int R>
__global__ void __launch_bounds__(256)
    k_rec_cones(const __grid_constant__ LevelDev L, const uint2* __restrict__ chunk,
                const uint32_t* __restrict__ nchunk, uint32_t* __restrict__ rec_g, uint32_t b_lo,
                uint32_t b_hi, uint32_t p_lo, uint32_t p_hi, int* err) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= *nchunk) return;
  const uint2 ch = chunk[t];
  const uint32_t b = ch.y;
  if (b < b_lo || b > b_hi) return;
  const uint32_t fb = L.first[b], cnt = L.count[b];
  // a rank plan's window holds whole boxes: points of [b_lo, b_hi] outside the
  // rank's [p_lo, p_hi) may see cones the rank does not store (never read)
  bool mine[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t i = ch.x + ((uint32_t)j < fb + cnt - ch.x ? j : 0);
    mine[j] = i >= p_lo && i < p_hi;
  }
  const uint32_t cntp = (cnt + R - 1) / R * R;
  uint64_t idx = L.pair_off[b] + (ch.x - fb);
  for (uint32_t k = L.cous_off[b]; k < L.cous_off[b + 1]; ++k, idx += cntp) {
    const uint32_t cb = L.cous[k];
    uint32_t g[R];
    if constexpr (R == 2) {
      const uint2 v = *reinterpret_cast<const uint2*>(rec_g + idx);
      g[0] = v.x;
      g[1] = v.y;
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) g[j] = rec_g[idx + j];
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      g[j] = find_cone(L, cb, g[j]);
      if (g[j] == 0xffffffffu && mine[j]) {
        raise_err(err, kErrInterpCover);
        return;
      }
    }
    rec_store<R>(rec_g, idx, g);
  }
}

// Clause 2 (cones.cpp:108-119): nodes of every relevant cone of the parent box
// mark the containing segment of each child box.
__global__ void k_mark_nodes(const __grid_constant__ LevelDev L, const __grid_constant__ LevelDev U,
                             const __grid_constant__ InterpConsts K, uint64_t* bits, int* err) {
  __shared__ double2 trig[kTrigEntries];
  stage_trig(trig, L.trig);
  __syncthreads();
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)U.nc * K.P) return;
  const uint32_t q = (uint32_t)(t / K.P);
  const int m = (int)(t % K.P);
  const int jp = m % K.pp, jt = (m / K.pp) % K.pt, js = m / (K.pp * K.pt);
  const uint32_t pb = U.cone_box[q];
  const SegMid sm = segment_mid(U, U.cone_gamma[q]);
  double x, y, z;
  node_position(sm, U.rad, U.cx[pb], U.cy[pb], U.cz[pb], K.ns[js], K.nt[jt], K.np[jp], x, y, z);
  for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb) {
    const double cx = L.cx[cb], cy = L.cy[cb], cz = L.cz[cb];
    uint32_t g;
    if (!cone_index_f32(L, cx, cy, cz, x, y, z, g)) {
      const int e = cone_of_point_fast(L, trig, cx, cy, cz, x, y, z, g);
      if (e) {
        raise_err(err, e);
        return;
      }
    }
    set_bit_warp(bits, (uint64_t)cb * L.G + g);
  }
}

__global__ void k_popc(const uint64_t* __restrict__ bits, size_t nw, uint32_t* cnt) {
  const size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (w < nw) cnt[w] = __popcll(bits[w]);
  else if (w == nw) cnt[w] = 0;
}

__global__ void k_compact(const __grid_constant__ LevelDev L, size_t nw, uint32_t* cone_box, uint32_t* cone_gamma) {
  const size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint64_t v = L.bits[w];
  uint32_t o = L.rank[w];
  while (v) {
    const int bit = __ffsll((long long)v) - 1;
    v &= v - 1;
    const uint64_t idx = (uint64_t)w * 64 + bit;
    cone_box[o] = (uint32_t)(idx / L.G);
    cone_gamma[o] = (uint32_t)(idx % L.G);
    ++o;
  }
}

__global__ void k_box_cone(const __grid_constant__ LevelDev L, uint32_t* box_cone) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > L.nb) return;
  const uint64_t idx = (uint64_t)b * L.G;
  const uint64_t w = idx >> 6;
  const uint64_t m = (1ull << (idx & 63)) - 1;
  box_cone[b] = L.rank[w] + (uint32_t)__popcll(L.bits[w] & m);
}

// grows the plan's CUB scratch buffer
struct Scratch {
  ifgf_plan* P;
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t b) {
    if (b > bytes) {
      if (p) IFGF_CUDA(cudaFreeAsync(p, P->s_main));
      bytes = b + (b >> 2) + 256;
      IFGF_CUDA(cudaMallocAsync(&p, bytes, P->s_main));
    }
    return p;
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, P->s_main);
  }
};

}  // namespace

void check_device_error(ifgf_plan* P) {
  int e = 0;
  IFGF_CUDA(cudaMemcpyAsync(&e, P->err, sizeof(int), cudaMemcpyDeviceToHost, P->s_main));
  IFGF_CUDA(cudaStreamSynchronize(P->s_main));
  if (!e) return;
  IFGF_CUDA(cudaMemsetAsync(P->err, 0, sizeof(int), P->s_main));
  switch (e) {
    case kErrSMax:
      throw Error(IFGF_EDOMAIN, "cone_of_point: point inside the neighbor zone (s > s_max)");
    case kErrCenter:
      throw Error(IFGF_EDOMAIN, "cone_coords: point at box center");
    case kErrPropCover:
      throw Error(IFGF_ELOGIC, "propagation: node not covered by a relevant child cone");
    case kErrInterpCover:
      throw Error(IFGF_ELOGIC, "interpolation: cousin point not covered by a relevant cone");
    case kErrOutside:
      throw Error(IFGF_EDOMAIN, "point outside bounding cube");
    case kErrNonFinite:
      throw Error(IFGF_EINVAL, "cheb_fit: non-finite node value");
    case kErrBadCone:
      throw Error(IFGF_EINVAL, "block exchange: cone ordinal out of range");
    default:
      throw Error(IFGF_ERUNTIME, "unknown device error " + std::to_string(e));
  }
}

namespace {

template <bool MARK>
void launch_locate_range(ifgf_plan* P, int d, uint32_t b_lo, uint32_t b_hi, cudaStream_t s) {
  const Level& L = P->lv[d];
  const unsigned g = (unsigned)((L.chunk_cap + 255) / 256);
  auto go = [&](auto kern) {
    kern<<<g, 256, 0, s>>>(L.dev(), L.chunk, L.nchunk, P->xs, P->ys, P->zs, P->kappa, L.bits,
                           L.rec_g, L.rec, b_lo, b_hi, P->err);
  };
  const bool lap = P->kappa == 0.0;
  switch (interp_points(P->K.P)) {
    case 1: lap ? go(k_locate_points<true, 1, MARK>) : go(k_locate_points<false, 1, MARK>); break;
    case 2: lap ? go(k_locate_points<true, 2, MARK>) : go(k_locate_points<false, 2, MARK>); break;
    case 3: lap ? go(k_locate_points<true, 3, MARK>) : go(k_locate_points<false, 3, MARK>); break;
    default: lap ? go(k_locate_points<true, 4, MARK>) : go(k_locate_points<false, 4, MARK>); break;
  }
  ++P->launches;
}

void launch_rec_cones(ifgf_plan* P, int d, uint32_t b_lo, uint32_t b_hi, uint32_t p_lo,
                      uint32_t p_hi, cudaStream_t s) {
  const Level& L = P->lv[d];
  auto conv = [&](auto kern) {
    kern<<<grid_for(L.chunk_cap), kT, 0, s>>>(L.dev(), L.chunk, L.nchunk, L.rec_g, b_lo, b_hi,
                                              p_lo, p_hi, P->err);
  };
  switch (interp_points(P->K.P)) {
    case 1: conv(k_rec_cones<1>); break;
    case 2: conv(k_rec_cones<2>); break;
    case 3: conv(k_rec_cones<3>); break;
    default: conv(k_rec_cones<4>); break;
  }
  ++P->launches;
}

// Record storage of levels 3..D: `pairs[d]` pairs per level, all levels or
// none.  An allocation failure (memory taken by others since the budget's
// sample) only costs the records: K4 falls back to k_interp.
bool alloc_records(ifgf_plan* P, const std::vector<unsigned long long>& pairs, cudaStream_t s) {
  const int D = P->depth, planes = P->kappa == 0.0 ? 4 : 5;
  bool ok = true;
  std::vector<void*> got;
  size_t got_bytes = 0;
  for (int d = 3; d <= D && ok; ++d) {
    Level& L = P->lv[d];
    const size_t b[2] = {((size_t)planes * pairs[d] + 2) * sizeof(double) + 16,
                         ((size_t)pairs[d] + 2) * sizeof(uint32_t) + 16};
    void* p[2] = {nullptr, nullptr};
    for (int i = 0; i < 2 && ok; ++i) {
      if (cudaMallocAsync(&p[i], b[i], s) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
      } else {
        got.push_back(p[i]);
        got_bytes += b[i];
      }
    }
    L.npairs = pairs[d];
    L.rec = static_cast<double*>(p[0]);
    L.rec_g = static_cast<uint32_t*>(p[1]);
  }
  if (ok) {
    P->allocs.insert(P->allocs.end(), got.begin(), got.end());
    P->bytes += got_bytes;
  } else {
    for (void* q : got) cudaFreeAsync(q, s);
    for (int d = 3; d <= D; ++d) {
      P->lv[d].rec = nullptr;
      P->lv[d].rec_g = nullptr;
      P->lv[d].npairs = 0;
    }
  }
  return ok;
}

double records_fraction() {
  static const double f = [] {
    const char* v = std::getenv("IFGF_K4_REC_FRAC");
    return v ? std::atof(v) : 0.15;
  }();
  return f;
}

}  // namespace

void launch_locate_points(ifgf_plan* P, int d, cudaStream_t s) {
  launch_locate_range<true>(P, d, 0u, 0xffffffffu, s);
}

// K4 records of a rank plan: for the boxes that hold the rank's points
// [p0, p1) at every level (1/R of the single-GPU plan's records), built after
// dist_prepare has made the level bitmaps rank-local, so the stored ordinals
// are the rank's block slots.
void build_rank_records(ifgf_plan* P, uint32_t p0, uint32_t p1) {
  const int D = P->depth;
  if (p1 <= p0 || D < 3 || !P->lv[D].pair_off) return;
  cudaStream_t s = P->s_main;
  std::vector<uint32_t> blo(D + 1, 0), bhi(D + 1, 0);
  std::vector<unsigned long long> off(D + 1, 0), end(D + 1, 0);
  for (int d = 3; d <= D; ++d) {
    IFGF_CUDA(cudaMemcpyAsync(&blo[d], P->lv[d].ptbox + p0, 4, cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaMemcpyAsync(&bhi[d], P->lv[d].ptbox + (p1 - 1), 4, cudaMemcpyDeviceToHost, s));
  }
  IFGF_CUDA(cudaStreamSynchronize(s));
  for (int d = 3; d <= D; ++d) {
    IFGF_CUDA(cudaMemcpyAsync(&off[d], P->lv[d].pair_off + blo[d], 8, cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaMemcpyAsync(&end[d], P->lv[d].pair_off + bhi[d] + 1, 8, cudaMemcpyDeviceToHost, s));
  }
  IFGF_CUDA(cudaStreamSynchronize(s));
  const int planes = P->kappa == 0.0 ? 4 : 5;
  std::vector<unsigned long long> win(D + 1, 0);
  unsigned long long pairs = 0;
  for (int d = 3; d <= D; ++d) pairs += (win[d] = end[d] - off[d]);
  const double need = (double)pairs * (planes * sizeof(double) + sizeof(uint32_t));
  if (pairs == 0 || need > records_fraction() * (double)mem_available(P)) return;
  if (!alloc_records(P, win, s)) return;
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    L.rec -= off[d];  // indexed by the level's global pair offsets
    L.rec_g -= off[d];
    launch_locate_range<false>(P, d, blo[d], bhi[d], s);
    launch_rec_cones(P, d, blo[d], bhi[d], p0, p1, s);
  }
  IFGF_CUDA(cudaStreamSynchronize(s));
  check_device_error(P);
}

void build_plan(ifgf_plan* P, const double* d_x, const double* d_y, const double* d_z) {
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = P->s_main;
  const size_t n = P->n;
  Scratch scratch{P};
  // IFGF_SETUP_TRACE=1: synchronise and print the elapsed time at each phase;
  // IFGF_SETUP_TRACE=2: no extra syncs -- record an event per phase on the
  // main stream and print, per phase, when the host passed it and when the
  // GPU did (a GPU time just after the host time means the GPU was waiting).
  static const int trace = [] {
    const char* v = std::getenv("IFGF_SETUP_TRACE");
    return v ? std::atoi(v) : 0;
  }();
  struct Mark {
    const char* what;
    double host_ms;
    cudaEvent_t ev;
  };
  std::vector<Mark> marks;
  cudaEvent_t ev0 = nullptr;
  if (trace == 2) {
    cudaEventCreate(&ev0);
    cudaEventRecord(ev0, s);
  }
  auto mark = [&](const char* what) {
    const double hm =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3;
    if (trace == 1) {
      cudaStreamSynchronize(s);
      std::fprintf(stderr, "[setup] %-28s %8.3f ms\n", what,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() *
                       1e3);
    } else if (trace == 2) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      marks.push_back({what, hm, e});
    }
  };
  auto dump_marks = [&] {
    if (trace != 2) return;
    cudaStreamSynchronize(s);
    for (auto& m : marks) {
      float g = 0.f;
      cudaEventElapsedTime(&g, ev0, m.ev);
      std::fprintf(stderr, "[setup] %-28s host %8.3f ms  gpu %8.3f ms\n", m.what, m.host_ms, g);
      cudaEventDestroy(m.ev);
    }
    cudaEventDestroy(ev0);
  };

  // -- bounding cube (geometry.cpp:95-114)
  const int nparts = 296;
  double* part = P->alloc<double>(nparts * 6 + 6);
  k_bbox_partial<<<nparts, kT, 0, s>>>(d_x, d_y, d_z, n, part);
  k_bbox_final<<<1, 32, 0, s>>>(part, nparts, part + nparts * 6);
  P->launches += 2;
  double bb[6];
  IFGF_CUDA(cudaMemcpyAsync(bb, part + nparts * 6, sizeof bb, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  for (int c = 0; c < 6; ++c)
    if (!std::isfinite(bb[c])) throw Error(IFGF_EDOMAIN, "point outside bounding cube");
  const double extent = std::max({bb[3] - bb[0], bb[4] - bb[1], bb[5] - bb[2]});
  const double side = std::max((1.0 + 1e-6) * extent, 1e-9);
  P->cube[3] = side;
  for (int c = 0; c < 3; ++c) P->cube[c] = 0.5 * (bb[c] + bb[3 + c]) - 0.5 * side;

  mark("bounding cube");
  // -- depth (engine.cpp:55-72)
  int D = 0;
  {
    const int rc = ifgf_choose_depth(n, side, P->kappa, &P->params, &D);
    if (rc) throw Error(rc, ifgf_last_error());
  }
  P->depth = D;
  {
    // angle seed table for the fast locate (ifgf_common.cuh fast_angles)
    std::vector<double2> trig(kTrigEntries);
    for (int k = 0; k < kTrigPhi; ++k) {
      const double a = (double)k * kTrigHPhi;  // same rounded product as fast_angles
      trig[k] = make_double2(std::cos(a), std::sin(a));
    }
    for (int k = 0; k <= kTrigTheta; ++k) {
      const double a = (double)k * kTrigHTheta;
      trig[kTrigPhi + k] = make_double2(std::cos(a), std::sin(a));
    }
    // phase table for sincos_tab: {cos, sin}(k 2 pi / kPhaseEntries), rounded
    // from long double
    for (int k = 0; k < kPhaseEntries; ++k) {
      const long double a =
          (long double)k * 6.28318530717958647692528676655900577L / (long double)kPhaseEntries;
      trig.push_back(make_double2((double)cosl(a), (double)sinl(a)));
    }
    double2* d_trig = P->alloc<double2>(trig.size());
    IFGF_CUDA(cudaMemcpyAsync(d_trig, trig.data(), trig.size() * sizeof(double2),
                              cudaMemcpyHostToDevice, s));
    for (int d = 0; d < IFGF_MAX_LEVELS; ++d) P->lv[d].trig = d_trig;
    P->phase = d_trig + kTrigEntries;
    IFGF_CUDA(cudaStreamSynchronize(s));  // trig lives on the stack until copied
  }
  {
    // bitmap indices of the coarsest cone level must fit the u32 gamma
    const double G3 = (double)P->params.base_s * P->params.base_theta * P->params.base_phi *
                      std::pow(8.0, D - 3);
    if (G3 >= 4294967296.0)
      throw Error(IFGF_EINVAL, "depth " + std::to_string(D) +
                                   " needs cone indices beyond 32 bits (unsupported)");
  }

  mark("trig table");
  // -- Morton codes + stable sort (morton.cpp:70-95)
  const uint32_t ngrid = 1u << (D - 1);
  const double hD = side / static_cast<double>(ngrid);
  uint64_t* codes_in = P->alloc<uint64_t>(n);
  uint64_t* codes = P->alloc<uint64_t>(n);
  uint32_t* idx_in = P->alloc<uint32_t>(n);
  P->perm = P->alloc<uint32_t>(n);
  k_morton<<<grid_for(n), kT, 0, s>>>(d_x, d_y, d_z, n, P->cube[0], P->cube[1], P->cube[2], side,
                                      hD, ngrid, codes_in, idx_in, P->err);
  ++P->launches;
  {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, codes_in, codes, idx_in, P->perm, (int)n, 0,
                                    3 * (D - 1), s);
    IFGF_CUDA(cub::DeviceRadixSort::SortPairs(scratch.get(tb), tb, codes_in, codes, idx_in,
                                              P->perm, (int)n, 0, 3 * (D - 1), s));
  }
  P->xs = P->alloc<double>(n);
  P->ys = P->alloc<double>(n);
  P->zs = P->alloc<double>(n);
  k_gather3<<<grid_for(n), kT, 0, s>>>(P->perm, d_x, d_y, d_z, n, P->xs, P->ys, P->zs);
  ++P->launches;

  mark("morton sort");
  // -- octree levels (octree.cpp:18-94)
  uint8_t* start = P->alloc<uint8_t>(n);
  uint32_t* hist = P->alloc<uint32_t>(32);
  IFGF_CUDA(cudaMemsetAsync(hist, 0, 32 * sizeof(uint32_t), s));
  k_start_level<<<grid_for(n), kT, 0, s>>>(codes, n, D, start, hist);
  ++P->launches;
  uint32_t h_hist[32];
  IFGF_CUDA(cudaMemcpyAsync(h_hist, hist, sizeof h_hist, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  mark("level sizes sync");
  {
    uint32_t acc = 0;
    for (int d = 1; d <= D; ++d) {
      acc += h_hist[d];
      P->lv[d].nb = acc;
      P->lv[d].d = d;
      P->lv[d].h = side / static_cast<double>(1u << (d - 1));
    }
  }
  for (int d = 1; d <= D; ++d) {
    Level& L = P->lv[d];
    L.ptbox = P->alloc<uint32_t>(n);
    cub::TransformInputIterator<uint32_t, StartsAt, cub::CountingInputIterator<size_t>> it(
        cub::CountingInputIterator<size_t>(0), StartsAt{start, d});
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, it, L.ptbox, (int)n, s);
    IFGF_CUDA(cub::DeviceScan::InclusiveSum(scratch.get(tb), tb, it, L.ptbox, (int)n, s));
    L.first = P->alloc<uint32_t>(L.nb);
    L.count = P->alloc<uint32_t>(L.nb);
    L.code = P->alloc<uint64_t>(L.nb);
    L.cx = P->alloc<double>(L.nb);
    L.cy = P->alloc<double>(L.nb);
    L.cz = P->alloc<double>(L.nb);
    k_boxes<<<grid_for(n), kT, 0, s>>>(L.ptbox, start, codes, n, d, D, P->cube[0], P->cube[1],
                                       P->cube[2], L.h, L.first, L.code, L.cx, L.cy, L.cz);
    ++P->launches;
  }
  mark("boxes");
  for (int d = 1; d <= D; ++d) {
    Level& L = P->lv[d];
    L.parent = P->alloc<uint32_t>(L.nb);
    L.child_begin = d < D ? P->alloc<uint32_t>(L.nb + 1) : nullptr;
    k_box_links<<<grid_for(L.nb + 1), kT, 0, s>>>(
        L.nb, n, L.first, L.count, d > 1 ? P->lv[d - 1].ptbox : nullptr, L.parent,
        d < D ? P->lv[d + 1].ptbox : nullptr, L.child_begin, d < D ? P->lv[d + 1].nb : 0);
    L.nbr = P->alloc<uint32_t>((size_t)L.nb * 27);
    L.nbr_cnt = P->alloc<uint32_t>(L.nb);
    k_neighbors<<<grid_for(L.nb), kT, 0, s>>>(L.nb, d, L.code, L.nbr, L.nbr_cnt);
    P->launches += 2;
  }
  // cousin CSR for d = 3..D
  std::vector<uint32_t> cous_total(D + 1, 0);
  // K4 records (k_locate_points): kept when all levels' records fit in
  // IFGF_K4_REC_FRAC (default 0.15) of the plan's memory budget;
  // IFGF_K4_RECORDS=0 turns them off.
  static const bool rec_env = [] {
    const char* v = std::getenv("IFGF_K4_RECORDS");
    return !v || std::atoi(v) != 0;
  }();
  const double rec_frac = records_fraction();
  // rank plans get the offsets here and their records from build_rank_records
  const bool want_records = rec_env && D >= 3;
  std::vector<unsigned long long> pair_total(D + 1, 0);
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    uint32_t* cnt = P->alloc<uint32_t>(L.nb + 1);
    L.cous_off = P->alloc<uint32_t>(L.nb + 1);
    IFGF_CUDA(cudaMemsetAsync(cnt + L.nb, 0, sizeof(uint32_t), s));
    k_cousins<<<grid_for(L.nb), kT, 0, s>>>(L.dev(), P->lv[d - 1].dev(), cnt, nullptr);
    ++P->launches;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, L.cous_off, (int)(L.nb + 1), s);
    IFGF_CUDA(
        cub::DeviceScan::ExclusiveSum(scratch.get(tb), tb, cnt, L.cous_off, (int)(L.nb + 1), s));
    IFGF_CUDA(cudaMemcpyAsync(&cous_total[d], L.cous_off + L.nb, sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, s));
    if (want_records) {
      // K4 record offsets: exclusive sum of points x cousins per box
      uint64_t* pc = P->alloc<uint64_t>(L.nb + 1);
      L.pair_off = P->alloc<uint64_t>(L.nb + 1);
      k_pair_count<<<grid_for(L.nb + 1), kT, 0, s>>>(L.count, cnt, L.nb,
                                                     (uint32_t)interp_points(P->K.P), pc);
      ++P->launches;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, pc, L.pair_off, (int)(L.nb + 1), s);
      IFGF_CUDA(
          cub::DeviceScan::ExclusiveSum(scratch.get(tb), tb, pc, L.pair_off, (int)(L.nb + 1), s));
      IFGF_CUDA(cudaMemcpyAsync(&pair_total[d], L.pair_off + L.nb, sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, s));
    }
  }
  // neighbour-list totals (ifgf_plan_info), read back with the cousin totals
  std::vector<unsigned long long> nbr_total(D + 1, 0);
  {
    unsigned long long* d_tot = P->alloc<unsigned long long>(D + 1);
    for (int d = 1; d <= D; ++d) {
      size_t tb = 0;
      cub::DeviceReduce::Sum(nullptr, tb, P->lv[d].nbr_cnt, d_tot + d, (int)P->lv[d].nb, s);
      IFGF_CUDA(cub::DeviceReduce::Sum(scratch.get(tb), tb, P->lv[d].nbr_cnt, d_tot + d,
                                       (int)P->lv[d].nb, s));
    }
    IFGF_CUDA(cudaMemcpyAsync(nbr_total.data() + 1, d_tot + 1, D * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
  }
  mark("neighbours + cousin counts");
  // K4 work items per level
  {
    const int R = interp_points(P->K.P);
    for (int d = 3; d <= D; ++d) {
      Level& L = P->lv[d];
      uint32_t* cnt = P->alloc<uint32_t>(L.nb + 1);
      uint32_t* off = P->alloc<uint32_t>(L.nb + 1);
      IFGF_CUDA(cudaMemsetAsync(cnt + L.nb, 0, sizeof(uint32_t), s));
      k_chunk_count<<<grid_for(L.nb), kT, 0, s>>>(L.count, L.nb, R, cnt);
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(L.nb + 1), s);
      IFGF_CUDA(cub::DeviceScan::ExclusiveSum(scratch.get(tb), tb, cnt, off, (int)(L.nb + 1), s));
      L.chunk_cap = (n + R - 1) / R + L.nb;
      L.chunk = P->alloc<uint2>(L.chunk_cap);
      L.nchunk = off + L.nb;
      k_chunk_fill<<<grid_for(L.chunk_cap), kT, 0, s>>>(L.first, L.nb, R, off, L.chunk_cap,
                                                         L.chunk);
      P->launches += 3;
    }
  }
  mark("K4 work items");
  IFGF_CUDA(cudaStreamSynchronize(s));
  mark("cousin sync");
  for (int d = 1; d <= D; ++d) P->lv[d].n_nbr = (size_t)nbr_total[d];
  if (want_records) {
    const int planes = P->kappa == 0.0 ? 4 : 5;
    unsigned long long pairs = 0;
    for (int d = 3; d <= D; ++d) pairs += pair_total[d];
    const double need = (double)pairs * (planes * sizeof(double) + sizeof(uint32_t));
    if (!P->rank_plan && pairs > 0 && need <= rec_frac * (double)mem_available(P))
      alloc_records(P, pair_total, s);
  }
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    L.n_cous = cous_total[d];
    L.cous = P->alloc<uint32_t>(L.n_cous + 1);
    k_cousins<<<grid_for(L.nb), kT, 0, s>>>(L.dev(), P->lv[d - 1].dev(), L.cous_off, L.cous);
    ++P->launches;
  }

  mark("octree + cousins");
  // -- relevant cones, d = 3..D (cones.cpp:90-150)
  // Clause 1 (points) of every level depends only on the octree: all levels
  // are marked up front on the aux stream, overlapping clause 2 (parent
  // nodes, level by level, which needs the parent level's cones), the tile
  // builds and the host round trips for the cone counts on the main stream.
  const ifgf_params& p = P->params;
  cudaStream_t sa = P->s_aux;
  cudaEvent_t ev_tree, ev_pts[IFGF_MAX_LEVELS];
  IFGF_CUDA(cudaEventCreateWithFlags(&ev_tree, cudaEventDisableTiming));
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    const int f = 1 << (D - d);
    L.n0 = p.base_s * f;
    L.n1 = p.base_theta * f;
    L.n2 = p.base_phi * f;
    L.w0 = kSMax / L.n0;
    L.w1 = kPi / L.n1;
    L.w2 = 2.0 * kPi / L.n2;
    L.iw0 = 1.0 / L.w0;
    L.iw1 = 1.0 / L.w1;
    L.iw2 = 1.0 / L.w2;
    L.rad = std::sqrt(3.0) * L.h / 2.0;
    L.G = (uint64_t)L.n0 * L.n1 * L.n2;
    L.nwords = ((uint64_t)L.nb * L.G + 63) / 64;
    L.bits = P->alloc<uint64_t>(L.nwords);
    L.rank = P->alloc<uint32_t>(L.nwords + 1);
  }
  IFGF_CUDA(cudaEventRecord(ev_tree, s));
  IFGF_CUDA(cudaStreamWaitEvent(sa, ev_tree, 0));
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    IFGF_CUDA(cudaMemsetAsync(L.bits, 0, L.nwords * sizeof(uint64_t), sa));
    if (L.rec) {
      launch_locate_points(P, d, sa);
    } else {
      k_mark_points<<<grid_for(n), kT, 0, sa>>>(L.dev(), L.ptbox, P->xs, P->ys, P->zs, n, L.bits,
                                                P->err);
      ++P->launches;
    }
    IFGF_CUDA(cudaEventCreateWithFlags(&ev_pts[d], cudaEventDisableTiming));
    IFGF_CUDA(cudaEventRecord(ev_pts[d], sa));
  }
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    IFGF_CUDA(cudaStreamWaitEvent(s, ev_pts[d], 0));
    mark("  mark points");
    if (d > 3 && P->lv[d - 1].nc > 0) {
      build_prop_tiles(
          P, d, [](void* ctx, size_t b) { return static_cast<Scratch*>(ctx)->get(b); }, &scratch);
      mark("  tiles");
      if (P->tiles[d].enabled) {
        launch_mark_nodes_tiles(P, d, L.bits);
      } else {
        const size_t work = (size_t)P->lv[d - 1].nc * P->K.P;
        k_mark_nodes<<<grid_for(work), kT, 0, s>>>(L.dev(), P->lv[d - 1].dev(), P->K, L.bits,
                                                   P->err);
        ++P->launches;
      }
    }
    mark("  mark nodes");
    uint32_t* cnt = P->alloc<uint32_t>(L.nwords + 1);
    k_popc<<<grid_for(L.nwords + 1), kT, 0, s>>>(L.bits, L.nwords, cnt);
    ++P->launches;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, L.rank, (int)(L.nwords + 1), s);
    IFGF_CUDA(
        cub::DeviceScan::ExclusiveSum(scratch.get(tb), tb, cnt, L.rank, (int)(L.nwords + 1), s));
    uint32_t nc = 0;
    IFGF_CUDA(
        cudaMemcpyAsync(&nc, L.rank + L.nwords, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaStreamSynchronize(s));
    mark("  count sync");
    L.nc = nc;
    L.cone_box = P->alloc<uint32_t>(nc + 1);
    L.cone_gamma = P->alloc<uint32_t>(nc + 1);
    L.box_cone = P->alloc<uint32_t>(L.nb + 1);
    k_compact<<<grid_for(L.nwords), kT, 0, s>>>(L.dev(), L.nwords, L.cone_box, L.cone_gamma);
    k_box_cone<<<grid_for(L.nb + 1), kT, 0, s>>>(L.dev(), L.box_cone);
    P->launches += 2;
    if (L.rec) {  // records: segment -> cone ordinal, on the aux stream
      IFGF_CUDA(cudaEventRecord(ev_pts[d], s));
      IFGF_CUDA(cudaStreamWaitEvent(sa, ev_pts[d], 0));
      launch_rec_cones(P, d, 0u, 0xffffffffu, 0u, 0xffffffffu, sa);
    }
    mark("  compact");
  }
  IFGF_CUDA(cudaEventRecord(ev_tree, sa));
  IFGF_CUDA(cudaStreamWaitEvent(s, ev_tree, 0));
  IFGF_CUDA(cudaStreamSynchronize(s));
  cudaEventDestroy(ev_tree);
  for (int d = 3; d <= D; ++d) cudaEventDestroy(ev_pts[d]);
  mark("end");
  dump_marks();
  check_device_error(P);
  P->setup_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace ifgf_b200
