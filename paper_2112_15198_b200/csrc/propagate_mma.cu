// propagate_mma.cu -- K3 (propagation_pass) from precomputed tile geometry:
// the row kernel (default), its on-the-fly form for levels without tiles,
// and the box-batched FP64 tensor-core GEMM (IFGF_PROP_DMMA).
//
// propagation_pass (engine.cpp:138-189) evaluates, for every parent cone q of
// level d-1 and every child box of q's box, the child interpolants at q's P
// interpolation nodes.  The nodes relative to a child centre depend only on
// the parent segment gamma and the child's octant in the parent box (child
// centres sit at parent centre +-h_child/2 per axis), not on the box.  So per
// (gamma, octant) "tile" the plan precomputes, once:
//   * the child cone gamma_c, local coordinates (ts, tt, tp) and re-centring
//     factor (rp/rc) e^{i kappa (rc - rp)} of every node (fast locate with the
//     exact-fallback margin; entries within the margin are flagged and
//     recomputed per box with the reference's exact formulas),
//   * the nodes grouped by gamma_c into row tiles of 8.
// k_propagate_rows evaluates rows of <= 3 nodes sharing a child cone per
// block load; k_propagate_gemm (IFGF_PROP_DMMA) batches up to 32 parent cones
// that share gamma and computes V[node][cone] = sum_k B_k(t_node) *
// C_{child cone}[k] with mma.sync.m8n8k4.f64.  Same result up to rounding.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "plan.hpp"

namespace ifgf_b200 {
namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kFlag = 0x80000000u;
constexpr uint32_t kFlagTask = 0xfffffffeu;  // task meta: flagged node (exact path)
// 12 warps of <= 168 registers per SM (measured best at C2 among 256/320/384
// threads and 1-2 CTAs per SM)
#ifndef IFGF_ROWS_THREADS
#define IFGF_ROWS_THREADS 384
#endif
#ifndef IFGF_ROWS_MINB
#define IFGF_ROWS_MINB 1
#endif
constexpr int kRowThreads = IFGF_ROWS_THREADS;
// L1 prefetch of the next task's child block
#ifndef IFGF_ROWS_PF
#define IFGF_ROWS_PF 1
#endif
// L1 prefetch of the round's blocks and row data after phase A
#ifndef IFGF_ROWS_PFA
#define IFGF_ROWS_PFA 1
#endif
constexpr int kRowMaxCpw = 16;  // parent cones per warp

struct TilesDev {
  uint32_t ngamma;
  const uint32_t* cone_gidx;
  const uint32_t* gamma_of;
  const double* e_t;
  const double2* e_T;
  const uint32_t* e_gc;
  const uint32_t* rt_off;
  const uint4* rt;
  const uint32_t* fl_cnt;   // flagged nodes of tile t: fl_node[t * P + i], i < fl_cnt[t]
  const uint16_t* fl_node;
  const uint8_t* e_perm;
  const uint32_t* rw_cnt;   // rows of tile t: rw[t * P + i], i < rw_cnt[t]
  const uint2* rw;
  const double* rdat;
  const uint32_t* rnode;
  const uint32_t* usorted;
  const uint32_t* unit_start;
};

TilesDev tiles_dev(const PropTiles& t) {
  return {t.ngamma,   t.cone_gidx,   t.gamma_of, t.e_t,    t.e_T,  t.e_gc, t.rt_off,
          t.rt,       t.fl_cnt,      t.fl_node,  t.e_perm,
          t.rw_cnt,   t.rw,          t.rdat,     t.rnode,   t.usorted, t.unit_start};
}

inline unsigned nblk(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ int rt_node(const uint4& R, int r) {
  const uint32_t w = r < 4 ? R.y : R.z;
  return (int)((w >> (8 * (r & 3))) & 0xffu);
}

// ---------------------------------------------------------------- building
__global__ void k_gamma_mark(const __grid_constant__ LevelDev U, uint64_t* gbits) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= U.nc) return;
  const uint32_t g = U.cone_gamma[q];
  const uint64_t m = 1ull << (g & 63);
  // most cones of a level share few gammas: test before the atomic
  if (!(gbits[g >> 6] & m)) atomicOr((unsigned long long*)&gbits[g >> 6], m);
}

__global__ void k_gamma_popc(const uint64_t* gbits, size_t nw, uint32_t* cnt) {
  const size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (w < nw) cnt[w] = __popcll(gbits[w]);
  else if (w == nw) cnt[w] = 0;
}

__global__ void k_gamma_index(const __grid_constant__ LevelDev U, const uint64_t* gbits,
                              const uint32_t* grank, uint32_t* cone_gidx, uint32_t* gamma_of) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= U.nc) return;
  const uint32_t g = U.cone_gamma[q];
  const uint64_t w = gbits[g >> 6];
  const uint32_t idx = grank[g >> 6] + __popcll(w & ((1ull << (g & 63)) - 1));
  cone_gidx[q] = idx;
  gamma_of[idx] = g;  // same value from every cone of this gamma
}

// One thread per (gamma index, octant, node).
__global__ void k_tile_entries(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                               const __grid_constant__ InterpConsts K, const uint32_t* gamma_of,
                               uint32_t ngamma, double kappa, double* e_t, double2* e_T,
                               uint32_t* e_gc) {
  __shared__ double2 trig[kTrigEntries];
  stage_trig(trig, L.trig);
  __syncthreads();
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)ngamma * 8 * K.P) return;
  const int m = (int)(t % K.P);
  const uint32_t tile = (uint32_t)(t / K.P);
  const int oct = (int)(tile & 7);
  const uint32_t gi = tile >> 3;
  const int jp = m % K.pp, jt = (m / K.pp) % K.pt, js = m / (K.pp * K.pt);
  const SegMid sg = segment_mid(U, gamma_of[gi]);
  // node relative to the parent centre (reference order without the centre)
  double x, y, z;
  node_position(sg, U.rad, 0.0, 0.0, 0.0, K.ns[js], K.nt[jt], K.np[jp], x, y, z);
  const double hc = L.h;
  const double ox = ((oct & 1) ? 0.5 : -0.5) * hc, oy = ((oct & 2) ? 0.5 : -0.5) * hc,
               oz = ((oct & 4) ? 0.5 : -0.5) * hc;
  const double rp = sqrt(fma(z, z, fma(y, y, x * x)));
  // fast locate relative to the child centre; flag anything near a boundary
  const double dx = x - ox, dy = y - oy, dz = z - oz;
  const double rho2 = fma(dy, dy, dx * dx), r2 = fma(dz, dz, rho2);
  const double rinv = rsqrt_nr(r2), s = L.rad * rinv, rho_inv = rsqrt_nr(rho2);
  double theta, phi;
  fast_angles(trig, dx, dy, dz, rho2 * rho_inv, rinv, rho_inv, theta, phi);
  const double fs = s * L.iw0, ft = theta * L.iw1, fp = phi * L.iw2;
  const bool flag = !(rho2 > 1e-300) || s > kSMaxTol * (1.0 - 1e-12) || near_boundary(fs) ||
                    near_boundary(ft) || near_boundary(fp);
  int is = (int)fs, it = (int)ft, ip = (int)fp;
  is = is < L.n0 - 1 ? is : L.n0 - 1;
  it = it < L.n1 - 1 ? it : L.n1 - 1;
  ip = ip < L.n2 - 1 ? ip : L.n2 - 1;
  const uint32_t gc = ((uint32_t)is * (uint32_t)L.n1 + (uint32_t)it) * (uint32_t)L.n2 + (uint32_t)ip;
  e_gc[t] = flag ? (kFlag | gc) : gc;
  e_t[3 * t] = 2.0 * (fs - is) - 1.0;
  e_t[3 * t + 1] = 2.0 * (ft - it) - 1.0;
  e_t[3 * t + 2] = 2.0 * (fp - ip) - 1.0;
  const double rc = r2 * rinv, ratio = rp * rinv;
  double sn = 0.0, cn = 1.0;
  if (kappa != 0.0) sincos_fast(kappa * (rc - rp), sn, cn);
  e_T[t] = make_double2(ratio * cn, ratio * sn);
}

// One thread per tile: group its non-flagged nodes by child gamma (stable in
// node order) into row tiles of 8; list flagged nodes.  Pass 1 counts.
__global__ void k_tile_rows(uint32_t ntiles, int P, const uint32_t* e_gc, uint32_t* rt_cnt,
                            uint32_t* fl_cnt, const uint32_t* rt_off, uint4* rt,
                            const uint32_t* fl_off, uint16_t* fl_node, uint8_t* e_perm,
                            uint32_t* rt_tile = nullptr) {
  uint32_t wp = 0;
  const uint32_t tile = blockIdx.x * blockDim.x + threadIdx.x;
  if (tile >= ntiles) return;
  const uint32_t* g = e_gc + (size_t)tile * P;
  uint32_t nrt = 0, nfl = 0;
  uint32_t wr = rt ? rt_off[tile] : 0;
  uint32_t wfl = fl_node ? fl_off[tile] : 0;
  // nodes in ascending (gamma, node) order: repeated min-scan (P <= 255)
  uint32_t last = 0;
  bool first = true;
  for (;;) {
    uint32_t cur = kNone;
    for (int m = 0; m < P; ++m) {
      const uint32_t v = g[m];
      if (v & kFlag) continue;
      if ((first || v > last) && v < cur) cur = v;
    }
    if (cur == kNone) break;
    first = false;
    last = cur;
    // group size in nodes -> row tiles; the group's first row tile carries the count
    int gsz = 0;
    for (int m = 0; m < P; ++m) gsz += g[m] == cur;
    const uint32_t ngt = (uint32_t)(gsz + 7) / 8;
    uint4 R = make_uint4(cur, 0xffffffffu, 0xffffffffu, ngt);
    int k = 0;
    for (int m = 0; m < P; ++m) {
      if (g[m] != cur) continue;
      if (e_perm) e_perm[(size_t)tile * P + wp++] = (uint8_t)m;
      const uint32_t sh = 8 * (k & 3);
      if (k < 4) R.y = (R.y & ~(0xffu << sh)) | ((uint32_t)m << sh);
      else R.z = (R.z & ~(0xffu << sh)) | ((uint32_t)m << sh);
      if (++k == 8) {
        if (rt_tile) rt_tile[wr] = tile;
        if (rt) rt[wr++] = R;
        ++nrt;
        R = make_uint4(cur, 0xffffffffu, 0xffffffffu, 0);
        k = 0;
      }
    }
    if (k) {
      if (rt_tile) rt_tile[wr] = tile;
      if (rt) rt[wr++] = R;
      ++nrt;
    }
  }
  for (int m = 0; m < P; ++m)
    if (g[m] & kFlag) {
      if (fl_node) fl_node[wfl++] = (uint16_t)m;
      if (e_perm) e_perm[(size_t)tile * P + wp++] = (uint8_t)m;
      ++nfl;
    }
  if (rt_cnt) {
    rt_cnt[tile] = nrt;
    fl_cnt[tile] = nfl;
  }
}

// Row data layout: the rows of a tile in chunks of 32; inside a chunk one
// 32-double column per field, so the lanes of a warp (consecutive rows)
// read every field with one coalesced 256-byte access, and a tile's rows
// stay within a few contiguous kilobytes (tiles are re-read by every parent
// cone of their gamma).
__host__ __device__ __forceinline__ size_t row_field(size_t tile, int P, int nf, int r, int f) {
  const size_t chunks = (size_t)(P + 31) / 32;
  return (((tile * chunks + (size_t)(r >> 5)) * nf + f) << 5) + (r & 31);
}

// Warp per tile: nodes ordered by raw e_gc (child gamma ascending, flagged
// ones last), node order within a gamma -- ranks by all-pairs comparison in
// registers (no serial scans).  Writes e_perm, the rows of <= R nodes
// {gamma, position | count << 16 | first-of-group << 24}, the flagged list
// (node order), both at a fixed stride of P per tile with their counts, and
// the rows' node data (local coordinates, transfer factors, node ids).
template <int NS>
__global__ void __launch_bounds__(256)
    k_tile_sort(uint32_t ntiles, int P, int R, const uint32_t* __restrict__ e_gc,
                const double* __restrict__ e_t, const double2* __restrict__ e_T,
                uint32_t* rw_cnt, uint32_t* fl_cnt, uint2* rw, uint16_t* fl_node,
                uint8_t* e_perm, double* rdat, uint8_t* rnode) {
  const uint32_t tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (tile >= ntiles) return;
  const size_t base = (size_t)tile * P;
  uint32_t key[NS];
  int less[NS], eqb[NS], eqn[NS];
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    const int m = lane + 32 * sl;
    key[sl] = m < P ? e_gc[base + m] : 0xffffffffu;
    less[sl] = eqb[sl] = eqn[sl] = 0;
  }
#pragma unroll
  for (int s2 = 0; s2 < NS; ++s2)
    for (int l2 = 0; l2 < 32; ++l2) {
      const uint32_t kj = __shfl_sync(0xffffffffu, key[s2], l2);
      const int j = 32 * s2 + l2;
      if (j >= P) break;
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        const int m = lane + 32 * sl;
        less[sl] += kj < key[sl];
        const bool eq = kj == key[sl];
        eqn[sl] += eq;
        eqb[sl] += eq && j < m;
      }
    }
  // rows start at every R-th node of a gamma group
  bool valid[NS], flag[NS], start[NS];
  int nrows = 0, nflag = 0;
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    valid[sl] = lane + 32 * sl < P;
    flag[sl] = valid[sl] && (key[sl] & kFlag);
    start[sl] = valid[sl] && !flag[sl] && eqb[sl] % R == 0;
    nrows += __popc(__ballot_sync(0xffffffffu, start[sl]));
    nflag += __popc(__ballot_sync(0xffffffffu, flag[sl]));
  }
  if (lane == 0) {
    rw_cnt[tile] = (uint32_t)nrows;
    fl_cnt[tile] = (uint32_t)nflag;
  }
  // row index = rows of smaller gammas + rows before this node in its group
  int rows_before[NS];
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) rows_before[sl] = eqb[sl] / R;
#pragma unroll
  for (int s2 = 0; s2 < NS; ++s2) {
    const bool lead = valid[s2] && !flag[s2] && eqb[s2] == 0;
    const int nr = lead ? (eqn[s2] + R - 1) / R : 0;
    for (int l2 = 0; l2 < 32; ++l2) {
      const uint32_t kj = __shfl_sync(0xffffffffu, key[s2], l2);
      const int rj = __shfl_sync(0xffffffffu, nr, l2);
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) rows_before[sl] += (rj && kj < key[sl]) ? rj : 0;
    }
  }
  const size_t r0 = base, f0 = base;  // fixed stride P per tile
  int fbase = 0;
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    const int m = lane + 32 * sl;
    const uint32_t fb = __ballot_sync(0xffffffffu, flag[sl]);
    if (valid[sl]) {
      const int rank = less[sl] + eqb[sl];
      e_perm[base + rank] = (uint8_t)m;
      if (!flag[sl]) {
        // row data: slot j of row r, field f (ts, tt, tp, tr, ti) at
        // rdat[row_field(tile, r, f * R + j)] -- 32-row chunks, SoA inside
        const size_t e = base + m;
        const int r = rows_before[sl], j = eqb[sl] % R;
        const int nf = 5 * R;
        rdat[row_field(tile, P, nf, r, 0 * R + j)] = e_t[3 * e];
        rdat[row_field(tile, P, nf, r, 1 * R + j)] = e_t[3 * e + 1];
        rdat[row_field(tile, P, nf, r, 2 * R + j)] = e_t[3 * e + 2];
        rdat[row_field(tile, P, nf, r, 3 * R + j)] = e_T[e].x;
        rdat[row_field(tile, P, nf, r, 4 * R + j)] = e_T[e].y;
        rnode[4 * (base + r) + j] = (uint8_t)m;
      }
      if (start[sl]) {
        const int cnt = min(R, eqn[sl] - eqb[sl]);
        rw[r0 + rows_before[sl]] =
            make_uint2(key[sl], (uint32_t)rank | ((uint32_t)cnt << 16) |
                                    ((eqb[sl] == 0 ? 1u : 0u) << 24));
      }
      if (flag[sl]) fl_node[f0 + fbase + __popc(fb & ((1u << lane) - 1u))] = (uint16_t)m;
    }
    fbase += __popc(fb);
  }
}

__global__ void k_chunk_flags(const uint64_t* gsorted, uint32_t n, uint32_t chunk, uint32_t* flag,
                              int shift = 0) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    flag[i] = 0;
    return;
  }
  // chunk starts: every chunk-th element of each run of equal gamma index
  uint32_t lo = 0, hi = i;
  const uint64_t g = gsorted[i] >> shift;
  while (lo < hi) {  // run start = lower_bound(g)
    const uint32_t mid = (lo + hi) >> 1;
    if ((gsorted[mid] >> shift) < g) lo = mid + 1;
    else hi = mid;
  }
  flag[i] = ((i - lo) % chunk == 0) ? 1u : 0u;
}

__global__ void k_chunk_starts(const uint32_t* flag, const uint32_t* pos, uint32_t n,
                               uint32_t* chunk_start, uint32_t nchunks) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) chunk_start[pos[i]] = i;
  if (i == 0) chunk_start[nchunks] = n;
}


// Warp-GEMM keys: (box group, gamma index, child-octant mask).  Sorting by the
// mask inside a (group, gamma) run puts cones whose boxes have the same
// children next to each other, so the 8 columns of an MMA column tile mostly
// share their present octants.
__global__ void k_wgemm_keys(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                             const uint32_t* __restrict__ gidx, uint32_t ngamma,
                             uint32_t box_group, uint32_t qb, uint32_t qe, uint64_t* key,
                             uint32_t* qidx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= qe - qb) return;
  const uint32_t q = qb + i;
  const uint32_t pb = U.cone_box[q];
  uint32_t mask = 0;
  for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb)
    mask |= 1u << (uint32_t)(L.code[cb] & 7);
  key[i] = (((uint64_t)(pb / box_group) * ngamma + gidx[q]) << 8) | mask;
  qidx[i] = q;
}

// Per row tile and node slot: the node's local coordinates in its child cone,
// its re-centring factor and its index (-1: empty slot) in one 48-byte
// record, so the warp GEMM reads a row tile's node data with one dependent
// load instead of three.
struct WgRow {
  double ts, tt, tp, tfx, tfy;
  long long m;
};

__global__ void k_wgemm_rtab(uint32_t nrt, int P, const uint4* __restrict__ rt,
                             const uint32_t* __restrict__ rt_tile, const double* __restrict__ e_t,
                             const double2* __restrict__ e_T, WgRow* __restrict__ rtab) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrt * 8) return;
  const uint32_t r = i >> 3;
  const int m = rt_node(rt[r], (int)(i & 7));
  WgRow w = {0.0, 0.0, 0.0, 0.0, 0.0, -1};
  if (m != 0xff) {
    const size_t e = (size_t)rt_tile[r] * P + m;
    w.ts = e_t[3 * e];
    w.tt = e_t[3 * e + 1];
    w.tp = e_t[3 * e + 2];
    w.tfx = e_T[e].x;
    w.tfy = e_T[e].y;
    w.m = m;
  }
  rtab[i] = w;
}

// Clause 2 of compute_relevant_cones (cones.cpp:108-119) from the tiles: a
// (parent cone, child box) pair marks the distinct child gammas of its tile
// (one per node group, ~2-3 instead of P), flagged nodes are recomputed per
// box with cone_of_point.
__global__ void k_mark_nodes_tiles(const __grid_constant__ LevelDev L,
                                   const __grid_constant__ LevelDev U,
                                   const __grid_constant__ InterpConsts K, TilesDev T,
                                   uint64_t* bits, int* err) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= U.nc) return;
  const uint32_t pb = U.cone_box[q];
  const uint32_t gi = T.cone_gidx[q];
  for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb) {
    const uint32_t tile = gi * 8 + (uint32_t)(L.code[cb] & 7);
    for (uint32_t r = 0; r < T.rw_cnt[tile]; ++r) {
      const uint2 R = T.rw[(size_t)tile * K.P + r];
      if (!(R.y >> 24)) continue;  // not the first row of its gamma group
      const uint64_t idx = (uint64_t)cb * L.G + R.x;
      const uint64_t msk = 1ull << (idx & 63);
      uint64_t* w = bits + (idx >> 6);
      if (!(*w & msk)) atomicOr((unsigned long long*)w, (unsigned long long)msk);
    }
    for (uint32_t f = 0; f < T.fl_cnt[tile]; ++f) {
      const int m = T.fl_node[(size_t)tile * K.P + f];
      const int jp = m % K.pp, jt = (m / K.pp) % K.pt, js = m / (K.pp * K.pt);
      const SegMid sg = segment_mid(U, U.cone_gamma[q]);
      double x, y, z;
      node_position(sg, U.rad, U.cx[pb], U.cy[pb], U.cz[pb], K.ns[js], K.nt[jt], K.np[jp], x,
                    y, z);
      uint32_t gc;
      const int e = cone_of_point(L, L.cx[cb], L.cy[cb], L.cz[cb], x, y, z, gc);
      if (e) {
        raise_err(err, e);
        return;
      }
      const uint64_t idx = (uint64_t)cb * L.G + gc;
      atomicOr((unsigned long long*)(bits + (idx >> 6)), 1ull << (idx & 63));
    }
  }
}

// ---------------------------------------------------------------- apply
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------ K3 warp GEMM
// A warp owns a unit of <= 8 * kG4Nct parent cones that share gamma (and,
// mostly, the octants of their children) from start to finish: node values
// in its own shared-memory accumulator, children in Morton order, then the
// fit.  No CTA barriers and no work shared between warps, so a warp's stalls
// are its own.  Per child octant and row tile (<= 8 nodes sharing a child
// cone):
//   V[node][cone] = sum_k A[node][k] C_{cone's child, gamma_c}[k]
// with mma.sync.m8n8k4.f64.  K runs over the child block in memory order, 8
// coefficients per chunk: one 256-bit load per lane brings two complex
// coefficients (a quad covers 128 contiguous bytes of one block, so a warp's
// load touches 8 lines for 1 KB -- the 128-bit version touched 8 lines for
// 512 B and was bound by L1 wavefronts), feeding four MMAs (2 K steps x re,
// im).  The loads run PF chunks ahead in a register ring that continues into
// the next row tile.  A (basis products of the lane's node at its own 2
// coefficients per chunk) is formed in registers per row tile: the 25
// theta-phi products once, then a 4-way select by the lane's position in the
// quad -- no table, no memory traffic.
// Measured at C2 (DESIGN.md sections 3 and 9): 8 warps x 2 column tiles is the
// optimum (12 warps x 15 cones at 168 registers, 16 warps x 1 tile, 6 and 4
// warps are all slower); the macros below exist for those sweeps.
#ifndef IFGF_G4_WARPS
#define IFGF_G4_WARPS 8
#endif
#ifndef IFGF_G4_NCT
#define IFGF_G4_NCT 2
#endif
constexpr int kG4Warps = IFGF_G4_WARPS;
constexpr int kG4Nct = IFGF_G4_NCT;       // column tiles (of 8 cones) per warp unit
#ifndef IFGF_G4_CONES
#define IFGF_G4_CONES (8 * IFGF_G4_NCT)
#endif
constexpr int kG4Cones = IFGF_G4_CONES;   // cones per unit (<= 8 * kG4Nct)
constexpr int kG4Cols = 8 * kG4Nct;
#ifndef IFGF_G4_PF
#define IFGF_G4_PF 6   // largest ring depth tried; the ring takes a divisor of the chunk count
#endif

constexpr int g4_prefetch(int nch) {
  for (int pf = IFGF_G4_PF; pf > 1; --pf)
    if (nch % pf == 0) return pf;
  return 1;
}

template <int PS, int PT, int PP>
struct G4Shape {
  static constexpr int P = PS * PT * PP;
  static constexpr size_t per_warp = (size_t)kG4Cones * P * sizeof(double2);
  static constexpr int warps = kG4Warps;
  static constexpr bool ok = P <= 80;  // A fragments and the load ring in registers
};

// a if p else b, as a select (the compiler turns ?: chains of doubles into
// divergent branches)
__device__ __forceinline__ double selp_f64(double a, double b, int p) {
  double d;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(d)
      : "d"(a), "d"(b), "r"(p));
  return d;
}
__device__ __forceinline__ double sel4(int kq, double a, double b, double c, double d) {
  return selp_f64(a, selp_f64(b, selp_f64(c, d, kq == 2), kq == 1), kq == 0);
}

template <int PS, int PT, int PP, bool LAP>
__global__ void __launch_bounds__(kG4Warps * 32, 1)
    k_propagate_wgemm(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                      const __grid_constant__ InterpConsts K, const TilesDev T,
                      const WgRow* __restrict__ rtab, double kappa, uint32_t nunits,
                      const double2* __restrict__ child, const double2* __restrict__ zblock,
                      double2* parent, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  constexpr int P = PS * PT * PP, NCH = (BL::Pst + 7) / 8, PF = g4_prefetch(NCH);
  constexpr bool kTail = (BL::Pst % 8) != 0;  // last chunk reaches past the block
  extern __shared__ double2 smem[];
  __shared__ uint32_t s_q[kG4Warps][kG4Cols];
  __shared__ uint32_t s_cb[kG4Warps][8][kG4Cols];   // child box per octant (kNone: absent)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int kq = lane & 3, nn = lane >> 2;
  double2* acc = smem + (size_t)w * kG4Cones * P;  // [kG4Cones][P] node values
  // chunk cc of the block at p (already offset by the lane's 2 kq coefficients)
  auto bload = [&](const double2* p, int cc) -> double4 {
    if (kTail && cc == NCH - 1) {
      double4 b = make_double4(0.0, 0.0, 0.0, 0.0);
      if (8 * cc + 2 * kq < BL::Pst) b = ldg256(p + 8 * cc);
      return b;
    }
    return ldg256(p + 8 * cc);
  };
  for (uint32_t unit = blockIdx.x * NW + w; unit < nunits; unit += gridDim.x * NW) {
    const uint32_t c0 = T.unit_start[unit], c1 = T.unit_start[unit + 1];
    const int nq = (int)(c1 - c0);
    for (int i = lane; i < kG4Cones * P; i += 32) acc[i] = make_double2(0.0, 0.0);
    uint32_t omask = 0;
    if (lane < kG4Cols) {
      const uint32_t q = lane < nq ? T.usorted[c0 + lane] : kNone;
      s_q[w][lane] = q;
      uint32_t cbo[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) cbo[o] = kNone;
      if (q != kNone) {
        const uint32_t pb = U.cone_box[q];
        for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb) {
          const int o = (int)(L.code[cb] & 7);
          omask |= 1u << o;
#pragma unroll
          for (int oo = 0; oo < 8; ++oo)
            if (oo == o) cbo[oo] = cb;
        }
      }
#pragma unroll
      for (int o = 0; o < 8; ++o) s_cb[w][o][lane] = cbo[o];
    }
    omask = __reduce_or_sync(0xffffffffu, omask);
    const uint32_t tbase = T.cone_gidx[T.usorted[c0]] * 8;
    __syncwarp();
    // The unit's row tiles, octant after octant, as one stream of instances
    // (octant, row tile).  Everything an instance needs from memory is
    // requested ahead of its turn: its child gamma three instances ahead,
    // its cones' bitmap words two ahead (find_cone), its node record and the
    // first kPF block chunks one ahead.
    struct Inst {
      int o;
      uint32_t r, r1;
    };
    auto advance = [&](Inst& it) {  // o = 8: past the end
      ++it.r;
      while (it.o < 8 && it.r >= it.r1) {
        do ++it.o;
        while (it.o < 8 && !((omask >> it.o) & 1u));
        if (it.o < 8) {
          it.r = T.rt_off[tbase + it.o];
          it.r1 = T.rt_off[tbase + it.o + 1];
        }
      }
    };
    // NU column tiles: units of <= 8 cones skip the second tile
    auto run_stream = [&](auto NUc) {
      constexpr int NU = decltype(NUc)::value;
      struct Pend {  // find_cone in flight: bitmap word, rank, bit (64: absent child)
        uint64_t wd;
        uint32_t rk, bit;
      };
      auto lookup = [&](const Inst& it, uint32_t gc, Pend (&pd)[NU]) {
  #pragma unroll
        for (int u = 0; u < NU; ++u) {
          const uint32_t cb = it.o < 8 ? s_cb[w][it.o][u * 8 + nn] : kNone;
          pd[u].wd = 0;
          pd[u].rk = 0;
          pd[u].bit = 64;
          if (cb != kNone) {
            const uint64_t idx = (uint64_t)cb * L.G + gc;
            pd[u].wd = __ldg(&L.bits[idx >> 6]);
            pd[u].rk = __ldg(&L.rank[idx >> 6]);
            pd[u].bit = (uint32_t)(idx & 63);
          }
        }
      };
      auto resolve = [&](const Pend (&pd)[NU], const double2* (&bpo)[NU]) {
  #pragma unroll
        for (int u = 0; u < NU; ++u) {
          const double2* p = zblock;
          if (pd[u].bit < 64) {
            const uint64_t bit = 1ull << pd[u].bit;
            if (pd[u].wd & bit)
              p = child + (size_t)(pd[u].rk + (uint32_t)__popcll(pd[u].wd & (bit - 1))) * BL::Pst;
            else
              raise_err(err, kErrPropCover);
          }
          bpo[u] = p + 2 * kq;
        }
      };
      Inst i0 = {-1, 0, 0};
      advance(i0);
      Inst i1 = i0;
      if (i1.o < 8) advance(i1);
      Inst i2 = i1;
      if (i2.o < 8) advance(i2);
      uint32_t g2 = i2.o < 8 ? __ldg(&T.rt[i2.r].x) : 0;
      const double2* bp[NU];
      double4 bq[PF][NU];
      Pend pd[NU];
      WgRow rec = {0.0, 0.0, 0.0, 0.0, 0.0, -1};
      if (i0.o < 8) {
        lookup(i0, __ldg(&T.rt[i0.r].x), pd);
        rec = rtab[(size_t)i0.r * 8 + nn];
      } else {
        lookup(i0, 0, pd);
      }
      resolve(pd, bp);
  #pragma unroll
      for (int c = 0; c < PF; ++c)
  #pragma unroll
        for (int u = 0; u < NU; ++u) bq[c][u] = bload(bp[u], c);
      lookup(i1, i1.o < 8 ? __ldg(&T.rt[i1.r].x) : 0, pd);
      while (i0.o < 8) {
        // instance i1: its cones are resolved now (requested one instance ago);
        // instance i2: request its bitmap words; instance i3: its child gamma
        const double2* bpn[NU];
        resolve(pd, bpn);
        lookup(i2, g2, pd);
        Inst i3 = i2;
        if (i3.o < 8) advance(i3);
        g2 = i3.o < 8 ? __ldg(&T.rt[i3.r].x) : 0;
        const WgRow recn = rtab[(size_t)(i1.o < 8 ? i1.r : i0.r) * 8 + nn];
        // basis of this lane's node: Ts and the theta-phi products
        double Ts[PS], WP[PT * PP];
        {
          double Tt[PT], Tp[PP];
          cheb_basis<PS>(rec.ts, Ts);
          cheb_basis<PT>(rec.tt, Tt);
          cheb_basis<PP>(rec.tp, Tp);
          if (rec.m < 0) {
  #pragma unroll
            for (int k2 = 0; k2 < PS; ++k2) Ts[k2] = 0.0;
          }
  #pragma unroll
          for (int t = 0; t < PT; ++t)
  #pragma unroll
            for (int p2 = 0; p2 < PP; ++p2) WP[t * PP + p2] = Tt[t] * Tp[p2];
        }
        double dr[NU][2], di[NU][2];
  #pragma unroll
        for (int u = 0; u < NU; ++u) dr[u][0] = dr[u][1] = di[u][0] = di[u][1] = 0.0;
  #pragma unroll
        for (int c = 0; c < NCH; ++c) {
          // A fragments of the chunk: the lane's two coefficients
          double a[2];
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            double wv[4], sv[4];
  #pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
              const int e = 8 * c + 2 * k2 + h;
              const bool real = e < BL::Pst && e % BL::PL < PT * PP;
              wv[k2] = real ? WP[real ? e % BL::PL : 0] : 0.0;
              sv[k2] = real ? Ts[real ? e / BL::PL : 0] : 0.0;
            }
            a[h] = sel4(kq, sv[0], sv[1], sv[2], sv[3]) * sel4(kq, wv[0], wv[1], wv[2], wv[3]);
          }
          double4 b[NU];
  #pragma unroll
          for (int u = 0; u < NU; ++u) b[u] = bq[c % PF][u];
  #pragma unroll
          for (int u = 0; u < NU; ++u) {
            dmma(dr[u][0], dr[u][1], a[0], b[u].x);
            dmma(di[u][0], di[u][1], a[0], b[u].y);
          }
  #pragma unroll
          for (int u = 0; u < NU; ++u) {
            dmma(dr[u][0], dr[u][1], a[1], b[u].z);
            dmma(di[u][0], di[u][1], a[1], b[u].w);
            bq[c % PF][u] = c + PF < NCH ? bload(bp[u], c + PF) : bload(bpn[u], c + PF - NCH);
          }
        }
        // epilogue: D row nn = node m, columns 2 kq + h = cones of the tile
        if (rec.m >= 0) {
          const int m = (int)rec.m;
  #pragma unroll
          for (int u = 0; u < NU; ++u)
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (kG4Cones < kG4Cols && u * 8 + 2 * kq + h >= kG4Cones) continue;
              const double vr = dr[u][h], vi = di[u][h];
              double2* p = acc + (size_t)(u * 8 + 2 * kq + h) * P + m;
              double2 v = *p;
              if (LAP) {
                v.x = fma(vr, rec.tfx, v.x);
                v.y = fma(vi, rec.tfx, v.y);
              } else {
                v.x = fma(vr, rec.tfx, fma(-vi, rec.tfy, v.x));
                v.y = fma(vr, rec.tfy, fma(vi, rec.tfx, v.y));
              }
              *p = v;
            }
        }
        // the next octant's row tiles touch the same (cone, node) slots from other lanes
        if (i1.o != i0.o) __syncwarp();
        i0 = i1;
        i1 = i2;
        i2 = i3;
        rec = recn;
  #pragma unroll
        for (int u = 0; u < NU; ++u) bp[u] = bpn[u];
      }
    };
    if (kG4Nct == 2 && nq <= 8) run_stream(std::integral_constant<int, 1>{});
    else run_stream(std::integral_constant<int, kG4Nct>{});
    __syncwarp();
    // flagged nodes: per-box exact locate + evaluation (rare), after the MMA
    // contributions, octants in Morton order
    for (int o = 0; o < 8; ++o) {
      if (!((omask >> o) & 1u)) continue;
      const uint32_t tile = tbase + (uint32_t)o;
      const size_t f0 = (size_t)tile * P;
      const uint32_t nfl = T.fl_cnt[tile];
      for (uint32_t i = lane; i < nfl * (uint32_t)kG4Cones; i += 32) {
        const int c = (int)(i % kG4Cones);
        const uint32_t cb = s_cb[w][o][c];
        if (cb == kNone) continue;
        const int m = T.fl_node[f0 + i / kG4Cones];
        const uint32_t q = s_q[w][c], pb = U.cone_box[q];
        const int jp = m % PP, jt = (m / PP) % PT, js = m / (PP * PT);
        const SegMid sg = segment_mid(U, U.cone_gamma[q]);
        const double pcx = U.cx[pb], pcy = U.cy[pb], pcz = U.cz[pb];
        double x, y, z;
        node_position(sg, U.rad, pcx, pcy, pcz, K.ns[js], K.nt[jt], K.np[jp], x, y, z);
        const double ux = x - pcx, uy = y - pcy, uz = z - pcz;
        const double rp = sqrt(fma(uz, uz, fma(uy, uy, ux * ux)));
        Loc lo;
        const int e = locate_fast(L, L.cx[cb], L.cy[cb], L.cz[cb], x, y, z, lo);
        if (e) {
          raise_err(err, e);
          continue;
        }
        const uint32_t cq = find_cone(L, cb, lo.gamma);
        if (cq == kNone) {
          raise_err(err, kErrPropCover);
          continue;
        }
        double vr, vi;
        eval_block<PS, PT, PP>(child + (size_t)cq * BL::Pst, lo.ts, lo.tt, lo.tp, vr, vi);
        const double ratio = rp * lo.rinv;
        double sn = 0.0, cn = 1.0;
        if (!LAP) sincos_fast(kappa * (lo.r - rp), sn, cn);
        const double tr = ratio * cn, ti = ratio * sn;
        double2 v = acc[(size_t)c * P + m];
        v.x = fma(vr, tr, fma(-vi, ti, v.x));
        v.y = fma(vr, ti, fma(vi, tr, v.y));
        acc[(size_t)c * P + m] = v;
      }
      __syncwarp();
    }
    fit_cones_inplace<PS, PT, PP>(K, acc, nq, parent, err, s_q[w]);
    __syncwarp();
  }
}

// K3 with register-blocked rows: task = (parent cone, child k, row of <= R
// nodes whose child cone coincides -- box-independent, from the tiles).  The
// thread loads the child block once and evaluates all nodes of the row
// (eval_block_multi), so a coefficient load feeds R FMA chains instead of
// one; the per-node kernel is bound by L1->register bandwidth (16 B per
// 2 FMAs, also for broadcast loads).  Flagged nodes (within the margin of a
// cone boundary) take the exact per-box path.  Each warp works alone on
// `cpw` consecutive parent cones at a time: it walks their children in
// Morton order with a warp barrier in between (every node receives one
// contribution per child, in the reference's child order: deterministic
// sums), then fits them (fit_cones_warp).  No CTA barriers, so load
// imbalance stays within the warp.
template <int PS, int PT, int PP, bool LAP, int R>
__global__ void __launch_bounds__(kRowThreads, IFGF_ROWS_MINB)
    k_propagate_rows(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                     const __grid_constant__ InterpConsts K, const TilesDev T, double kappa,
                     uint32_t qb, uint32_t qe, int cpw, int groups,
                     const double2* __restrict__ child, double2* parent, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  constexpr int P = PS * PT * PP;
  constexpr int NW = kRowThreads / 32;
  extern __shared__ double2 smem[];
  __shared__ uint32_t s_cb0[NW][kRowMaxCpw], s_tile[NW][kRowMaxCpw], s_nrow[NW][kRowMaxCpw],
      s_pre[NW][kRowMaxCpw + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // per warp: sv (cpw * P values), task meta (<= cpw * P tasks)
  double2* sv = smem + (size_t)w * 2 * cpw * P;
  uint2* meta = reinterpret_cast<uint2*>(sv + cpw * P);
  for (int g = 0; g < groups; ++g) {
    const uint32_t q0 = qb + (((uint32_t)g * gridDim.x + blockIdx.x) * NW + w) * cpw;
    if (q0 >= qe) break;
    const int nw = (int)min((uint32_t)cpw, qe - q0);
    for (int i = lane; i < nw * P; i += 32) sv[i] = make_double2(0.0, 0.0);
    uint32_t cb0 = 0, nch = 0, tbase = 0;
    if (lane < nw) {
      const uint32_t q = q0 + lane;
      const uint32_t pb = U.cone_box[q];
      cb0 = U.child_begin[pb];
      nch = U.child_begin[pb + 1] - cb0;
      tbase = T.cone_gidx[q] * 8;
    }
    if (lane < cpw) s_cb0[w][lane] = cb0;
    uint32_t kmax = nch;
#pragma unroll
    for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    for (uint32_t kc = 0; kc < kmax; ++kc) {  // k-th child, ascending Morton order
      uint32_t n = 0, tile = 0, nrow = 0;
      if (lane < nw && kc < nch) {
        const uint32_t cb = cb0 + kc;
        tile = tbase + (uint32_t)(L.code[cb] & 7);
        nrow = T.rw_cnt[tile];
        n = nrow + T.fl_cnt[tile];
      }
      uint32_t incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();  // previous child's readers of s_* are done
      if (lane < cpw) {
        s_tile[w][lane] = tile;
        s_nrow[w][lane] = nrow;
        s_pre[w][lane + 1] = incl;
      }
      if (lane == 0) s_pre[w][0] = 0;
      __syncwarp();
      // phase A: every task's child cone ordinal and row (independent loads
      // across lanes), into shared memory: {cq, c << 24 | cnt << 16 | row},
      // flagged tasks {kFlagTask, c << 24 | index}
      for (uint32_t t = lane; t < total; t += 32) {
        int c = 0;
        while (s_pre[w][c + 1] <= t) ++c;
        const uint32_t tl = s_tile[w][c], loc = t - s_pre[w][c];
        uint2 mt;
        if (loc < s_nrow[w][c]) {
          const uint2 rw = T.rw[(size_t)tl * P + loc];
          mt = make_uint2(find_cone(L, s_cb0[w][c] + kc, rw.x),
                          ((uint32_t)c << 24) | (rw.y & 0xff0000u) | loc);
#if IFGF_ROWS_PFA
          // the whole round's data into L1 before phase B: each child-cone
          // group's block once (its first row), each 16-row run of row data
          if ((rw.y >> 24) & 1u && mt.x != kNone) {
            const char* pf = (const char*)(child + (size_t)mt.x * BL::Pst);
#pragma unroll
            for (int l = 0; l < (BL::Pst * 16 + 127) / 128; ++l)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(pf + 128 * l));
          }
          if ((loc & 15u) == 0) {
            const char* rd = (const char*)(T.rdat + row_field(tl, P, 5 * R, (int)loc, 0));
#pragma unroll
            for (int f = 0; f < 5 * R; ++f) asm volatile("prefetch.global.L1 [%0];" ::"l"(rd + 256 * f));
          }
#endif
        } else {
          mt = make_uint2(kFlagTask, ((uint32_t)c << 24) | (loc - s_nrow[w][c]));
        }
        meta[t] = mt;
      }
      __syncwarp();
      // phase B: evaluate; the next task's block is prefetched into L1 while
      // the current one is evaluated
      for (uint32_t t = lane; t < total; t += 32) {
        const uint2 mt = meta[t];
        const int c = (int)(mt.y >> 24);
        const uint32_t cq = mt.x;
#if IFGF_ROWS_PF >= 1
        if (t + 32 < total) {
          const uint2 mn = meta[t + 32];
          if (mn.x < kFlagTask) {
            const char* pf = (const char*)(child + (size_t)mn.x * BL::Pst);
#pragma unroll
            for (int l = 0; l < (BL::Pst * 16 + 127) / 128; ++l)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(pf + 128 * l));
          }
        }
#endif
        const uint32_t rwy = mt.y;
        const uint32_t tl = s_tile[w][c], cb = s_cb0[w][c] + kc;
        double2* acc = sv + c * P;
        if (cq != kFlagTask) {
          if (cq == kNone) {
            raise_err(err, kErrPropCover);
            continue;
          }
          const int r = (int)(rwy & 0xffffu), cnt = (int)((rwy >> 16) & 0xffu);
          const double* rd = T.rdat + row_field(tl, P, 5 * R, r, 0);
          double ts[R], tt[R], tp[R];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            if (j < cnt) {
              ts[j] = __ldg(rd + 32 * (0 * R + j));
              tt[j] = __ldg(rd + 32 * (1 * R + j));
              tp[j] = __ldg(rd + 32 * (2 * R + j));
            } else {
              ts[j] = tt[j] = tp[j] = 0.0;
            }
          }
          double vr[R], vi[R];
          eval_block_multi<PS, PT, PP, R>(child + (size_t)cq * BL::Pst, ts, tt, tp, vr, vi);
          const uint32_t nodes = __ldg(T.rnode + (size_t)tl * P + r);
#pragma unroll
          for (int j = 0; j < R; ++j) {
            if (j < cnt) {
              const double tr = __ldg(rd + 32 * (3 * R + j)), ti = __ldg(rd + 32 * (4 * R + j));
              const int m = (int)((nodes >> (8 * j)) & 0xffu);
              double2 v = acc[m];
              v.x = fma(vr[j], tr, fma(-vi[j], ti, v.x));
              v.y = fma(vr[j], ti, fma(vi[j], tr, v.y));
              acc[m] = v;
            }
          }
        } else {
          // flagged node: the exact per-box path
          const uint32_t q = q0 + c;
          const int m = T.fl_node[(size_t)tl * P + (mt.y & 0xffffffu)];
          const uint32_t pb = U.cone_box[q];
          const int jp = m % PP, jt = (m / PP) % PT, js = m / (PP * PT);
          const SegMid sg = segment_mid(U, U.cone_gamma[q]);
          const double pcx = U.cx[pb], pcy = U.cy[pb], pcz = U.cz[pb];
          double x, y, z;
          node_position(sg, U.rad, pcx, pcy, pcz, K.ns[js], K.nt[jt], K.np[jp], x, y, z);
          const double ux = x - pcx, uy = y - pcy, uz = z - pcz;
          const double rp = sqrt(fma(uz, uz, fma(uy, uy, ux * ux)));
          Loc lo;
          const int er = locate_fast(L, L.cx[cb], L.cy[cb], L.cz[cb], x, y, z, lo);
          if (er) {
            raise_err(err, er);
            continue;
          }
          const uint32_t cq = find_cone(L, cb, lo.gamma);
          if (cq == kNone) {
            raise_err(err, kErrPropCover);
            continue;
          }
          double vr, vi;
          eval_block<PS, PT, PP>(child + (size_t)cq * BL::Pst, lo.ts, lo.tt, lo.tp, vr, vi);
          const double ratio = rp * lo.rinv;
          double sn = 0.0, cn = 1.0;
          if (!LAP) sincos_fast(kappa * (lo.r - rp), sn, cn);
          const double tr = ratio * cn, ti = ratio * sn;
          double2 v = acc[m];
          v.x = fma(vr, tr, fma(-vi, ti, v.x));
          v.y = fma(vr, ti, fma(vi, tr, v.y));
          acc[m] = v;
        }
      }
      __syncwarp();
    }
    fit_cones_inplace<PS, PT, PP>(K, sv, nw, parent + (size_t)q0 * BL::Pst, err);
    __syncwarp();
  }
}

// K3 rows without precomputed tiles (levels whose parent cones mostly have
// distinct gammas, where tiles would cost more than they save): warp = one
// parent cone at a time.  Per child box the warp locates all P nodes
// (locate_fast, exact fallback near boundaries -- the reference's cone per
// node), groups them by child cone in node order (warp min-reduction +
// ballots) into rows of <= R, and evaluates each row with one block load
// (eval_block_multi).  Children in Morton order, one contribution per node
// and child: deterministic sums.  Then fit_cones_warp on the cone.
template <int P>
struct FlyWarp {
  double2 sv[P], st[P];
  double nx[P], ny[P], nz[P], nrp[P];      // node positions, distance to parent centre
  double ts[P], tt[P], tp[P], tr[P], ti[P];  // per node for the current child
  uint32_t key[P];                         // child gamma (kNone: error)
  uint32_t rkey[P];                        // per row: child gamma
  uint8_t rcnt[P];
  uint8_t rnode[P][4];
};

template <int PS, int PT, int PP, bool LAP, int R>
__global__ void __launch_bounds__(kRowThreads, IFGF_ROWS_MINB)
    k_propagate_fly(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                    const __grid_constant__ InterpConsts K, double kappa, uint32_t qb,
                    uint32_t qe, const double2* __restrict__ child, double2* parent, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  constexpr int P = PS * PT * PP;
  static_assert(R <= 4, "rows hold <= 4 nodes");
  const int NW = blockDim.x >> 5;
  extern __shared__ __align__(16) unsigned char fly_smem[];
  __shared__ double2 trig[kTrigEntries];
  stage_trig(trig, L.trig);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  FlyWarp<P>& F = reinterpret_cast<FlyWarp<P>*>(fly_smem)[w];
  const uint32_t nwarps = gridDim.x * NW;
  for (uint32_t q = qb + blockIdx.x * NW + w; q < qe; q += nwarps) {
    const uint32_t pb = U.cone_box[q];
    const SegMid sg = segment_mid(U, U.cone_gamma[q]);
    const double pcx = U.cx[pb], pcy = U.cy[pb], pcz = U.cz[pb];
    for (int m = lane; m < P; m += 32) {
      const int jp = m % PP, jt = (m / PP) % PT, js = m / (PP * PT);
      double x, y, z;
      node_position(sg, U.rad, pcx, pcy, pcz, K.ns[js], K.nt[jt], K.np[jp], x, y, z);
      const double ux = x - pcx, uy = y - pcy, uz = z - pcz;
      F.nx[m] = x;
      F.ny[m] = y;
      F.nz[m] = z;
      F.nrp[m] = sqrt(fma(uz, uz, fma(uy, uy, ux * ux)));
      F.sv[m] = make_double2(0.0, 0.0);
    }
    __syncwarp();
    for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb) {
      const double cx = L.cx[cb], cy = L.cy[cb], cz = L.cz[cb];
      // a. locate every node in the child box
      for (int m = lane; m < P; m += 32) {
        Loc o;
        const int e = locate_fast(L, trig, cx, cy, cz, F.nx[m], F.ny[m], F.nz[m], o);
        if (e) {
          raise_err(err, e);
          F.key[m] = kNone;
          continue;
        }
        F.key[m] = o.gamma;
        F.ts[m] = o.ts;
        F.tt[m] = o.tt;
        F.tp[m] = o.tp;
        const double rp = F.nrp[m], ratio = rp * o.rinv;
        double sn = 0.0, cn = 1.0;
        if (!LAP) sincos_fast(kappa * (o.r - rp), sn, cn);
        F.tr[m] = ratio * cn;
        F.ti[m] = ratio * sn;
      }
      __syncwarp();
      // b. rows: nodes grouped by child gamma (ascending), node order within
      constexpr int NS = (P + 31) / 32;
      uint32_t k[NS];
      bool done[NS];
#pragma unroll
      for (int sl = 0; sl < NS; ++sl) {
        const int m = lane + 32 * sl;
        k[sl] = m < P ? F.key[m] : kNone;
        done[sl] = k[sl] == kNone;
      }
      int nrows = 0;
      for (;;) {
        uint32_t mn = kNone;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl)
          if (!done[sl]) mn = min(mn, k[sl]);
        mn = __reduce_min_sync(0xffffffffu, mn);
        if (mn == kNone) break;
        int total = 0;
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          const bool mine = !done[sl] && k[sl] == mn;
          const uint32_t bal = __ballot_sync(0xffffffffu, mine);
          if (mine) {
            const int rank = total + __popc(bal & lt);
            const int row = nrows + rank / R;
            F.rnode[row][rank % R] = (uint8_t)(lane + 32 * sl);
            done[sl] = true;
          }
          total += __popc(bal);
        }
        const int nr = (total + R - 1) / R;
        for (int r = lane; r < nr; r += 32) {
          F.rkey[nrows + r] = mn;
          F.rcnt[nrows + r] = (uint8_t)min(R, total - r * R);
        }
        nrows += nr;
      }
      __syncwarp();
      // c. one block load per row
      for (int r = lane; r < nrows; r += 32) {
        const uint32_t cq = find_cone(L, cb, F.rkey[r]);
        if (cq == kNone) {
          raise_err(err, kErrPropCover);
          continue;
        }
        const int cnt = F.rcnt[r];
        double ts[R], tt[R], tp[R];
        int nd[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          nd[j] = j < cnt ? F.rnode[r][j] : 0;
          ts[j] = j < cnt ? F.ts[nd[j]] : 0.0;
          tt[j] = j < cnt ? F.tt[nd[j]] : 0.0;
          tp[j] = j < cnt ? F.tp[nd[j]] : 0.0;
        }
        double vr[R], vi[R];
        eval_block_multi<PS, PT, PP, R>(child + (size_t)cq * BL::Pst, ts, tt, tp, vr, vi);
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j < cnt) {
            const int m = nd[j];
            const double tr = F.tr[m], ti = F.ti[m];
            double2 v = F.sv[m];
            v.x = fma(vr[j], tr, fma(-vi[j], ti, v.x));
            v.y = fma(vr[j], ti, fma(vi[j], tr, v.y));
            F.sv[m] = v;
          }
        }
      }
      __syncwarp();
    }
    fit_cones_inplace<PS, PT, PP>(K, F.sv, 1, parent + (size_t)q * BL::Pst, err);
    __syncwarp();
  }
}

template <class F>
bool dispatch_mma_orders(int ps, int pt, int pp, F&& f) {
#define IFGF_MMA_CASE(a, b, c)          \
  if (ps == a && pt == b && pp == c) {  \
    f(std::integral_constant<int, a>{}, std::integral_constant<int, b>{}, \
      std::integral_constant<int, c>{}); \
    return true;                        \
  }
  IFGF_MMA_CASE(3, 5, 5)
  IFGF_MMA_CASE(4, 6, 6)
  IFGF_MMA_CASE(5, 7, 7)
  IFGF_MMA_CASE(3, 3, 3)
  IFGF_MMA_CASE(4, 4, 4)
#undef IFGF_MMA_CASE
  return false;
}

// Orders served by the tiles and the row kernel: every shipped order triple
// (passes.cu dispatch_orders).
template <class F>
bool dispatch_rows_orders(int ps, int pt, int pp, F&& f) {
#define IFGF_ROWS_CASE(a, b, c)         \
  if (ps == a && pt == b && pp == c) {  \
    f(std::integral_constant<int, a>{}, std::integral_constant<int, b>{}, \
      std::integral_constant<int, c>{}); \
    return true;                        \
  }
  IFGF_ROWS_CASE(3, 5, 5)
  IFGF_ROWS_CASE(4, 6, 6)
  IFGF_ROWS_CASE(5, 7, 7)
  IFGF_ROWS_CASE(1, 1, 1)
  IFGF_ROWS_CASE(2, 2, 2)
  IFGF_ROWS_CASE(3, 3, 3)
  IFGF_ROWS_CASE(4, 4, 4)
  IFGF_ROWS_CASE(2, 3, 3)
  IFGF_ROWS_CASE(3, 4, 4)
#undef IFGF_ROWS_CASE
  return false;
}


}  // namespace

void build_prop_tiles(ifgf_plan* P, int d, void* (*scratch)(void*, size_t), void* sctx) {
  PropTiles& T = P->tiles[d];
  T = PropTiles{};
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  cudaStream_t s = P->s_main;
  if (U.nc == 0 || K.P > 255) return;
  if (!dispatch_rows_orders(K.ps, K.pt, K.pp, [](auto, auto, auto) {})) return;
  if (U.G > (1ull << 28)) return;  // gamma bitmap too large: per-node kernel
  // distinct parent gammas
  const size_t nw = (U.G + 63) / 64;
  uint64_t* gbits = P->alloc<uint64_t>(nw);
  uint32_t* gcnt = P->alloc<uint32_t>(nw + 1);
  uint32_t* grank = P->alloc<uint32_t>(nw + 1);
  IFGF_CUDA(cudaMemsetAsync(gbits, 0, nw * 8, s));
  k_gamma_mark<<<nblk(U.nc), 256, 0, s>>>(U.dev(), gbits);
  k_gamma_popc<<<nblk(nw + 1), 256, 0, s>>>(gbits, nw, gcnt);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, gcnt, grank, (int)(nw + 1), s);
    IFGF_CUDA(cub::DeviceScan::ExclusiveSum(scratch(sctx, tb), tb, gcnt, grank, (int)(nw + 1), s));
  }
  uint32_t ng = 0;
  IFGF_CUDA(cudaMemcpyAsync(&ng, grank + nw, 4, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  // worth it only if a (gamma, octant) tile serves several parent cones
  const double uses = (double)U.nc / ng;
  P->launches += 2;
  static const double min_uses = [] {
    const char* v = std::getenv("IFGF_TILE_MIN_USES");
    return v ? std::atof(v) : 3.0;
  }();
  if (uses < min_uses) return;
  // memory: ~103 B per (gamma, octant, node) entry; above min(8 GB, free / 4)
  // the on-the-fly rows are the better deal (a Laplace or high-kappa coarse
  // level can have millions of distinct gammas)
  {
    const size_t fr = mem_available(P);
    const double rows_bytes = (double)((K.P + 31) / 32 * 32) / K.P * 15.0 * sizeof(double);
    const double bytes = (double)ng * 8.0 * K.P *
                         (rows_bytes + 3 * sizeof(double) + sizeof(double2) +
                          2 * sizeof(uint32_t) + sizeof(uint2) + sizeof(uint16_t) + 1);
    static const double max_gb = [] {
      const char* v = std::getenv("IFGF_TILE_MAX_GB");
      return v ? std::atof(v) : 8.0;
    }();
    if (bytes > std::min(max_gb * (1ull << 30), 0.25 * (double)fr)) return;
  }
  T.ngamma = ng;
  T.cone_gidx = P->alloc<uint32_t>(U.nc);
  T.gamma_of = P->alloc<uint32_t>(ng);
  k_gamma_index<<<nblk(U.nc), 256, 0, s>>>(U.dev(), gbits, grank, T.cone_gidx, T.gamma_of);
  const uint32_t ntiles = ng * 8;
  const size_t ne = (size_t)ntiles * K.P;
  T.e_t = P->alloc<double>(3 * ne);
  T.e_T = P->alloc<double2>(ne);
  T.e_gc = P->alloc<uint32_t>(ne);
  k_tile_entries<<<nblk(ne, 256), 256, 0, s>>>(U.dev(), L.dev(), K, T.gamma_of, ng, P->kappa, T.e_t,
                                          T.e_T, T.e_gc);
  // order, rows of <= row_nodes (IFGF_PROP_ROWS), flagged lists, row-ordered entries
  {
    static const int rn_env = [] {
      const char* v = std::getenv("IFGF_ROWS_R");
      return v ? std::atoi(v) : 0;
    }();
    // nodes per row: register budget of eval_block_multi (~17 doubles per node)
    T.row_nodes = rn_env >= 2 && rn_env <= 3 ? rn_env : (K.P <= 100 ? 3 : 2);
  }
  T.rw_cnt = P->alloc<uint32_t>(ntiles);
  T.fl_cnt = P->alloc<uint32_t>(ntiles);
  T.rw = P->alloc<uint2>(ne);
  T.fl_node = P->alloc<uint16_t>(ne);
  T.e_perm = P->alloc<uint8_t>(ne);
  T.rdat = P->alloc<double>(row_field(ntiles, K.P, 5 * T.row_nodes, 0, 0));
  T.rnode = P->alloc<uint32_t>(ne);
  {
    const unsigned g = nblk((size_t)ntiles * 32, 256);
    auto go = [&](auto kern) {
      kern<<<g, 256, 0, s>>>(ntiles, K.P, T.row_nodes, T.e_gc, T.e_t, T.e_T, T.rw_cnt, T.fl_cnt,
                             T.rw, T.fl_node, T.e_perm, T.rdat,
                             reinterpret_cast<uint8_t*>(T.rnode));
    };
    switch ((K.P + 31) / 32) {
      case 1: go(k_tile_sort<1>); break;
      case 2: go(k_tile_sort<2>); break;
      case 3: go(k_tile_sort<3>); break;
      case 4: go(k_tile_sort<4>); break;
      case 5: go(k_tile_sort<5>); break;
      case 6: go(k_tile_sort<6>); break;
      case 7: go(k_tile_sort<7>); break;
      default: go(k_tile_sort<8>); break;
    }
  }
  IFGF_CUDA(cudaGetLastError());
  P->launches += 1;
  T.enabled = true;
}

void launch_mark_nodes_tiles(ifgf_plan* P, int d, uint64_t* bits) {
  const PropTiles& T = P->tiles[d];
  const Level& U = P->lv[d - 1];
  k_mark_nodes_tiles<<<nblk(U.nc, 128), 128, 0, P->s_main>>>(P->lv[d].dev(), U.dev(), P->K,
                                                             tiles_dev(T), bits, P->err);
  ++P->launches;
}

bool launch_propagation_fly(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, const double2* child,
                            double2* parent, cudaStream_t s) {
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  if (K.P > 255) return false;
  return dispatch_rows_orders(K.ps, K.pt, K.pp, [&](auto A, auto B, auto C) {
    constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
    constexpr int Pn = PS * PT * PP;
    // warps per CTA: kRowThreads / 32, fewer when the per-warp scratch
    // would exceed ~200 KB of shared memory (large orders)
    const int NW = (int)std::max<size_t>(
        1, std::min<size_t>(kRowThreads / 32, 200 * 1024 / sizeof(FlyWarp<Pn>)));
    const size_t sm = NW * sizeof(FlyWarp<Pn>);
    const uint32_t nq = qe - qb;
    const unsigned grid = (unsigned)std::max<size_t>(
        1, std::min<size_t>((nq + NW - 1) / NW, (size_t)148 * 8));
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<grid, NW * 32, sm, s>>>(U.dev(), L.dev(), K, P->kappa, qb, qe, child, parent,
                                     P->err);
    };
    const bool lap = P->kappa == 0.0;
    constexpr int R = Pn <= 100 ? 3 : 2;
    lap ? launch(k_propagate_fly<PS, PT, PP, true, R>)
        : launch(k_propagate_fly<PS, PT, PP, false, R>);
    ++P->launches;
  });
}

// Warp-GEMM tables of child level d, built on first use: row tiles of <= 8
// nodes sharing a child cone (CSR over tiles), one node record per row tile
// slot, the zero block, and the parent cones sorted (stably) by (gamma index,
// child mask) and cut into warp units of <= kG4Cones cones sharing gamma.
// (The build-time scratch stays with the plan: returning it to the pool with
// cudaFreeAsync cost 0.4 ms per C2 plan build.)
void build_wgemm_extras(ifgf_plan* P, int d, cudaStream_t s) {
  PropTiles& T = P->tiles[d];
  const InterpConsts& K = P->K;
  const uint32_t ntiles = T.ngamma * 8;
  uint32_t* rt_cnt = P->alloc<uint32_t>(ntiles + 1);
  uint32_t* fl_cnt = P->alloc<uint32_t>(ntiles + 1);
  IFGF_CUDA(cudaMemsetAsync(rt_cnt + ntiles, 0, 4, s));
  k_tile_rows<<<nblk(ntiles, 64), 64, 0, s>>>(ntiles, K.P, T.e_gc, rt_cnt, fl_cnt, nullptr,
                                              nullptr, nullptr, nullptr, nullptr);
  T.rt_off = P->alloc<uint32_t>(ntiles + 1);
  auto tmp = [&](size_t b) { return (void*)P->alloc<char>(b); };
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, rt_cnt, T.rt_off, (int)(ntiles + 1), s);
    IFGF_CUDA(cub::DeviceScan::ExclusiveSum(tmp(tb), tb, rt_cnt, T.rt_off, (int)(ntiles + 1), s));
  }
  uint32_t nrt = 0;
  IFGF_CUDA(cudaMemcpyAsync(&nrt, T.rt_off + ntiles, 4, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  T.rt = P->alloc<uint4>(nrt + 1);
  uint32_t* rt_tile = P->alloc<uint32_t>(nrt + 1);
  k_tile_rows<<<nblk(ntiles, 64), 64, 0, s>>>(ntiles, K.P, T.e_gc, nullptr, nullptr, T.rt_off,
                                              T.rt, nullptr, nullptr, nullptr, rt_tile);
  T.rtab = P->alloc<char>((size_t)(nrt + 1) * 8 * sizeof(WgRow));
  k_wgemm_rtab<<<nblk((size_t)nrt * 8, 256), 256, 0, s>>>(nrt, K.P, T.rt, rt_tile, T.e_t, T.e_T,
                                                        reinterpret_cast<WgRow*>(T.rtab));
  T.zblock = P->alloc<double2>((size_t)K.Pst + 8);
  IFGF_CUDA(cudaMemsetAsync(T.zblock, 0, ((size_t)K.Pst + 8) * sizeof(double2), s));
  P->launches += 4;
}

// Warp units of the parent cones [qb, qe) of level d - 1 (the whole level, or
// a rank's interval): sorted (stably) by (gamma index, child mask), cut into
// units of <= kG4Cones cones sharing gamma.  A cone's result does not depend
// on the unit it lands in (MMA columns are independent), so a rank plan's
// blocks equal the single-GPU plan's bitwise.
void build_wgemm_units(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, cudaStream_t s) {
  PropTiles& T = P->tiles[d];
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const uint32_t n = qe - qb;
  auto tmp = [&](size_t b) { return (void*)P->alloc<char>(b); };
  // One box group = the whole level (gamma-major order) measured best at C2
  // (d = 8: 5.8 ms against 6.8 ms with 193-box groups sized for L2): longer
  // (gamma, mask) runs fill the units and align their child masks, and the
  // child blocks' re-reads come from DRAM at a rate the kernel does not feel.
  static const int bg_env = [] {
    const char* v = std::getenv("IFGF_G4_BOXGROUP");
    return v ? std::atoi(v) : 0;
  }();
  const uint32_t bg = bg_env > 0 ? (uint32_t)bg_env : std::max<uint32_t>(1, U.nb);
  uint32_t* qidx = P->alloc<uint32_t>(n);
  uint64_t* key = P->alloc<uint64_t>(n);
  uint64_t* gsorted = P->alloc<uint64_t>(n);
  T.usorted = P->alloc<uint32_t>(n);
  {
    k_wgemm_keys<<<nblk(n), 256, 0, s>>>(U.dev(), L.dev(), T.cone_gidx, T.ngamma, bg, qb, qe, key,
                                         qidx);
    size_t tb = 0;
    int bits = 1;
    const uint64_t kmax = (((uint64_t)U.nb / bg + 1) * T.ngamma) << 8;
    while ((1ull << bits) < kmax && bits < 64) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, gsorted, qidx, T.usorted, (int)n, 0, bits,
                                    s);
    IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp(tb), tb, key, gsorted, qidx, T.usorted,
                                              (int)n, 0, bits, s));
  }
  uint32_t* flag = P->alloc<uint32_t>(n + 1);
  uint32_t* pos = P->alloc<uint32_t>(n + 1);
  // units end where (group, gamma) changes; cutting at mask changes as well
  // (IFGF_G4_MASKCUT=1) leaves units of ~6 cones at C2 and is 2-3x slower
  static const bool maskcut = [] {
    const char* v = std::getenv("IFGF_G4_MASKCUT");
    return v && std::atoi(v) != 0;
  }();
  k_chunk_flags<<<nblk(n + 1), 256, 0, s>>>(gsorted, n, kG4Cones, flag, maskcut ? 0 : 8);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, (int)(n + 1), s);
    IFGF_CUDA(cub::DeviceScan::ExclusiveSum(tmp(tb), tb, flag, pos, (int)(n + 1), s));
  }
  uint32_t nu = 0;
  IFGF_CUDA(cudaMemcpyAsync(&nu, pos + n, 4, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  T.nunits = nu;
  T.unit_start = P->alloc<uint32_t>(nu + 1);
  k_chunk_starts<<<nblk(n + 1), 256, 0, s>>>(flag, pos, n, T.unit_start, nu);
  IFGF_CUDA(cudaGetLastError());
  P->launches += 5;
  T.wg_qb = qb;
  T.wg_qe = qe;
  if (std::getenv("IFGF_G4_TRACE"))
    std::fprintf(stderr, "[wgemm] d=%d cones [%u, %u) of %u gammas %u units %u (%.2f cones/unit)\n",
                 d, qb, qe, U.nc, T.ngamma, nu, (double)n / std::max(1u, nu));
}

bool launch_propagation_wgemm(ifgf_plan* P, int d, const double2* child, double2* parent,
                              cudaStream_t s) {
  PropTiles& T = P->tiles[d];
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  bool done = false;
  dispatch_mma_orders(K.ps, K.pt, K.pp, [&](auto A, auto B, auto C) {
    constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
    using S4 = G4Shape<PS, PT, PP>;
    if constexpr (S4::ok) {
      constexpr int NW = S4::warps;
      const size_t sm = S4::per_warp * NW;
      const unsigned grid = (unsigned)std::max<size_t>(
          1, std::min<size_t>((T.nunits + NW - 1) / NW, (size_t)148));
      auto launch = [&](auto kern) {
        IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        kern<<<grid, NW * 32, sm, s>>>(U.dev(), L.dev(), K, tiles_dev(T),
                                       reinterpret_cast<const WgRow*>(T.rtab), P->kappa, T.nunits,
                                       child, T.zblock, parent, P->err);
        IFGF_CUDA(cudaGetLastError());
      };
      P->kappa == 0.0 ? launch(k_propagate_wgemm<PS, PT, PP, true>)
                      : launch(k_propagate_wgemm<PS, PT, PP, false>);
      ++P->launches;
      done = true;
    }
  });
  return done;
}

bool launch_propagation_mma(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, const double2* child,
                            double2* parent, cudaStream_t s) {
  PropTiles& T = P->tiles[d];
  if (P->prop_kernel == IFGF_PROP_FLY || !T.enabled)
    return launch_propagation_fly(P, d, qb, qe, child, parent, s);
  // The warp GEMM runs on the cone range its units were built for -- the
  // first range a plan propagates at this level (the whole level, or a rank
  // plan's interval); other ranges (pass-level API) run the rows kernel.
  // IFGF_PROP_AUTO takes it where enough parent cones share each gamma to
  // fill the units (C2: d = 8, 7, 6 with 12,280 / 1,679 / 216 cones per gamma;
  // d = 5 with 23 stays with the rows: 12 cones per unit, 7.4 ms against 6.8)
  if (P->prop_kernel == IFGF_PROP_DMMA || P->prop_kernel == IFGF_PROP_AUTO) {
    // (the level's totals, not the range's: every rank plan of a group takes
    // the same kernel as the single-GPU plan, so their blocks agree bitwise).
    // IFGF_G4_MIN_SHARE / IFGF_G4_MIN_CONES override the thresholds (tests).
    const char* ev = std::getenv("IFGF_G4_MIN_SHARE");
    const double min_share = ev ? std::atof(ev) : 100.0;
    ev = std::getenv("IFGF_G4_MIN_CONES");
    // several units per resident warp (C1's 44,522-cone level: rows 0.30 ms,
    // warp GEMM 0.36)
    const double min_cones = ev ? std::atof(ev) : 4.0 * 148 * kG4Warps * kG4Cones;
    const double lnc = (double)P->lv[d - 1].nc;
    const bool want = P->prop_kernel == IFGF_PROP_DMMA ||
                      (lnc >= min_share * (double)T.ngamma && lnc >= min_cones);
    bool ok = false;
    dispatch_mma_orders(P->K.ps, P->K.pt, P->K.pp, [&](auto A, auto B, auto C) {
      ok = G4Shape<decltype(A)::value, decltype(B)::value, decltype(C)::value>::ok;
    });
    if (want && ok) {
      if (!T.rtab) build_wgemm_extras(P, d, s);
      if (!T.usorted) build_wgemm_units(P, d, qb, qe, s);
      if (T.wg_qb == qb && T.wg_qe == qe && T.nunits > 0 &&
          launch_propagation_wgemm(P, d, child, parent, s))
        return true;
    }
  }
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  return dispatch_rows_orders(K.ps, K.pt, K.pp, [&](auto A, auto B, auto C) {
    constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
    constexpr int Pn = PS * PT * PP;
    constexpr int NW = kRowThreads / 32;
    static const int cpw_env = [] {
      const char* v = std::getenv("IFGF_ROWS_CPW");
      return v ? std::atoi(v) : 0;
    }();
    // shared memory for sv + task meta: ~64 KB per CTA (the rest of the SRAM is L1)
    const int per_cone = 2 * Pn * (int)sizeof(double2);
    const int cpw_fit = (int)(64 * 1024 / IFGF_ROWS_MINB / per_cone / NW);
    const int cpw = std::max(1, std::min(kRowMaxCpw, cpw_env > 0 ? cpw_env : std::max(1, cpw_fit)));
    const int cpb = NW * cpw;
    const uint32_t nq = qe - qb;
    const int groups = (int)std::min<size_t>(8, std::max<size_t>(1, nq / ((size_t)cpb * 148 * 4)));
    const unsigned grid = (unsigned)((nq + (size_t)cpb * groups - 1) / ((size_t)cpb * groups));
    const size_t sm = (size_t)cpb * per_cone;
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<grid, kRowThreads, sm, s>>>(U.dev(), L.dev(), K, tiles_dev(T), P->kappa, qb, qe, cpw,
                                        groups, child, parent, P->err);
    };
    const bool lap = P->kappa == 0.0;
    if (T.row_nodes == 2)
      lap ? launch(k_propagate_rows<PS, PT, PP, true, 2>) : launch(k_propagate_rows<PS, PT, PP, false, 2>);
    else
      lap ? launch(k_propagate_rows<PS, PT, PP, true, 3>) : launch(k_propagate_rows<PS, PT, PP, false, 3>);
    ++P->launches;
  });
}

}  // namespace ifgf_b200
