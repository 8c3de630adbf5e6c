// propagate_mma.cu -- K3 as batched FP64 tensor-core GEMMs.
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
// With IFGF_PROP_DMMA a warp takes up to kChunk = 8 parent cones that share
// one gamma (cones sorted by gamma) and, octant by octant in Morton order,
// computes V[node][cone] = sum_k B_k(t_node) * C_{child cone}[k] with
// mma.sync.m8n8k4.f64 (k_propagate_gemm).  Same result as the per-node
// evaluation up to rounding (the basis is evaluated at identical t).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "plan.hpp"

namespace ifgf_b200 {
namespace {

constexpr int kChunk = 8;  // IFGF_PROP_DMMA: parent cones per warp (the B / D columns)
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
  const uint32_t* qsorted;
  const uint32_t* chunk_start;
  const uint8_t* e_perm;
  const uint32_t* rw_cnt;   // rows of tile t: rw[t * P + i], i < rw_cnt[t]
  const uint2* rw;
  const double* rdat;
  const uint32_t* rnode;
};

TilesDev tiles_dev(const PropTiles& t) {
  return {t.ngamma,   t.cone_gidx,   t.gamma_of, t.e_t,    t.e_T,  t.e_gc, t.rt_off,
          t.rt,       t.fl_cnt,      t.fl_node,  t.qsorted, t.chunk_start, t.e_perm,
          t.rw_cnt,   t.rw,          t.rdat,     t.rnode};
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
                            const uint32_t* fl_off, uint16_t* fl_node, uint8_t* e_perm) {
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
        if (rt) rt[wr++] = R;
        ++nrt;
        R = make_uint4(cur, 0xffffffffu, 0xffffffffu, 0);
        k = 0;
      }
    }
    if (k) {
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

#ifndef IFGF_GEMM_BOXGROUP
#define IFGF_GEMM_BOXGROUP 32
#endif
constexpr uint32_t kGemmBoxGroup = IFGF_GEMM_BOXGROUP;

__global__ void k_gemm_keys(const __grid_constant__ LevelDev U, const uint32_t* __restrict__ gidx,
                            uint32_t ngamma, uint64_t* key, uint32_t* qidx) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= U.nc) return;
  key[q] = (uint64_t)(U.cone_box[q] / kGemmBoxGroup) * ngamma + gidx[q];
  qidx[q] = q;
}

__global__ void k_chunk_flags(const uint64_t* gsorted, uint32_t n, uint32_t* flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    flag[i] = 0;
    return;
  }
  // chunk starts: every kChunk-th element of each run of equal gamma index
  uint32_t lo = 0, hi = i;
  const uint64_t g = gsorted[i];
  while (lo < hi) {  // run start = lower_bound(g)
    const uint32_t mid = (lo + hi) >> 1;
    if (gsorted[mid] < g) lo = mid + 1;
    else hi = mid;
  }
  flag[i] = ((i - lo) % kChunk == 0) ? 1u : 0u;
}

__global__ void k_chunk_starts(const uint32_t* flag, const uint32_t* pos, uint32_t n,
                               uint32_t* chunk_start, uint32_t nchunks) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) chunk_start[pos[i]] = i;
  if (i == 0) chunk_start[nchunks] = n;
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

// K3 as FP64 tensor-core GEMMs (IFGF_PROP_DMMA).  For one tile (gamma,
// octant) and one of its child-gamma groups, the evaluation of the child
// interpolants at the group's nodes for 8 parent cones that share gamma is
//   V[node][cone] = sum_k A[node][k] C_cone[k],
//   A[node][k]   = T_ks(ts) T_kt(tt) T_kp(tp)   (box-independent),
// C the child cone's complex coefficients, re and im as two
// mma.sync.m8n8k4.f64 that share A and one 16-byte load of B.  A warp owns
// 8 cones (the B / D columns); A fragments are formed in registers from each
// lane's node basis, B fragments come straight from the child blocks, so
// there is no shared-memory staging and no CTA barrier.  K order (GemmK):
// part 1 steps (ks, kt, c), lane k of the quad -> kp = 4c + k; part 2 packs
// the remaining kp >= 4 floor(PP/4) over (kp, ks, kt), four per step.  The
// dense contraction does 2 (PS PT PP + pad) FMA per node and cone (160 at
// (3,5,5), against 186 for the separable scalar evaluation).
template <int PS, int PT, int PP>
struct GemmK {
  static constexpr int NC = PP / 4;           // full kp chunks of 4
  static constexpr int PPF = 4 * NC;
  static constexpr int N1 = PS * PT * NC;      // part-1 steps
  static constexpr int N2R = (PP - PPF) * PS * PT;
  static constexpr int N2 = (N2R + 3) / 4;     // part-2 steps
  static constexpr int NS = N1 + N2;           // K steps of 4
  static constexpr int P = PS * PT * PP;
  // warps per CTA: node values of 8 cones + one cone of fit scratch per warp
  static constexpr int NW = (200 * 1024) / (9 * P * 16) >= 4 ? 4
                          : ((200 * 1024) / (9 * P * 16) < 1 ? 1 : (200 * 1024) / (9 * P * 16));
  static constexpr size_t smem = (size_t)NW * 9 * P * sizeof(double2);
};

// Coefficient (device block offset, or -1 for a pad entry) of K step st,
// quad lane k (GemmK order).
template <int PS, int PT, int PP>
__host__ __device__ __forceinline__ int gemm_koff(int st, int k, int& ks, int& kt, int& kp) {
  using G = GemmK<PS, PT, PP>;
  constexpr int PL = BlockLayout<PS, PT, PP>::PL;
  if (st < G::N1) {
    const int c = st % G::NC, pair = st / G::NC;
    ks = pair / PT;
    kt = pair % PT;
    kp = 4 * c + k;
  } else {
    const int p = 4 * (st - G::N1) + k;
    if (p >= G::N2R) return -1;
    const int e = p / (PS * PT), pr = p % (PS * PT);
    ks = pr / PT;
    kt = pr % PT;
    kp = G::PPF + e;
  }
  return ks * PL + kt * PP + kp;
}

#ifndef IFGF_GEMM_RB
#define IFGF_GEMM_RB 2
#endif
constexpr int kGemmRB = IFGF_GEMM_RB;  // row tiles per batch (one B load feeds 2 RB MMAs)
#ifndef IFGF_GEMM_KS
#define IFGF_GEMM_KS 1
#endif
constexpr int kGemmKS = IFGF_GEMM_KS;  // accumulator sets (MMA chains split over K)
constexpr int kGemmMaxRt = 16;      // row tiles per tile resolved ahead (more: resolved in the loop)
constexpr int kGemmMaxGroups = 16;  // child-gamma groups per tile resolved ahead

template <int PS, int PT, int PP, bool LAP>
__global__ void __launch_bounds__(GemmK<PS, PT, PP>::NW * 32)
    k_propagate_gemm(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                     const __grid_constant__ InterpConsts K, const TilesDev T, double kappa,
                     uint32_t nchunks, const double2* __restrict__ child, double2* parent,
                     int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  using G = GemmK<PS, PT, PP>;
  constexpr int P = G::P, PL = BL::PL, NW = G::NW;
  extern __shared__ double2 smem[];
  __shared__ double sM[PP * PP + PT * PT + PS * PS];
  __shared__ uint32_t s_q[NW][8];
  __shared__ uint32_t s_cb[NW][8][8];
  __shared__ uint4 s_rt[NW][8][kGemmMaxRt];             // row tiles of each octant's tile
  __shared__ uint32_t s_cq[NW][8][kGemmMaxGroups][8];   // child cone per (octant, group, cone)
  __shared__ uint32_t s_off[NW][9];
  stage_fit_matrices<PS, PT, PP>(K, sM);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t ch = blockIdx.x * NW + w;
  if (ch >= nchunks) return;
  const uint32_t c0 = T.chunk_start[ch], c1 = T.chunk_start[ch + 1];
  const int nq = (int)(c1 - c0);
  double2* acc = smem + (size_t)w * 9 * P;
  double2* scr = acc + 8 * P;
  for (int i = lane; i < 8 * P; i += 32) acc[i] = make_double2(0.0, 0.0);
  const uint32_t q0 = T.qsorted[c0];
  const uint32_t gi = T.cone_gidx[q0];
  if (lane < 8) {
    const uint32_t q = lane < nq ? T.qsorted[c0 + lane] : kNone;
    s_q[w][lane] = q;
    uint32_t cbo[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) cbo[o] = kNone;
    if (q != kNone) {
      const uint32_t pb = U.cone_box[q];
      for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb) {
        const int o = (int)(L.code[cb] & 7);
#pragma unroll
        for (int oo = 0; oo < 8; ++oo)
          if (oo == o) cbo[oo] = cb;
      }
    }
#pragma unroll
    for (int o = 0; o < 8; ++o) s_cb[w][lane][o] = cbo[o];
  }
  if (lane < 9) s_off[w][lane] = T.rt_off[gi * 8 + lane];
  __syncwarp();
  // phase A1: the row tiles of all eight tiles (independent loads)
#pragma unroll
  for (int i = 0; i < 8 * kGemmMaxRt / 32; ++i) {
    const int t = lane + 32 * i, o = t / kGemmMaxRt, rel = t % kGemmMaxRt;
    if (s_off[w][o] + rel < s_off[w][o + 1]) s_rt[w][o][rel] = T.rt[s_off[w][o] + rel];
  }
  __syncwarp();
  // phase A2: every (octant, cone) walks its tile's groups: child cone
  // ordinals into s_cq, the blocks prefetched into L2
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = lane + 32 * i, o = t >> 3, c = t & 7;
    const uint32_t cb = s_cb[w][c][o];
    const int n = (int)min(s_off[w][o + 1] - s_off[w][o], (uint32_t)kGemmMaxRt);
    int gidx = 0;
    for (int rel = 0; rel < n && gidx < kGemmMaxGroups; ++gidx) {
      const uint4 R = s_rt[w][o][rel];
      uint32_t cq = kNone;
      if (cb != kNone) {
        cq = find_cone(L, cb, R.x);
        if (cq != kNone) {
          const char* pf = (const char*)(child + (size_t)cq * BL::Pst);
#pragma unroll
          for (int l = 0; l < (BL::Pst * 16 + 127) / 128; ++l)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + 128 * l));
        } else {
          raise_err(err, kErrPropCover);
        }
      }
      s_cq[w][o][gidx][c] = cq;
      rel += (int)max(R.w, 1u);
    }
  }
  __syncwarp();
  const int kq = lane & 3, nn = lane >> 2;  // A/D row (node slot) = nn; B row k = kq, column = nn
  for (int o = 0; o < 8; ++o) {
    const uint32_t cbn = s_cb[w][nn][o];  // child box of this lane's B column cone
    if (!__any_sync(0xffffffffu, cbn != kNone)) continue;
    const uint32_t tile = gi * 8 + (uint32_t)o;
    const uint32_t r0 = s_off[w][o], r1 = s_off[w][o + 1];
    int gidx = 0;
    for (uint32_t ga = r0; ga < r1; ++gidx) {
      // group [ga, gb): row tiles sharing one child gamma
      const uint32_t rel = ga - r0;
      const uint4 RG = rel < kGemmMaxRt ? s_rt[w][o][rel] : T.rt[ga];
      const uint32_t gb = ga + max(RG.w, 1u);
      const double2* bb = child;  // unresolved column: any finite block (ignored)
      if (cbn != kNone) {
        uint32_t cq;
        if (rel < kGemmMaxRt && gidx < kGemmMaxGroups) {
          cq = s_cq[w][o][gidx][nn];
        } else {
          cq = find_cone(L, cbn, RG.x);
          if (cq == kNone) raise_err(err, kErrPropCover);
        }
        if (cq != kNone) bb = child + (size_t)cq * BL::Pst;
      }
      for (uint32_t rb = ga; rb < gb; rb += kGemmRB) {
        const int nrb = (int)min(gb - rb, (uint32_t)kGemmRB);
        double Ts[kGemmRB][PS], Tt[kGemmRB][PT], Tp[kGemmRB][PP], TpL[kGemmRB][G::NC + 1];
        int m[kGemmRB];
        // kGemmKS accumulator sets over alternating K steps: independent MMA chains
        double dr[kGemmKS][kGemmRB][2], di[kGemmKS][kGemmRB][2];
#pragma unroll
        for (int j = 0; j < kGemmRB; ++j) {
          const uint32_t rj = rb + j - r0;
          m[j] = j < nrb ? rt_node(rj < kGemmMaxRt ? s_rt[w][o][rj] : T.rt[rb + j], nn) : 0xff;
          double ts = 0.0, tt = 0.0, tp = 0.0;
          if (m[j] != 0xff) {
            const double* tv = T.e_t + ((size_t)tile * P + m[j]) * 3;
            ts = tv[0];
            tt = tv[1];
            tp = tv[2];
          }
          cheb_basis<PS>(ts, Ts[j]);
          cheb_basis<PT>(tt, Tt[j]);
          cheb_basis<PP>(tp, Tp[j]);
#pragma unroll
          for (int k2 = 0; k2 < PS; ++k2)
            if (m[j] == 0xff) Ts[j][k2] = 0.0;  // empty node slot: zero row of A
#pragma unroll
          for (int c = 0; c < G::NC; ++c) {
            double v = Tp[j][4 * c];
#pragma unroll
            for (int kk = 1; kk < 4; ++kk)
              if (kq == kk) v = Tp[j][4 * c + kk];
            TpL[j][c] = v;
          }
#pragma unroll
          for (int u = 0; u < kGemmKS; ++u) dr[u][j][0] = dr[u][j][1] = di[u][j][0] = di[u][j][1] = 0.0;
        }
        // part 1: (ks, kt, c), lane kp = 4c + kq; A formed in registers
#pragma unroll
        for (int ks = 0; ks < PS; ++ks)
#pragma unroll
          for (int kt = 0; kt < PT; ++kt)
#pragma unroll
            for (int c = 0; c < G::NC; ++c) {
              const double2 b = __ldg(bb + ks * PL + kt * PP + 4 * c + kq);
#pragma unroll
              for (int j = 0; j < kGemmRB; ++j)
                if (j < nrb) {
                  const double a = Ts[j][ks] * Tt[j][kt] * TpL[j][c];
                  const int u = ((ks * PT + kt) * G::NC + c) % kGemmKS;
                  dmma(dr[u][j][0], dr[u][j][1], a, b.x);
                  dmma(di[u][j][0], di[u][j][1], a, b.y);
                }
            }
        // part 2: entries p = 4g + kq over (kp >= PPF, ks, kt); pad entries
        // (A = 0) read coefficient 0 (finite, contributes exactly 0)
#pragma unroll
        for (int st = G::N1; st < G::NS; ++st) {
          int ks, kt, kp, off = 0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int o2 = gemm_koff<PS, PT, PP>(st, kk, ks, kt, kp);
            if (kq == kk && o2 >= 0) off = o2;
          }
          const double2 b = __ldg(bb + off);
#pragma unroll
          for (int j = 0; j < kGemmRB; ++j)
            if (j < nrb) {
              double a = 0.0;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                if (gemm_koff<PS, PT, PP>(st, kk, ks, kt, kp) >= 0) {
                  const double v = Ts[j][ks] * Tt[j][kt] * Tp[j][kp];
                  if (kq == kk) a = v;
                }
              }
              const int u = st % kGemmKS;
              dmma(dr[u][j][0], dr[u][j][1], a, b.x);
              dmma(di[u][j][0], di[u][j][1], a, b.y);
            }
        }
#pragma unroll
        for (int u = 1; u < kGemmKS; ++u)
#pragma unroll
          for (int j = 0; j < kGemmRB; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              dr[0][j][h] += dr[u][j][h];
              di[0][j][h] += di[u][j][h];
            }
        // epilogue: D row nn = node m[j], columns 2 kq + h = cones
#pragma unroll
        for (int j = 0; j < kGemmRB; ++j) {
          if (j < nrb && m[j] != 0xff) {
            const double2 Tf = __ldg(&T.e_T[(size_t)tile * P + m[j]]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cn = 2 * kq + h;
              if (s_cb[w][cn][o] != kNone) {
                double2 v = acc[cn * P + m[j]];
                if (LAP) {
                  v.x = fma(dr[0][j][h], Tf.x, v.x);
                  v.y = fma(di[0][j][h], Tf.x, v.y);
                } else {
                  v.x = fma(dr[0][j][h], Tf.x, fma(-di[0][j][h], Tf.y, v.x));
                  v.y = fma(dr[0][j][h], Tf.y, fma(di[0][j][h], Tf.x, v.y));
                }
                acc[cn * P + m[j]] = v;
              }
            }
          }
        }
      }
      ga = gb;
    }
    // flagged nodes: per-box exact locate + evaluation (rare); lanes over
    // (flagged node, cone)
    const size_t f0 = (size_t)tile * P;
    const uint32_t nfl = T.fl_cnt[tile];
    for (uint32_t i = lane; i < nfl * 8u; i += 32) {
      const int c = (int)(i & 7u);
      const uint32_t cb = s_cb[w][c][o];
      if (cb == kNone) continue;
      const int m = T.fl_node[f0 + (i >> 3)];
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
      double2 v = acc[c * P + m];
      v.x = fma(vr, tr, fma(-vi, ti, v.x));
      v.y = fma(vr, ti, fma(vi, tr, v.y));
      acc[c * P + m] = v;
    }
    __syncwarp();
  }
  for (int c = 0; c < nq; ++c) {  // one cone at a time: one cone of scratch per warp
    fit_cones_warp<PS, PT, PP>(sM, acc + c * P, scr, 1, parent, err, &s_q[w][c]);
    __syncwarp();
  }
}

// K3 per node with the tile geometry: thread = (parent cone, lane j); for
// child octant o the lane takes the j-th node of tile (gamma, o) in child-cone
// order, so neighbouring lanes read the same child block (broadcast loads --
// the per-node evaluation is L1-throughput bound when lanes diverge).  The
// (child gamma, t, transfer) entry replaces locate + node trigonometry +
// sincos; flagged entries take the per-box exact path.  Node sums live in
// shared memory; octants are processed in Morton order with a CTA barrier in
// between, which keeps the reference's child summation order.
template <int PS, int PT, int PP, bool LAP>
__global__ void __launch_bounds__(320, 2)
    k_propagate_tab(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                    const __grid_constant__ InterpConsts K, const TilesDev T, double kappa,
                    uint32_t qb, uint32_t qe, int cpb, int groups,
                    const double2* __restrict__ child, double2* parent, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  constexpr int P = PS * PT * PP;
  extern __shared__ double2 smem[];
  double2* sv = smem;
  double2* st = smem + cpb * P;
  __shared__ uint32_t cfirst[16], cnum[16];
  __shared__ int kmax_s;
  const int c = threadIdx.x / P, j = threadIdx.x % P;
  for (int g = 0; g < groups; ++g) {
    const uint32_t q0 = qb + ((uint32_t)g * gridDim.x + blockIdx.x) * cpb;
    if (q0 >= qe) break;
    const int ncon = (int)min((uint32_t)cpb, qe - q0);
    if (threadIdx.x < cpb) {
      const int cc = threadIdx.x;
      cfirst[cc] = 0;
      cnum[cc] = 0;
      if (cc < ncon) {
        const uint32_t pb = U.cone_box[q0 + cc];
        cfirst[cc] = U.child_begin[pb];
        cnum[cc] = U.child_begin[pb + 1] - U.child_begin[pb];
      }
    }
    for (int i = threadIdx.x; i < cpb * P; i += blockDim.x) sv[i] = make_double2(0.0, 0.0);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t k = 0;
      for (int cc = 0; cc < ncon; ++cc) k = max(k, cnum[cc]);
      kmax_s = (int)k;
    }
    __syncthreads();
    const bool active = c < ncon;
    const uint32_t q = q0 + c;
    const size_t tbase = active ? (size_t)T.cone_gidx[q] * 8 : 0;
    const int kmax = kmax_s;
    for (int kc = 0; kc < kmax; ++kc) {  // k-th child, ascending Morton order
      const uint32_t cb = (active && (uint32_t)kc < cnum[c]) ? cfirst[c] + kc : kNone;
      if (cb != kNone) {
        const size_t tile = tbase + (L.code[cb] & 7);
        const int m = T.e_perm[tile * P + j];
        const size_t e = tile * P + m;
        const uint32_t gc = T.e_gc[e];
        double ts, tt, tp, tr, ti;
        uint32_t cq;
        bool ok = true;
        if (!(gc & kFlag)) {
          cq = find_cone(L, cb, gc);
          ts = T.e_t[3 * e];
          tt = T.e_t[3 * e + 1];
          tp = T.e_t[3 * e + 2];
          const double2 Tf = T.e_T[e];
          tr = Tf.x;
          ti = Tf.y;
        } else {
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
            ok = false;
          }
          cq = ok ? find_cone(L, cb, lo.gamma) : kNone;
          ts = lo.ts;
          tt = lo.tt;
          tp = lo.tp;
          const double ratio = rp * lo.rinv;
          double sn = 0.0, cn = 1.0;
          if (!LAP && ok) sincos_fast(kappa * (lo.r - rp), sn, cn);
          tr = ratio * cn;
          ti = ratio * sn;
        }
        if (ok && cq == kNone) {
          raise_err(err, kErrPropCover);
          ok = false;
        }
        if (ok) {
          double vr, vi;
          eval_block<PS, PT, PP>(child + (size_t)cq * BL::Pst, ts, tt, tp, vr, vi);
          double2 v = sv[c * P + m];
          v.x = fma(vr, tr, fma(-vi, ti, v.x));
          v.y = fma(vr, ti, fma(vi, tr, v.y));
          sv[c * P + m] = v;
        }
      }
      __syncthreads();
    }
    fit_cones<PS, PT, PP>(K, sv, st, ncon, parent + (size_t)q0 * BL::Pst, err);
    __syncthreads();
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
  __shared__ double sM[PP * PP + PT * PT + PS * PS];
  stage_fit_matrices<PS, PT, PP>(K, sM);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // per warp: sv, st (cpw * P values each), task meta (<= cpw * P tasks)
  double2* sv = smem + (size_t)w * 3 * cpw * P;
  double2* st = sv + cpw * P;
  uint2* meta = reinterpret_cast<uint2*>(st + cpw * P);
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
    fit_cones_warp<PS, PT, PP>(sM, sv, st, nw, parent + (size_t)q0 * BL::Pst, err);
    __syncwarp();
  }
}

// K3 pipelined (IFGF_PROP_PIPE): warp-specialised CTA, one per SM.  Work
// unit = <= kPpCh consecutive parent cones of one parent box (same
// children); a stage = (unit, child), held in a ring of kPpStages
// shared-memory buffers.
//   producer warp: per stage, TMA bulk copies (cp.async.bulk + mbarrier
//     transaction counts) of everything the stage reads that does not
//     depend on the child blocks: each cone's tile rows (first 32-row chunk
//     of local coordinates and transfer factors, the row list, the node map,
//     row and flagged counts) and the child box's cone bitmap.  It never
//     waits on what it copies, so it runs stages ahead.
//   consumer warps, software-pipelined one stage apart:
//     A(i+1): the rows' child cones from the staged bitmap, one shared slot
//       per distinct cone (atomicCAS table), TMA copies of those blocks;
//     B(i):   every row evaluated from shared memory only (eval_block_multi
//       over LDS; ~47 of 64 DFMA/clk/SM measured for 3-node rows), the
//       contributions added to the unit's node values, then the stage is
//       released; after a unit's last child its cones are fitted.
// The block copies of stage i+1 thus land while stage i is evaluated.  Named
// barriers order the consumer phases; every node gets one contribution per
// child, in child order: the sums of k_propagate_rows, bitwise.  Rows past
// the first 32 of a tile, cones beyond the slot capacity and bitmaps wider
// than kPpBitWords fall back to global memory; flagged nodes take the exact
// per-box path.
#ifndef IFGF_PP_CH
#define IFGF_PP_CH 11
#endif
#ifndef IFGF_PP_STAGES
#define IFGF_PP_STAGES 3
#endif
constexpr int kPpCh = IFGF_PP_CH;          // parent cones per unit (<= 18: unit records)
constexpr int kPpConsumers = IFGF_PP_CH;   // one consumer warp per unit cone
constexpr int kPpThreads = (kPpConsumers + 1) * 32;
constexpr int kPpStages = IFGF_PP_STAGES;
static_assert(kPpCh <= 18, "unit records hold 18 cones");
constexpr int kPpBitWords = 72;   // staged bitmap words per child box
constexpr int kPpTab = 2048;      // child cones covered by the slot table
constexpr uint32_t kPpEmpty = 0xffffffffu, kPpPending = 0xfffffffeu;
constexpr uint32_t kPpGlobal = 0xffu;

__device__ __forceinline__ void pp_mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
               "r"(count));
}
__device__ __forceinline__ void pp_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(m))
               : "memory");
}
__device__ __forceinline__ void pp_wait(uint64_t* m, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile(
      "{\n .reg .pred p;\n"
      "PPW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PPW;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// expected bytes are added before each copy is issued, so the transaction
// count never goes negative; the phase completes at the producer's final
// arrive once every copy has landed
__device__ __forceinline__ void pp_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(m)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m))
      : "memory");
}

// Units of <= ch consecutive cones of one parent box, the box's cones split
// evenly: unit_start[u] .. unit_start[u + 1].
__global__ void k_pp_units_count(const __grid_constant__ LevelDev U, uint32_t ch, uint32_t* cnt) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > U.nb) return;
  cnt[b] = b == U.nb ? 0u : (U.box_cone[b + 1] - U.box_cone[b] + ch - 1) / ch;
}
__global__ void k_pp_units_fill(const __grid_constant__ LevelDev U, uint32_t ch, const uint32_t* off,
                                uint32_t* ustart, uint32_t* nunits) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= U.nb) {
    if (b == U.nb) {
      ustart[off[b]] = U.nc;
      *nunits = off[b];
    }
    return;
  }
  const uint32_t q0 = U.box_cone[b], n = U.box_cone[b + 1] - q0;
  const uint32_t parts = (n + ch - 1) / ch;
  for (uint32_t j = 0; j < parts; ++j)
    ustart[off[b] + j] = q0 + (uint32_t)(((uint64_t)j * n) / parts);
}

// Per-unit record for the producer (32 words, one coalesced load per unit):
// [0] q0, [1] ncon, [2] first child, [3] children, [4] child octants (3 bits
// each), [5 .. 5+nch] the children's first cone ordinals (box_cone), [14 ..
// 14+ncon) the cones' gamma indices (ncon <= 18).
constexpr int kPpRec = 32;
// Optional record order (IFGF_PP_ORDER=1): units sorted by their first
// cone's gamma (stable in box order), so CTAs working at the same time on
// the same gamma range of neighbouring boxes share the (gamma, octant) tiles
// in L2.
__global__ void k_pp_units_keys(const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ ustart,
                                const uint32_t* __restrict__ nunits, uint32_t umax, uint32_t* key,
                                uint32_t* id) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= umax) return;
  key[u] = u < *nunits ? gidx[ustart[u]] : 0xffffffffu;
  id[u] = u;
}
__global__ void k_pp_units_info(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                                const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ ustart,
                                const uint32_t* __restrict__ nunits, const uint32_t* __restrict__ order,
                                uint32_t* rec) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *nunits) return;
  const uint32_t u = order ? order[v] : v;
  uint32_t* o = rec + (size_t)v * kPpRec;
  const uint32_t q0 = ustart[u], ncon = ustart[u + 1] - q0;
  const uint32_t pb = U.cone_box[q0];
  const uint32_t cb0 = U.child_begin[pb], nch = U.child_begin[pb + 1] - cb0;
  uint32_t octs = 0;
  for (uint32_t k = 0; k < nch; ++k) octs |= (uint32_t)(L.code[cb0 + k] & 7) << (3 * k);
  o[0] = q0;
  o[1] = ncon;
  o[2] = cb0;
  o[3] = nch;
  o[4] = octs;
  for (uint32_t k = 0; k <= nch; ++k) o[5 + k] = L.box_cone[cb0 + k];
  for (uint32_t c = 0; c < ncon; ++c) o[14 + c] = gidx[q0 + c];
}

template <int PS, int PT, int PP, int R>
struct PipeShape {
  static constexpr int P = PS * PT * PP;
  static constexpr int Pst = BlockLayout<PS, PT, PP>::Pst;
  static constexpr int NF = 5 * R;              // row fields
  static constexpr int RowBytes = NF * 32 * 8;  // one 32-row chunk
  static constexpr int RwBytes = 32 * 8 + 16;   // 32 row entries + alignment slack
  static constexpr int NodeBytes = 32 * 4 + 16;
  static constexpr int CntBytes = 32;           // rw_cnt and fl_cnt words, 16 B each
  static constexpr int BitBytes = kPpBitWords * 8 + 16, RankBytes = kPpBitWords * 4 + 16;
  static constexpr int NB = P <= 80 ? 12 : 4;   // block slots per stage
  static constexpr int MaxTask = kPpCh * P;
  static constexpr int off_row = 0;
  static constexpr int off_rw = off_row + kPpCh * RowBytes;
  static constexpr int off_node = off_rw + kPpCh * RwBytes;
  static constexpr int off_cnt = off_node + kPpCh * NodeBytes;
  static constexpr int off_bits = off_cnt + kPpCh * CntBytes;
  static constexpr int off_rank = off_bits + BitBytes;
  static constexpr int off_blk = (off_rank + RankBytes + 15) / 16 * 16;
  static constexpr int off_task = off_blk + NB * Pst * 16;
  static constexpr int off_cq = (off_task + MaxTask + 15) / 16 * 16;  // u8 slots, then u32 cones
  static constexpr int stage_bytes = ((off_cq + MaxTask * 4) + 127) / 128 * 128;
  static constexpr size_t smem = (size_t)kPpStages * stage_bytes  // stages
                                 + (size_t)kPpCh * P * 16          // sv
                                 + (size_t)kPpTab * 4;             // slot table
  static constexpr bool fits = RowBytes >= P * 16;  // fit scratch in the cone's row chunk
};

struct PipeHdr {
  uint32_t q0, ncon, cb, cbase, ncb, last, nwd, sbm;
  uint64_t w0;
  uint32_t tile[kPpCh], rwoff[kPpCh], nodeoff[kPpCh], rcoff[kPpCh], fcoff[kPpCh];
  uint32_t bitoff, rankoff;
  // consumers
  uint32_t nslot;
};

// 16-byte-aligned window [lo, lo + size) covering [p, p + bytes)
__device__ __forceinline__ const void* pp_window(const void* p, uint32_t bytes, uint32_t& off,
                                                 uint32_t& size) {
  const uintptr_t a = (uintptr_t)p, lo = a & ~(uintptr_t)15;
  off = (uint32_t)(a - lo);
  size = (off + bytes + 15) & ~15u;
  return (const void*)lo;
}

template <int PS, int PT, int PP, bool LAP, int R>
__global__ void __launch_bounds__(kPpThreads, 1)
    k_propagate_pipe(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                     const __grid_constant__ InterpConsts K, const TilesDev T, double kappa,
                     const uint32_t* __restrict__ ustart, const uint32_t* __restrict__ nunits,
                     const uint32_t* __restrict__ urec, const double2* __restrict__ child,
                     double2* parent, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  using SH = PipeShape<PS, PT, PP, R>;
  constexpr int P = SH::P;
  constexpr uint32_t kBlkBytes = BL::Pst * 16;
  extern __shared__ __align__(128) unsigned char pp_smem[];
  double2* sv = reinterpret_cast<double2*>(pp_smem + (size_t)kPpStages * SH::stage_bytes);
  uint32_t* tab = reinterpret_cast<uint32_t*>(sv + kPpCh * P);
  __shared__ PipeHdr hdr[kPpStages];
  __shared__ __align__(8) uint64_t full[kPpStages], blk[kPpStages], empty[kPpStages];
  __shared__ double sM[PP * PP + PT * PT + PS * PS];
  stage_fit_matrices<PS, PT, PP>(K, sM);
  for (int i = threadIdx.x; i < kPpTab; i += blockDim.x) tab[i] = kPpEmpty;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPpStages; ++i) {
      pp_mbar_init(&full[i], 1);
      pp_mbar_init(&blk[i], kPpConsumers);
      pp_mbar_init(&empty[i], kPpConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nu = *nunits;
  if (w == kPpConsumers) {
    // ------------------------------------------------------------ producer
    // unit records loaded one unit ahead; per stage no global loads, only
    // the copies
    uint32_t it = 0;
    uint32_t rnext = blockIdx.x < nu ? urec[(size_t)blockIdx.x * kPpRec + lane] : 0u;
    for (uint32_t u = blockIdx.x; u < nu; u += gridDim.x) {
      const uint32_t rec = rnext;
      if (u + gridDim.x < nu) rnext = urec[(size_t)(u + gridDim.x) * kPpRec + lane];
      const uint32_t q0 = __shfl_sync(0xffffffffu, rec, 0), ncon = __shfl_sync(0xffffffffu, rec, 1);
      const uint32_t cb0 = __shfl_sync(0xffffffffu, rec, 2), nch = __shfl_sync(0xffffffffu, rec, 3);
      const uint32_t octs = __shfl_sync(0xffffffffu, rec, 4);
      const uint32_t gid = __shfl_sync(0xffffffffu, rec, 14 + min(lane, kPpCh - 1));
      for (uint32_t kc = 0; kc < nch; ++kc, ++it) {
        const int st = (int)(it % kPpStages);
        const uint32_t round = it / kPpStages;
        const uint32_t cbase = __shfl_sync(0xffffffffu, rec, 5 + kc);
        const uint32_t cend = __shfl_sync(0xffffffffu, rec, 6 + kc);
        if (round > 0) pp_wait(&empty[st], (round - 1) & 1u);
        unsigned char* sb = pp_smem + (size_t)st * SH::stage_bytes;
        PipeHdr& H = hdr[st];
        const uint32_t cb = cb0 + kc;
        const uint32_t oct = (octs >> (3 * kc)) & 7u;
        if ((uint32_t)lane < ncon) {
          const uint32_t tile = gid * 8 + oct;
          H.tile[lane] = tile;
          uint32_t off, size;
          pp_bulk(sb + SH::off_row + lane * SH::RowBytes, T.rdat + row_field(tile, P, SH::NF, 0, 0),
                  SH::RowBytes, &full[st]);
          const void* src = pp_window(T.rw + (size_t)tile * P, 32 * 8, off, size);
          pp_bulk(sb + SH::off_rw + lane * SH::RwBytes, src, size, &full[st]);
          H.rwoff[lane] = off;
          src = pp_window(T.rnode + (size_t)tile * P, 32 * 4, off, size);
          pp_bulk(sb + SH::off_node + lane * SH::NodeBytes, src, size, &full[st]);
          H.nodeoff[lane] = off;
          src = pp_window(T.rw_cnt + tile, 4, off, size);
          pp_bulk(sb + SH::off_cnt + lane * SH::CntBytes, src, 16, &full[st]);
          H.rcoff[lane] = off;
          src = pp_window(T.fl_cnt + tile, 4, off, size);
          pp_bulk(sb + SH::off_cnt + lane * SH::CntBytes + 16, src, 16, &full[st]);
          H.fcoff[lane] = off;
        }
        if (lane == 0) {
          const uint64_t i0 = (uint64_t)cb * L.G, i1 = i0 + L.G;
          const uint64_t w0 = i0 >> 6, nwd = ((i1 - 1) >> 6) - w0 + 1;
          H.q0 = q0;
          H.ncon = ncon;
          H.cb = cb;
          H.nslot = 0;
          H.cbase = cbase;
          H.ncb = cend - cbase;
          H.last = kc + 1 == nch;
          H.w0 = w0;
          H.nwd = (uint32_t)nwd;
          H.sbm = nwd <= (uint64_t)kPpBitWords;
          if (H.sbm) {
            uint32_t off, size;
            const void* src = pp_window(L.bits + w0, (uint32_t)nwd * 8, off, size);
            pp_bulk(sb + SH::off_bits, src, size, &full[st]);
            H.bitoff = off;
            src = pp_window(L.rank + w0, (uint32_t)nwd * 4, off, size);
            pp_bulk(sb + SH::off_rank, src, size, &full[st]);
            H.rankoff = off;
          }
        }
        __syncwarp();
        if (lane == 0) pp_arrive(&full[st]);
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  // consumer warp w owns cone w of every unit: it alone writes sv[w], so the
  // warps need no barrier among themselves -- they meet only at the stage
  // mbarriers (blocks staged by all eight, stage released by all eight).
  static_assert(kPpConsumers == kPpCh, "one consumer warp per unit cone");
  const uint32_t c = (uint32_t)w;
  double2* acc = sv + (size_t)c * P;
  // A(i): this cone's rows of stage i -> child cones, one slot per distinct
  // cone (tagged table entries: tag = stage sequence, no clearing), copies
  auto phaseA = [&](uint32_t i) {
    const int st = (int)(i % kPpStages);
    pp_wait(&full[st], (i / kPpStages) & 1u);
    unsigned char* sb = pp_smem + (size_t)st * SH::stage_bytes;
    PipeHdr& H = hdr[st];
    if (c < H.ncon) {
      const unsigned char* cw = sb + SH::off_cnt + c * SH::CntBytes;
      const uint32_t nrow = *reinterpret_cast<const uint32_t*>(cw + H.rcoff[c]);
      const uint32_t cb = H.cb, cbase = H.cbase;
      const bool use_tab = H.ncb <= (uint32_t)kPpTab;
      const uint32_t tag = (i & 0x7fffffu) << 9;
      uint8_t* tslot = sb + SH::off_task + c * P;
      uint32_t* tcq = reinterpret_cast<uint32_t*>(sb + SH::off_cq) + c * P;
      for (uint32_t r0 = 0; r0 < nrow; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint32_t cq = kNone;
        if (r < nrow) {
          const uint2 rw = r < 32 ? *reinterpret_cast<const uint2*>(sb + SH::off_rw + c * SH::RwBytes +
                                                                     H.rwoff[c] + 8 * r)
                                  : T.rw[(size_t)H.tile[c] * P + r];
          if (H.sbm) {
            const uint64_t idx = (uint64_t)cb * L.G + rw.x;
            const uint32_t wi = (uint32_t)((idx >> 6) - H.w0);
            const uint64_t wd = *reinterpret_cast<const uint64_t*>(sb + SH::off_bits + H.bitoff + 8 * wi);
            const uint32_t rk = *reinterpret_cast<const uint32_t*>(sb + SH::off_rank + H.rankoff + 4 * wi);
            const uint64_t bit = 1ull << (idx & 63);
            cq = (wd & bit) ? rk + (uint32_t)__popcll(wd & (bit - 1)) : kNone;
          } else {
            cq = find_cone(L, cb, rw.x);
          }
        }
        // one claim per distinct cone of the warp; the leader resolves it
        const unsigned grp = __match_any_sync(0xffffffffu, cq);
        const int leader = __ffs(grp) - 1;
        uint32_t slot = kPpGlobal;
        if (leader == lane && cq != kNone && use_tab) {
          uint32_t* e = tab + (cq - cbase);
          for (;;) {
            const uint32_t old = *(volatile uint32_t*)e;
            if ((old & ~0x1ffu) == tag) {  // this stage's entry
              if (old & 0x100u) continue;   // claimed, slot not yet written
              slot = old & 0xffu;
              break;
            }
            if (atomicCAS(e, old, tag | 0x100u) == old) {
              const uint32_t sl = atomicAdd(&H.nslot, 1u);
              if (sl < (uint32_t)SH::NB) {
                pp_bulk(sb + SH::off_blk + sl * kBlkBytes, child + (size_t)cq * BL::Pst, kBlkBytes,
                        &blk[st]);
                slot = sl;
              }
              __threadfence_block();
              atomicExch(e, tag | slot);
              break;
            }
          }
        }
        slot = __shfl_sync(0xffffffffu, slot, leader);
        if (r < nrow) {
          tslot[r] = (uint8_t)slot;
          tcq[r] = cq;
        }
      }
    }
    __syncwarp();
    if (lane == 0) pp_arrive(&blk[st]);
  };
  // B(i): evaluate this cone's rows of stage i, release the stage; returns
  // whether it ended a unit (the cone is then fitted)
  auto phaseB = [&](uint32_t i) -> bool {
    const int st = (int)(i % kPpStages);
    pp_wait(&blk[st], (i / kPpStages) & 1u);
    const unsigned char* sb = pp_smem + (size_t)st * SH::stage_bytes;
    const PipeHdr& H = hdr[st];
    const bool last = H.last;
    const uint32_t q0 = H.q0, ncon = H.ncon, cb = H.cb;
    if (c < ncon) {
      const unsigned char* cw = sb + SH::off_cnt + c * SH::CntBytes;
      const uint32_t nrow = *reinterpret_cast<const uint32_t*>(cw + H.rcoff[c]);
      const uint32_t nfl = *reinterpret_cast<const uint32_t*>(cw + 16 + H.fcoff[c]);
      const uint32_t tl = H.tile[c];
      const uint8_t* tslot = sb + SH::off_task + c * P;
      const uint32_t* tcq = reinterpret_cast<const uint32_t*>(sb + SH::off_cq) + c * P;
      for (uint32_t r = lane; r < nrow; r += 32) {
        const uint32_t cq = tcq[r];
        if (cq == kNone) {
          raise_err(err, kErrPropCover);
          continue;
        }
        const uint32_t slot = tslot[r];
        double rv[SH::NF];
        uint32_t nodes;
        if (r < 32) {
          const double* rd = reinterpret_cast<const double*>(sb + SH::off_row + c * SH::RowBytes) + r;
#pragma unroll
          for (int f = 0; f < SH::NF; ++f) rv[f] = rd[32 * f];
          nodes = *reinterpret_cast<const uint32_t*>(sb + SH::off_node + c * SH::NodeBytes +
                                                     H.nodeoff[c] + 4 * r);
        } else {
          const double* rd = T.rdat + row_field(tl, P, SH::NF, (int)r, 0);
#pragma unroll
          for (int f = 0; f < SH::NF; ++f) rv[f] = __ldg(rd + 32 * f);
          nodes = __ldg(T.rnode + (size_t)tl * P + r);
        }
        const uint2 rw = r < 32 ? *reinterpret_cast<const uint2*>(sb + SH::off_rw + c * SH::RwBytes +
                                                                   H.rwoff[c] + 8 * r)
                                : T.rw[(size_t)tl * P + r];
        const int cnt = (int)((rw.y >> 16) & 0xffu);
        double ts[R], tt[R], tp[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const bool on = j < cnt;
          ts[j] = on ? rv[0 * R + j] : 0.0;
          tt[j] = on ? rv[1 * R + j] : 0.0;
          tp[j] = on ? rv[2 * R + j] : 0.0;
        }
        double vr[R], vi[R];
        if (slot != kPpGlobal)
          eval_block_multi<PS, PT, PP, R, true>(
              reinterpret_cast<const double2*>(sb + SH::off_blk + slot * kBlkBytes), ts, tt, tp, vr, vi);
        else
          eval_block_multi<PS, PT, PP, R>(child + (size_t)cq * BL::Pst, ts, tt, tp, vr, vi);
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j < cnt) {
            const double tr = rv[3 * R + j], ti = rv[4 * R + j];
            const int m = (int)((nodes >> (8 * j)) & 0xffu);
            double2 v = acc[m];
            v.x = fma(vr[j], tr, fma(-vi[j], ti, v.x));
            v.y = fma(vr[j], ti, fma(vi[j], tr, v.y));
            acc[m] = v;
          }
        }
      }
      // flagged nodes of this cone: the exact per-box path
      const uint32_t q = q0 + c;
      for (uint32_t f = lane; f < nfl; f += 32) {
        const uint32_t pb = U.cone_box[q];
        const int m = T.fl_node[(size_t)tl * P + f];
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
    if (last && c < ncon) {
      // scratch: this cone's (consumed) row chunk of the stage; the generic
      // writes are fenced against the producer's next bulk copies into it
      double2* sf = reinterpret_cast<double2*>(const_cast<unsigned char*>(sb) + SH::off_row +
                                               c * SH::RowBytes);
      fit_cones_warp<PS, PT, PP>(sM, acc, sf, 1, parent + (size_t)(q0 + c) * BL::Pst, err);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    if (lane == 0) pp_arrive(&empty[st]);
    if (last)
      for (int k = lane; k < P; k += 32) acc[k] = make_double2(0.0, 0.0);
    __syncwarp();
    return last;
  };
  uint32_t nstage = 0;
  for (uint32_t u = blockIdx.x; u < nu; u += gridDim.x) nstage += urec[(size_t)u * kPpRec + 3];
  for (int k = lane; k < P; k += 32) acc[k] = make_double2(0.0, 0.0);
  __syncwarp();
  if (nstage) phaseA(0);
  for (uint32_t i = 0; i < nstage; ++i) {
    if (i + 1 < nstage) phaseA(i + 1);
    phaseB(i);
  }
}


// K3 streaming (IFGF_PROP_STREAM, an option; measured slower than rows): the child block stays in
// registers while the nodes that fall into it stream past.  A child cone of
// a parent box collects ~25 nodes of each parent cone (the child's cone
// grid is 2x coarser per axis), so a block loaded once serves a whole run
// of rows instead of one row of <= 3 nodes: the rows kernel moves 1,248 B
// from L1 into registers for every 3 evaluations and saturates the L1 data
// path at ~35 % of the FP64 pipe.
//
// Warp = cpw parent cones, children in Morton order.  Lanes 0..29 form ten
// groups of PS = 3; lane a of a group holds s-plane a of the current child
// block (PT*PP complex coefficients in registers).  A child round's rows
// (the tiles' rows of every owned cone, in cone then row order) are
// concatenated and their nodes split evenly over the groups; a group walks
// its node span, reloading its plane only where the child cone changes.
// Per node every lane of the group contracts its plane (phi then theta),
// weights it by T_a(ts), and the three partials are summed on the group's
// first lane ((a0 + a1) + a2), which applies the transfer factor and adds
// the contribution to the node's slot in shared memory.  Each slot gets one
// contribution per child, children in order: deterministic sums.  Flagged
// nodes (exact per-box path) follow each round, one lane each.
// Node record of a streaming round (48 B): local coordinates, transfer
// factor, child cone ordinal, accumulator slot (cone * P + node).
struct SNode {
  double t[3];
  double tr, ti;
  uint32_t cq, slot;
};
// shared memory per warp and owned parent cone, in double2 units of P:
// sv + st (P each) + P node records (3 double2 each)
constexpr int kStreamSmem = 5;

template <int PS, int PT, int PP>
struct StreamShape {
  static constexpr int NG = 32 / PS;              // lane groups per warp
  static constexpr int NR = PT * PP;              // complex coefficients per plane
  static constexpr bool ok = PS <= 4 && NR <= 25;  // plane fits in registers
};

template <int PS, int PT, int PP, bool LAP, int R>
__global__ void __launch_bounds__(kRowThreads, IFGF_ROWS_MINB)
    k_propagate_stream(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                       const __grid_constant__ InterpConsts K, const TilesDev T, double kappa,
                       uint32_t qb, uint32_t qe, int cpw, int groups,
                       const double2* __restrict__ child, double2* parent, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  using SS = StreamShape<PS, PT, PP>;
  constexpr int P = PS * PT * PP;
  constexpr int NW = kRowThreads / 32;
  constexpr int NR = SS::NR;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ double2 smem[];
  __shared__ uint32_t s_cb0[NW][kRowMaxCpw], s_tile[NW][kRowMaxCpw], s_nrow[NW][kRowMaxCpw],
      s_nfl[NW][kRowMaxCpw], s_pre[NW][kRowMaxCpw + 1], s_fpre[NW][kRowMaxCpw + 1];
  __shared__ double sM[PP * PP + PT * PT + PS * PS];
  stage_fit_matrices<PS, PT, PP>(K, sM);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = lane / PS, pa = lane - grp * PS;  // group, plane
  const int lead = grp * PS;
  const bool in_grp = grp < SS::NG;
  double2* sv = smem + (size_t)w * kStreamSmem * cpw * P;
  double2* st = sv + cpw * P;
  SNode* nd = reinterpret_cast<SNode*>(st + cpw * P);  // the round's nodes
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
    for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(FULL, kmax, o));
    for (uint32_t kc = 0; kc < kmax; ++kc) {  // k-th child, ascending Morton order
      uint32_t nrow = 0, nfl = 0, tile = 0;
      if (lane < nw && kc < nch) {
        const uint32_t cb = cb0 + kc;
        tile = tbase + (uint32_t)(L.code[cb] & 7);
        nrow = T.rw_cnt[tile];
        nfl = T.fl_cnt[tile];
      }
      uint32_t incl = nrow, fincl = nfl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, o), f = __shfl_up_sync(FULL, fincl, o);
        if (lane >= o) {
          incl += v;
          fincl += f;
        }
      }
      const uint32_t rtot = __shfl_sync(FULL, incl, 31), ftot = __shfl_sync(FULL, fincl, 31);
      __syncwarp();  // previous round's readers of s_* / meta are done
      if (lane < cpw) {
        s_tile[w][lane] = tile;
        s_nrow[w][lane] = nrow;
        s_nfl[w][lane] = nfl;
        s_pre[w][lane + 1] = incl;
        s_fpre[w][lane + 1] = fincl;
      }
      if (lane == 0) s_pre[w][0] = s_fpre[w][0] = 0;
      __syncwarp();
      // phase A: rows -> per-node records in shared memory, node order
      // (lanes = rows: coalesced reads of the tiles' 32-row SoA chunks)
      uint32_t carry = 0;
      for (uint32_t t0 = 0; t0 < rtot; t0 += 32) {
        const uint32_t t = t0 + lane;
        uint32_t cnt = 0, c = 0, loc = 0, tl = 0;
        uint2 rw = make_uint2(0, 0);
        if (t < rtot) {
          while (s_pre[w][c + 1] <= t) ++c;
          tl = s_tile[w][c];
          loc = t - s_pre[w][c];
          rw = T.rw[(size_t)tl * P + loc];
          cnt = (rw.y >> 16) & 0xffu;
        }
        uint32_t ci = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(FULL, ci, o);
          if (lane >= o) ci += v;
        }
        if (t < rtot) {
          const uint32_t n0 = carry + ci - cnt;
          const uint32_t cq = find_cone(L, s_cb0[w][c] + kc, rw.x);
          const double* rd = T.rdat + row_field(tl, P, 5 * R, (int)loc, 0);
          const uint32_t nodes = __ldg(T.rnode + (size_t)tl * P + loc);
#pragma unroll
          for (int j = 0; j < R; ++j)
            if (j < (int)cnt) {
              SNode& sn = nd[n0 + j];
              sn.t[0] = __ldg(rd + 32 * (0 * R + j));
              sn.t[1] = __ldg(rd + 32 * (1 * R + j));
              sn.t[2] = __ldg(rd + 32 * (2 * R + j));
              sn.tr = __ldg(rd + 32 * (3 * R + j));
              sn.ti = __ldg(rd + 32 * (4 * R + j));
              sn.cq = cq;
              sn.slot = c * P + ((nodes >> (8 * j)) & 0xffu);
            }
        }
        carry += __shfl_sync(FULL, ci, 31);
      }
      __syncwarp();
      // phase B: the groups split the round's nodes evenly
      const uint32_t ntot = carry;
      const uint32_t per = (ntot + SS::NG - 1) / SS::NG;
      const uint32_t n_lo = in_grp ? min(ntot, (uint32_t)grp * per) : ntot;
      const uint32_t n_hi = in_grp ? min(ntot, n_lo + per) : ntot;
      uint32_t cur = kNone;  // child cone ordinal held in registers
      double pr[NR], pi[NR];
      for (uint32_t it = 0; it < per; ++it) {
        const uint32_t n = n_lo + it;
        const bool act = n < n_hi;
        const SNode* sn = nd + (act ? n : 0);
        const uint32_t cq = act ? sn->cq : kNone;
        if (act && cq == kNone && pa == 0) raise_err(err, kErrPropCover);
        const bool ev = act && cq != kNone;
        if (ev && cq != cur) {  // load plane pa of the child block
          const double2* plane = child + (size_t)cq * BL::Pst + pa * BL::PL;
#pragma unroll
          for (int q = 0; q < BL::PL / 2; ++q) {
            const double4 v = ldg256(plane + 2 * q);
            if (2 * q < NR) {
              pr[2 * q] = v.x;
              pi[2 * q] = v.y;
            }
            if (2 * q + 1 < NR) {
              pr[2 * q + 1] = v.z;
              pi[2 * q + 1] = v.w;
            }
          }
          cur = cq;
        }
        double vr = 0.0, vi = 0.0;
        if (ev) {
          const double ts = sn->t[0], tt = sn->t[1], tp = sn->t[2];
          double Tt[PT], Tp[PP];
          cheb_basis<PT>(tt, Tt);
          cheb_basis<PP>(tp, Tp);
          double cr = 0.0, ci = 0.0;
#pragma unroll
          for (int b = 0; b < PT; ++b) {
            double rr = pr[b * PP], ri = pi[b * PP];
#pragma unroll
            for (int k = 1; k < PP; ++k) {
              rr = fma(pr[b * PP + k], Tp[k], rr);
              ri = fma(pi[b * PP + k], Tp[k], ri);
            }
            if (b == 0) {
              cr = rr;
              ci = ri;
            } else {
              cr = fma(rr, Tt[b], cr);
              ci = fma(ri, Tt[b], ci);
            }
          }
          // T_a(ts), the reference's recurrence
          double Ta = 1.0, Tm = 1.0;
#pragma unroll
          for (int k = 1; k < PS; ++k) {
            const double Tn = k == 1 ? ts : fma(2.0 * ts, Ta, -Tm);
            Tm = Ta;
            Ta = k <= pa ? Tn : Ta;
          }
          vr = cr * Ta;
          vi = ci * Ta;
        }
        // group sum on the first lane: ((a0 + a1) + a2)
#pragma unroll
        for (int k = 1; k < PS; ++k) {
          const int src = min(lead + k, 31);
          const double ur = __shfl_sync(FULL, vr, src), ui = __shfl_sync(FULL, vi, src);
          if (pa == 0) {
            vr += ur;
            vi += ui;
          }
        }
        if (ev && pa == 0) {
          const double tr = sn->tr, ti = sn->ti;
          double2* acc = sv + sn->slot;
          double2 v = *acc;
          v.x = fma(vr, tr, fma(-vi, ti, v.x));
          v.y = fma(vr, ti, fma(vi, tr, v.y));
          *acc = v;
        }
      }
      // flagged nodes: the exact per-box path, one lane each
      for (uint32_t f = lane; f < ftot; f += 32) {
        int c = 0;
        while (s_fpre[w][c + 1] <= f) ++c;
        const uint32_t tl = s_tile[w][c], cb = s_cb0[w][c] + kc;
        const uint32_t q = q0 + c;
        const int m = T.fl_node[(size_t)tl * P + (f - s_fpre[w][c])];
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
        double2* acc = sv + c * P;
        double2 v = acc[m];
        v.x = fma(vr, tr, fma(-vi, ti, v.x));
        v.y = fma(vr, ti, fma(vi, tr, v.y));
        acc[m] = v;
      }
      __syncwarp();
    }
    fit_cones_warp<PS, PT, PP>(sM, sv, st, nw, parent + (size_t)q0 * BL::Pst, err);
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
  __shared__ double sM[PP * PP + PT * PT + PS * PS];
  stage_trig(trig, L.trig);
  stage_fit_matrices<PS, PT, PP>(K, sM);
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
        int below = 0, total = 0;
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
    fit_cones_warp<PS, PT, PP>(sM, F.sv, F.st, 1, parent + (size_t)q * BL::Pst, err);
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
    size_t fr = 0, tot = 0;
    IFGF_CUDA(cudaMemGetInfo(&fr, &tot));
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

// Row tiles of 8 and gamma-sorted cone chunks for IFGF_PROP_DMMA, built on
// first use (the default kernels do not need them).
void build_dmma_extras(ifgf_plan* P, int d, cudaStream_t s) {
  PropTiles& T = P->tiles[d];
  const Level& U = P->lv[d - 1];
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
  k_tile_rows<<<nblk(ntiles, 64), 64, 0, s>>>(ntiles, K.P, T.e_gc, nullptr, nullptr, T.rt_off,
                                              T.rt, nullptr, nullptr, nullptr);
  // parent cones sorted (stably) by (group of kGemmBoxGroup consecutive parent
  // boxes, gamma index) -> chunks of <= kChunk cones sharing gamma.  Box
  // groups keep the child blocks that neighbouring gammas share in L2 (gamma
  // order alone re-reads them from DRAM: 10 GB per C2 launch).
  uint32_t* qidx = P->alloc<uint32_t>(U.nc);
  uint64_t* key = P->alloc<uint64_t>(U.nc);
  uint64_t* gsorted = P->alloc<uint64_t>(U.nc);
  T.qsorted = P->alloc<uint32_t>(U.nc);
  {
    k_gemm_keys<<<nblk(U.nc), 256, 0, s>>>(U.dev(), T.cone_gidx, T.ngamma, key, qidx);
    size_t tb = 0;
    int bits = 1;
    const uint64_t kmax = ((uint64_t)U.nb / kGemmBoxGroup + 1) * T.ngamma;
    while ((1ull << bits) < kmax && bits < 64) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, gsorted, qidx, T.qsorted, (int)U.nc, 0,
                                    bits, s);
    IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp(tb), tb, key, gsorted, qidx, T.qsorted,
                                              (int)U.nc, 0, bits, s));
    IFGF_CUDA(cudaStreamSynchronize(s));
  }
  uint32_t* flag = P->alloc<uint32_t>(U.nc + 1);
  uint32_t* pos = P->alloc<uint32_t>(U.nc + 1);
  k_chunk_flags<<<nblk(U.nc + 1), 256, 0, s>>>(gsorted, U.nc, flag);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, (int)(U.nc + 1), s);
    IFGF_CUDA(cub::DeviceScan::ExclusiveSum(tmp(tb), tb, flag, pos, (int)(U.nc + 1), s));
  }
  uint32_t nch = 0;
  IFGF_CUDA(cudaMemcpyAsync(&nch, pos + U.nc, 4, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  T.nchunks = nch;
  T.chunk_start = P->alloc<uint32_t>(nch + 1);
  k_chunk_starts<<<nblk(U.nc + 1), 256, 0, s>>>(flag, pos, U.nc, T.chunk_start, nch);
  IFGF_CUDA(cudaGetLastError());
  P->launches += 5;
}

bool launch_propagation_mma(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, const double2* child,
                            double2* parent, cudaStream_t s) {
  PropTiles& T = P->tiles[d];
  if (P->prop_kernel == IFGF_PROP_FLY ||
      ((P->prop_kernel == IFGF_PROP_ROWS || P->prop_kernel == IFGF_PROP_STREAM ||
        P->prop_kernel == IFGF_PROP_PIPE) &&
       !T.enabled))
    return launch_propagation_fly(P, d, qb, qe, child, parent, s);
  if (!T.enabled) return false;
  if (P->prop_kernel == IFGF_PROP_DMMA && !T.rt) build_dmma_extras(P, d, s);
  if (T.nchunks == 0 && P->prop_kernel == IFGF_PROP_DMMA) return false;
  const bool full = qb == 0 && qe == P->lv[d - 1].nc;
  bool piped = false;
  if (P->prop_kernel == IFGF_PROP_PIPE && full &&
      dispatch_rows_orders(P->K.ps, P->K.pt, P->K.pp, [&](auto A, auto B, auto C) {
        constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
        // orders whose stages do not fit in shared memory run the rows kernel
        constexpr size_t kMaxSmem = 220 * 1024;
        if constexpr (PipeShape<PS, PT, PP, 2>::smem > kMaxSmem ||
                      PipeShape<PS, PT, PP, 3>::smem > kMaxSmem ||
                      !PipeShape<PS, PT, PP, 2>::fits || !PipeShape<PS, PT, PP, 3>::fits) {
          return;
        } else {
        const Level& U = P->lv[d - 1];
        const Level& L = P->lv[d];
        if (!T.ustart) {  // units, built on first use (device only, no host sync)
          uint32_t* cnt = P->alloc<uint32_t>(U.nb + 1);
          uint32_t* off = P->alloc<uint32_t>(U.nb + 1);
          T.ustart = P->alloc<uint32_t>((size_t)U.nc / kPpCh + U.nb + 2);
          T.nunits = P->alloc<uint32_t>(1);
          k_pp_units_count<<<nblk(U.nb + 1), 256, 0, s>>>(U.dev(), kPpCh, cnt);
          size_t tb = 0;
          cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(U.nb + 1), s);
          void* tmp = P->alloc<unsigned char>(tb);
          IFGF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)(U.nb + 1), s));
          k_pp_units_fill<<<nblk(U.nb + 1), 256, 0, s>>>(U.dev(), kPpCh, off, T.ustart, T.nunits);
          const size_t umax = (size_t)U.nc / kPpCh + U.nb + 1;
          T.urec = P->alloc<uint32_t>(umax * kPpRec);
          static const int by_gamma = [] {
            // 1: units by first gamma (measured 40.7 ms at C2 vs 39.3 in box order:
            // the child blocks then miss L2 more than the tiles gain)
            const char* v = std::getenv("IFGF_PP_ORDER");
            return v ? std::atoi(v) : 0;
          }();
          uint32_t* order = nullptr;
          if (by_gamma) {
            uint32_t* key = P->alloc<uint32_t>(umax);
            uint32_t* key2 = P->alloc<uint32_t>(umax);
            uint32_t* id = P->alloc<uint32_t>(umax);
            order = P->alloc<uint32_t>(umax);
            k_pp_units_keys<<<nblk(umax), 256, 0, s>>>(T.cone_gidx, T.ustart, T.nunits,
                                                       (uint32_t)umax, key, id);
            size_t tb2 = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb2, key, key2, id, order, (int)umax, 0, 32, s);
            void* tmp2 = P->alloc<unsigned char>(tb2);
            IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, tb2, key, key2, id, order, (int)umax, 0,
                                                      32, s));
            P->launches += 1;
          }
          k_pp_units_info<<<nblk(umax), 256, 0, s>>>(U.dev(), L.dev(), T.cone_gidx, T.ustart,
                                                     T.nunits, order, T.urec);
          IFGF_CUDA(cudaGetLastError());
          P->launches += 3;
        }
        auto launch = [&](auto kern, size_t sm) {
          IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          kern<<<148, kPpThreads, sm, s>>>(U.dev(), L.dev(), P->K, tiles_dev(T), P->kappa, T.ustart,
                                           T.nunits, T.urec, child, parent, P->err);
          IFGF_CUDA(cudaGetLastError());
        };
        const bool lap = P->kappa == 0.0;
        if (T.row_nodes == 2) {
          const size_t sm = PipeShape<PS, PT, PP, 2>::smem;
          lap ? launch(k_propagate_pipe<PS, PT, PP, true, 2>, sm)
              : launch(k_propagate_pipe<PS, PT, PP, false, 2>, sm);
        } else {
          const size_t sm = PipeShape<PS, PT, PP, 3>::smem;
          lap ? launch(k_propagate_pipe<PS, PT, PP, true, 3>, sm)
              : launch(k_propagate_pipe<PS, PT, PP, false, 3>, sm);
        }
        ++P->launches;
        piped = true;
        }
      }) &&
      piped)
    return true;
  if (P->prop_kernel == IFGF_PROP_ROWS || P->prop_kernel == IFGF_PROP_STREAM ||
      P->prop_kernel == IFGF_PROP_PIPE) {
    const Level& U = P->lv[d - 1];
    const Level& L = P->lv[d];
    const InterpConsts& K = P->K;
    return dispatch_rows_orders(K.ps, K.pt, K.pp, [&](auto A, auto B, auto C) {
      constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
      constexpr int Pn = PS * PT * PP;
      // orders whose planes do not fit in registers run the rows kernel
      const bool stream = P->prop_kernel == IFGF_PROP_STREAM && StreamShape<PS, PT, PP>::ok;
      constexpr int NW = kRowThreads / 32;
      static const int cpw_env = [] {
        const char* v = std::getenv("IFGF_ROWS_CPW");
        return v ? std::atoi(v) : 0;
      }();
      // shared memory for sv + st + task meta: ~96 KB per CTA (the rest of the SRAM is L1)
      // stream: sv + st + node records, ~150 KB per CTA
      const int per_cone = (stream ? kStreamSmem : 3) * Pn * (int)sizeof(double2);
      const int cpw_fit = (int)((stream ? 150 : 96) * 1024 / IFGF_ROWS_MINB / per_cone / NW);
      const int cpw = std::max(1, std::min(kRowMaxCpw, cpw_env > 0 ? cpw_env : std::max(1, cpw_fit)));
      const int cpb = NW * cpw;
      const uint32_t nq = qe - qb;
      const int groups =
          (int)std::min<size_t>(8, std::max<size_t>(1, nq / ((size_t)cpb * 148 * 4)));
      const unsigned grid = (unsigned)((nq + (size_t)cpb * groups - 1) / ((size_t)cpb * groups));
      const size_t sm = (size_t)cpb * per_cone;
      auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<grid, kRowThreads, sm, s>>>(U.dev(), L.dev(), K, tiles_dev(T), P->kappa, qb, qe,
                                          cpw, groups, child, parent, P->err);
      };
      const bool lap = P->kappa == 0.0;
      if constexpr (StreamShape<PS, PT, PP>::ok) {
        if (stream) {
          if (T.row_nodes == 2)
            lap ? launch(k_propagate_stream<PS, PT, PP, true, 2>)
                : launch(k_propagate_stream<PS, PT, PP, false, 2>);
          else
            lap ? launch(k_propagate_stream<PS, PT, PP, true, 3>)
                : launch(k_propagate_stream<PS, PT, PP, false, 3>);
          ++P->launches;
          return;
        }
      }
      if (T.row_nodes == 2)
        lap ? launch(k_propagate_rows<PS, PT, PP, true, 2>)
            : launch(k_propagate_rows<PS, PT, PP, false, 2>);
      else
        lap ? launch(k_propagate_rows<PS, PT, PP, true, 3>)
            : launch(k_propagate_rows<PS, PT, PP, false, 3>);
      ++P->launches;
    });
  }
  if (P->prop_kernel == IFGF_PROP_TILES || !full) {  // per node from the tiles (any range)
    const Level& U = P->lv[d - 1];
    const Level& L = P->lv[d];
    const InterpConsts& K = P->K;
    return dispatch_mma_orders(K.ps, K.pt, K.pp, [&](auto A, auto B, auto C) {
      constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
      constexpr int Pn = PS * PT * PP;
      int cpb = std::max(1, std::min(16, 320 / Pn));
      const uint32_t nq = qe - qb;
      const int groups =
          (int)std::min<size_t>(8, std::max<size_t>(1, nq / ((size_t)cpb * 148 * 8)));
      const unsigned grid = (unsigned)((nq + (size_t)cpb * groups - 1) / ((size_t)cpb * groups));
      const unsigned thr = (unsigned)(((cpb * Pn + 31) / 32) * 32);
      const size_t sm = 2 * (size_t)cpb * Pn * sizeof(double2);
      if (P->kappa == 0.0)
        k_propagate_tab<PS, PT, PP, true><<<grid, thr, sm, s>>>(
            U.dev(), L.dev(), K, tiles_dev(T), P->kappa, qb, qe, cpb, groups, child, parent,
            P->err);
      else
        k_propagate_tab<PS, PT, PP, false><<<grid, thr, sm, s>>>(
            U.dev(), L.dev(), K, tiles_dev(T), P->kappa, qb, qe, cpb, groups, child, parent,
            P->err);
      ++P->launches;
    });
  }
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  return dispatch_mma_orders(K.ps, K.pt, K.pp, [&](auto A, auto B, auto C) {
    constexpr int PS = decltype(A)::value, PT = decltype(B)::value, PP = decltype(C)::value;
    using G = GemmK<PS, PT, PP>;
    const size_t sm = G::smem;
    auto launch = [&](auto kern) {
      IFGF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      kern<<<(T.nchunks + G::NW - 1) / G::NW, G::NW * 32, sm, s>>>(U.dev(), L.dev(), K, tiles_dev(T),
                                                                  P->kappa, T.nchunks, child, parent, P->err);
      IFGF_CUDA(cudaGetLastError());
    };
    P->kappa == 0.0 ? launch(k_propagate_gemm<PS, PT, PP, true>)
                    : launch(k_propagate_gemm<PS, PT, PP, false>);
    ++P->launches;
  });
}

}  // namespace ifgf_b200
