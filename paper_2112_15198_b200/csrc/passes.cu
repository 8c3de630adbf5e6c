// passes.cu -- the four IFGF passes of ifgf::apply (engine.cpp:233-325) as
// sm_100a kernels, FP64 throughout.
//
//   K1 k_singular     singular_pass + green_sum       engine.cpp:233-258, kernels_scalar.cpp:12-30
//   K2 k_level_d      eval_level_d + factored_sum     engine.cpp:107-136, kernels_scalar.cpp:32-52
//                     + cheb_fit                      interp.cpp:68-91
//   K3 k_propagate    propagation_pass                engine.cpp:138-189
//   K4 k_interp       interpolation_pass              engine.cpp:191-231
//   K6 gather/scatter density gather, apply tail     engine.cpp:312-315
//
// Every work item writes only its own output slot, in a fixed order, so the
// result is bitwise reproducible run to run (parallel.hpp:17-19 contract).
#include <algorithm>

#include "plan.hpp"

namespace ifgf_b200 {
namespace {

template <int A, int B, int C>
struct Orders {
  static constexpr int PS = A, PT = B, PP = C, P = A * B * C;
};

// Interpolation orders instantiated in this build (the hot default first).
#define IFGF_FOR_ORDERS(X) \
  X(3, 5, 5) X(4, 6, 6) X(5, 7, 7) X(1, 1, 1) X(2, 2, 2) X(3, 3, 3) X(4, 4, 4) X(2, 3, 3) X(3, 4, 4)

template <class F>
bool dispatch_orders(int ps, int pt, int pp, F&& f) {
#define IFGF_CASE(a, b, c)                 \
  if (ps == a && pt == b && pp == c) {     \
    f(Orders<a, b, c>{});                  \
    return true;                           \
  }
  IFGF_FOR_ORDERS(IFGF_CASE)
#undef IFGF_CASE
  return false;
}

inline unsigned blocks_for(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Occupancy targets (CTAs per SM) handed to __launch_bounds__; tuned on B200.
#ifndef IFGF_PROP_MINB
#define IFGF_PROP_MINB 2
#endif
#ifndef IFGF_INTERP_MINB
#define IFGF_INTERP_MINB 3
#endif



// ---------------------------------------------------------------- K1 near field
template <bool LAP>
__global__ void __launch_bounds__(128) k_singular(const __grid_constant__ LevelDev L, const uint32_t* __restrict__ ptbox,
                                                  const double* __restrict__ xs,
                                                  const double* __restrict__ ys,
                                                  const double* __restrict__ zs,
                                                  const double* __restrict__ ar,
                                                  const double* __restrict__ ai, double kappa,
                                                  size_t b0, size_t e0, double* ir, double* ii) {
  const size_t i = b0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= e0) return;
  const uint32_t b = ptbox[i];
  const double tx = xs[i], ty = ys[i], tz = zs[i];
  double sr = 0.0, si = 0.0;
  const uint32_t nn = L.nbr_cnt[b];
  for (uint32_t a = 0; a < nn; ++a) {
    const uint32_t o = L.nbr[(size_t)b * 27 + a];
    const uint32_t f = L.first[o], e = f + L.count[o];
    for (uint32_t m = f; m < e; ++m) {
      if (m == i) continue;
      const double dx = tx - __ldg(&xs[m]), dy = ty - __ldg(&ys[m]), dz = tz - __ldg(&zs[m]);
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double rinv = rsqrt_nr(r2);
      const double inv = kQuarterInvPi * rinv;
      const double a_r = __ldg(&ar[m]), a_i = __ldg(&ai[m]);
      if (LAP) {
        sr = fma(a_r, inv, sr);
        si = fma(a_i, inv, si);
      } else {
        double sn, cs;
        sincos_fast(kappa * (r2 * rinv), sn, cs);
        const double gr = cs * inv, gi = sn * inv;
        sr = fma(a_r, gr, fma(-a_i, gi, sr));
        si = fma(a_r, gi, fma(a_i, gr, si));
      }
    }
  }
  ir[i] += sr;
  ii[i] += si;
}

// K1, box form (default): warps of a persistent grid take target boxes of
// level D from a work counter.  A box's neighbour sources (the same list for
// every target of the box) are staged once in shared memory, in chunks of
// CH, with the density pre-scaled by 1/(4 pi).  The lanes split the sources
// (lane k takes sources k, k+32, ...) and each pass carries T = 4, 2 or 1
// targets, so every staged source feeds T pairs and all 32 lanes stay busy
// whatever the box population (the thread-per-target form runs 2-3 boxes per
// warp with divergent neighbour loops).  The pair is branch-free: rsqrt_nr,
// and e^{i kappa r} from sincos_tab.  Rounds that hold a self pair or tail
// lanes take a masked copy of the body.  The T complex partial sums are
// combined with a transposing butterfly and written by 2T lanes.  Sums run
// in a fixed order, so results are bitwise reproducible; they differ from
// the reference's sequential green_sum (kernels_scalar.cpp:12-30) by
// rounding only.
constexpr int kNearWarps = 4;

// One near-field pair: (vr, vi) += q e^{i kappa r} / r for the offset
// (dx, dy, dz); q carries the 1/(4 pi).  A skipped pair passes q = 0 with a
// unit offset.  (Laplace: q / r.)
template <bool LAP>
__device__ __forceinline__ void near_pair(const double2* ptab, double dx, double dy, double dz,
                                          double qr, double qi, double kappa, double& vr,
                                          double& vi) {
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double rinv = rsqrt_nr(r2);
  const double br = qr * rinv, bi = qi * rinv;
  if (LAP) {
    vr += br;
    vi += bi;
  } else {
    double sn, cs;
    sincos_tab(ptab, kappa * (r2 * rinv), sn, cs);  // kappa carries kPhaseScale
    vr = fma(br, cs, fma(-bi, sn, vr));
    vi = fma(br, sn, fma(bi, cs, vi));
  }
}

// Sum NV values per lane over the warp.  Each step halves the values a lane
// carries (the half it keeps is picked by its lane bit), so NV values cost
// NV - 1 + log2(32 / NV) shuffles instead of 5 NV.  On return lanes with
// lane % (32 / NV) == 0 hold the sum of value `idx` in v[0].
template <int NV>
__device__ __forceinline__ void warp_transpose_sum(double* v, int lane, int& idx) {
  idx = 0;
#pragma unroll
  for (int m = 16, h = NV / 2; h >= 1; m >>= 1, h >>= 1) {
    const bool up = lane & m;
#pragma unroll
    for (int q = 0; q < h; ++q) {
      const double send = up ? v[q] : v[q + h], keep = up ? v[q + h] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
    if (up) idx += h;
  }
#pragma unroll
  for (int m = 16 / NV; m >= 1; m >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
}

// One pass: targets t0 .. t0+T-1 of the box against the cn staged sources.
template <bool LAP, int T>
__device__ __forceinline__ void near_pass(const double* sx, const double* sy, const double* sz,
                                          const double* sar, const double* sai,
                                          const double2* ptab, uint32_t cn, uint32_t js0,
                                          const double* __restrict__ xs,
                                          const double* __restrict__ ys,
                                          const double* __restrict__ zs, size_t t0,
                                          double kappa, int lane, double* ir, double* ii) {
  double tx[T], ty[T], tz[T], v[2 * T];
#pragma unroll
  for (int u = 0; u < T; ++u) {
    tx[u] = xs[t0 + u];
    ty[u] = ys[t0 + u];
    tz[u] = zs[t0 + u];
    v[2 * u] = 0.0;
    v[2 * u + 1] = 0.0;
  }
  for (uint32_t kb = 0; kb < cn; kb += 32) {
    const uint32_t k = kb + lane;
    const bool valid = k < cn;
    const uint32_t kk = valid ? k : cn - 1;
    const double px = sx[kk], py = sy[kk], pz = sz[kk], qr = sar[kk], qi = sai[kk];
    // own slot of target u in this chunk is js0 + u (wrapped when outside)
    const bool hit = !valid || (k - js0 < (uint32_t)T);
    if (!__any_sync(0xffffffffu, hit)) {
#pragma unroll
      for (int u = 0; u < T; ++u)
        near_pair<LAP>(ptab, tx[u] - px, ty[u] - py, tz[u] - pz, qr, qi, kappa, v[2 * u],
                       v[2 * u + 1]);
    } else {
#pragma unroll
      for (int u = 0; u < T; ++u) {
        const bool skip = !valid || k == js0 + u;
        near_pair<LAP>(ptab, skip ? 1.0 : tx[u] - px, ty[u] - py, tz[u] - pz, skip ? 0.0 : qr,
                       skip ? 0.0 : qi, kappa, v[2 * u], v[2 * u + 1]);
      }
    }
  }
  int idx;
  warp_transpose_sum<2 * T>(v, lane, idx);
  if ((lane & (16 / T - 1)) == 0) {
    const size_t i = t0 + (idx >> 1);
    (idx & 1 ? ii : ir)[i] += v[0];
  }
}

template <bool LAP, int CH>
__global__ void __launch_bounds__(kNearWarps * 32)
    k_near_box(const __grid_constant__ LevelDev L, const double2* __restrict__ phase,
               const double* __restrict__ xs, const double* __restrict__ ys,
               const double* __restrict__ zs, const double* __restrict__ ar,
               const double* __restrict__ ai, double kappa, size_t b0, size_t e0, double* ir,
               double* ii, uint32_t* ctr) {
  extern __shared__ double nsm[];
  __shared__ double2 ptab[kPhaseEntries];
  constexpr unsigned FULL = 0xffffffffu;
  for (int k = threadIdx.x; k < kPhaseEntries; k += blockDim.x) ptab[k] = phase[k];
  __syncthreads();
  kappa *= kPhaseScale;  // sincos_tab takes the phase in units of pi/256
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sx = nsm + (size_t)w * 5 * CH;
  double* sy = sx + CH;
  double* sz = sy + CH;
  double* sar = sz + CH;
  double* sai = sar + CH;
  for (;;) {
    uint32_t b = 0;
    if (lane == 0) b = atomicAdd(ctr, 1u);
    b = __shfl_sync(FULL, b, 0);
    if (b >= L.nb) break;
    const size_t tf = L.first[b];
    const size_t lo = max(tf, b0), hi = min(tf + L.count[b], e0);
    if (lo >= hi) continue;
    // neighbour segments (ascending, own box included): lane a holds segment a
    const uint32_t nn = L.nbr_cnt[b];
    uint32_t o = 0, f = 0, c = 0;
    if (lane < (int)nn) {
      o = L.nbr[(size_t)b * 27 + lane];
      f = L.first[o];
      c = L.count[o];
    }
    uint32_t inc = c;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t v = __shfl_up_sync(FULL, inc, k);
      if (lane >= k) inc += v;
    }
    const uint32_t off = inc - c;
    const uint32_t S = __shfl_sync(FULL, inc, 31);
    const unsigned selfm = __ballot_sync(FULL, lane < (int)nn && o == b);
    const uint32_t self_off = __shfl_sync(FULL, off, __ffs(selfm) - 1);
    for (uint32_t cs = 0; cs < S; cs += CH) {
      const uint32_t cn = min((uint32_t)CH, S - cs);
      __syncwarp();
      for (uint32_t a = 0; a < nn; ++a) {
        const uint32_t oa = __shfl_sync(FULL, off, a), ca = __shfl_sync(FULL, c, a),
                       fa = __shfl_sync(FULL, f, a);
        const uint32_t jl = max(oa, cs), jh = min(oa + ca, cs + cn);
        for (uint32_t j = jl + lane; j < jh; j += 32) {
          const uint32_t m = fa + (j - oa), k = j - cs;
          sx[k] = __ldg(&xs[m]);
          sy[k] = __ldg(&ys[m]);
          sz[k] = __ldg(&zs[m]);
          sar[k] = kQuarterInvPi * __ldg(&ar[m]);
          sai[k] = kQuarterInvPi * __ldg(&ai[m]);
        }
      }
      __syncwarp();
      // own slot of target t in this chunk: self_off + (t - tf) - cs
      const uint32_t jbase = self_off - (uint32_t)tf - cs;
      size_t t0 = lo;
      for (; t0 + 4 <= hi; t0 += 4)
        near_pass<LAP, 4>(sx, sy, sz, sar, sai, ptab, cn, jbase + (uint32_t)t0, xs, ys, zs, t0,
                          kappa, lane, ir, ii);
      if (t0 + 2 <= hi) {
        near_pass<LAP, 2>(sx, sy, sz, sar, sai, ptab, cn, jbase + (uint32_t)t0, xs, ys, zs, t0,
                          kappa, lane, ir, ii);
        t0 += 2;
      }
      if (t0 < hi)
        near_pass<LAP, 1>(sx, sy, sz, sar, sai, ptab, cn, jbase + (uint32_t)t0, xs, ys, zs, t0,
                          kappa, lane, ir, ii);
    }
  }
}

// ------------------------------------------------------- K2 level-D seeding
template <int PS, int PT, int PP, bool LAP>
__global__ void __launch_bounds__(320)
    k_level_d(const __grid_constant__ LevelDev L, const __grid_constant__ InterpConsts K, const double* __restrict__ xs,
              const double* __restrict__ ys, const double* __restrict__ zs,
              const double* __restrict__ ar, const double* __restrict__ ai, double kappa,
              uint32_t qb, uint32_t qe, int cpb, double2* out, int* err) {
  constexpr int P = PS * PT * PP;
  extern __shared__ double2 smem[];
  double2* sv = smem;
  double2* st = smem + cpb * P;
  double2* ptab = st + cpb * P;  // sincos_tab phase table
  if (!LAP) {
    for (int k = threadIdx.x; k < kPhaseEntries; k += blockDim.x) ptab[k] = L.trig[kTrigEntries + k];
    __syncthreads();
  }
  const double ks = kappa * kPhaseScale;
  const uint32_t q0 = qb + blockIdx.x * cpb;
  const int ncon = (int)min((uint32_t)cpb, qe - q0);
  const int c = threadIdx.x / P, m = threadIdx.x % P;
  if (c < ncon) {
    const uint32_t q = q0 + c;
    const uint32_t b = L.cone_box[q];
    const int jp = m % PP, jt = (m / PP) % PT, js = m / (PP * PT);
    const SegMid sg = segment_mid(L, L.cone_gamma[q]);
    const double cx = L.cx[b], cy = L.cy[b], cz = L.cz[b];
    double tx, ty, tz;
    node_position(sg, L.rad, cx, cy, cz, K.ns[js], K.nt[jt], K.np[jp], tx, ty, tz);
    const double ux = tx - cx, uy = ty - cy, uz = tz - cz;
    const double rc = sqrt(fma(uz, uz, fma(uy, uy, ux * ux)));
    double sr = 0.0, si = 0.0;
    const uint32_t f = L.first[b], e = f + L.count[b];
    for (uint32_t j = f; j < e; ++j) {
      const double dx = tx - __ldg(&xs[j]), dy = ty - __ldg(&ys[j]), dz = tz - __ldg(&zs[j]);
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double rinv = rsqrt_nr(r2);
      const double ratio = rc * rinv;
      const double a_r = __ldg(&ar[j]), a_i = __ldg(&ai[j]);
      if (LAP) {
        sr = fma(a_r, ratio, sr);
        si = fma(a_i, ratio, si);
      } else {
        double sn, cs;
        sincos_tab(ptab, ks * (r2 * rinv - rc), sn, cs);
        const double gr = cs * ratio, gi = sn * ratio;
        sr = fma(a_r, gr, fma(-a_i, gi, sr));
        si = fma(a_r, gi, fma(a_i, gr, si));
      }
    }
    sv[c * P + m] = make_double2(sr, si);
  }
  __syncthreads();
  fit_cones_inplace<PS, PT, PP, true>(K, sv, ncon, out + (size_t)q0 * BlockLayout<PS, PT, PP>::Pst,
                                      err);
}

// ------------------------------------------------------------ K3 propagation
// One CTA = `groups` consecutive groups of `cpb` parent cones (cone order is
// box-major, so a CTA mostly stays inside one parent box and re-reads the
// same child blocks from L1); thread = (cone, node).
template <int PS, int PT, int PP, bool LAP>
__global__ void __launch_bounds__(320, IFGF_PROP_MINB)
    k_propagate(const __grid_constant__ LevelDev U, const __grid_constant__ LevelDev L,
                const __grid_constant__ InterpConsts K, double kappa, uint32_t qb, uint32_t qe,
                int cpb, int groups, const double2* __restrict__ child, double2* parent,
                int* err) {
  constexpr int P = PS * PT * PP;
  extern __shared__ double2 smem[];
  double2* sv = smem;
  double2* st = smem + cpb * P;
  __shared__ double2 trig[kTrigEntries];
  stage_trig(trig, L.trig);
  __syncthreads();
  const int c = threadIdx.x / P, m = threadIdx.x % P;
  const int jp = m % PP, jt = (m / PP) % PT, js = m / (PP * PT);
  for (int g = 0; g < groups; ++g) {
    const uint32_t q0 = qb + ((uint32_t)g * gridDim.x + blockIdx.x) * cpb;
    if (q0 >= qe) break;
    const int ncon = (int)min((uint32_t)cpb, qe - q0);
    if (c < ncon) {
      const uint32_t q = q0 + c;
      const uint32_t pb = U.cone_box[q];
      const SegMid sg = segment_mid(U, U.cone_gamma[q]);
      const double pcx = U.cx[pb], pcy = U.cy[pb], pcz = U.cz[pb];
      double x, y, z;
      node_position(sg, U.rad, pcx, pcy, pcz, K.ns[js], K.nt[jt], K.np[jp], x, y, z);
      const double ux = x - pcx, uy = y - pcy, uz = z - pcz;
      const double rp = sqrt(fma(uz, uz, fma(uy, uy, ux * ux)));
      double acr = 0.0, aci = 0.0;
      const uint32_t c0 = U.child_begin[pb], c1 = U.child_begin[pb + 1];
      for (uint32_t cb = c0; cb < c1; ++cb) {
        Loc o;
        const int e = locate_fast(L, trig, L.cx[cb], L.cy[cb], L.cz[cb], x, y, z, o);
        if (e) {
          raise_err(err, e);
          break;
        }
        const uint32_t cq = find_cone(L, cb, o.gamma);
        if (cq == 0xffffffffu) {
          raise_err(err, kErrPropCover);
          break;
        }
        double vr, vi;
        eval_block<PS, PT, PP>(child + (size_t)cq * BlockLayout<PS, PT, PP>::Pst, o.ts, o.tt, o.tp, vr, vi);
        const double ratio = rp * o.rinv;
        if (LAP) {
          acr = fma(vr, ratio, acr);
          aci = fma(vi, ratio, aci);
        } else {
          double sn, cn;
          sincos_fast(kappa * (o.r - rp), sn, cn);
          const double tr = ratio * cn, ti = ratio * sn;
          acr = fma(vr, tr, fma(-vi, ti, acr));
          aci = fma(vr, ti, fma(vi, tr, aci));
        }
      }
      sv[c * P + m] = make_double2(acr, aci);
    }
    __syncthreads();
    fit_cones<PS, PT, PP>(K, sv, st, ncon, parent + (size_t)q0 * BlockLayout<PS, PT, PP>::Pst, err);
    __syncthreads();
  }
}

// ---------------------------------------------------------- K4 interpolation
// Thread = one run of <= R consecutive (Morton-sorted) points of one box
// (Level::chunk), clipped to [b0, e0).  They share the cousin list, and per
// cousin they nearly always fall into the same cone: that block is loaded once
// and evaluated at all R points (eval_block_multi), which takes the evaluation
// off the L1->register bandwidth limit.  Points that land in another cone of
// the cousin are evaluated singly.  Per point, cousins are summed in list
// order.
template <int PS, int PT, int PP, bool LAP, int R>
__global__ void __launch_bounds__(128, IFGF_INTERP_MINB)
    k_interp(const __grid_constant__ LevelDev L, const uint2* __restrict__ chunk,
             const uint32_t* __restrict__ nchunk, const double* __restrict__ xs,
             const double* __restrict__ ys, const double* __restrict__ zs, double kappa,
             size_t b0, size_t e0, const double2* __restrict__ blocks, double* ir, double* ii,
             int* err) {
  using BL = BlockLayout<PS, PT, PP>;
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
  const size_t lo = max((size_t)ch.x, b0);
  const size_t hi = min(min((size_t)ch.x + R, (size_t)L.first[b] + L.count[b]), e0);
  if (lo >= hi) return;
  const size_t i0 = lo;
  const int n = (int)(hi - lo);
  double px[R], py[R], pz[R], acr[R], aci[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const size_t i = i0 + (j < n ? j : 0);
    px[j] = xs[i];
    py[j] = ys[i];
    pz[j] = zs[i];
    acr[j] = aci[j] = 0.0;
  }
  const uint32_t k0 = L.cous_off[b], k1 = L.cous_off[b + 1];
  // cousin index and centre loaded one iteration ahead
  uint32_t cbn = k0 < k1 ? L.cous[k0] : 0;
  double cxn = L.cx[cbn], cyn = L.cy[cbn], czn = L.cz[cbn];
  for (uint32_t k = k0; k < k1; ++k) {
    const uint32_t cb = cbn;
    const double cx = cxn, cy = cyn, cz = czn;
    if (k + 1 < k1) {
      cbn = L.cous[k + 1];
      cxn = L.cx[cbn];
      cyn = L.cy[cbn];
      czn = L.cz[cbn];
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
    const uint32_t q = find_cone(L, cb, o[0].gamma);
    if (q == 0xffffffffu) {
      raise_err(err, kErrInterpCover);
      return;
    }
    double ts[R], tt[R], tp[R], vr[R], vi[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      ts[j] = o[j].ts;
      tt[j] = o[j].tt;
      tp[j] = o[j].tp;
    }
#if IFGF_K4_NOEVAL  // experiment: locate + factor only
#pragma unroll
    for (int j = 0; j < R; ++j) vr[j] = ts[j] + q, vi[j] = tt[j] + tp[j];
#else
    eval_block_multi<PS, PT, PP, R>(blocks + (size_t)q * BL::Pst, ts, tt, tp, vr, vi);
#endif
#pragma unroll
    for (int j = 1; j < R; ++j) {
      if (j < n && o[j].gamma != o[0].gamma) {  // another cone of this cousin
        const uint32_t qj = find_cone(L, cb, o[j].gamma);
        if (qj == 0xffffffffu) {
          raise_err(err, kErrInterpCover);
          return;
        }
        eval_block<PS, PT, PP>(blocks + (size_t)qj * BL::Pst, o[j].ts, o[j].tt, o[j].tp, vr[j],
                               vi[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const double inv = kQuarterInvPi * o[j].rinv;
      if (LAP) {
        acr[j] = fma(vr[j], inv, acr[j]);
        aci[j] = fma(vi[j], inv, aci[j]);
      } else {
        double sn, cn;
        sincos_tab<true>(ptab, ks * o[j].r, sn, cn);
        const double gr = cn * inv, gi = sn * inv;
        acr[j] = fma(vr[j], gr, fma(-vi[j], gi, acr[j]));
        aci[j] = fma(vr[j], gi, fma(vi[j], gr, aci[j]));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (j < n) {
      ir[i0 + j] += acr[j];
      ii[i0 + j] += aci[j];
    }
}

// K4 from the plan's locate records (LevelDev::rec / rec_g, setup.cu
// k_locate_points + k_rec_cones): the same work items, cousin order and sums
// as k_interp with the cone ordinal, the local coordinates and the kernel
// factor of every (point, cousin) pair read back instead of recomputed --
// bitwise the same result.
//
// k_interp_rec: blocks streamed per thread from global memory (any orders).
// k_interp_stg: blocks staged in shared memory.  Without the locate K4 is
// bound by the L1 tag stage: every lane streams its own 1.2 KB block, ~30
// different lines per warp load (ncu: L1 wavefronts 74 %, FP64 pipe 28 %).
// Neighbouring points mostly see the same few cones of a cousin, so per
// cousin step the warp finds the distinct blocks among its 64 (lane, point)
// pairs (match.any), copies each once with coalesced cp.async into one of S
// padded slots (slot stride = block + 16 B, so the lanes' reads of different
// slots fall into different banks), one step ahead of the evaluation (two
// slot sets per warp), and every lane evaluates from its slot.  Pairs beyond
// S distinct blocks read from global memory as before.  No CTA barriers.
// The records of one work item and cousin: R slots per plane, read with one
// aligned vector load per plane for R = 2.
template <int R, bool LAP>
struct RecSet {
  uint32_t g[R];
  double ts[R], tt[R], tp[R], gr[R], gi[R];
  __device__ __forceinline__ void load(const uint32_t* __restrict__ rec_g,
                                       const double* __restrict__ rec, uint64_t np, uint64_t idx) {
    if constexpr (R == 2) {
      const uint2 q = *reinterpret_cast<const uint2*>(rec_g + idx);
      g[0] = q.x, g[1] = q.y;
      double2 v = *reinterpret_cast<const double2*>(rec + idx);
      ts[0] = v.x, ts[1] = v.y;
      v = *reinterpret_cast<const double2*>(rec + np + idx);
      tt[0] = v.x, tt[1] = v.y;
      v = *reinterpret_cast<const double2*>(rec + 2 * np + idx);
      tp[0] = v.x, tp[1] = v.y;
      v = *reinterpret_cast<const double2*>(rec + 3 * np + idx);
      gr[0] = v.x, gr[1] = v.y;
      if (!LAP) {
        v = *reinterpret_cast<const double2*>(rec + 4 * np + idx);
        gi[0] = v.x, gi[1] = v.y;
      } else {
        gi[0] = gi[1] = 0.0;
      }
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        g[j] = rec_g[idx + j];
        ts[j] = rec[idx + j];
        tt[j] = rec[np + idx + j];
        tp[j] = rec[2 * np + idx + j];
        gr[j] = rec[3 * np + idx + j];
        gi[j] = LAP ? 0.0 : rec[4 * np + idx + j];
      }
    }
  }
  __device__ __forceinline__ void get(int slot, uint32_t& g_, double& ts_, double& tt_, double& tp_,
                                      double& gr_, double& gi_) const {
    g_ = g[0], ts_ = ts[0], tt_ = tt[0], tp_ = tp[0], gr_ = gr[0], gi_ = gi[0];
#pragma unroll
    for (int j = 1; j < R; ++j)
      if (slot == j) g_ = g[j], ts_ = ts[j], tt_ = tt[j], tp_ = tp[j], gr_ = gr[j], gi_ = gi[j];
  }
};

#ifndef IFGF_INTERP_REC_MINB
#define IFGF_INTERP_REC_MINB 3
#endif
template <int PS, int PT, int PP, bool LAP, int R>
__global__ void __launch_bounds__(128, IFGF_INTERP_REC_MINB)
    k_interp_rec(const __grid_constant__ LevelDev L, const uint2* __restrict__ chunk,
                 const uint32_t* __restrict__ nchunk, size_t b0, size_t e0,
                 const double2* __restrict__ blocks, double* ir, double* ii, int* err) {
  using BL = BlockLayout<PS, PT, PP>;
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= *nchunk) return;
  const uint2 ch = chunk[t];
  const uint32_t b = ch.y;
  const uint32_t fb = L.first[b], cnt = L.count[b];
  const size_t lo = max((size_t)ch.x, b0);
  const size_t hi = min(min((size_t)ch.x + R, (size_t)fb + cnt), e0);
  if (lo >= hi) return;
  const int n = (int)(hi - lo);
  const uint32_t k0 = L.cous_off[b], k1 = L.cous_off[b + 1];
  if (k0 == k1) return;
  const uint64_t np = L.npairs;
  const double* __restrict__ rec = L.rec;
  const uint32_t* __restrict__ rec_g = L.rec_g;
  const uint32_t cntp = (cnt + R - 1) / R * R;
  uint64_t idx = L.pair_off[b] + (ch.x - fb);
  // record slot of evaluation j: the item's points from lo on, the first repeated
  int off[R];
#pragma unroll
  for (int j = 0; j < R; ++j) off[j] = (int)(lo - ch.x) + (j < n ? j : 0);
  double acr[R], aci[R];
#pragma unroll
  for (int j = 0; j < R; ++j) acr[j] = aci[j] = 0.0;
  RecSet<R, LAP> nx;
  nx.load(rec_g, rec, np, idx);
  for (uint32_t k = k0; k < k1; ++k) {
    uint32_t g[R];
    double ts[R], tt[R], tp[R], gr[R], gi[R], vr[R], vi[R];
#pragma unroll
    for (int j = 0; j < R; ++j) nx.get(off[j], g[j], ts[j], tt[j], tp[j], gr[j], gi[j]);
    if (k + 1 < k1) {
      idx += cntp;
      nx.load(rec_g, rec, np, idx);
    }
    eval_block_multi<PS, PT, PP, R>(blocks + (size_t)g[0] * BL::Pst, ts, tt, tp, vr, vi);
#pragma unroll
    for (int j = 1; j < R; ++j)
      if (j < n && g[j] != g[0])  // another cone of this cousin
        eval_block<PS, PT, PP>(blocks + (size_t)g[j] * BL::Pst, ts[j], tt[j], tp[j], vr[j], vi[j]);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (LAP) {
        acr[j] = fma(vr[j], gr[j], acr[j]);
        aci[j] = fma(vi[j], gr[j], aci[j]);
      } else {
        acr[j] = fma(vr[j], gr[j], fma(-vi[j], gi[j], acr[j]));
        aci[j] = fma(vr[j], gi[j], fma(vi[j], gr[j], aci[j]));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (j < n) {
      ir[lo + j] += acr[j];
      ii[lo + j] += aci[j];
    }
}

__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

#ifndef IFGF_STG_WARPS
#define IFGF_STG_WARPS 2
#endif
#ifndef IFGF_STG_MINB
#define IFGF_STG_MINB 5
#endif
constexpr int kStgWarps = IFGF_STG_WARPS;
// slots per set: 8 blocks of <= 80 coefficients, 4 of <= 160
#ifndef IFGF_STG_SLOTS
#define IFGF_STG_SLOTS 8
#endif
constexpr int stg_slots(int Pst) { return Pst <= 80 ? IFGF_STG_SLOTS : (Pst <= 160 ? IFGF_STG_SLOTS / 2 : 0); }

template <int PS, int PT, int PP, bool LAP>
__global__ void __launch_bounds__(kStgWarps * 32, IFGF_STG_MINB)
    k_interp_stg(const __grid_constant__ LevelDev L, const uint2* __restrict__ chunk,
                 const uint32_t* __restrict__ nchunk, size_t b0, size_t e0,
                 const double2* __restrict__ blocks, double* ir, double* ii) {
  using BL = BlockLayout<PS, PT, PP>;
  constexpr int R = 2;
  constexpr int S = stg_slots(BL::Pst);
  constexpr int ST = BL::Pst + 1;  // slot stride (double2): odd, so slots start in different banks
  constexpr unsigned FULL = 0xffffffffu;
  constexpr uint32_t NONE = 0xffffffffu;
  extern __shared__ double2 stg_smem[];
  const int lane = threadIdx.x & 31;
  double2* const buf = stg_smem + (size_t)(threadIdx.x >> 5) * 2 * S * ST;
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const uint32_t nch = *nchunk;
  if (t - lane >= nch) return;  // whole warp past the work list
  // lanes without work stay for the cooperative copies
  uint32_t cntp = 0, len = 0;
  size_t lo = 0;
  int n = 0;
  bool sel0 = false, sel1 = false;  // record slot (0 / 1) of the two evaluations
  uint64_t idx = 0;
  if (t < nch) {
    const uint2 ch = chunk[t];
    const uint32_t b = ch.y;
    const uint32_t fb = L.first[b], cnt = L.count[b];
    cntp = (cnt + 1u) & ~1u;
    lo = max((size_t)ch.x, b0);
    const size_t hi = min(min((size_t)ch.x + R, (size_t)fb + cnt), e0);
    if (lo < hi) {
      n = (int)(hi - lo);
      len = L.cous_off[b + 1] - L.cous_off[b];
      idx = L.pair_off[b] + (ch.x - fb);
      sel0 = lo > ch.x;
      sel1 = sel0 || n > 1;
    }
  }
  const uint32_t maxlen = __reduce_max_sync(FULL, len);
  if (maxlen == 0) return;
  const uint64_t np = L.npairs;
  const double* __restrict__ rec = L.rec;
  const uint32_t* __restrict__ rec_g = L.rec_g;
  double acr[R] = {0.0, 0.0}, aci[R] = {0.0, 0.0};

  // cone ordinals of step kk (NONE: no work), from the records
  auto load_q = [&](uint32_t kk, uint32_t& q0, uint32_t& q1) {
    q0 = q1 = NONE;
    if (kk < len) {
      const uint2 v = *reinterpret_cast<const uint2*>(rec_g + idx + (uint64_t)kk * cntp);
      q0 = sel0 ? v.y : v.x;
      q1 = sel1 ? v.y : v.x;
    }
  };
  // slots of the step's distinct blocks, and their copies into slot set `set`
  auto stage = [&](uint32_t q0, uint32_t q1, int set, int& s0, int& s1) {
    const bool act = q0 != NONE;
    const unsigned pa = __match_any_sync(FULL, q0);
    const int la = __ffs(pa) - 1;
    const unsigned leadA = __ballot_sync(FULL, act && la == lane);
    s0 = __popc(leadA & ((1u << la) - 1u));
    const int nA = __popc(leadA);
    const bool diff = act && q1 != q0;
    const unsigned dm = __ballot_sync(FULL, diff);
    s1 = s0;
    unsigned leadB = 0;
    if (dm) {  // warp-uniform
      const uint32_t v = diff ? q1 : q0;
      const unsigned pb = __match_any_sync(FULL, v);
      const unsigned same0 = pb & ~dm;  // lanes whose first block is this one
      const int src = same0 ? __ffs(same0) - 1 : lane;
      const int sfrom = __shfl_sync(FULL, s0, src);
      const int lb = __ffs(pb & dm) - 1;
      leadB = __ballot_sync(FULL, diff && !same0 && lb == lane);
      if (diff) s1 = same0 ? sfrom : nA + __popc(leadB & ((1u << lb) - 1u));
    }
    const int ntot = min(nA + __popc(leadB), S);
    double2* const dst0 = buf + (size_t)set * S * ST;
    for (int s = 0; s < ntot; ++s) {
      const bool fromA = s < nA;
      const int src = (int)__fns(fromA ? leadA : leadB, 0, (fromA ? s : s - nA) + 1);
      const uint32_t q = __shfl_sync(FULL, fromA ? q0 : q1, src);
      const double2* g = blocks + (size_t)q * BL::Pst;
      double2* d = dst0 + (size_t)s * ST;
#pragma unroll
      for (int c = 0; c < (BL::Pst + 31) / 32; ++c)
        if (c * 32 + lane < BL::Pst) cp_async16(d + c * 32 + lane, g + c * 32 + lane);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // The cone ordinals run three steps ahead of the evaluation through a
  // per-lane ring in shared memory (cp.async with the block copies: a
  // register prefetch leaves the loop's register rotation waiting on the load)
  uint2* const qring = reinterpret_cast<uint2*>(stg_smem + (size_t)kStgWarps * 2 * S * ST) +
                       (size_t)(threadIdx.x >> 5) * 4 * 32 + lane;
  auto fetch_q = [&](uint32_t kk) {  // async: lands with the next committed group
    uint2* dst = qring + (kk & 3) * 32;
    if (kk < len) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d),
                   "l"(rec_g + idx + (uint64_t)kk * cntp)
                   : "memory");
    } else {
      *dst = make_uint2(NONE, NONE);
    }
  };
  auto read_q = [&](uint32_t kk, uint32_t& q0, uint32_t& q1) {
    const uint2 v = qring[(kk & 3) * 32];
    q0 = sel0 ? v.y : v.x;
    q1 = sel1 ? v.y : v.x;
  };
  uint32_t q0, q1, q0n, q1n;
  int s0, s1, s0n = 0, s1n = 0;
  load_q(0, q0, q1);
  fetch_q(1);
  fetch_q(2);
  stage(q0, q1, 0, s0, s1);  // commits group 0 (blocks of step 0, ordinals of steps 1 and 2)
  // the step's record pairs as loaded (the slot selects wait until the
  // evaluation, a whole step after the loads were issued)
  double2 raw[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) raw[i] = make_double2(0.0, 0.0);
  auto load_rec = [&](uint32_t kk) {
    if (kk < len) {
      const double* r = rec + idx + (uint64_t)kk * cntp;
#pragma unroll
      for (int i = 0; i < (LAP ? 4 : 5); ++i)
        raw[i] = *reinterpret_cast<const double2*>(r + i * np);
    }
  };
  load_rec(0);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  for (uint32_t kk = 0; kk < maxlen; ++kk) {
    // next step's blocks into the other slot set (its readers finished at the
    // __syncwarp that closed the previous iteration), ordinals of step kk + 3
    read_q(kk + 1, q0n, q1n);
    fetch_q(kk + 3);
    if (kk + 1 < maxlen) stage(q0n, q1n, (kk + 1) & 1, s0n, s1n);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    if (q0 != NONE) {
      const double2* const set = buf + (size_t)(kk & 1) * S * ST;
      double vr[R], vi[R];
      const double ts[R] = {sel0 ? raw[0].y : raw[0].x, sel1 ? raw[0].y : raw[0].x};
      const double tt[R] = {sel0 ? raw[1].y : raw[1].x, sel1 ? raw[1].y : raw[1].x};
      const double tp[R] = {sel0 ? raw[2].y : raw[2].x, sel1 ? raw[2].y : raw[2].x};
      const double gr[R] = {sel0 ? raw[3].y : raw[3].x, sel1 ? raw[3].y : raw[3].x};
      const double gi[R] = {sel0 ? raw[4].y : raw[4].x, sel1 ? raw[4].y : raw[4].x};
      if (s0 < S)
        eval_block_multi<PS, PT, PP, R, true>(set + (size_t)s0 * ST, ts, tt, tp, vr, vi);
      else
        eval_block_multi<PS, PT, PP, R>(blocks + (size_t)q0 * BL::Pst, ts, tt, tp, vr, vi);
      if (q1 != q0) {  // the second point sees another cone of this cousin
        if (s1 < S)
          eval_block<PS, PT, PP, true>(set + (size_t)s1 * ST, ts[1], tt[1], tp[1], vr[1], vi[1]);
        else
          eval_block<PS, PT, PP>(blocks + (size_t)q1 * BL::Pst, ts[1], tt[1], tp[1], vr[1], vi[1]);
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (LAP) {
          acr[j] = fma(vr[j], gr[j], acr[j]);
          aci[j] = fma(vi[j], gr[j], aci[j]);
        } else {
          acr[j] = fma(vr[j], gr[j], fma(-vi[j], gi[j], acr[j]));
          aci[j] = fma(vr[j], gi[j], fma(vi[j], gr[j], aci[j]));
        }
      }
    }
    load_rec(kk + 1);
    __syncwarp();
    q0 = q0n;
    q1 = q1n;
    s0 = s0n;
    s1 = s1n;
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (j < n) {
      ir[lo + j] += acr[j];
      ii[lo + j] += aci[j];
    }
}

// --------------------------------------------------------------- K6 permutes
__global__ void k_gather_density(const uint32_t* __restrict__ perm, const double* __restrict__ a_re,
                                 const double* __restrict__ a_im, size_t n, double* ar, double* ai,
                                 double* ir, double* ii) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  ar[i] = a_re[j];
  ai[i] = a_im ? a_im[j] : 0.0;
  if (ir) {
    ir[i] = 0.0;
    ii[i] = 0.0;
  }
}

__global__ void k_scatter_result(const uint32_t* __restrict__ perm, const double* __restrict__ ir,
                                 const double* __restrict__ ii, size_t n, double* o_re,
                                 double* o_im) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = perm[i];
  o_re[j] = ir[i];
  o_im[j] = ii[i];
}

__global__ void k_pack(const double2* __restrict__ blocks, const uint32_t* __restrict__ cones,
                       size_t m, int Pst, uint32_t nc, double2* buf, int unpack,
                       double2* blocks_out, int* err) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= m * Pst) return;
  const size_t j = t / Pst, k = t % Pst;
  const uint32_t q = cones[j];
  if (q >= nc) {  // caller-supplied ordinal out of range: invalid_argument
    if (k == 0) raise_err(err, kErrBadCone);
    return;
  }
  const size_t g = (size_t)q * Pst + k;
  if (unpack) blocks_out[g] = buf[t];
  else buf[t] = blocks[g];
}

inline int cones_per_cta(int P) {
  int c = 320 / P;
  if (c < 1) c = 1;
  while (c > 1 && ((c * P + 31) / 32) * 32 > 320) --c;
  return c;
}

inline unsigned threads_for(int cpb, int P) { return (unsigned)(((cpb * P + 31) / 32) * 32); }

}  // namespace

bool orders_supported(int ps, int pt, int pp) {
  return dispatch_orders(ps, pt, pp, [](auto) {});
}

void launch_gather_density(ifgf_plan* P, const double* a_re, const double* a_im, cudaStream_t s) {
  k_gather_density<<<blocks_for(P->n, 256), 256, 0, s>>>(P->perm, a_re, a_im, P->n, P->ar, P->ai,
                                                         P->ir, P->ii);
  ++P->launches;
}

void launch_scatter_result(ifgf_plan* P, double* o_re, double* o_im, cudaStream_t s) {
  k_scatter_result<<<blocks_for(P->n, 256), 256, 0, s>>>(P->perm, P->ir, P->ii, P->n, o_re, o_im);
  ++P->launches;
}

template <bool LAP, int CH>
void launch_near_box(ifgf_plan* P, const Level& L, size_t b, size_t e, cudaStream_t s) {
  const size_t smem = (size_t)kNearWarps * 5 * CH * sizeof(double);
  static int ctas_per_sm = 0;  // per instantiation
  if (!ctas_per_sm) {
    IFGF_CUDA(cudaFuncSetAttribute(k_near_box<LAP, CH>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    IFGF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k_near_box<LAP, CH>,
                                                            kNearWarps * 32, smem));
    ctas_per_sm = std::max(ctas_per_sm, 1);
  }
  int sms = 0;
  IFGF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device));
  const unsigned grid =
      std::min<unsigned>(blocks_for(L.nb, kNearWarps), (unsigned)(sms * ctas_per_sm));
  uint32_t* ctr = P->work_ctr + ifgf_plan::kCtrNear;
  IFGF_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), s));
  k_near_box<LAP, CH><<<grid, kNearWarps * 32, smem, s>>>(
      L.dev(), P->phase, P->xs, P->ys, P->zs, P->ar, P->ai, P->kappa, b, e, P->ir, P->ii, ctr);
}

#ifndef IFGF_NEAR_CHUNK
#define IFGF_NEAR_CHUNK 192
#endif

void launch_singular(ifgf_plan* P, size_t b, size_t e, cudaStream_t s) {
  if (e <= b) return;
  const Level& L = P->lv[P->depth];
  // the box form needs populated leaves: below ~12 points per box (Laplace
  // depth rule, C3) its per-box staging and reductions cost more than the
  // divergence they remove
  if (P->near_kernel == IFGF_NEAR_BOX && P->n >= 12 * (size_t)L.nb) {
    if (P->kappa == 0.0) launch_near_box<true, IFGF_NEAR_CHUNK>(P, L, b, e, s);
    else launch_near_box<false, IFGF_NEAR_CHUNK>(P, L, b, e, s);
    ++P->launches;
    return;
  }
  const unsigned g = blocks_for(e - b, 128);
  if (P->kappa == 0.0)
    k_singular<true><<<g, 128, 0, s>>>(L.dev(), L.ptbox, P->xs, P->ys, P->zs, P->ar, P->ai,
                                       P->kappa, b, e, P->ir, P->ii);
  else
    k_singular<false><<<g, 128, 0, s>>>(L.dev(), L.ptbox, P->xs, P->ys, P->zs, P->ar, P->ai,
                                        P->kappa, b, e, P->ir, P->ii);
  ++P->launches;
}

void launch_level_d(ifgf_plan* P, uint32_t qb, uint32_t qe, double2* out, cudaStream_t s) {
  if (qe <= qb) return;
  const Level& L = P->lv[P->depth];
  const InterpConsts& K = P->K;
  dispatch_orders(K.ps, K.pt, K.pp, [&](auto o) {
    using O = decltype(o);
    const int cpb = cones_per_cta(O::P);
    const unsigned grid = blocks_for(qe - qb, cpb);
    const size_t smem = (2 * (size_t)cpb * O::P + kPhaseEntries) * sizeof(double2);
    if (P->kappa == 0.0)
      k_level_d<O::PS, O::PT, O::PP, true><<<grid, threads_for(cpb, O::P), smem, s>>>(
          L.dev(), K, P->xs, P->ys, P->zs, P->ar, P->ai, P->kappa, qb, qe, cpb, out, P->err);
    else
      k_level_d<O::PS, O::PT, O::PP, false><<<grid, threads_for(cpb, O::P), smem, s>>>(
          L.dev(), K, P->xs, P->ys, P->zs, P->ar, P->ai, P->kappa, qb, qe, cpb, out, P->err);
  });
  ++P->launches;
}

void launch_propagation(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, const double2* child,
                        double2* parent, cudaStream_t s) {
  if (qe <= qb) return;
  // precomputed (gamma, octant) geometry kernels when selected and the plan
  // built tiles for this level (IFGF_OPT_PROP_KERNEL)
  if (P->prop_kernel != IFGF_PROP_NODE && launch_propagation_mma(P, d, qb, qe, child, parent, s))
    return;
  const Level& U = P->lv[d - 1];
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  dispatch_orders(K.ps, K.pt, K.pp, [&](auto o) {
    using O = decltype(o);
    const int cpb = cones_per_cta(O::P);
    // enough CTAs for ~8 per SM, at most 8 groups each
    int groups = (int)std::min<size_t>(8, std::max<size_t>(1, (qe - qb) / ((size_t)cpb * 148 * 8)));
    const unsigned grid = blocks_for(qe - qb, cpb * groups);
    const size_t smem = 2 * (size_t)cpb * O::P * sizeof(double2);
    if (P->kappa == 0.0)
      k_propagate<O::PS, O::PT, O::PP, true><<<grid, threads_for(cpb, O::P), smem, s>>>(
          U.dev(), L.dev(), K, P->kappa, qb, qe, cpb, groups, child, parent, P->err);
    else
      k_propagate<O::PS, O::PT, O::PP, false><<<grid, threads_for(cpb, O::P), smem, s>>>(
          U.dev(), L.dev(), K, P->kappa, qb, qe, cpb, groups, child, parent, P->err);
  });
  ++P->launches;
}

void launch_interpolation(ifgf_plan* P, int d, size_t b, size_t e, const double2* blocks,
                          cudaStream_t s) {
  if (e <= b) return;
  const Level& L = P->lv[d];
  const InterpConsts& K = P->K;
  dispatch_orders(K.ps, K.pt, K.pp, [&](auto o) {
    using O = decltype(o);
    constexpr int R = interp_points(O::P);
    const unsigned g = blocks_for(L.chunk_cap, 128);
    if (L.rec && P->k4_records) {
      using BL = BlockLayout<O::PS, O::PT, O::PP>;
      static const bool no_stage = [] {
        const char* v = std::getenv("IFGF_K4_STAGE");
        return v && std::atoi(v) == 0;
      }();
      if constexpr (R == 2 && stg_slots(BL::Pst) > 0) {
        if (!no_stage) {
          auto kern = P->kappa == 0.0 ? k_interp_stg<O::PS, O::PT, O::PP, true>
                                      : k_interp_stg<O::PS, O::PT, O::PP, false>;
          const size_t smem =
              (size_t)kStgWarps * 2 * stg_slots(BL::Pst) * (BL::Pst + 1) * sizeof(double2) +
              (size_t)kStgWarps * 4 * 32 * sizeof(uint2);  // slot sets + ordinal rings
          static bool attr_set = false;  // per instantiation (orders, kernel kind share the size)
          if (!attr_set) {
            IFGF_CUDA(cudaFuncSetAttribute(k_interp_stg<O::PS, O::PT, O::PP, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            IFGF_CUDA(cudaFuncSetAttribute(k_interp_stg<O::PS, O::PT, O::PP, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_set = true;
          }
          kern<<<blocks_for(L.chunk_cap, kStgWarps * 32), kStgWarps * 32, smem, s>>>(
              L.dev(), L.chunk, L.nchunk, b, e, blocks, P->ir, P->ii);
          return;
        }
      }
      auto kern = P->kappa == 0.0 ? k_interp_rec<O::PS, O::PT, O::PP, true, R>
                                  : k_interp_rec<O::PS, O::PT, O::PP, false, R>;
      kern<<<g, 128, 0, s>>>(L.dev(), L.chunk, L.nchunk, b, e, blocks, P->ir, P->ii, P->err);
      return;
    }
    auto kern = P->kappa == 0.0 ? k_interp<O::PS, O::PT, O::PP, true, R>
                                : k_interp<O::PS, O::PT, O::PP, false, R>;
    kern<<<g, 128, 0, s>>>(L.dev(), L.chunk, L.nchunk, P->xs, P->ys, P->zs, P->kappa, b, e,
                           blocks, P->ir, P->ii, P->err);
  });
  ++P->launches;
}

void launch_pack(ifgf_plan* P, const double2* blocks, const uint32_t* cones, size_t m,
                 uint32_t nc, double* buf, int unpack, double2* blocks_out, cudaStream_t s) {
  if (!m) return;
  const int Pn = P->K.Pst;
  k_pack<<<blocks_for(m * Pn, 256), 256, 0, s>>>(blocks, cones, m, Pn, nc,
                                                 reinterpret_cast<double2*>(buf), unpack,
                                                 blocks_out, P->err);
  ++P->launches;
}

}  // namespace ifgf_b200
