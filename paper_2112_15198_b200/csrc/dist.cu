// dist.cu -- multi-GPU IFGF matvec behind the C ABI: the reference's rank
// algorithm (dist.cpp:241-361; PAPER.md "IFGF Method" in MPI form) with real
// per-level exchanges of cone-segment interpolant blocks.
//
// Layout (dist.cpp:78-130, partition_host): a rank owns a contiguous Morton
// interval of level-D boxes (its points) and, per level, an equal-count
// interval [c0, c1) of that level's cones -- whole boxes at fine levels,
// cone segments of one box split across ranks at coarse levels.  The octree
// and the relevant-cone structure are built on every rank (replicated
// setup, ~10 ms at C2); the interpolant BLOCKS are partitioned:
//
//   per level d, rank storage = the cones the rank owns + its halo, the
//   foreign cones it reads: the cones of its points seen from their cousins
//   (interpolation data, dist.cpp:179-201) and the child cones hit by the
//   nodes of its owned parent cones (propagation data, dist.cpp:206-237).
//   Slots follow the global cone order: [halo below c0 | owned | halo above].
//   The rank's level bitmap keeps only these cones, so the unchanged K3/K4
//   kernels' find_cone (bitmap word + prefix popcount) returns the local
//   slot directly, and a cone missing from the halo fails loudly
//   (kErrPropCover / kErrInterpCover) instead of reading a wrong block.
//
// Exchange (per level, once its blocks are final on every rank): each owner
// packs the blocks its peers asked for (k_pack over the owner's local slots)
// and one NCCL group of send/recv moves them over NVLink; the receiver's
// halo cones from one owner are contiguous slots, so they land in place (no
// unpack).  The request lists are exchanged once per plan.  NCCL's stream
// semantics order everything: pack after the level's kernels, the level's
// consumers after the group.  In-process rank groups (ifgf_run_distributed,
// the analogue of dist::run_distributed, used by the tests on one GPU) run
// the same partition, halos, pack kernel and slot layout with device copies
// in place of NCCL.
//
// Why not read foreign blocks straight from peer memory inside K3/K4 (no
// halo copy): at the coarse levels every point's ~45 cousin blocks are
// (R-1)/R foreign and are re-read by every point of a box; over NVLink
// without local L2 caching that is ~58 GB per C2 matvec, against the tens of
// MB a halo copy moves once.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"

namespace ifgf_b200 {

// --------------------------------------------------------------- NCCL (dlopen)
// Loaded on first use so single-GPU users of libifgf_b200.so never need it.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    auto sym = [&](const char* s) { return dlsym(a.h, s); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.h || !api.CommInitRank || !api.Send || !api.Recv || !api.GroupStart)
    throw Error(IFGF_ERUNTIME, "NCCL (libnccl.so.2) not loadable: multi-process rank groups "
                               "need it");
  return api;
}

#define IFGF_NCCL(call)                                                                          \
  do {                                                                                           \
    const ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                       \
      throw ::ifgf_b200::Error(IFGF_ERUNTIME, std::string("NCCL: ") +                            \
                                                  nccl().GetErrorString(r_) + " at " __FILE__ ":" + \
                                                  std::to_string(__LINE__));                     \
  } while (0)

}  // namespace ifgf_b200

static inline ncclComm_t nccl_of(const ifgf_comm* C) { return static_cast<ncclComm_t>(C->nccl); }

namespace ifgf_b200 {

struct DistLevel {
  uint32_t c0 = 0, c1 = 0;  // owned cone interval (global ordinals)
  uint32_t hb = 0;          // halo cones below c0
  uint32_t nh = 0;          // halo cones
  uint32_t nslot = 0;       // c1 - c0 + nh
  uint64_t interp_need = 0, prop_need = 0;  // per-kind foreign cones (CommStats counters)
  std::vector<uint32_t> recv_off;  // R+1: halo entries [recv_off[p], recv_off[p+1]) owned by p
  std::vector<uint32_t> send_off;  // R+1: my send list entries for requester r
  uint32_t* d_halo = nullptr;      // nh sorted global ordinals
  uint32_t* d_send = nullptr;      // send list: my local slots, concatenated over requesters
  double2* store = nullptr;        // nslot * Pst
  double2* sendbuf = nullptr;      // send_off[R] * Pst
  uint64_t* gbits = nullptr;       // the plan's global bitmap / prefix (restored on free)
  uint32_t* grank = nullptr;
  uint64_t* lbits = nullptr;       // the rank's bitmap / prefix of present cones
  uint32_t* lrank = nullptr;
  uint32_t slot_of(uint32_t j) const { return j < hb ? j : j + (c1 - c0); }
  // write base for owned cone q: slot = hb + q - c0
  double2* owned_base(int Pst) const {
    return store + (ptrdiff_t)((int64_t)hb - (int64_t)c0) * Pst;
  }
};

struct DistState {
  ifgf_comm* comm = nullptr;  // multi-process (NCCL); null in an in-process group
  int rank = 0, world = 1;
  std::vector<uint32_t> box_begin, point_begin;  // R+1
  std::vector<uint32_t> cone_begin;              // (D-2)*(R+1), level-major from d=3
  DistLevel lv[IFGF_MAX_LEVELS];
  size_t block_bytes = 0;
  double compute_seconds = 0.0;  // IFGF_DIST_RANK_TIMING (run_local_group)
  std::vector<cudaEvent_t> evs;  // scratch events of the in-process schedule
  ~DistState() {
    for (auto e : evs) cudaEventDestroy(e);
  }
};

namespace {

inline unsigned nblocks(size_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ int owner_of(uint32_t q, const uint32_t* cb, int R) {
  int r = 0;
  while (r < R - 1 && q >= cb[r + 1]) ++r;
  return r;
}

// dist.cpp:179-201: cones of level d holding (via cone_of_point) the rank's
// points as seen from their cousins; foreign ones flagged (bit 0).
__global__ void k_need_interp(const __grid_constant__ LevelDev L, const uint32_t* __restrict__ ptbox,
                              const double* xs, const double* ys, const double* zs, uint32_t p0,
                              uint32_t p1, const uint32_t* bounds, int R, int rank, uint8_t* need,
                              int* err) {
  const uint32_t i = p0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p1) return;
  const uint32_t b = ptbox[i];
  for (uint32_t k = L.cous_off[b]; k < L.cous_off[b + 1]; ++k) {
    const uint32_t cb = L.cous[k];
    uint32_t g;
    const int e = cone_of_point_fast(L, L.cx[cb], L.cy[cb], L.cz[cb], xs[i], ys[i], zs[i], g);
    if (e) {
      raise_err(err, e);
      return;
    }
    const uint32_t q = find_cone(L, cb, g);
    if (q == 0xffffffffu) {
      raise_err(err, kErrInterpCover);
      return;
    }
    if (owner_of(q, bounds, R) != rank) need[q] |= 1;
  }
}

// dist.cpp:206-237: child cones of level d hit by the nodes of the rank's
// parent cones [q0, q1) of level d-1 (bit 1).
__global__ void k_need_prop(const __grid_constant__ LevelDev L, const __grid_constant__ LevelDev U,
                            const __grid_constant__ InterpConsts K, uint32_t q0, uint32_t q1,
                            const uint32_t* bounds, int R, int rank, uint8_t* need, int* err) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)(q1 - q0) * K.P) return;
  const uint32_t q = q0 + (uint32_t)(t / K.P);
  const int m = (int)(t % K.P);
  const int jp = m % K.pp, jt = (m / K.pp) % K.pt, js = m / (K.pp * K.pt);
  const uint32_t pb = U.cone_box[q];
  const SegMid sg = segment_mid(U, U.cone_gamma[q]);
  double x, y, z;
  node_position(sg, U.rad, U.cx[pb], U.cy[pb], U.cz[pb], K.ns[js], K.nt[jt], K.np[jp], x, y, z);
  for (uint32_t cb = U.child_begin[pb]; cb < U.child_begin[pb + 1]; ++cb) {
    uint32_t g;
    const int e = cone_of_point_fast(L, L.cx[cb], L.cy[cb], L.cz[cb], x, y, z, g);
    if (e) {
      raise_err(err, e);
      return;
    }
    const uint32_t cq = find_cone(L, cb, g);
    if (cq == 0xffffffffu) {
      raise_err(err, kErrPropCover);
      return;
    }
    if (owner_of(cq, bounds, R) != rank) need[cq] |= 2;
  }
}

// counts of the two kinds and of their union
__global__ void k_need_count(const uint8_t* need, uint32_t nc, unsigned long long* cnt) {
  uint32_t a = 0, b = 0, u = 0;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nc; q += gridDim.x * blockDim.x) {
    const uint8_t v = need[q];
    a += v & 1;
    b += (v >> 1) & 1;
    u += v != 0;
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    u += __shfl_xor_sync(0xffffffffu, u, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&cnt[0], a);
    atomicAdd(&cnt[1], b);
    atomicAdd(&cnt[2], u);
  }
}

struct NeedFlag {
  const uint8_t* need;
  __device__ __forceinline__ bool operator()(uint32_t q) const { return need[q] != 0; }
};

// local bitmap: the owned interval and the halo cones of a level
__global__ void k_local_bits(const __grid_constant__ LevelDev L, uint32_t c0, uint32_t c1,
                             const uint32_t* halo, uint32_t nh, uint64_t* bits) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t no = c1 - c0;
  if (t >= no + nh) return;
  const uint32_t q = t < no ? c0 + t : halo[t - no];
  const uint64_t idx = (uint64_t)L.cone_box[q] * L.G + L.cone_gamma[q];
  atomicOr((unsigned long long*)(bits + (idx >> 6)), 1ull << (idx & 63));
}

__global__ void k_popc_words(const uint64_t* bits, size_t nw, uint32_t* cnt) {
  const size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (w < nw) cnt[w] = __popcll(bits[w]);
  else if (w == nw) cnt[w] = 0;
}

// requested global ordinals -> this rank's local slots (owned: hb + q - c0)
__global__ void k_to_slots(uint32_t* v, size_t m, uint32_t c0, uint32_t c1, uint32_t hb, int* err) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t q = v[i];
  if (q < c0 || q >= c1) {
    raise_err(err, kErrBadCone);
    v[i] = 0;
    return;
  }
  v[i] = hb + (q - c0);
}

template <class T>
T* dalloc(ifgf_plan* P, size_t n) {
  return P->alloc<T>(n ? n : 1);
}

}  // namespace

// ------------------------------------------------------------------ building
// Phase 1 (every rank alone): layout, need sets, halo, local bitmaps, storage.
void dist_prepare(ifgf_plan* P, int R, int rank) {
  static const bool trace = std::getenv("IFGF_ALLOC_TRACE") != nullptr;
  const auto tp0 = std::chrono::steady_clock::now();
  struct TraceEnd {
    bool on;
    std::chrono::steady_clock::time_point t0;
    ~TraceEnd() {
      if (on)
        std::fprintf(stderr, "[dist_prepare] %8.3f ms\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);
    }
  } trace_end{trace, tp0};
  auto* S = new DistState;
  P->dist = S;
  S->rank = rank;
  S->world = R;
  const int D = P->depth;
  cudaStream_t s = P->s_main;
  S->box_begin.resize(R + 1);
  S->point_begin.resize(R + 1);
  S->cone_begin.resize((size_t)(D - 2) * (R + 1));
  partition_host(P, R, S->box_begin.data(), S->point_begin.data(), S->cone_begin.data());
  const int Pst = P->K.Pst;
  const uint32_t p0 = S->point_begin[rank], p1 = S->point_begin[rank + 1];
  uint32_t* d_cb = dalloc<uint32_t>(P, S->cone_begin.size());
  IFGF_CUDA(cudaMemcpyAsync(d_cb, S->cone_begin.data(), S->cone_begin.size() * 4,
                            cudaMemcpyHostToDevice, s));
  unsigned long long* d_cnt = dalloc<unsigned long long>(P, 3 * (D + 1));
  IFGF_CUDA(cudaMemsetAsync(d_cnt, 0, 3 * (D + 1) * sizeof(unsigned long long), s));
  size_t need_max = 0;
  for (int d = 3; d <= D; ++d) need_max = std::max<size_t>(need_max, P->lv[d].nc);
  uint8_t* need = dalloc<uint8_t>(P, need_max + 1);
  uint32_t* nsel = dalloc<uint32_t>(P, 1);
  std::vector<unsigned long long> cnt(3 * (D + 1), 0);
  for (int d = 3; d <= D; ++d) {
    Level& L = P->lv[d];
    DistLevel& V = S->lv[d];
    const uint32_t* cb = S->cone_begin.data() + (size_t)(d - 3) * (R + 1);
    V.c0 = cb[rank];
    V.c1 = cb[rank + 1];
    IFGF_CUDA(cudaMemsetAsync(need, 0, L.nc + 1, s));
    const uint32_t* d_cbl = d_cb + (size_t)(d - 3) * (R + 1);
    if (R > 1 && p1 > p0) {
      k_need_interp<<<nblocks(p1 - p0, 128), 128, 0, s>>>(L.dev(), L.ptbox, P->xs, P->ys, P->zs,
                                                         p0, p1, d_cbl, R, rank, need, P->err);
      ++P->launches;
    }
    if (R > 1 && d > 3) {
      const uint32_t* cu = S->cone_begin.data() + (size_t)(d - 4) * (R + 1);
      const uint32_t q0 = cu[rank], q1 = cu[rank + 1];
      const size_t work = (size_t)(q1 - q0) * P->K.P;
      if (work) {
        k_need_prop<<<nblocks(work, 128), 128, 0, s>>>(L.dev(), P->lv[d - 1].dev(), P->K, q0, q1,
                                                       d_cbl, R, rank, need, P->err);
        ++P->launches;
      }
    }
    k_need_count<<<std::min<unsigned>(nblocks(L.nc, 256), 1184), 256, 0, s>>>(need, L.nc,
                                                                          d_cnt + 3 * d);
    ++P->launches;
    IFGF_CUDA(cudaMemcpyAsync(&cnt[3 * d], d_cnt + 3 * d, 3 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaStreamSynchronize(s));
    check_device_error(P);
    V.interp_need = cnt[3 * d];
    V.prop_need = cnt[3 * d + 1];
    V.nh = (uint32_t)cnt[3 * d + 2];
    V.nslot = V.c1 - V.c0 + V.nh;
    // halo = the flagged cones in ascending order
    V.d_halo = dalloc<uint32_t>(P, V.nh);
    {
      cub::CountingInputIterator<uint32_t> it(0);
      cub::TransformInputIterator<bool, NeedFlag, cub::CountingInputIterator<uint32_t>> fl(
          it, NeedFlag{need});
      size_t tb = 0;
      cub::DeviceSelect::Flagged(nullptr, tb, it, fl, V.d_halo, nsel, (int)L.nc, s);
      void* tmp = nullptr;
      IFGF_CUDA(cudaMallocAsync(&tmp, tb ? tb : 16, s));
      IFGF_CUDA(cub::DeviceSelect::Flagged(tmp, tb, it, fl, V.d_halo, nsel, (int)L.nc, s));
      IFGF_CUDA(cudaFreeAsync(tmp, s));
    }
    // owners' ranges in the sorted halo (owner intervals are contiguous)
    std::vector<uint32_t> halo(V.nh);
    if (V.nh)
      IFGF_CUDA(cudaMemcpyAsync(halo.data(), V.d_halo, V.nh * 4, cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaStreamSynchronize(s));
    V.recv_off.assign(R + 1, 0);
    for (int p = 0; p <= R; ++p)
      V.recv_off[p] = p == R ? V.nh
                             : (uint32_t)(std::lower_bound(halo.begin(), halo.end(), cb[p]) -
                                          halo.begin());
    V.hb = V.recv_off[rank];
    if (V.recv_off[rank + 1] != V.hb)
      throw Error(IFGF_ELOGIC, "dist: a rank's halo contains its own cones");
    // storage and the rank's bitmap of present cones
    // every slot is written each apply (owned: K2/K3, halo: the exchange)
    V.store = dalloc<double2>(P, (size_t)V.nslot * Pst + 2);
    S->block_bytes += (size_t)V.nslot * Pst * sizeof(double2);
    uint64_t* lb = dalloc<uint64_t>(P, L.nwords);
    uint32_t* lr = dalloc<uint32_t>(P, L.nwords + 1);
    uint32_t* wc = dalloc<uint32_t>(P, L.nwords + 1);
    IFGF_CUDA(cudaMemsetAsync(lb, 0, L.nwords * 8, s));
    if (V.nslot) {
      k_local_bits<<<nblocks(V.nslot, 256), 256, 0, s>>>(L.dev(), V.c0, V.c1, V.d_halo, V.nh, lb);
      ++P->launches;
    }
    k_popc_words<<<nblocks(L.nwords + 1, 256), 256, 0, s>>>(lb, L.nwords, wc);
    ++P->launches;
    {
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, wc, lr, (int)(L.nwords + 1), s);
      void* tmp = nullptr;
      IFGF_CUDA(cudaMallocAsync(&tmp, tb ? tb : 16, s));
      IFGF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, wc, lr, (int)(L.nwords + 1), s));
      IFGF_CUDA(cudaFreeAsync(tmp, s));
    }
    V.gbits = L.bits;
    V.grank = L.rank;
    V.lbits = lb;
    V.lrank = lr;
  }
  IFGF_CUDA(cudaStreamSynchronize(s));
  // the apply kernels look cones up in the rank's bitmaps from here on: the
  // unchanged find_cone returns local slots, absent cones fail loudly
  for (int d = 3; d <= D; ++d) {
    P->lv[d].bits = S->lv[d].lbits;
    P->lv[d].rank = S->lv[d].lrank;
  }
  // K4 locate records of the rank's own points (ordinals = local block slots)
  build_rank_records(P, p0, p1);
}

namespace {

// Phase 2, multi-process: tell every owner which of its cones this rank needs
// (counts, then lists, all levels in one NCCL group each) and turn the
// received requests into this rank's pack lists.
void connect_nccl(ifgf_plan* P, DistState* S) {
  const int R = S->world, me = S->rank, D = P->depth;
  ifgf_comm* C = S->comm;
  cudaStream_t s = P->s_main;
  NcclApi& N = nccl();
  const int L = D - 2;
  // counts: out[d][p] = cones I need from p; in[d][r] = cones r needs from me
  std::vector<uint32_t> h_out((size_t)L * R, 0), h_in((size_t)L * R, 0);
  for (int d = 3; d <= D; ++d)
    for (int p = 0; p < R; ++p)
      h_out[(size_t)(d - 3) * R + p] = S->lv[d].recv_off[p + 1] - S->lv[d].recv_off[p];
  uint32_t* d_out = dalloc<uint32_t>(P, h_out.size());
  uint32_t* d_in = dalloc<uint32_t>(P, h_in.size());
  IFGF_CUDA(cudaMemcpyAsync(d_out, h_out.data(), h_out.size() * 4, cudaMemcpyHostToDevice, s));
  IFGF_CUDA(cudaMemsetAsync(d_in, 0, h_in.size() * 4, s));
  IFGF_NCCL(N.GroupStart());
  for (int d = 3; d <= D; ++d)
    for (int p = 0; p < R; ++p) {
      if (p == me) continue;
      const size_t k = (size_t)(d - 3) * R + p;
      IFGF_NCCL(N.Send(d_out + k, 1, ncclUint32, p, nccl_of(C), s));
      IFGF_NCCL(N.Recv(d_in + k, 1, ncclUint32, p, nccl_of(C), s));
    }
  IFGF_NCCL(N.GroupEnd());
  IFGF_CUDA(cudaMemcpyAsync(h_in.data(), d_in, h_in.size() * 4, cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  // lists
  for (int d = 3; d <= D; ++d) {
    DistLevel& V = S->lv[d];
    V.send_off.assign(R + 1, 0);
    for (int r = 0; r < R; ++r) V.send_off[r + 1] = V.send_off[r] + h_in[(size_t)(d - 3) * R + r];
    V.d_send = dalloc<uint32_t>(P, V.send_off[R]);
    V.sendbuf = dalloc<double2>(P, (size_t)V.send_off[R] * P->K.Pst);
  }
  IFGF_NCCL(N.GroupStart());
  for (int d = 3; d <= D; ++d) {
    DistLevel& V = S->lv[d];
    for (int p = 0; p < R; ++p) {
      if (p == me) continue;
      const uint32_t no = V.recv_off[p + 1] - V.recv_off[p];
      if (no) IFGF_NCCL(N.Send(V.d_halo + V.recv_off[p], no, ncclUint32, p, nccl_of(C), s));
      const uint32_t ni = V.send_off[p + 1] - V.send_off[p];
      if (ni) IFGF_NCCL(N.Recv(V.d_send + V.send_off[p], ni, ncclUint32, p, nccl_of(C), s));
    }
  }
  IFGF_NCCL(N.GroupEnd());
  for (int d = 3; d <= D; ++d) {
    DistLevel& V = S->lv[d];
    if (V.send_off[R]) {
      k_to_slots<<<nblocks(V.send_off[R], 256), 256, 0, s>>>(V.d_send, V.send_off[R], V.c0, V.c1,
                                                             V.hb, P->err);
      ++P->launches;
    }
  }
  IFGF_CUDA(cudaStreamSynchronize(s));
  check_device_error(P);
}

// Phase 2, in-process group: the same lists read from the peers directly.
void connect_local(std::vector<ifgf_plan*>& G) {
  const int R = (int)G.size();
  for (int me = 0; me < R; ++me) {
    ifgf_plan* P = G[me];
    DistState* S = P->dist;
    cudaStream_t s = P->s_main;
    IFGF_CUDA(cudaSetDevice(P->device));
    for (int d = 3; d <= P->depth; ++d) {
      DistLevel& V = S->lv[d];
      V.send_off.assign(R + 1, 0);
      for (int r = 0; r < R; ++r) {
        const DistLevel& W = G[r]->dist->lv[d];
        V.send_off[r + 1] = V.send_off[r] + (r == me ? 0 : W.recv_off[me + 1] - W.recv_off[me]);
      }
      V.d_send = dalloc<uint32_t>(P, V.send_off[R]);
      V.sendbuf = dalloc<double2>(P, (size_t)V.send_off[R] * P->K.Pst);
      for (int r = 0; r < R; ++r) {
        const uint32_t m = V.send_off[r + 1] - V.send_off[r];
        if (!m) continue;
        const DistLevel& W = G[r]->dist->lv[d];
        IFGF_CUDA(cudaMemcpyAsync(V.d_send + V.send_off[r], W.d_halo + W.recv_off[me], m * 4,
                                  cudaMemcpyDefault, s));
      }
      if (V.send_off[R]) {
        k_to_slots<<<nblocks(V.send_off[R], 256), 256, 0, s>>>(V.d_send, V.send_off[R], V.c0,
                                                               V.c1, V.hb, P->err);
        ++P->launches;
      }
    }
  }
  for (ifgf_plan* P : G) {
    IFGF_CUDA(cudaSetDevice(P->device));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
    check_device_error(P);
  }
}

}  // namespace

// ------------------------------------------------------------------ apply
namespace {

void pack_level(ifgf_plan* P, int d, cudaStream_t s) {
  DistLevel& V = P->dist->lv[d];
  const int R = P->dist->world;
  if (V.send_off[R])
    launch_pack(P, V.store, V.d_send, V.send_off[R], V.nslot, reinterpret_cast<double*>(V.sendbuf),
                0, nullptr, s);
}

void exchange_nccl(ifgf_plan* P, int d, cudaStream_t s) {
  DistState* S = P->dist;
  DistLevel& V = S->lv[d];
  const int R = S->world, me = S->rank;
  const size_t bd = 2 * (size_t)P->K.Pst;  // doubles per block
  pack_level(P, d, s);
  NcclApi& N = nccl();
  IFGF_NCCL(N.GroupStart());
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    const uint32_t ns = V.send_off[p + 1] - V.send_off[p];
    if (ns)
      IFGF_NCCL(N.Send(reinterpret_cast<const double*>(V.sendbuf) + V.send_off[p] * bd, ns * bd,
                       ncclFloat64, p, nccl_of(S->comm), s));
    const uint32_t nr = V.recv_off[p + 1] - V.recv_off[p];
    if (nr)
      IFGF_NCCL(N.Recv(reinterpret_cast<double*>(V.store) + (size_t)V.slot_of(V.recv_off[p]) * bd,
                       nr * bd, ncclFloat64, p, nccl_of(S->comm), s));
  }
  IFGF_NCCL(N.GroupEnd());
}

// owned sorted results to every rank, then the caller's order
void gather_results_nccl(ifgf_plan* P, double* o_re, double* o_im, cudaStream_t s) {
  DistState* S = P->dist;
  const int R = S->world, me = S->rank;
  NcclApi& N = nccl();
  const uint32_t p0 = S->point_begin[me], p1 = S->point_begin[me + 1];
  IFGF_NCCL(N.GroupStart());
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    if (p1 > p0) {
      IFGF_NCCL(N.Send(P->ir + p0, p1 - p0, ncclFloat64, p, nccl_of(S->comm), s));
      IFGF_NCCL(N.Send(P->ii + p0, p1 - p0, ncclFloat64, p, nccl_of(S->comm), s));
    }
    const uint32_t b = S->point_begin[p], e = S->point_begin[p + 1];
    if (e > b) {
      IFGF_NCCL(N.Recv(P->ir + b, e - b, ncclFloat64, p, nccl_of(S->comm), s));
      IFGF_NCCL(N.Recv(P->ii + b, e - b, ncclFloat64, p, nccl_of(S->comm), s));
    }
  }
  IFGF_NCCL(N.GroupEnd());
  launch_scatter_result(P, o_re, o_im, s);
}

}  // namespace

// One rank's apply (multi-process), every kernel stream-ordered against the
// NCCL groups: s_main = gather, K2, X(D), K3(D), X(D-1), ..., K3(4), X(3),
// result all-gather + scatter; s_aux = K1, K4(D..3), each K4(d) after X(d).
void dist_apply_device(ifgf_plan* P, const double* a_re, const double* a_im, double* i_re,
                       double* i_im, cudaStream_t caller, ifgf_report* rep) {
  DistState* S = P->dist;
  if (!S || !S->comm) throw Error(IFGF_EINVAL, "dist apply: not a multi-process rank plan");
  const auto t0 = std::chrono::steady_clock::now();
  IFGF_CUDA(cudaSetDevice(P->device));
  const int D = P->depth, me = S->rank, Pst = P->K.Pst;
  const size_t launches0 = P->launches;
  cudaStream_t sm = P->s_main, sa = P->s_aux;
  std::vector<cudaEvent_t> evs;
  auto mk = [&]() {
    cudaEvent_t e;
    IFGF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evs.push_back(e);
    return e;
  };
  struct Guard {
    std::vector<cudaEvent_t>& v;
    ~Guard() {
      for (auto e : v) cudaEventDestroy(e);
    }
  } guard{evs};
  const uint32_t p0 = S->point_begin[me], p1 = S->point_begin[me + 1];
  cudaEvent_t start = mk();
  IFGF_CUDA(cudaEventRecord(start, caller));
  IFGF_CUDA(cudaStreamWaitEvent(sm, start, 0));
  launch_gather_density(P, a_re, a_im, sm);
  cudaEvent_t g = mk();
  IFGF_CUDA(cudaEventRecord(g, sm));
  IFGF_CUDA(cudaStreamWaitEvent(sa, g, 0));
  launch_singular(P, p0, p1, sa);
  {
    const DistLevel& V = S->lv[D];
    launch_level_d(P, V.c0, V.c1, V.owned_base(Pst), sm);
  }
  exchange_nccl(P, D, sm);
  for (int d = D; d >= 3; --d) {
    cudaEvent_t x = mk();
    IFGF_CUDA(cudaEventRecord(x, sm));
    IFGF_CUDA(cudaStreamWaitEvent(sa, x, 0));
    launch_interpolation(P, d, p0, p1, S->lv[d].store, sa);
    if (d > 3) {
      const DistLevel& U = S->lv[d - 1];
      launch_propagation(P, d, U.c0, U.c1, S->lv[d].store, U.owned_base(Pst), sm);
      exchange_nccl(P, d - 1, sm);
    }
  }
  cudaEvent_t k4 = mk();
  IFGF_CUDA(cudaEventRecord(k4, sa));
  IFGF_CUDA(cudaStreamWaitEvent(sm, k4, 0));
  gather_results_nccl(P, i_re, i_im, sm);
  cudaEvent_t done = mk();
  IFGF_CUDA(cudaEventRecord(done, sm));
  IFGF_CUDA(cudaGetLastError());
  IFGF_CUDA(cudaStreamWaitEvent(caller, done, 0));
  IFGF_CUDA(cudaEventSynchronize(done));
  check_device_error(P);
  if (rep) {
    std::memset(rep, 0, sizeof *rep);
    rep->total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep->depth = D;
    rep->n = P->n;
    rep->h_level_d = P->lv[D].h;
    rep->n_levels = D - 2;
    for (int d = 3; d <= D; ++d) {
      rep->level_boxes[d - 3] = P->lv[d].nb;
      rep->level_cones[d - 3] = P->lv[d].nc;
    }
    rep->peak_live_blocks = S->block_bytes / (Pst * sizeof(double2));
    rep->gpu_launches = P->launches - launches0;
  }
}

// ifgf_run_distributed: R rank plans in this process, advanced phase by phase
// across ranks (no kernel ever waits on another rank's pending kernel), the
// exchanges as device copies from the owners' pack buffers.  Host in/out.
void run_local_group(std::vector<ifgf_plan*>& G, const double* a_re, const double* a_im,
                     double* i_re, double* i_im, ifgf_report* rep) {
  const int R = (int)G.size();
  ifgf_plan* P0 = G[0];
  const int D = P0->depth, Pst = P0->K.Pst;
  const size_t n = P0->n;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<double*> dens(R, nullptr);
  for (int r = 0; r < R; ++r) {
    ifgf_plan* P = G[r];
    IFGF_CUDA(cudaSetDevice(P->device));
    double* buf = P->staging ? P->staging : (P->staging = P->alloc<double>(2 * n));
    IFGF_CUDA(cudaMemcpyAsync(buf, a_re, n * 8, cudaMemcpyHostToDevice, P->s_main));
    if (a_im) IFGF_CUDA(cudaMemcpyAsync(buf + n, a_im, n * 8, cudaMemcpyHostToDevice, P->s_main));
    dens[r] = buf;
  }
  auto ev_on = [&](ifgf_plan* P, cudaStream_t s) {
    cudaEvent_t e;
    IFGF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P->dist->evs.push_back(e);
    IFGF_CUDA(cudaEventRecord(e, s));
    return e;
  };
  auto exchange_all = [&](int d) {
    std::vector<cudaEvent_t> packed(R);
    for (int r = 0; r < R; ++r) {
      ifgf_plan* P = G[r];
      IFGF_CUDA(cudaSetDevice(P->device));
      pack_level(P, d, P->s_main);
      packed[r] = ev_on(P, P->s_main);
    }
    for (int r = 0; r < R; ++r) {
      ifgf_plan* P = G[r];
      IFGF_CUDA(cudaSetDevice(P->device));
      DistLevel& V = P->dist->lv[d];
      for (int p = 0; p < R; ++p) {
        const uint32_t nr = V.recv_off[p + 1] - V.recv_off[p];
        if (p == r || !nr) continue;
        const DistLevel& W = G[p]->dist->lv[d];
        IFGF_CUDA(cudaStreamWaitEvent(P->s_main, packed[p], 0));
        IFGF_CUDA(cudaMemcpyAsync(V.store + (size_t)V.slot_of(V.recv_off[p]) * Pst,
                                  W.sendbuf + (size_t)W.send_off[r] * Pst,
                                  (size_t)nr * Pst * sizeof(double2), cudaMemcpyDefault,
                                  P->s_main));
      }
    }
  };
  // IFGF_DIST_RANK_TIMING=1: ranks' compute phases serialised and timed one
  // by one (the load-balance measure of ifgf_dist_info.compute_seconds;
  // exchanges excluded), else ranks overlap on the device(s)
  static const bool timing = [] {
    const char* v = std::getenv("IFGF_DIST_RANK_TIMING");
    return v && std::atoi(v) != 0;
  }();
  std::vector<double> secs(R, 0.0);
  std::chrono::steady_clock::time_point tr;
  auto t_begin = [&](ifgf_plan* P) {
    if (!timing) return;
    IFGF_CUDA(cudaDeviceSynchronize());
    tr = std::chrono::steady_clock::now();
    (void)P;
  };
  auto t_end = [&](int r) {
    if (!timing) return;
    IFGF_CUDA(cudaDeviceSynchronize());
    secs[r] += std::chrono::duration<double>(std::chrono::steady_clock::now() - tr).count();
  };
  for (int r = 0; r < R; ++r) {
    ifgf_plan* P = G[r];
    DistState* S = P->dist;
    IFGF_CUDA(cudaSetDevice(P->device));
    t_begin(P);
    launch_gather_density(P, dens[r], a_im ? dens[r] + n : nullptr, P->s_main);
    IFGF_CUDA(cudaStreamWaitEvent(P->s_aux, ev_on(P, P->s_main), 0));
    launch_singular(P, S->point_begin[r], S->point_begin[r + 1], P->s_aux);
    launch_level_d(P, S->lv[D].c0, S->lv[D].c1, S->lv[D].owned_base(Pst), P->s_main);
    t_end(r);
  }
  exchange_all(D);
  for (int d = D; d >= 3; --d) {
    for (int r = 0; r < R; ++r) {
      ifgf_plan* P = G[r];
      DistState* S = P->dist;
      IFGF_CUDA(cudaSetDevice(P->device));
      t_begin(P);
      IFGF_CUDA(cudaStreamWaitEvent(P->s_aux, ev_on(P, P->s_main), 0));
      launch_interpolation(P, d, S->point_begin[r], S->point_begin[r + 1], S->lv[d].store,
                           P->s_aux);
      if (d > 3) {
        const DistLevel& U = S->lv[d - 1];
        launch_propagation(P, d, U.c0, U.c1, S->lv[d].store, U.owned_base(Pst), P->s_main);
      }
      t_end(r);
    }
    if (d > 3) exchange_all(d - 1);
  }
  std::vector<double> sr(n, 0.0), si(n, 0.0);
  for (int r = 0; r < R; ++r) {
    ifgf_plan* P = G[r];
    DistState* S = P->dist;
    IFGF_CUDA(cudaSetDevice(P->device));
    IFGF_CUDA(cudaStreamWaitEvent(P->s_main, ev_on(P, P->s_aux), 0));
    const uint32_t b = S->point_begin[r], e = S->point_begin[r + 1];
    if (e > b) {
      IFGF_CUDA(cudaMemcpyAsync(sr.data() + b, P->ir + b, (e - b) * 8, cudaMemcpyDeviceToHost,
                                P->s_main));
      IFGF_CUDA(cudaMemcpyAsync(si.data() + b, P->ii + b, (e - b) * 8, cudaMemcpyDeviceToHost,
                                P->s_main));
    }
  }
  for (int r = 0; r < R; ++r) {
    IFGF_CUDA(cudaSetDevice(G[r]->device));
    IFGF_CUDA(cudaStreamSynchronize(G[r]->s_main));
    check_device_error(G[r]);
    for (auto e : G[r]->dist->evs) cudaEventDestroy(e);
    G[r]->dist->evs.clear();
  }
  for (int r = 0; r < R; ++r) G[r]->dist->compute_seconds = secs[r];
  std::vector<uint32_t> perm(n);
  IFGF_CUDA(cudaSetDevice(P0->device));
  IFGF_CUDA(cudaMemcpy(perm.data(), P0->perm, n * 4, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    i_re[perm[i]] = sr[i];
    i_im[perm[i]] = si[i];
  }
  if (rep) {
    std::memset(rep, 0, sizeof *rep);
    rep->total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep->depth = D;
    rep->n = n;
    rep->h_level_d = P0->lv[D].h;
    rep->n_levels = D - 2;
    size_t peak = 0;
    for (int d = 3; d <= D; ++d) {
      rep->level_boxes[d - 3] = P0->lv[d].nb;
      rep->level_cones[d - 3] = P0->lv[d].nc;
    }
    for (ifgf_plan* P : G) {
      peak = std::max(peak, P->dist->block_bytes / (Pst * sizeof(double2)));
      rep->gpu_launches += P->launches;
    }
    rep->peak_live_blocks = peak;
  }
}

void dist_connect(ifgf_plan* P) { connect_nccl(P, P->dist); }
void dist_connect_local(std::vector<ifgf_plan*>& G) { connect_local(G); }

void dist_free(ifgf_plan* P) {
  if (!P->dist) return;
  // restore the global bitmaps (the plan frees every allocation itself)
  for (int d = 3; d <= P->depth; ++d)
    if (P->dist->lv[d].gbits) {
      P->lv[d].bits = P->dist->lv[d].gbits;
      P->lv[d].rank = P->dist->lv[d].grank;
    }
  delete P->dist;
  P->dist = nullptr;
}

ifgf_comm* comm_create(const void* id, int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(IFGF_EINVAL, "comm: bad rank/world");
  if (!id) throw Error(IFGF_EINVAL, "comm: null unique id");
  NcclApi& N = nccl();
  auto C = std::make_unique<ifgf_comm>();
  C->rank = rank;
  C->world = world;
  C->device = device;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  IFGF_CUDA(cudaSetDevice(device));
  ncclComm_t nc = nullptr;
  IFGF_NCCL(N.CommInitRank(&nc, world, uid, rank));
  C->nccl = nc;
  return C.release();
}

void comm_unique_id(void* out) {
  NcclApi& N = nccl();
  ncclUniqueId uid;
  IFGF_NCCL(N.GetUniqueId(&uid));
  std::memcpy(out, &uid, sizeof uid);
}

void comm_destroy(ifgf_comm* C) {
  if (!C) return;
  if (C->nccl) {
    cudaSetDevice(C->device);
    nccl().CommDestroy(nccl_of(C));
  }
  delete C;
}

}  // namespace ifgf_b200

namespace ifgf_b200 {

// Exchange sets of one rank and kind (ifgf_plan_exchange_set): kind 0 over the
// sorted points [lo, hi), kind 1 over the parent cones [lo, hi) of level d-1.
void launch_need(ifgf_plan* P, int d, int kind, const uint32_t* d_bounds, int R, int rank,
                 uint32_t lo, uint32_t hi, uint8_t* need, cudaStream_t s) {
  const Level& L = P->lv[d];
  if (hi <= lo) return;
  if (kind == 0) {
    k_need_interp<<<nblocks(hi - lo, 128), 128, 0, s>>>(L.dev(), L.ptbox, P->xs, P->ys, P->zs, lo,
                                                       hi, d_bounds, R, rank, need, P->err);
  } else {
    const size_t work = (size_t)(hi - lo) * P->K.P;
    k_need_prop<<<nblocks(work, 128), 128, 0, s>>>(L.dev(), P->lv[d - 1].dev(), P->K, lo, hi,
                                                   d_bounds, R, rank, need, P->err);
  }
  ++P->launches;
}

void comm_attach(ifgf_plan* P, ifgf_comm* C) { P->dist->comm = C; }

void dist_fill_info(const ifgf_plan* P, ifgf_dist_info* info) {
  std::memset(info, 0, sizeof *info);
  const DistState* S = P->dist;
  if (!S) throw Error(IFGF_EINVAL, "dist_info: not a rank plan");
  info->rank = S->rank;
  info->world = S->world;
  info->point_begin = S->point_begin[S->rank];
  info->point_end = S->point_begin[S->rank + 1];
  info->depth = P->depth;
  for (int d = 3; d <= P->depth; ++d) {
    const DistLevel& V = S->lv[d];
    ifgf_dist_level& o = info->levels[d - 3];
    o.owned_cones = V.c1 - V.c0;
    o.halo_cones = V.nh;
    o.interp_needed = V.interp_need;
    o.prop_needed = V.prop_need;
    o.sent_cones = V.send_off.empty() ? 0 : V.send_off.back();
  }
  info->block_bytes = S->block_bytes;
  info->device_bytes = P->bytes;
  info->compute_seconds = S->compute_seconds;
}

}  // namespace ifgf_b200
