// capi.cu -- the C ABI (include/ifgf_b200.h): plan lifecycle, the apply
// orchestration (engine.cpp:260-325) on two CUDA streams, the pass-level API
// (engine.hpp:91-110), structure export, rank layout and exchange sets
// (dist.cpp:78-237), and the device-side direct sums.
//
// Apply schedule (one plan, one GPU):
//   s_main: gather densities -> K2 level-D blocks -> K3(D) -> K3(D-1) -> ... -> K3(4)
//   s_aux : K1 near field -> K4(D) -> K4(D-1) -> ... -> K4(3)        (all += into i)
//   K4(d) waits for "blocks of level d ready"; K3(d) overwrites the slot of
//   level d-1+n_slots and therefore waits for K4 of that level.  With one slot
//   per level (the default whenever the blocks fit) K3 never waits on K4, so
//   propagation and interpolation of a level overlap.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "plan.hpp"

using namespace ifgf_b200;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return IFGF_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return IFGF_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return IFGF_ERUNTIME;
  }
}

using clk = std::chrono::steady_clock;
double since(clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); }

void tune_pool(int device);

void require_device(int device) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw Error(IFGF_ERUNTIME, std::string("no CUDA device visible (") +
                                   (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                                   "); libifgf_b200 has no CPU path");
  if (device < 0 || device >= count) throw Error(IFGF_EINVAL, "device ordinal out of range");
  // cudaGetDeviceProperties costs ~1 ms per call: query the major version only
  int major = 0;
  IFGF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) {
    cudaDeviceProp prop;
    IFGF_CUDA(cudaGetDeviceProperties(&prop, device));
    throw Error(IFGF_ERUNTIME, std::string("device ") + prop.name +
                                   " is not sm_100 (this build targets sm_100a only)");
  }
  IFGF_CUDA(cudaSetDevice(device));
  tune_pool(device);
}

// Keep freed stream-ordered memory in each device's default pool (a release
// threshold of 0 returns it to the driver at every sync point: 20-80 ms setup
// spikes).  Once per device ordinal.
void tune_pool(int device) {
  static std::mutex mu;
  static uint64_t tuned = 0;  // bit per device ordinal
  if (device < 0 || device >= 64) return;
  std::lock_guard<std::mutex> g(mu);
  if (tuned >> device & 1) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  tuned |= 1ull << device;
}

// Restores the caller's current device when an entry point returns (the C
// ABI switches to the plan's device internally).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Device memory a new plan may count on.  cudaMemGetInfo stalls for 10-78 ms
// in a good fraction of calls while other driver clients are active (NCCL's
// proxy thread, the NVML sampler; IFGF_ALLOC_TRACE,
// profiles/r02/meminfo_spikes_c2.log), which was the whole setup-time
// spread.  So it is sampled at most every 30 s per device; in between the
// budget follows the stream-ordered pool's own counters (cheap attribute
// reads): free memory at the sample, plus what the pool had reserved then,
// minus what the pool has in use now.  Allocations by other allocators
// after the sample are not seen, so the block-storage decision also
// recovers from an out-of-memory by falling back to two rotating slots.
size_t device_memory_budget(int device) {
  struct Sample {
    bool valid = false;
    size_t free = 0;
    uint64_t reserved = 0;
    clk::time_point when;
  };
  static std::mutex mu;
  static Sample cache[64];
  auto pool_counters = [&](uint64_t& reserved, uint64_t& used) {
    reserved = used = 0;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
  };
  std::lock_guard<std::mutex> g(mu);
  Sample& c = cache[device >= 0 && device < 64 ? device : 0];
  uint64_t reserved = 0, used = 0;
  if (!c.valid || since(c.when) > 30.0) {
    static const bool trace = std::getenv("IFGF_ALLOC_TRACE") != nullptr;
    const auto t0 = clk::now();
    size_t fr = 0, tot = 0;
    IFGF_CUDA(cudaMemGetInfo(&fr, &tot));
    if (trace) std::fprintf(stderr, "[meminfo] %8.3f ms\n", since(t0) * 1e3);
    pool_counters(reserved, used);
    c = {true, fr, reserved, clk::now()};
  }
  pool_counters(reserved, used);
  const uint64_t have = (uint64_t)c.free + c.reserved;
  return have > used ? (size_t)(have - used) : 0;
}

void validate_params(const ifgf_params* p) {
  if (!p) throw Error(IFGF_EINVAL, "null params");
  if (p->p_s < 1 || p->p_theta < 1 || p->p_phi < 1 || p->p_s > kMaxOrder ||
      p->p_theta > kMaxOrder || p->p_phi > kMaxOrder)
    throw Error(IFGF_EINVAL, "unsupported interpolation orders");
  if (!orders_supported(p->p_s, p->p_theta, p->p_phi))
    throw Error(IFGF_EINVAL, "interpolation orders (" + std::to_string(p->p_s) + "," +
                                 std::to_string(p->p_theta) + "," + std::to_string(p->p_phi) +
                                 ") are not instantiated in this build");
  if (p->base_s < 1 || p->base_theta < 1 || p->base_phi < 1)
    throw Error(IFGF_EINVAL, "cone base counts must be positive");
}

// interp.hpp:29-31 nodes and interp.cpp:19-34 transforms, host libm.
InterpConsts make_consts(const ifgf_params* p) {
  InterpConsts K{};
  K.ps = p->p_s;
  K.pt = p->p_theta;
  K.pp = p->p_phi;
  K.P = K.ps * K.pt * K.pp;
  K.PL = (K.pt * K.pp + 1) & ~1;
  K.Pst = K.ps * K.PL;
  const auto fill = [](int q, double* nodes, double* M) {
    for (int j = 0; j < q; ++j) nodes[j] = std::cos(kPi * (2.0 * j + 1.0) / (2.0 * q));
    for (int k = 0; k < q; ++k) {
      const double w = (k == 0 ? 1.0 : 2.0) / q;
      for (int j = 0; j < q; ++j) M[k * q + j] = w * std::cos(k * kPi * (2.0 * j + 1.0) / (2.0 * q));
    }
  };
  fill(K.ps, K.ns, K.Ms);
  fill(K.pt, K.nt, K.Mt);
  fill(K.pp, K.np, K.Mp);
  return K;
}

// Streams are recycled per device instead of created per plan: blocks a plan
// frees into the stream-ordered pool are reused without new physical
// mappings only when the next plan allocates on the same stream (a fresh
// stream per plan made the pool grow and remap: 20-80 ms setup spikes).
struct StreamCache {
  std::mutex mu;
  std::vector<std::pair<int, cudaStream_t>> free;
};
StreamCache& stream_cache() {
  static StreamCache* c = new StreamCache;  // leaked: streams outlive static destructors
  return *c;
}
cudaStream_t take_stream(int device) {
  {
    StreamCache& c = stream_cache();
    std::lock_guard<std::mutex> g(c.mu);
    for (size_t k = c.free.size(); k-- > 0;)
      if (c.free[k].first == device) {
        cudaStream_t s = c.free[k].second;
        c.free.erase(c.free.begin() + k);
        return s;
      }
  }
  cudaStream_t s = nullptr;
  IFGF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}
void give_stream(int device, cudaStream_t s) {
  if (!s) return;
  StreamCache& c = stream_cache();
  std::lock_guard<std::mutex> g(c.mu);
  c.free.emplace_back(device, s);
}

void plan_free(ifgf_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  dist_free(P);
  if (P->s_aux) cudaStreamSynchronize(P->s_aux);
  // stream-ordered frees back into the pool (a cudaFree per allocation would
  // synchronise the device ~150 times)
  for (void* a : P->allocs) {
    if (P->s_main) cudaFreeAsync(a, P->s_main);
    else cudaFree(a);
  }
  if (P->s_main) cudaStreamSynchronize(P->s_main);
  // aux first, main last: take_stream pops from the back, so the next plan
  // gets this plan's main stream back as its main stream
  give_stream(P->device, P->s_aux);
  give_stream(P->device, P->s_main);
  delete P;
}

// Plans of a rank group keep K4 locate records for their own points only
// (build_rank_records, after dist_prepare), not the whole cloud's.
thread_local bool tl_rank_plan = false;
struct RankPlanScope {
  RankPlanScope() { tl_rank_plan = true; }
  ~RankPlanScope() { tl_rank_plan = false; }
};

ifgf_plan* new_plan(size_t n, int kind, double wavenumber, const ifgf_params* p) {
  if (n < 1) throw Error(IFGF_EINVAL, "empty point cloud");
  if (n > 0xffffffffull) throw Error(IFGF_EINVAL, "more than 2^32 points");
  if (kind != IFGF_HELMHOLTZ && kind != IFGF_LAPLACE) throw Error(IFGF_EINVAL, "bad kernel kind");
  if (!(wavenumber >= 0.0) || !std::isfinite(wavenumber))
    throw Error(IFGF_EINVAL, "wavenumber must be finite and >= 0");
  validate_params(p);
  require_device(p->device);
  auto* P = new ifgf_plan;
  P->device = p->device;
  P->n = n;
  P->kind = kind;
  P->kappa = kind == IFGF_LAPLACE ? 0.0 : wavenumber;  // KernelConfig::kappa, kernel.hpp:20
  P->params = *p;
  P->K = make_consts(p);
  if (p->partition != IFGF_PARTITION_COUNT && p->partition != IFGF_PARTITION_WORK)
    throw Error(IFGF_EINVAL, "unknown partition mode");
  P->partition_mode = p->partition;
  P->mem_budget = device_memory_budget(P->device);
  P->rank_plan = tl_rank_plan;
  try {
    P->s_main = take_stream(P->device);
    P->s_aux = take_stream(P->device);
    P->err = P->alloc<int>(1);
    P->work_ctr = P->alloc<uint32_t>(ifgf_plan::kWorkCtrs);
    IFGF_CUDA(cudaMemsetAsync(P->err, 0, sizeof(int), P->s_main));
  } catch (...) {
    plan_free(P);
    throw;
  }
  return P;
}

void finish_create(ifgf_plan* P, const double* dx, const double* dy, const double* dz) {
  build_plan(P, dx, dy, dz);
  P->setup_launches = P->launches;
  P->ar = P->alloc<double>(P->n);
  P->ai = P->alloc<double>(P->n);
  P->ir = P->alloc<double>(P->n);
  P->ii = P->alloc<double>(P->n);
  IFGF_CUDA(cudaStreamSynchronize(P->s_main));
}

// Block storage for apply: one slot per level when it fits in half of the
// free memory, else two slots sized for the largest level.
void ensure_slots(ifgf_plan* P) {
  if (P->n_slots) return;
  const int D = P->depth;
  const size_t bpc = (size_t)P->K.Pst * sizeof(double2);
  size_t total = 0, mx = 0;
  for (int d = 3; d <= D; ++d) {
    total += P->lv[d].nc;
    mx = std::max<size_t>(mx, P->lv[d].nc);
  }
  const size_t fr = mem_available(P);
  double2* base = nullptr;
  if (total * bpc < fr / 2) {
    // one slot per level; an out-of-memory (memory taken by other allocators
    // since the budget's sample) falls back to the two rotating slots
    void* p = nullptr;
    const size_t b = (total * P->K.Pst + 2) * sizeof(double2) + 16;
    if (cudaMallocAsync(&p, b, P->s_main) == cudaSuccess) {
      P->allocs.push_back(p);
      P->bytes += b;
      base = static_cast<double2*>(p);
    } else {
      cudaGetLastError();
    }
  }
  if (base) {
    size_t off = 0;
    for (int d = 3; d <= D; ++d) {
      P->slots[d] = base + off * P->K.Pst;
      off += P->lv[d].nc;
    }
    P->n_slots = D - 2;
  } else {
    double2* a = P->alloc<double2>(mx * P->K.Pst + 2);
    double2* b = P->alloc<double2>(mx * P->K.Pst + 2);
    for (int d = 3; d <= D; ++d) P->slots[d] = (d % 2) ? a : b;
    P->n_slots = 2;
  }
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

// The operator on device buffers (densities/results in caller order).
void apply_device(ifgf_plan* P, const double* a_re, const double* a_im, double* i_re,
                  double* i_im, cudaStream_t caller, ifgf_report* rep) {
  const auto t0 = clk::now();
  IFGF_CUDA(cudaSetDevice(P->device));
  ensure_slots(P);
  const int D = P->depth;
  const size_t launches0 = P->launches;
  cudaStream_t sm = P->s_main, sa = P->serial ? P->s_main : P->s_aux;

  std::vector<cudaEvent_t> evs;
  auto mk = [&](bool timing) {
    cudaEvent_t e;
    IFGF_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    evs.push_back(e);
    return e;
  };
  struct Guard {
    std::vector<cudaEvent_t>& v;
    ~Guard() {
      for (auto e : v) cudaEventDestroy(e);
    }
  } guard{evs};

  cudaEvent_t start = mk(false);
  IFGF_CUDA(cudaEventRecord(start, caller));
  IFGF_CUDA(cudaStreamWaitEvent(sm, start, 0));
  launch_gather_density(P, a_re, a_im, sm);
  cudaEvent_t gathered = mk(false);
  IFGF_CUDA(cudaEventRecord(gathered, sm));
  IFGF_CUDA(cudaStreamWaitEvent(sa, gathered, 0));

  EventPair t_sing{mk(true), mk(true)}, t_ld{mk(true), mk(true)};
  std::vector<EventPair> t_int(D + 1), t_prop(D + 1);
  std::vector<cudaEvent_t> blk_ready(D + 1), int_done(D + 1);

  IFGF_CUDA(cudaEventRecord(t_sing.a, sa));
  launch_singular(P, 0, P->n, sa);
  IFGF_CUDA(cudaEventRecord(t_sing.b, sa));

  IFGF_CUDA(cudaEventRecord(t_ld.a, sm));
  launch_level_d(P, 0, P->lv[D].nc, P->slots[D], sm);
  IFGF_CUDA(cudaEventRecord(t_ld.b, sm));
  blk_ready[D] = t_ld.b;

  // K4 from the locate records stages its blocks in 212 KB of shared memory
  // per SM: next to K3 on a second stream it costs both kernels their L1
  // (C2 apply 50.1 ms on two streams against 48.4 ms in line), so it runs on
  // the main stream between the propagation levels; K1 keeps the aux stream.
  const bool k4_staged = P->k4_records && P->lv[D].rec != nullptr;
  cudaStream_t s4 = k4_staged ? sm : sa;
  // K1 and K4 both add into the result: K4 starts after K1 on either stream
  if (s4 != sa) IFGF_CUDA(cudaStreamWaitEvent(s4, t_sing.b, 0));
  for (int d = D; d >= 3; --d) {
    IFGF_CUDA(cudaStreamWaitEvent(s4, blk_ready[d], 0));
    t_int[d] = {mk(true), mk(true)};
    IFGF_CUDA(cudaEventRecord(t_int[d].a, s4));
    launch_interpolation(P, d, 0, P->n, P->slots[d], s4);
    IFGF_CUDA(cudaEventRecord(t_int[d].b, s4));
    int_done[d] = t_int[d].b;
    if (d > 3) {
      const int prev = d - 1 + P->n_slots;  // previous occupant of level d-1's slot
      if (P->n_slots < D - 2 && prev <= D) IFGF_CUDA(cudaStreamWaitEvent(sm, int_done[prev], 0));
      t_prop[d] = {mk(true), mk(true)};
      IFGF_CUDA(cudaEventRecord(t_prop[d].a, sm));
      launch_propagation(P, d, 0, P->lv[d - 1].nc, P->slots[d], P->slots[d - 1], sm);
      IFGF_CUDA(cudaEventRecord(t_prop[d].b, sm));
      blk_ready[d - 1] = t_prop[d].b;
    }
  }
  IFGF_CUDA(cudaStreamWaitEvent(sm, int_done[3], 0));
  IFGF_CUDA(cudaStreamWaitEvent(sm, t_sing.b, 0));
  launch_scatter_result(P, i_re, i_im, sm);
  cudaEvent_t done = mk(false);
  IFGF_CUDA(cudaEventRecord(done, sm));
  IFGF_CUDA(cudaGetLastError());
  IFGF_CUDA(cudaStreamWaitEvent(caller, done, 0));
  IFGF_CUDA(cudaEventSynchronize(done));
  check_device_error(P);

  if (rep) {
    auto ms = [](const EventPair& e) {
      float v = 0.f;
      if (e.a && e.b) cudaEventElapsedTime(&v, e.a, e.b);
      return 1e-3 * v;
    };
    rep->singular = ms(t_sing);
    rep->level_d = ms(t_ld);
    rep->interpolation = rep->propagation = 0.0;
    for (int d = 3; d <= D; ++d) {
      rep->interpolation += ms(t_int[d]);
      if (d > 3) rep->propagation += ms(t_prop[d]);
    }
    rep->total = since(t0);
    rep->depth = D;
    rep->n = P->n;
    rep->h_level_d = P->lv[D].h;
    rep->n_levels = D - 2;
    size_t peak = P->lv[D].nc;
    for (int d = 3; d <= D; ++d) {
      rep->level_boxes[d - 3] = P->lv[d].nb;
      rep->level_cones[d - 3] = P->lv[d].nc;
      if (d > 3) peak = std::max<size_t>(peak, P->lv[d].nc + P->lv[d - 1].nc);
    }
    rep->peak_live_blocks = peak;  // the reference's two-level figure (engine.cpp:280-308)
    rep->setup = 0.0;
    rep->gpu_launches = P->launches - launches0;
  }
}

// 2n doubles of host<->device staging for the pass-level API, allocated once
// per plan (each call synchronises before returning, so calls can share it).
double* staging(ifgf_plan* P) {
  if (!P->staging) P->staging = P->alloc<double>(2 * P->n);
  return P->staging;
}

// nrhs densities (vector r at offset r * n, caller's order) against one
// plan, one after another on the plan's streams: the setup is shared, the
// passes run per rhs.  Kernel-level batching (K4 / K3 sharing each step's
// locate, cone lookup, node data and phase factor across two rhs) was built
// and measured at C2: 66.5 ms per rhs against 65.9 ms for single applies --
// both kernels are bound by the L1->register path of the block loads, which
// batching does not reduce, so it was not kept.
void apply_batch_device(ifgf_plan* P, int nrhs, const double* a_re, const double* a_im,
                        double* i_re, double* i_im, cudaStream_t caller, ifgf_report* rep) {
  const auto t0 = clk::now();
  const size_t n = P->n;
  size_t launches = 0;
  ifgf_report r1{};
  for (int r = 0; r < nrhs; ++r) {
    apply_device(P, a_re + r * n, a_im ? a_im + r * n : nullptr, i_re + r * n, i_im + r * n,
                 caller, &r1);
    launches += r1.gpu_launches;
  }
  if (rep) {
    *rep = r1;
    rep->gpu_launches = launches;
    rep->total = since(t0);
  }
}

double2* stage_blocks(ifgf_plan* P, int d) {
  if (d < 3 || d > P->depth) throw Error(IFGF_EINVAL, "level out of range");
  if (!P->stage_blocks[d]) {
    P->stage_blocks[d] = P->alloc<double2>((size_t)P->lv[d].nc * P->K.Pst + 2);
    IFGF_CUDA(cudaMemsetAsync(P->stage_blocks[d], 0,
                              ((size_t)P->lv[d].nc * P->K.Pst + 2) * sizeof(double2), P->s_main));
  }
  return P->stage_blocks[d];
}

template <class T>
std::vector<T> d2h(const T* d, size_t count, cudaStream_t s) {
  std::vector<T> h(count);
  if (count) IFGF_CUDA(cudaMemcpyAsync(h.data(), d, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  IFGF_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

namespace ifgf_b200 {

// dist.cpp:78-130 (partition), on host arrays of the level-D boxes.
// Cut [0, n) into R contiguous intervals of about equal weight (w: per unit,
// prefix over units); every interval gets >= min_units units when possible.
void cut_weighted(const std::vector<double>& w, int R, size_t min_units, uint32_t* begin) {
  const size_t n = w.size();
  std::vector<double> pre(n + 1, 0.0);
  for (size_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + w[i];
  begin[0] = 0;
  size_t b = 0;
  for (int r = 0; r < R - 1; ++r) {
    const double target = pre[n] * (r + 1) / R;
    const size_t rest = (size_t)(R - 1 - r) * min_units;
    const size_t max_end = n >= rest ? n - rest : b;
    size_t e = std::min(b + min_units, max_end);
    // first e with pre[e] >= target, then the nearer of e-1 / e
    while (e < max_end && pre[e] < target) ++e;
    if (e > b + min_units && e - 1 >= b + min_units && target - pre[e - 1] < pre[e] - target) --e;
    begin[r + 1] = (uint32_t)e;
    b = e;
  }
  begin[R] = (uint32_t)n;
}

// Rank layout (dist.cpp:78-130).  IFGF_PARTITION_COUNT (the reference):
// contiguous Morton intervals of finest-level boxes balanced by point count,
// equal-count cone intervals per level.  IFGF_PARTITION_WORK (the paper's
// future work): the same contiguous intervals balanced by
// evaluation work in the SURVEY.md 8(d) flop units -- per finest box its
// points' near-field pairs (57) and interpolation evaluations over all
// levels (429); per cone its block's construction: level-D seeding
// (58 per node and source) or propagation (430 per node and child) + the
// fit (3,900).
void partition_host(ifgf_plan* P, int R, uint32_t* box_begin, uint32_t* point_begin,
                    uint32_t* cone_begin) {
  if (R < 1) throw Error(IFGF_EINVAL, "partition: need at least one rank");
  const int D = P->depth;
  const Level& L = P->lv[D];
  const size_t nb = L.nb;
  if ((size_t)R > nb)
    throw Error(IFGF_EINVAL,
                "partition: more ranks than relevant finest-level boxes (the smallest "
                "distribution unit)");
  const auto first = d2h(L.first, nb, P->s_main);
  const auto count = d2h(L.count, nb, P->s_main);
  const size_t npts = (size_t)first[nb - 1] + count[nb - 1];
  const bool work = P->partition_mode == IFGF_PARTITION_WORK;
  if (!work) {
    box_begin[0] = point_begin[0] = 0;
    uint32_t b = 0;
    for (int r = 0; r < R - 1; ++r) {
      const double target = static_cast<double>(npts) * (r + 1) / R;
      const uint32_t max_end = (uint32_t)nb - (uint32_t)(R - 1 - r);
      uint32_t e = b + 1;
      while (e < max_end && static_cast<double>(first[e - 1] + count[e - 1]) < target) ++e;
      box_begin[r + 1] = e;
      point_begin[r + 1] = first[e - 1] + count[e - 1];
      b = e;
    }
    box_begin[R] = (uint32_t)nb;
    point_begin[R] = (uint32_t)npts;
  } else {
    // per finest box: sources seen by its near field, cousins per level
    const auto nbr = d2h(L.nbr, nb * 27, P->s_main);
    const auto nbr_cnt = d2h(L.nbr_cnt, nb, P->s_main);
    std::vector<double> cous(nb, 0.0);  // sum over levels of the ancestor's cousins
    std::vector<uint32_t> anc(nb);
    for (size_t b = 0; b < nb; ++b) anc[b] = (uint32_t)b;
    for (int d = D; d >= 3; --d) {
      const Level& V = P->lv[d];
      const auto off = d2h(V.cous_off, (size_t)V.nb + 1, P->s_main);
      for (size_t b = 0; b < nb; ++b) cous[b] += off[anc[b] + 1] - off[anc[b]];
      if (d > 3) {
        const auto par = d2h(V.parent, V.nb, P->s_main);
        for (size_t b = 0; b < nb; ++b) anc[b] = par[anc[b]];
      }
    }
    std::vector<double> w(nb);
    for (size_t b = 0; b < nb; ++b) {
      double src = 0.0;
      for (uint32_t a = 0; a < nbr_cnt[b]; ++a) src += count[nbr[b * 27 + a]];
      w[b] = (double)count[b] * (57.0 * (src - 1.0) + 429.0 * cous[b]);
    }
    cut_weighted(w, R, 1, box_begin);
    for (int r = 0; r <= R; ++r)
      point_begin[r] =
          box_begin[r] == nb ? (uint32_t)npts : first[box_begin[r]];
  }
  if (cone_begin)
    for (int d = 3; d <= D; ++d) {
      uint32_t* cb = cone_begin + (size_t)(d - 3) * (R + 1);
      const Level& V = P->lv[d];
      const size_t nc = V.nc;
      if (!work) {
        const size_t base = nc / R, extra = nc % R;
        cb[0] = 0;
        for (int r = 0; r < R; ++r)
          cb[r + 1] = cb[r] + (uint32_t)(base + ((size_t)r < extra ? 1 : 0));
        continue;
      }
      const auto cbox = d2h(V.cone_box, nc, P->s_main);
      std::vector<double> w(nc);
      const double Pn = P->K.P;
      if (d == D) {
        const auto cnt = d2h(V.count, V.nb, P->s_main);
        for (size_t q = 0; q < nc; ++q) w[q] = Pn * 58.0 * cnt[cbox[q]] + 3900.0;
      } else {
        const auto ch = d2h(V.child_begin, (size_t)V.nb + 1, P->s_main);
        for (size_t q = 0; q < nc; ++q)
          w[q] = Pn * 430.0 * (ch[cbox[q] + 1] - ch[cbox[q]]) + 3900.0;
      }
      cut_weighted(w, R, 0, cb);
    }
}


}  // namespace ifgf_b200

extern "C" {

const char* ifgf_last_error(void) { return g_err.c_str(); }
int ifgf_abi_version(void) { return IFGF_B200_ABI_VERSION; }

void ifgf_default_params(ifgf_params* p) {
  if (!p) return;
  p->depth = 0;
  p->box_lambda = 0.25;
  p->points_per_box = 64;
  p->base_s = 1;
  p->base_theta = 2;
  p->base_phi = 4;
  p->p_s = 3;
  p->p_theta = 5;
  p->p_phi = 5;
  p->device = 0;
  p->partition = IFGF_PARTITION_COUNT;
}

int ifgf_device_ok(void) {
  // the caller's current device (bench.py: torch.cuda.set_device(local_rank)),
  // left current on return
  DeviceGuard keep;
  return guarded([] {
           int dev = 0;
           if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
           require_device(dev);
         }) == IFGF_OK
             ? 1
             : 0;
}

int ifgf_choose_depth(size_t n, double side, double kappa, const ifgf_params* p, int* out) {
  return guarded([&] {
    if (!p || !out) throw Error(IFGF_EINVAL, "null argument");
    int d;
    if (p->depth > 0) {
      d = p->depth;
    } else if (kappa > 0.0) {
      const double lambda = 2.0 * kPi / kappa;
      const double ratio = side / (p->box_lambda * lambda);
      d = 1 + static_cast<int>(std::floor(std::log2(std::max(ratio, 1.0)) + 1e-4));
    } else {
      const double boxes = static_cast<double>(n) / std::max(1, p->points_per_box);
      d = 1 + static_cast<int>(std::ceil(0.5 * std::log2(std::max(boxes, 1.0)) - 1e-9));
    }
    *out = std::clamp(d, 3, 21);
  });
}

int ifgf_plan_create_device(const double* dx, const double* dy, const double* dz, size_t n,
                            int kind, double k, const ifgf_params* p, void* stream,
                            ifgf_plan** out) {
  DeviceGuard keep;
  return guarded([&] {
    if (!out) throw Error(IFGF_EINVAL, "null output");
    *out = nullptr;
    ifgf_plan* P = new_plan(n, kind, k, p);
    try {
      cudaEvent_t e;
      IFGF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      IFGF_CUDA(cudaEventRecord(e, static_cast<cudaStream_t>(stream)));
      IFGF_CUDA(cudaStreamWaitEvent(P->s_main, e, 0));
      cudaEventDestroy(e);
      finish_create(P, dx, dy, dz);
    } catch (...) {
      plan_free(P);
      throw;
    }
    *out = P;
  });
}

int ifgf_plan_create(const double* x1, const double* x2, const double* x3, size_t n, int kind,
                     double k, const ifgf_params* p, ifgf_plan** out) {
  DeviceGuard keep;
  return guarded([&] {
    if (!out) throw Error(IFGF_EINVAL, "null output");
    *out = nullptr;
    if (n >= 1 && (!x1 || !x2 || !x3)) throw Error(IFGF_EINVAL, "null coordinates");
    const auto t0 = clk::now();
    ifgf_plan* P = new_plan(n, kind, k, p);
    try {
      double* tmp = P->alloc<double>(3 * n);
      IFGF_CUDA(cudaMemcpyAsync(tmp, x1, n * sizeof(double), cudaMemcpyHostToDevice, P->s_main));
      IFGF_CUDA(cudaMemcpyAsync(tmp + n, x2, n * sizeof(double), cudaMemcpyHostToDevice, P->s_main));
      IFGF_CUDA(
          cudaMemcpyAsync(tmp + 2 * n, x3, n * sizeof(double), cudaMemcpyHostToDevice, P->s_main));
      finish_create(P, tmp, tmp + n, tmp + 2 * n);
      P->setup_seconds = since(t0);
    } catch (...) {
      plan_free(P);
      throw;
    }
    *out = P;
  });
}

void ifgf_plan_destroy(ifgf_plan* plan) {
  DeviceGuard keep;
  plan_free(plan);
}

int ifgf_plan_set_option(ifgf_plan* P, int option, int value) {
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    if (option == IFGF_OPT_SERIAL) {
      P->serial = value != 0;
    } else if (option == IFGF_OPT_PROP_KERNEL) {
      if (value != IFGF_PROP_NODE && value != IFGF_PROP_DMMA && value != IFGF_PROP_ROWS &&
          value != IFGF_PROP_FLY && value != IFGF_PROP_AUTO)
        throw Error(IFGF_EINVAL, "unknown propagation kernel (TILES, STREAM and PIPE were "
                                 "measured slower than ROWS and removed; DESIGN.md section 3)");
      P->prop_kernel = value;
    } else if (option == IFGF_OPT_PARTITION) {
      if (value < IFGF_PARTITION_COUNT || value > IFGF_PARTITION_WORK)
        throw Error(IFGF_EINVAL, "unknown partition mode");
      P->partition_mode = value;
    } else if (option == IFGF_OPT_NEAR_KERNEL) {
      if (value < IFGF_NEAR_POINT || value > IFGF_NEAR_BOX)
        throw Error(IFGF_EINVAL, "unknown near-field kernel");
      P->near_kernel = value;
    } else if (option == IFGF_OPT_K4_RECORDS) {
      P->k4_records = value != 0;
    } else {
      throw Error(IFGF_EINVAL, "unknown option");
    }
  });
}

int ifgf_plan_apply_device(ifgf_plan* P, const double* a_re, const double* a_im, double* i_re,
                           double* i_im, void* stream, ifgf_report* rep) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P || !a_re || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    if (P->n < 2) throw Error(IFGF_EINVAL, "apply: need at least two points");
    apply_device(P, a_re, a_im, i_re, i_im, static_cast<cudaStream_t>(stream), rep);
  });
}

int ifgf_plan_apply(ifgf_plan* P, const double* a_re, const double* a_im, double* i_re,
                    double* i_im, ifgf_report* rep) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P || !a_re || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    if (P->n < 2) throw Error(IFGF_EINVAL, "apply: need at least two points");
    const auto t0 = clk::now();
    IFGF_CUDA(cudaSetDevice(P->device));
    const size_t n = P->n;
    double* buf = nullptr;
    IFGF_CUDA(cudaMallocAsync(&buf, 4 * n * sizeof(double), P->s_main));
    struct F {
      double* b;
      cudaStream_t s;
      ~F() { cudaFreeAsync(b, s); }
    } f{buf, P->s_main};
    IFGF_CUDA(cudaMemcpyAsync(buf, a_re, n * sizeof(double), cudaMemcpyHostToDevice, P->s_main));
    if (a_im)
      IFGF_CUDA(
          cudaMemcpyAsync(buf + n, a_im, n * sizeof(double), cudaMemcpyHostToDevice, P->s_main));
    apply_device(P, buf, a_im ? buf + n : nullptr, buf + 2 * n, buf + 3 * n, P->s_main, rep);
    IFGF_CUDA(
        cudaMemcpyAsync(i_re, buf + 2 * n, n * sizeof(double), cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(
        cudaMemcpyAsync(i_im, buf + 3 * n, n * sizeof(double), cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
    if (rep) rep->total = since(t0);
  });
}

int ifgf_plan_apply_batch_device(ifgf_plan* P, int nrhs, const double* a_re, const double* a_im,
                                 double* i_re, double* i_im, void* stream, ifgf_report* rep) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P || !a_re || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    if (nrhs < 1) throw Error(IFGF_EINVAL, "apply_batch: need at least one right-hand side");
    if (P->n < 2) throw Error(IFGF_EINVAL, "apply: need at least two points");
    if (P->dist) throw Error(IFGF_EINVAL, "apply_batch: not on a rank plan");
    apply_batch_device(P, nrhs, a_re, a_im, i_re, i_im, static_cast<cudaStream_t>(stream), rep);
  });
}

int ifgf_plan_apply_batch(ifgf_plan* P, int nrhs, const double* a_re, const double* a_im,
                          double* i_re, double* i_im, ifgf_report* rep) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P || !a_re || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    if (nrhs < 1) throw Error(IFGF_EINVAL, "apply_batch: need at least one right-hand side");
    if (P->n < 2) throw Error(IFGF_EINVAL, "apply: need at least two points");
    if (P->dist) throw Error(IFGF_EINVAL, "apply_batch: not on a rank plan");
    const auto t0 = clk::now();
    IFGF_CUDA(cudaSetDevice(P->device));
    const size_t n = P->n, m = (size_t)nrhs * n;
    double* buf = nullptr;
    IFGF_CUDA(cudaMallocAsync(&buf, 4 * m * sizeof(double), P->s_main));
    struct F {
      double* b;
      cudaStream_t s;
      ~F() { cudaFreeAsync(b, s); }
    } f{buf, P->s_main};
    IFGF_CUDA(cudaMemcpyAsync(buf, a_re, m * 8, cudaMemcpyHostToDevice, P->s_main));
    if (a_im)
      IFGF_CUDA(cudaMemcpyAsync(buf + m, a_im, m * 8, cudaMemcpyHostToDevice, P->s_main));
    apply_batch_device(P, nrhs, buf, a_im ? buf + m : nullptr, buf + 2 * m, buf + 3 * m,
                       P->s_main, rep);
    IFGF_CUDA(cudaMemcpyAsync(i_re, buf + 2 * m, m * 8, cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaMemcpyAsync(i_im, buf + 3 * m, m * 8, cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
    if (rep) rep->total = since(t0);
  });
}

int ifgf_apply(size_t n, const double* x1, const double* x2, const double* x3, const double* a_re,
               const double* a_im, int kind, double k, const ifgf_params* p, double* i_re,
               double* i_im, ifgf_report* rep) {
  // engine.cpp:260-325: rebuild, apply, return in the caller's order.  The
  // densities travel to the device on the aux stream while the main stream
  // builds the plan from the coordinates (Problem::build), so their copy is
  // off the critical path.
  if (n < 2) {
    g_err = "apply: need at least two points";
    return IFGF_EINVAL;
  }
  DeviceGuard keep;
  ifgf_plan* P = nullptr;
  size_t setup_launches = 0;
  const int rc = guarded([&] {
    if (!x1 || !x2 || !x3 || !a_re || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    const auto t0 = clk::now();
    P = new_plan(n, kind, k, p);
    double* buf = nullptr;
    IFGF_CUDA(cudaMallocAsync(&buf, 4 * n * sizeof(double), P->s_aux));
    struct F {
      double* b;
      cudaStream_t s;
      ~F() {
        if (b) cudaFreeAsync(b, s);
      }
    } f{buf, P->s_main};
    IFGF_CUDA(cudaMemcpyAsync(buf, a_re, n * 8, cudaMemcpyHostToDevice, P->s_aux));
    if (a_im) IFGF_CUDA(cudaMemcpyAsync(buf + n, a_im, n * 8, cudaMemcpyHostToDevice, P->s_aux));
    cudaEvent_t dens;
    IFGF_CUDA(cudaEventCreateWithFlags(&dens, cudaEventDisableTiming));
    IFGF_CUDA(cudaEventRecord(dens, P->s_aux));
    double* tmp = P->alloc<double>(3 * n);
    IFGF_CUDA(cudaMemcpyAsync(tmp, x1, n * 8, cudaMemcpyHostToDevice, P->s_main));
    IFGF_CUDA(cudaMemcpyAsync(tmp + n, x2, n * 8, cudaMemcpyHostToDevice, P->s_main));
    IFGF_CUDA(cudaMemcpyAsync(tmp + 2 * n, x3, n * 8, cudaMemcpyHostToDevice, P->s_main));
    finish_create(P, tmp, tmp + n, tmp + 2 * n);
    P->setup_seconds = since(t0);
    setup_launches = P->launches;
    IFGF_CUDA(cudaStreamWaitEvent(P->s_main, dens, 0));
    cudaEventDestroy(dens);
    apply_device(P, buf, a_im ? buf + n : nullptr, buf + 2 * n, buf + 3 * n, P->s_main, rep);
    IFGF_CUDA(cudaMemcpyAsync(i_re, buf + 2 * n, n * 8, cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaMemcpyAsync(i_im, buf + 3 * n, n * 8, cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
    if (rep) {
      rep->setup = P->setup_seconds;
      rep->gpu_launches = P->launches;  // setup + apply kernels of this call
    }
    (void)setup_launches;
    f.b = nullptr;
    IFGF_CUDA(cudaFreeAsync(buf, P->s_main));
    const double total = since(t0);
    if (rep) rep->total = total;
  });
  if (P) plan_free(P);
  return rc;
}

int ifgf_plan_get_info(const ifgf_plan* P, ifgf_plan_info* info) {
  return guarded([&] {
    if (!P || !info) throw Error(IFGF_EINVAL, "null argument");
    std::memset(info, 0, sizeof *info);
    info->n = P->n;
    info->depth = P->depth;
    for (int c = 0; c < 3; ++c) info->cube_origin[c] = P->cube[c];
    info->cube_side = P->cube[3];
    info->kappa = P->kappa;
    info->p_s = P->K.ps;
    info->p_theta = P->K.pt;
    info->p_phi = P->K.pp;
    info->P = P->K.P;
    for (int d = 1; d <= P->depth; ++d) {
      const Level& L = P->lv[d];
      info->boxes[d] = L.nb;
      info->cones[d] = d >= 3 ? L.nc : 0;
      info->cousin_entries[d] = d >= 3 ? L.n_cous : 0;
      info->h[d] = L.h;
    }
    for (int d = 1; d <= P->depth; ++d) info->nbr_entries[d] = P->lv[d].n_nbr;
    info->setup_seconds = P->setup_seconds;
    info->device_bytes = P->bytes;
    info->setup_launches = P->setup_launches;
    info->launches = P->launches;
    info->k4_record_pairs = 0;
    for (int d = 3; d <= P->depth; ++d)
      if (P->lv[d].rec) info->k4_record_pairs += (size_t)P->lv[d].npairs;
    info->k4_record_bytes = info->k4_record_pairs *
                            ((P->kappa == 0.0 ? 4 : 5) * sizeof(double) + sizeof(uint32_t));
  });
}

int ifgf_plan_export_perm(const ifgf_plan* P, uint32_t* perm) {
  return guarded([&] {
    if (!P || !perm) throw Error(IFGF_EINVAL, "null argument");
    IFGF_CUDA(cudaMemcpy(perm, P->perm, P->n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  });
}

int ifgf_plan_export_level(const ifgf_plan* Pc, int d, uint64_t* codes, uint32_t* first,
                           uint32_t* count, double* centers3, uint32_t* parent,
                           uint32_t* child_begin, uint32_t* nbr_off, uint32_t* nbr,
                           uint32_t* cousin_off, uint32_t* cousin, uint32_t* cone_box,
                           uint64_t* cone_gamma, uint32_t* box_cone_begin) {
  return guarded([&] {
    ifgf_plan* P = const_cast<ifgf_plan*>(Pc);
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    if (d < 1 || d > P->depth) throw Error(IFGF_EINVAL, "level out of range");
    const Level& L = P->lv[d];
    cudaStream_t s = P->s_main;
    const size_t nb = L.nb;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && src && bytes)
        IFGF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    cp(codes, L.code, nb * 8);
    cp(first, L.first, nb * 4);
    cp(count, L.count, nb * 4);
    cp(parent, L.parent, nb * 4);
    if (d < P->depth) cp(child_begin, L.child_begin, (nb + 1) * 4);
    if (centers3) {
      const auto x = d2h(L.cx, nb, s), y = d2h(L.cy, nb, s), z = d2h(L.cz, nb, s);
      for (size_t b = 0; b < nb; ++b) {
        centers3[3 * b] = x[b];
        centers3[3 * b + 1] = y[b];
        centers3[3 * b + 2] = z[b];
      }
    }
    if (nbr_off || nbr) {
      const auto cnt = d2h(L.nbr_cnt, nb, s);
      const auto all = d2h(L.nbr, nb * 27, s);
      size_t o = 0;
      for (size_t b = 0; b < nb; ++b) {
        if (nbr_off) nbr_off[b] = (uint32_t)o;
        for (uint32_t a = 0; a < cnt[b]; ++a, ++o)
          if (nbr) nbr[o] = all[b * 27 + a];
      }
      if (nbr_off) nbr_off[nb] = (uint32_t)o;
    }
    if (d >= 3) {
      cp(cousin_off, L.cous_off, (nb + 1) * 4);
      cp(cousin, L.cous, L.n_cous * 4);
      cp(cone_box, L.cone_box, (size_t)L.nc * 4);
      cp(box_cone_begin, L.box_cone, (nb + 1) * 4);
      if (cone_gamma) {
        const auto g = d2h(L.cone_gamma, L.nc, s);
        for (size_t q = 0; q < L.nc; ++q) cone_gamma[q] = g[q];
      }
    }
    IFGF_CUDA(cudaStreamSynchronize(s));
  });
}

int ifgf_plan_set_density(ifgf_plan* P, const double* a_re, const double* a_im) {
  return guarded([&] {
    if (!P || !a_re) throw Error(IFGF_EINVAL, "null argument");
    IFGF_CUDA(cudaSetDevice(P->device));
    const size_t n = P->n;
    double* buf = staging(P);
    IFGF_CUDA(cudaMemcpyAsync(buf, a_re, n * 8, cudaMemcpyHostToDevice, P->s_main));
    if (a_im) IFGF_CUDA(cudaMemcpyAsync(buf + n, a_im, n * 8, cudaMemcpyHostToDevice, P->s_main));
    // gather without touching the result buffer
    double* ir = P->ir;
    double* ii = P->ii;
    P->ir = P->ii = nullptr;
    launch_gather_density(P, buf, a_im ? buf + n : nullptr, P->s_main);
    P->ir = ir;
    P->ii = ii;
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
  });
}

int ifgf_plan_zero_result(ifgf_plan* P) {
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    IFGF_CUDA(cudaMemsetAsync(P->ir, 0, P->n * 8, P->s_main));
    IFGF_CUDA(cudaMemsetAsync(P->ii, 0, P->n * 8, P->s_main));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
  });
}

int ifgf_plan_singular_pass(ifgf_plan* P, size_t b, size_t e) {
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    if (b > e || e > P->n) throw Error(IFGF_EINVAL, "point range out of bounds");
    launch_singular(P, b, e, P->s_main);
    IFGF_CUDA(cudaGetLastError());
    check_device_error(P);
  });
}

int ifgf_plan_level_d_pass(ifgf_plan* P, uint32_t qb, uint32_t qe) {
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    if (qb > qe || qe > P->lv[P->depth].nc) throw Error(IFGF_EINVAL, "cone range out of bounds");
    launch_level_d(P, qb, qe, stage_blocks(P, P->depth), P->s_main);
    IFGF_CUDA(cudaGetLastError());
    check_device_error(P);
  });
}

int ifgf_plan_propagation_pass(ifgf_plan* P, int d, uint32_t qb, uint32_t qe) {
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    if (d < 4 || d > P->depth) throw Error(IFGF_EINVAL, "propagation level out of range");
    if (qb > qe || qe > P->lv[d - 1].nc) throw Error(IFGF_EINVAL, "cone range out of bounds");
    double2* child = stage_blocks(P, d);
    double2* parent = stage_blocks(P, d - 1);
    launch_propagation(P, d, qb, qe, child, parent, P->s_main);
    IFGF_CUDA(cudaGetLastError());
    check_device_error(P);
  });
}

int ifgf_plan_interpolation_pass(ifgf_plan* P, int d, size_t b, size_t e) {
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    if (d < 3 || d > P->depth) throw Error(IFGF_EINVAL, "level out of range");
    if (b > e || e > P->n) throw Error(IFGF_EINVAL, "point range out of bounds");
    launch_interpolation(P, d, b, e, stage_blocks(P, d), P->s_main);
    IFGF_CUDA(cudaGetLastError());
    check_device_error(P);
  });
}

int ifgf_plan_read_blocks(ifgf_plan* P, int d, double* re, double* im) {
  return guarded([&] {
    if (!P || !re || !im) throw Error(IFGF_EINVAL, "null argument");
    const double2* blk = stage_blocks(P, d);
    const size_t nc = P->lv[d].nc, Pn = P->K.P, Ps = P->K.Pst;
    const auto h = d2h(blk, nc * Ps, P->s_main);
    const size_t plane = (size_t)P->K.pt * P->K.pp, PL = P->K.PL;
    for (size_t q = 0; q < nc; ++q)
      for (size_t k = 0; k < Pn; ++k) {
        const size_t dk = (k / plane) * PL + k % plane;
        re[q * Pn + k] = h[q * Ps + dk].x;
        im[q * Pn + k] = h[q * Ps + dk].y;
      }
  });
}

int ifgf_plan_write_blocks(ifgf_plan* P, int d, const double* re, const double* im) {
  return guarded([&] {
    if (!P || !re || !im) throw Error(IFGF_EINVAL, "null argument");
    double2* blk = stage_blocks(P, d);
    const size_t nc = P->lv[d].nc, Pn = P->K.P, Ps = P->K.Pst;
    std::vector<double2> h(nc * Ps, make_double2(0.0, 0.0));
    const size_t plane = (size_t)P->K.pt * P->K.pp, PL = P->K.PL;
    for (size_t q = 0; q < nc; ++q)
      for (size_t k = 0; k < Pn; ++k)
        h[q * Ps + (k / plane) * PL + k % plane] = make_double2(re[q * Pn + k], im[q * Pn + k]);
    IFGF_CUDA(cudaMemcpyAsync(blk, h.data(), nc * Ps * sizeof(double2), cudaMemcpyHostToDevice,
                              P->s_main));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
  });
}

int ifgf_plan_read_result(ifgf_plan* P, int sorted, double* i_re, double* i_im) {
  return guarded([&] {
    if (!P || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    const size_t n = P->n;
    if (sorted) {
      IFGF_CUDA(cudaMemcpyAsync(i_re, P->ir, n * 8, cudaMemcpyDeviceToHost, P->s_main));
      IFGF_CUDA(cudaMemcpyAsync(i_im, P->ii, n * 8, cudaMemcpyDeviceToHost, P->s_main));
      IFGF_CUDA(cudaStreamSynchronize(P->s_main));
      return;
    }
    double* buf = staging(P);
    launch_scatter_result(P, buf, buf + n, P->s_main);
    IFGF_CUDA(cudaMemcpyAsync(i_re, buf, n * 8, cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaMemcpyAsync(i_im, buf + n, n * 8, cudaMemcpyDeviceToHost, P->s_main));
    IFGF_CUDA(cudaStreamSynchronize(P->s_main));
  });
}

int ifgf_plan_block_stride(const ifgf_plan* P) { return P ? P->K.Pst : 0; }

// Pack/unpack run on the caller's stream but touch the plan's level storage,
// which the passes (and stage_blocks' first-use zero fill) use on s_main: the
// caller's stream first waits for s_main, and s_main then waits for the copy,
// so a pass issued after an unpack never reads blocks the unpack has not
// written, and an unpack never overwrites blocks a pending pass still reads.
void order_with_main(ifgf_plan* P, cudaStream_t s, bool before) {
  cudaEvent_t e;
  IFGF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (before) {
    IFGF_CUDA(cudaEventRecord(e, P->s_main));
    IFGF_CUDA(cudaStreamWaitEvent(s, e, 0));
  } else {
    IFGF_CUDA(cudaEventRecord(e, s));
    IFGF_CUDA(cudaStreamWaitEvent(P->s_main, e, 0));
  }
  cudaEventDestroy(e);
}

int ifgf_plan_pack_blocks(ifgf_plan* P, int d, const uint32_t* d_cones, size_t m, double* d_buf,
                          void* stream) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    IFGF_CUDA(cudaSetDevice(P->device));
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    double2* blk = stage_blocks(P, d);  // the pass-level API's level storage
    order_with_main(P, s, true);
    launch_pack(P, blk, d_cones, m, P->lv[d].nc, d_buf, 0, nullptr, s);
    IFGF_CUDA(cudaGetLastError());
    order_with_main(P, s, false);
  });
}

int ifgf_plan_unpack_blocks(ifgf_plan* P, int d, const uint32_t* d_cones, size_t m,
                            const double* d_buf, void* stream) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P) throw Error(IFGF_EINVAL, "null plan");
    IFGF_CUDA(cudaSetDevice(P->device));
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    double2* blk = stage_blocks(P, d);
    order_with_main(P, s, true);
    launch_pack(P, nullptr, d_cones, m, P->lv[d].nc, const_cast<double*>(d_buf), 1, blk, s);
    IFGF_CUDA(cudaGetLastError());
    order_with_main(P, s, false);
  });
}

int ifgf_plan_partition(const ifgf_plan* P, int R, uint32_t* box_begin, uint32_t* point_begin,
                        uint32_t* cone_begin) {
  return guarded([&] {
    if (!P || !box_begin || !point_begin) throw Error(IFGF_EINVAL, "null argument");
    partition_host(const_cast<ifgf_plan*>(P), R, box_begin, point_begin, cone_begin);
  });
}

int ifgf_plan_exchange_set(ifgf_plan* P, int R, int rank, int d, int kind, uint32_t* cones,
                           size_t* count) {
  return guarded([&] {
    if (!P || !count) throw Error(IFGF_EINVAL, "null argument");
    if (rank < 0 || rank >= R) throw Error(IFGF_EINVAL, "rank out of range");
    if (P->dist) throw Error(IFGF_EINVAL, "exchange_set: not on a rank plan of a group");
    if (d < 3 || d > P->depth || (kind == 1 && d < 4) || kind < 0 || kind > 1)
      throw Error(IFGF_EINVAL, "bad level or kind");
    std::vector<uint32_t> bb(R + 1), pb(R + 1), cb((size_t)(P->depth - 2) * (R + 1));
    partition_host(P, R, bb.data(), pb.data(), cb.data());
    const Level& L = P->lv[d];
    // call-scoped scratch, returned to the pool when the call ends
    struct Tmp {
      void* p = nullptr;
      cudaStream_t s;
      ~Tmp() {
        if (p) cudaFreeAsync(p, s);
      }
    } t_need{nullptr, P->s_main}, t_cb{nullptr, P->s_main};
    IFGF_CUDA(cudaMallocAsync(&t_need.p, L.nc + 1, P->s_main));
    IFGF_CUDA(cudaMallocAsync(&t_cb.p, (R + 1) * sizeof(uint32_t), P->s_main));
    uint8_t* need = static_cast<uint8_t*>(t_need.p);
    IFGF_CUDA(cudaMemsetAsync(need, 0, L.nc + 1, P->s_main));
    // this level's cone boundaries on the device (ownership test)
    uint32_t* d_cb = static_cast<uint32_t*>(t_cb.p);
    IFGF_CUDA(cudaMemcpyAsync(d_cb, cb.data() + (size_t)(d - 3) * (R + 1), (R + 1) * 4,
                              cudaMemcpyHostToDevice, P->s_main));
    if (kind == 0)
      launch_need(P, d, 0, d_cb, R, rank, pb[rank], pb[rank + 1], need, P->s_main);
    else
      launch_need(P, d, 1, d_cb, R, rank, cb[(size_t)(d - 4) * (R + 1) + rank],
                  cb[(size_t)(d - 4) * (R + 1) + rank + 1], need, P->s_main);
    IFGF_CUDA(cudaGetLastError());
    check_device_error(P);
    const auto h = d2h(need, L.nc, P->s_main);
    size_t k = 0;
    for (size_t q = 0; q < L.nc; ++q)
      if (h[q]) {
        if (cones) cones[k] = (uint32_t)q;
        ++k;
      }
    *count = k;
  });
}


// ---- multi-GPU (dist.cu) ----
int ifgf_comm_unique_id(void* id_out) {
  return guarded([&] {
    if (!id_out) throw Error(IFGF_EINVAL, "null id buffer");
    comm_unique_id(id_out);
  });
}

int ifgf_comm_create(const void* id, int rank, int world, int device, ifgf_comm** out) {
  DeviceGuard keep;
  return guarded([&] {
    if (!out) throw Error(IFGF_EINVAL, "null output");
    *out = nullptr;
    require_device(device);
    *out = comm_create(id, rank, world, device);
  });
}

void ifgf_comm_destroy(ifgf_comm* comm) {
  DeviceGuard keep;
  comm_destroy(comm);
}

int ifgf_dist_plan_create_device(ifgf_comm* comm, const double* dx, const double* dy,
                                 const double* dz, size_t n, int kind, double k,
                                 const ifgf_params* p, void* stream, ifgf_plan** out) {
  DeviceGuard keep;
  return guarded([&] {
    if (!out || !comm) throw Error(IFGF_EINVAL, "null argument");
    *out = nullptr;
    if (!p) throw Error(IFGF_EINVAL, "null params");
    ifgf_params q = *p;
    q.device = comm->device;
    RankPlanScope rank_scope;
    ifgf_plan* P = new_plan(n, kind, k, &q);
    try {
      cudaEvent_t e;
      IFGF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      IFGF_CUDA(cudaEventRecord(e, static_cast<cudaStream_t>(stream)));
      IFGF_CUDA(cudaStreamWaitEvent(P->s_main, e, 0));
      cudaEventDestroy(e);
      const auto t0 = clk::now();
      finish_create(P, dx, dy, dz);
      dist_prepare(P, comm->world, comm->rank);
      comm_attach(P, comm);
      dist_connect(P);
      P->setup_seconds = since(t0);
    } catch (...) {
      plan_free(P);
      throw;
    }
    *out = P;
  });
}

int ifgf_dist_plan_apply_device(ifgf_plan* P, const double* a_re, const double* a_im,
                                double* i_re, double* i_im, void* stream, ifgf_report* rep) {
  DeviceGuard keep;
  return guarded([&] {
    if (!P || !a_re || !i_re || !i_im) throw Error(IFGF_EINVAL, "null argument");
    if (P->n < 2) throw Error(IFGF_EINVAL, "apply: need at least two points");
    dist_apply_device(P, a_re, a_im, i_re, i_im, static_cast<cudaStream_t>(stream), rep);
  });
}

int ifgf_dist_plan_info(const ifgf_plan* P, ifgf_dist_info* info) {
  return guarded([&] {
    if (!P || !info) throw Error(IFGF_EINVAL, "null argument");
    dist_fill_info(P, info);
  });
}

int ifgf_run_distributed(size_t n, const double* x1, const double* x2, const double* x3,
                         const double* a_re, const double* a_im, int kind, double k,
                         const ifgf_params* p, int R, const int* devices, double* i_re,
                         double* i_im, ifgf_report* rep, ifgf_dist_info* info) {
  DeviceGuard keep;
  return guarded([&] {
    // dist.cpp:241-243
    if (n < 2) throw Error(IFGF_EINVAL, "run_distributed: need two points");
    if (R < 1) throw Error(IFGF_EINVAL, "run_distributed: need at least one rank");
    if (!x1 || !x2 || !x3 || !a_re || !i_re || !i_im || !p)
      throw Error(IFGF_EINVAL, "null argument");
    std::vector<ifgf_plan*> G;
    struct Free {
      std::vector<ifgf_plan*>& g;
      ~Free() {
        for (auto* P : g) plan_free(P);
      }
    } fr{G};
    const auto t0 = clk::now();
    RankPlanScope rank_scope;
    for (int r = 0; r < R; ++r) {
      ifgf_params q = *p;
      q.device = devices ? devices[r] : p->device;
      ifgf_plan* P = nullptr;
      const int rc = ifgf_plan_create(x1, x2, x3, n, kind, k, &q, &P);
      if (rc) throw Error(rc, g_err);
      G.push_back(P);
      dist_prepare(P, R, r);
    }
    dist_connect_local(G);
    const double setup = since(t0);
    run_local_group(G, a_re, a_im, i_re, i_im, rep);
    if (rep) {
      rep->setup = setup;
      rep->total += setup;
    }
    if (info)
      for (int r = 0; r < R; ++r) dist_fill_info(G[r], &info[r]);
  });
}

int ifgf_direct_eval(size_t n, const double* x1, const double* x2, const double* x3,
                     const double* a_re, const double* a_im, int kind, double k,
                     const uint32_t* targets, size_t m, int device, double* o_re, double* o_im) {
  DeviceGuard keep;
  return guarded([&] {
    if (n < 2) throw Error(IFGF_EINVAL, "direct_eval: need at least two points");
    require_device(device);
    const size_t cnt = targets ? m : n;
    for (size_t j = 0; targets && j < m; ++j)
      if (targets[j] >= n) throw Error(IFGF_EINVAL, "target index out of range");
    const double kappa = kind == IFGF_LAPLACE ? 0.0 : k;
    cudaStream_t s;
    IFGF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double* buf = nullptr;
    uint32_t* tg = nullptr;
    IFGF_CUDA(cudaMallocAsync(&buf, (5 * n + 2 * cnt) * sizeof(double), s));
    IFGF_CUDA(cudaMemcpyAsync(buf, x1, n * 8, cudaMemcpyHostToDevice, s));
    IFGF_CUDA(cudaMemcpyAsync(buf + n, x2, n * 8, cudaMemcpyHostToDevice, s));
    IFGF_CUDA(cudaMemcpyAsync(buf + 2 * n, x3, n * 8, cudaMemcpyHostToDevice, s));
    IFGF_CUDA(cudaMemcpyAsync(buf + 3 * n, a_re, n * 8, cudaMemcpyHostToDevice, s));
    if (a_im) IFGF_CUDA(cudaMemcpyAsync(buf + 4 * n, a_im, n * 8, cudaMemcpyHostToDevice, s));
    else IFGF_CUDA(cudaMemsetAsync(buf + 4 * n, 0, n * 8, s));
    if (targets) {
      IFGF_CUDA(cudaMallocAsync(&tg, m * 4, s));
      IFGF_CUDA(cudaMemcpyAsync(tg, targets, m * 4, cudaMemcpyHostToDevice, s));
    }
    double* o = buf + 5 * n;
    direct_sums(buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, n, kappa, tg, cnt, o,
                o + cnt, s);
    IFGF_CUDA(cudaMemcpyAsync(o_re, o, cnt * 8, cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaMemcpyAsync(o_im, o + cnt, cnt * 8, cudaMemcpyDeviceToHost, s));
    IFGF_CUDA(cudaFreeAsync(buf, s));
    if (tg) IFGF_CUDA(cudaFreeAsync(tg, s));
    IFGF_CUDA(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
  });
}

int ifgf_sample_indices(size_t n, size_t m, uint64_t seed, uint32_t* out) {
  // engine.cpp:341-352: partial Fisher-Yates with mt19937_64(seed)
  return guarded([&] {
    if (m > n) throw Error(IFGF_EINVAL, "sample_indices: m > n");
    std::vector<uint32_t> idx(n);
    for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
    std::mt19937_64 rng(seed);
    for (size_t j = 0; j < m; ++j) {
      const size_t k = j + static_cast<size_t>(rng() % (n - j));
      std::swap(idx[j], idx[k]);
    }
    std::memcpy(out, idx.data(), m * sizeof(uint32_t));
  });
}

int ifgf_error_at_indices(size_t n, const double* x1, const double* x2, const double* x3,
                          const double* a_re, const double* a_im, const double* i_re,
                          const double* i_im, int kind, double k, const uint32_t* idx, size_t m,
                          int device, double* eps) {
  // engine.cpp:354-376 with the exact sums on the device
  std::vector<double> dre(m ? m : 1), dim(m ? m : 1);
  const int rc = ifgf_direct_eval(n, x1, x2, x3, a_re, a_im, kind, k, idx, m, device, dre.data(),
                                  dim.data());
  if (rc) return rc;
  return guarded([&] {
    double num = 0.0, den = 0.0;
    for (size_t j = 0; j < m; ++j) {
      const double er = dre[j] - i_re[idx[j]], ei = dim[j] - i_im[idx[j]];
      num += er * er + ei * ei;
      den += dre[j] * dre[j] + dim[j] * dim[j];
    }
    if (den == 0.0) throw Error(IFGF_EDOMAIN, "estimate_error: zero reference norm");
    *eps = std::sqrt(num / den);
  });
}

}  // extern "C"
