// plan.hpp -- host-side plan object (device-resident Problem) shared by the
// translation units of libifgf_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ifgf_b200.h"
#include "ifgf_common.cuh"

// A multi-process rank group's handle (dist.cu): this process's rank and its
// NCCL communicator (ncclComm_t, opaque here).
struct ifgf_comm {
  int rank = 0, world = 1, device = 0;
  void* nccl = nullptr;
};

namespace ifgf_b200 {

struct DistState;  // dist.cu: a rank's share of a multi-GPU plan

// C++ exception carrying one of the IFGF_E* codes; caught at the C ABI.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define IFGF_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::ifgf_b200::Error(IFGF_ERUNTIME, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                                  " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

// One octree level: owned device arrays + the LevelDev view handed to kernels.
struct Level {
  int d = 0;
  uint32_t nb = 0;
  double h = 0.0;
  uint64_t* code = nullptr;
  uint32_t* first = nullptr;
  uint32_t* count = nullptr;
  double *cx = nullptr, *cy = nullptr, *cz = nullptr;
  uint32_t* parent = nullptr;
  uint32_t* child_begin = nullptr;
  uint32_t* nbr = nullptr;
  uint32_t* nbr_cnt = nullptr;
  uint32_t* cous_off = nullptr;
  uint32_t* cous = nullptr;
  size_t n_cous = 0;
  size_t n_nbr = 0;
  uint32_t* ptbox = nullptr;  // box ordinal of every sorted point at this level
  // K4 work items: runs of <= interp_points(P) points of one box, {first point, box}
  uint2* chunk = nullptr;
  const uint32_t* nchunk = nullptr;  // device count
  size_t chunk_cap = 0;              // upper bound n / R + nb (launch size)
  // cone set
  int n0 = 0, n1 = 0, n2 = 0;
  double w0 = 0, w1 = 0, w2 = 0, iw0 = 0, iw1 = 0, iw2 = 0, rad = 0;
  uint64_t G = 0;
  uint32_t nc = 0;
  uint32_t* cone_box = nullptr;
  uint32_t* cone_gamma = nullptr;
  uint32_t* box_cone = nullptr;
  uint64_t* bits = nullptr;
  uint32_t* rank = nullptr;
  size_t nwords = 0;
  const double2* trig = nullptr;
  // K4 records (null unless the plan keeps them for this level)
  uint64_t* pair_off = nullptr;
  uint32_t* rec_g = nullptr;
  double* rec = nullptr;
  uint64_t npairs = 0;

  LevelDev dev() const {
    LevelDev v;
    v.d = d;
    v.nb = nb;
    v.h = h;
    v.code = code;
    v.first = first;
    v.count = count;
    v.cx = cx;
    v.cy = cy;
    v.cz = cz;
    v.parent = parent;
    v.child_begin = child_begin;
    v.nbr = nbr;
    v.nbr_cnt = nbr_cnt;
    v.cous_off = cous_off;
    v.cous = cous;
    v.n0 = n0;
    v.n1 = n1;
    v.n2 = n2;
    v.w0 = w0;
    v.w1 = w1;
    v.w2 = w2;
    v.iw0 = iw0;
    v.iw1 = iw1;
    v.iw2 = iw2;
    v.rad = rad;
    v.G = G;
    v.nc = nc;
    v.cone_box = cone_box;
    v.cone_gamma = cone_gamma;
    v.box_cone = box_cone;
    v.bits = bits;
    v.rank = rank;
    v.trig = trig;
    v.pair_off = pair_off;
    v.rec_g = rec_g;
    v.rec = rec;
    v.npairs = npairs;
    return v;
  }
};

// Box-independent propagation geometry for child level d (parent level d-1).
// A parent cone's nodes seen from a child centre depend only on the parent
// segment gamma and the child's octant, so the child cone, the local
// Chebyshev coordinates and the re-centring factor of every (gamma, octant,
// node) are computed once per plan.  Entries within kIdxMargin of a segment
// boundary are flagged and recomputed per box exactly (the reference's
// absolute-coordinate rounding could move them).
// Points per K4 thread (register blocking of the interpolant evaluation;
// C2: R = 1 23.2 ms, 2 21.5 ms, 3 24.2 ms -- K4 is load-latency bound, and
// the extra registers of R = 3 cost more occupancy than the loads it saves).
#ifndef IFGF_INTERP_R
#define IFGF_INTERP_R 2
#endif
constexpr int interp_points(int P) { return P <= 100 ? IFGF_INTERP_R : 2; }

struct PropTiles {
  bool enabled = false;
  uint32_t ngamma = 0;          // distinct parent gammas in use
  uint32_t* cone_gidx = nullptr;   // parent cone -> gamma index
  uint32_t* gamma_of = nullptr;    // gamma index -> parent gamma
  // entries [(gidx * 8 + octant) * P + node]
  double* e_t = nullptr;        // ts, tt, tp
  double2* e_T = nullptr;       // transfer factor (rp/rc) e^{i kappa (rc - rp)}
  uint32_t* e_gc = nullptr;     // child gamma; bit 31 = flagged (exact per-box path)
  // per tile (gidx * 8 + octant), fixed stride P: nodes ordered by child
  // gamma (flagged last), flagged nodes, rows of <= row_nodes nodes sharing a
  // child gamma (IFGF_PROP_ROWS) {child gamma, first permuted position |
  // count << 16 | first-of-group << 24}; entry data permuted into row order
  uint8_t* e_perm = nullptr;
  uint32_t* fl_cnt = nullptr;
  uint16_t* fl_node = nullptr;
  int row_nodes = 3;
  uint32_t* rw_cnt = nullptr;
  uint2* rw = nullptr;
  // IFGF_PROP_DMMA only (built on first use): row tiles of 8, CSR over tiles
  uint32_t* rt_off = nullptr;
  uint4* rt = nullptr;          // {child gamma, nodes 0-3 (u8), nodes 4-7 (u8), group rows}
  double* rdat = nullptr;       // row data (ts, tt, tp, tr, ti per slot), 32-row chunks,
                                // SoA inside (propagate_mma.cu row_field)
  uint32_t* rnode = nullptr;    // per row (tile * P + r): node of slot j in byte j
  // warp GEMM (k_propagate_wgemm): per row tile and node slot one record of
  // node data; parent cones sorted by (box group, gamma, child mask) and cut
  // into warp units of <= 8 * kG4Nct cones sharing (group, gamma, mask)
  char* rtab = nullptr;
  uint32_t nunits = 0;
  uint32_t wg_qb = 0, wg_qe = 0;  // cone range of the units
  uint32_t* usorted = nullptr;
  uint32_t* unit_start = nullptr;
  double2* zblock = nullptr;   // one zero block (absent children's B operand)
};

}  // namespace ifgf_b200

struct ifgf_plan {
  int device = 0;
  cudaStream_t s_main = nullptr, s_aux = nullptr;
  size_t n = 0;
  int kind = IFGF_HELMHOLTZ;
  double kappa = 0.0;
  ifgf_params params{};
  ifgf_b200::InterpConsts K{};
  double cube[4] = {0, 0, 0, 0};
  int depth = 0;
  uint32_t* perm = nullptr;
  double *xs = nullptr, *ys = nullptr, *zs = nullptr;  // Morton-sorted coordinates
  double *ar = nullptr, *ai = nullptr;                 // sorted densities
  double *ir = nullptr, *ii = nullptr;                 // sorted results
  double* staging = nullptr;  // 2n doubles: pass-level API host<->device staging, reused

  int* err = nullptr;
  const double2* phase = nullptr;  // sincos_tab table (kPhaseEntries), after the trig table
  uint32_t* work_ctr = nullptr;    // persistent-kernel work counters (kWorkCtrs)
  static constexpr int kCtrNear = 0, kWorkCtrs = 4;
  ifgf_b200::Level lv[IFGF_MAX_LEVELS];
  double2* stage_blocks[IFGF_MAX_LEVELS] = {};  // pass-level API storage
  double2* slots[IFGF_MAX_LEVELS] = {};         // apply rotation
  ifgf_b200::PropTiles tiles[IFGF_MAX_LEVELS];  // index = child level d
  int n_slots = 0;
  size_t slot_cap = 0;
  std::vector<void*> allocs;
  size_t bytes = 0;
  double setup_seconds = 0.0;
  size_t launches = 0;  // kernels launched by this plan since the last reset
  bool serial = false;  // IFGF_OPT_SERIAL
  int prop_kernel = IFGF_PROP_AUTO;  // IFGF_OPT_PROP_KERNEL
  int near_kernel = IFGF_NEAR_BOX;   // IFGF_OPT_NEAR_KERNEL
  int partition_mode = IFGF_PARTITION_COUNT;  // IFGF_OPT_PARTITION
  size_t setup_launches = 0;
  bool k4_records = true;  // IFGF_OPT_K4_RECORDS: K4 reads the stored locate records where a level has them
  bool rank_plan = false;  // plan of a rank group: records only for its own points (build_rank_records)
  size_t mem_budget = 0;  // device memory available when the plan was created (capi.cu)
  ifgf_b200::DistState* dist = nullptr;  // rank plans of a multi-GPU group (dist.cu)

  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    const size_t b = count * sizeof(T) + 16;
    static const bool trace = std::getenv("IFGF_ALLOC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    IFGF_CUDA(cudaMallocAsync(&p, b, s_main));
    if (trace) {
      const double ms =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3;
      if (ms > 0.3) std::fprintf(stderr, "[alloc] %12zu B  %8.3f ms\n", b, ms);
    }
    allocs.push_back(p);
    bytes += b;
    return static_cast<T*>(p);
  }
  const ifgf_b200::Level& L(int d) const { return lv[d]; }
};

namespace ifgf_b200 {
// setup.cu
void build_plan(ifgf_plan* P, const double* d_x, const double* d_y, const double* d_z);
void check_device_error(ifgf_plan* P);
// passes.cu
void launch_gather_density(ifgf_plan* P, const double* a_re, const double* a_im, cudaStream_t s);
void launch_scatter_result(ifgf_plan* P, double* o_re, double* o_im, cudaStream_t s);
void launch_singular(ifgf_plan* P, size_t b, size_t e, cudaStream_t s);
void launch_level_d(ifgf_plan* P, uint32_t qb, uint32_t qe, double2* out, cudaStream_t s);
void launch_propagation(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, const double2* child,
                        double2* parent, cudaStream_t s);
void launch_interpolation(ifgf_plan* P, int d, size_t b, size_t e, const double2* blocks,
                          cudaStream_t s);
void launch_locate_points(ifgf_plan* P, int d, cudaStream_t s);
void build_rank_records(ifgf_plan* P, uint32_t p0, uint32_t p1);
void launch_pack(ifgf_plan* P, const double2* blocks, const uint32_t* cones, size_t m,
                 uint32_t nc, double* buf, int unpack, double2* blocks_out, cudaStream_t s);
bool orders_supported(int ps, int pt, int pp);
// propagate_mma.cu
void build_prop_tiles(ifgf_plan* P, int d, void* (*scratch)(void*, size_t), void* sctx);
void launch_mark_nodes_tiles(ifgf_plan* P, int d, uint64_t* bits);
bool launch_propagation_mma(ifgf_plan* P, int d, uint32_t qb, uint32_t qe, const double2* child,
                            double2* parent, cudaStream_t s);

// capi.cu
// the plan's creation-time memory budget less what it has allocated since
inline size_t mem_available(const ifgf_plan* P);
void partition_host(ifgf_plan* P, int R, uint32_t* box_begin, uint32_t* point_begin,
                    uint32_t* cone_begin);
// dist.cu
void launch_need(ifgf_plan* P, int d, int kind, const uint32_t* d_bounds, int R, int rank,
                 uint32_t lo, uint32_t hi, uint8_t* need, cudaStream_t s);
void dist_prepare(ifgf_plan* P, int R, int rank);
void dist_connect(ifgf_plan* P);
void dist_connect_local(std::vector<ifgf_plan*>& G);
void dist_apply_device(ifgf_plan* P, const double* a_re, const double* a_im, double* i_re,
                       double* i_im, cudaStream_t caller, ifgf_report* rep);
void run_local_group(std::vector<ifgf_plan*>& G, const double* a_re, const double* a_im,
                     double* i_re, double* i_im, ifgf_report* rep);
void dist_fill_info(const ifgf_plan* P, ifgf_dist_info* info);
void dist_free(ifgf_plan* P);
ifgf_comm* comm_create(const void* id, int rank, int world, int device);
void comm_unique_id(void* out);
void comm_destroy(ifgf_comm* C);
void comm_attach(ifgf_plan* P, ifgf_comm* C);
// direct.cu
void direct_sums(const double* x, const double* y, const double* z, const double* ar,
                 const double* ai, size_t n, double kappa, const uint32_t* targets, size_t m,
                 double* o_re, double* o_im, cudaStream_t s);
}  // namespace ifgf_b200

inline size_t ifgf_b200::mem_available(const ifgf_plan* P) {
  return P->mem_budget > P->bytes ? P->mem_budget - P->bytes : 0;
}
