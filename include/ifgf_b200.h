/* ifgf_b200.h -- C ABI of the B200-native IFGF matvec (libifgf_b200.so).
 *
 * Drop-in boundary for the reference's operator path (paths relative to
 * /root/reference/proj).  The reference is a C++ static library with no FFI;
 * each entry point below names the C++ interface it replaces:
 *
 *   ifgf_apply               ifgf::apply(PointCloud&, const KernelConfig&,
 *                                        const EngineParams&)   engine.hpp:112-114
 *   ifgf_plan_create         ifgf::Problem::build                engine.hpp:54-55
 *   ifgf_plan_apply          apply() minus the rebuild           engine.cpp:270-315
 *   ifgf_plan_*_pass         singular_pass / eval_level_d /
 *                            propagation_pass / interpolation_pass engine.hpp:91-110
 *   ifgf_direct_eval         ifgf::direct_eval                   engine.hpp:117
 *   ifgf_sample_indices      ifgf::sample_indices                engine.hpp:120
 *   ifgf_error_at_indices    ifgf::error_at_indices              engine.hpp:123-124
 *   ifgf_choose_depth        ifgf::choose_depth                  engine.hpp:21
 *   ifgf_plan_partition      ifgf::dist::partition               dist.hpp:23
 *   ifgf_run_distributed     ifgf::dist::run_distributed         dist.hpp:90
 *   ifgf_dist_plan_*         the rank loop of run_distributed    dist.cpp:241-361
 *                            as one process per GPU (MPI ranks, PAPER.md)
 *
 * Conventions: plain pointers and sizes, no CUDA or C++ types.  Functions
 * return 0 on success or an IFGF_E* code mirroring the reference's exception
 * classes (invalid_argument, domain_error, logic_error, runtime_error);
 * ifgf_last_error() returns the thread-local message.  Host-pointer entry
 * points are blocking.  "_device" entry points take device pointers and a
 * cudaStream_t passed as void* (NULL = legacy default stream); they order
 * themselves after that stream and make it wait for their completion.
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point fails with IFGF_ERUNTIME.
 */
#ifndef IFGF_B200_H
#define IFGF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IFGF_B200_ABI_VERSION 2

enum {
  IFGF_OK = 0,
  IFGF_EINVAL = 1,   /* std::invalid_argument */
  IFGF_EDOMAIN = 2,  /* std::domain_error     */
  IFGF_ELOGIC = 3,   /* std::logic_error      */
  IFGF_ERUNTIME = 4  /* std::runtime_error (CUDA, memory, device) */
};

enum { IFGF_HELMHOLTZ = 0, IFGF_LAPLACE = 1 }; /* KernelKind, kernel.hpp:13 */

/* EngineParams (engine.hpp:12-19) + InterpOrders (interp.hpp:11-14). */
typedef struct ifgf_params {
  int depth;          /* 0 = choose_depth */
  double box_lambda;  /* 0.25 */
  int points_per_box; /* 64 */
  int base_s, base_theta, base_phi; /* 1, 2, 4 */
  int p_s, p_theta, p_phi;          /* 3, 5, 5 */
  int device;                       /* CUDA ordinal (replaces `threads`) */
  int partition; /* rank layout of multi-GPU plans: IFGF_PARTITION_COUNT (0,
                    the reference's) or IFGF_PARTITION_WORK (1); see below */
} ifgf_params;

#define IFGF_MAX_LEVELS 22

/* ApplyReport (engine.hpp:23-42).  Seconds: setup is host wall clock around
 * the device setup; the pass times are CUDA-event durations. */
typedef struct ifgf_report {
  double setup, singular, level_d, interpolation, propagation, total;
  int depth;
  size_t n;
  double h_level_d;
  int n_levels;                           /* levels d = 3..depth */
  size_t level_boxes[IFGF_MAX_LEVELS];    /* index d - 3 */
  size_t level_cones[IFGF_MAX_LEVELS];
  size_t peak_live_blocks;
  size_t gpu_launches;                    /* kernels launched by this call */
} ifgf_report;

typedef struct ifgf_plan ifgf_plan;

void ifgf_default_params(ifgf_params* p);
const char* ifgf_last_error(void);
int ifgf_abi_version(void);
/* 1 if a usable sm_100 device is visible, else 0 (message in last_error). */
int ifgf_device_ok(void);

int ifgf_choose_depth(size_t n, double cube_side, double kappa, const ifgf_params* p,
                      int* depth_out);

/* ---- plan = Problem::build on the device ---- */
int ifgf_plan_create(const double* x1, const double* x2, const double* x3, size_t n,
                     int kernel_kind, double wavenumber, const ifgf_params* p,
                     ifgf_plan** out);
int ifgf_plan_create_device(const double* d_x1, const double* d_x2, const double* d_x3,
                            size_t n, int kernel_kind, double wavenumber,
                            const ifgf_params* p, void* stream, ifgf_plan** out);
void ifgf_plan_destroy(ifgf_plan* plan);

/* Plan options.
 * IFGF_OPT_SERIAL = 1: every apply kernel on one stream (no near-field /
 *   interpolation overlap) so per-pass event times are exclusive.
 * IFGF_OPT_PROP_KERNEL selects the propagation kernel:
 *   IFGF_PROP_NODE  (0) thread per (parent cone, node), locate per child
 *                       (the generic path: any orders);
 *   IFGF_PROP_DMMA  (2) warp-level FP64 tensor-core GEMM on every level with
 *                       the precomputed geometry: a warp owns 16 parent
 *                       cones that share gamma, mma.sync.m8n8k4.f64 over the
 *                       child blocks in memory order (whole levels only;
 *                       ranges and levels without the precomputed geometry
 *                       run ROWS / FLY);
 *   IFGF_PROP_ROWS  (3) thread per (parent cone, child, row of <= 3
 *                       nodes that share a child cone) from the precomputed
 *                       geometry, one block load per row; levels without
 *                       the precomputed geometry run IFGF_PROP_FLY;
 *   IFGF_PROP_FLY   (4) the same rows grouped per parent cone on the fly
 *                       (no precomputed geometry);
 *   IFGF_PROP_AUTO  (7, default) per level: the warp GEMM where at least
 *                       100 parent cones share each gamma (the fine
 *                       levels), ROWS / FLY elsewhere.
 *   Values 1, 5, 6 (TILES, STREAM, PIPE of ABI 1) were measured slower than
 *   ROWS and removed; they fail with IFGF_EINVAL.
 *   All agree to rounding; DESIGN.md records their measured times.
 * IFGF_OPT_NEAR_KERNEL selects the near-field kernel:
 *   IFGF_NEAR_POINT (0) thread per target point, neighbour sources in order;
 *   IFGF_NEAR_BOX   (1, default) warp per target box, the box's neighbour
 *                       sources staged in shared memory and split across
 *                       lanes, several targets per pass.
 *   Both agree to rounding.
 * IFGF_OPT_K4_RECORDS = 0: the interpolation pass locates every (point,
 *   cousin) pair again instead of reading the plan's locate records (kept
 *   when they fit in 15 % of the device memory -- a rank plan keeps only its
 *   own points'; same result bitwise).  Default 1. */
enum { IFGF_OPT_SERIAL = 1, IFGF_OPT_PROP_KERNEL = 2, IFGF_OPT_NEAR_KERNEL = 3,
       IFGF_OPT_PARTITION = 4, IFGF_OPT_K4_RECORDS = 5 };
enum { IFGF_NEAR_POINT = 0, IFGF_NEAR_BOX = 1 };
/* IFGF_OPT_PARTITION selects the rank layout of ifgf_plan_partition and
 * ifgf_plan_exchange_set:
 *   IFGF_PARTITION_COUNT (0, default) the reference's: finest boxes balanced
 *                        by point count, equal-count cone intervals
 *                        (dist.cpp:90-128);
 *   IFGF_PARTITION_WORK  (1) the same contiguous intervals balanced by
 *                        evaluation work (near-field pairs + interpolation
 *                        evaluations per box; seeding or propagation + fit
 *                        per cone) -- the paper's proposed extension
 *                        (PAPER.md:1648-1656). */
enum { IFGF_PARTITION_COUNT = 0, IFGF_PARTITION_WORK = 1 };
enum {
  IFGF_PROP_NODE = 0,
  IFGF_PROP_DMMA = 2,
  IFGF_PROP_ROWS = 3,
  IFGF_PROP_FLY = 4,
  IFGF_PROP_AUTO = 7
};
int ifgf_plan_set_option(ifgf_plan* plan, int option, int value);

/* ---- operator application; i_* in the caller's original point order ---- */
int ifgf_plan_apply(ifgf_plan* plan, const double* a_re, const double* a_im, double* i_re,
                    double* i_im, ifgf_report* rep);
int ifgf_plan_apply_device(ifgf_plan* plan, const double* d_a_re, const double* d_a_im,
                           double* d_i_re, double* d_i_im, void* stream, ifgf_report* rep);
/* Several right-hand sides against one plan (iterative solvers): nrhs
 * densities, vector r at offset r * n in each array (caller's order), applied
 * one after another with the setup shared; identical to nrhs calls of
 * ifgf_plan_apply. */
int ifgf_plan_apply_batch(ifgf_plan* plan, int nrhs, const double* a_re, const double* a_im,
                          double* i_re, double* i_im, ifgf_report* rep);
int ifgf_plan_apply_batch_device(ifgf_plan* plan, int nrhs, const double* d_a_re,
                                 const double* d_a_im, double* d_i_re, double* d_i_im,
                                 void* stream, ifgf_report* rep);
/* create + apply + destroy: the exact contract of ifgf::apply (a_im may be
 * NULL for a real density). */
int ifgf_apply(size_t n, const double* x1, const double* x2, const double* x3,
               const double* a_re, const double* a_im, int kernel_kind, double wavenumber,
               const ifgf_params* p, double* i_re, double* i_im, ifgf_report* rep);

/* ---- structure export (parity against Problem::build) ---- */
typedef struct ifgf_plan_info {
  size_t n;
  int depth;
  double cube_origin[3], cube_side;
  double kappa;
  int p_s, p_theta, p_phi, P;
  size_t boxes[IFGF_MAX_LEVELS];   /* index d (1..depth) */
  size_t cones[IFGF_MAX_LEVELS];   /* index d (3..depth) */
  size_t nbr_entries[IFGF_MAX_LEVELS];
  size_t cousin_entries[IFGF_MAX_LEVELS];
  double h[IFGF_MAX_LEVELS];
  double setup_seconds;
  size_t device_bytes;
  size_t setup_launches; /* our kernels launched by the plan's setup */
  size_t launches;       /* our kernels launched by the plan so far (setup + passes) */
  size_t k4_record_pairs; /* (point, cousin) pairs whose locate the plan keeps (0: none) */
  size_t k4_record_bytes; /* device bytes of those records */
} ifgf_plan_info;

int ifgf_plan_get_info(const ifgf_plan* plan, ifgf_plan_info* info);
int ifgf_plan_export_perm(const ifgf_plan* plan, uint32_t* perm);
/* Any pointer may be NULL.  Arrays are sized from ifgf_plan_info; child_begin
 * has boxes+1 entries for d < depth, CSR offsets have boxes+1 entries, and
 * cone arrays exist for d >= 3 (OctreeLevel octree.hpp:23-38, LevelConeSet
 * cones.hpp:97-104). */
int ifgf_plan_export_level(const ifgf_plan* plan, int d, uint64_t* codes, uint32_t* first,
                           uint32_t* count, double* centers3, uint32_t* parent,
                           uint32_t* child_begin, uint32_t* nbr_off, uint32_t* nbr,
                           uint32_t* cousin_off, uint32_t* cousin, uint32_t* cone_box,
                           uint64_t* cone_gamma, uint32_t* box_cone_begin);

/* ---- pass-level API (engine.hpp:91-110) over plan-owned device state ----
 * set_density takes host arrays in the caller's order; the result buffer is
 * in sorted order until read back.  Blocks are the reference BlockStore
 * layout on the host side: planar re and im, [cones][P]. */
int ifgf_plan_set_density(ifgf_plan* plan, const double* a_re, const double* a_im);
int ifgf_plan_zero_result(ifgf_plan* plan);
int ifgf_plan_singular_pass(ifgf_plan* plan, size_t pt_begin, size_t pt_end);
int ifgf_plan_level_d_pass(ifgf_plan* plan, uint32_t cone_begin, uint32_t cone_end);
int ifgf_plan_propagation_pass(ifgf_plan* plan, int d, uint32_t pcone_begin,
                               uint32_t pcone_end);
int ifgf_plan_interpolation_pass(ifgf_plan* plan, int d, size_t pt_begin, size_t pt_end);
int ifgf_plan_read_blocks(ifgf_plan* plan, int d, double* re, double* im);
int ifgf_plan_write_blocks(ifgf_plan* plan, int d, const double* re, const double* im);
int ifgf_plan_read_result(ifgf_plan* plan, int sorted_order, double* i_re, double* i_im);
/* Device-side block exchange for multi-GPU: pack/unpack the blocks of the
 * listed cone ordinals (device u32 array) to/from a contiguous device buffer
 * of m * 2 * Pst doubles, Pst = p_s * PL, PL = p_theta * p_phi rounded up to
 * even (the device block layout; see ifgf_plan_block_stride). */
int ifgf_plan_block_stride(const ifgf_plan* plan);
int ifgf_plan_pack_blocks(ifgf_plan* plan, int d, const uint32_t* d_cones, size_t m,
                          double* d_buf, void* stream);
int ifgf_plan_unpack_blocks(ifgf_plan* plan, int d, const uint32_t* d_cones, size_t m,
                            const double* d_buf, void* stream);
/* Rank layout (dist.cpp:78-130): box_begin and point_begin have n_ranks+1
 * entries, cone_begin has (depth-2)*(n_ranks+1), level-major from d = 3. */
int ifgf_plan_partition(const ifgf_plan* plan, int n_ranks, uint32_t* box_begin,
                        uint32_t* point_begin, uint32_t* cone_begin);
/* Deduplicated foreign cones rank `rank` needs at level d (kind 0:
 * interpolation data, dist.cpp:179-201; kind 1: propagation data,
 * dist.cpp:206-237), sorted.  Call with cones == NULL to get the count. */
int ifgf_plan_exchange_set(ifgf_plan* plan, int n_ranks, int rank, int d, int kind,
                           uint32_t* cones, size_t* count);

/* ---- multi-GPU: the reference's rank algorithm (dist.hpp, dist.cpp:241-361)
 * with partitioned block storage and per-level exchanges of the boundary
 * cone-segment interpolants.  Each rank builds the (replicated) structure and
 * owns its Morton interval of points and, per level, an equal-count interval
 * of cones (dist.cpp:78-130); it stores only its own blocks plus its halo.
 *
 * One process per GPU: rank 0 calls ifgf_comm_unique_id, the launcher
 * broadcasts the IFGF_COMM_ID_BYTES bytes, every rank calls ifgf_comm_create
 * (NCCL communicator over NVLink/NVSwitch, loaded on first use).  Then per
 * matvec configuration ifgf_dist_plan_create_device (collective) and
 * ifgf_dist_plan_apply_device (collective; full result in the caller's order
 * on every rank).  ifgf_plan_destroy frees a rank plan. */
#define IFGF_COMM_ID_BYTES 128
typedef struct ifgf_comm ifgf_comm;
int ifgf_comm_unique_id(void* id_out);
int ifgf_comm_create(const void* id, int rank, int world, int device, ifgf_comm** out);
void ifgf_comm_destroy(ifgf_comm* comm);
int ifgf_dist_plan_create_device(ifgf_comm* comm, const double* d_x1, const double* d_x2,
                                 const double* d_x3, size_t n, int kernel_kind,
                                 double wavenumber, const ifgf_params* p, void* stream,
                                 ifgf_plan** out);
int ifgf_dist_plan_apply_device(ifgf_plan* plan, const double* d_a_re, const double* d_a_im,
                                double* d_i_re, double* d_i_im, void* stream, ifgf_report* rep);

/* Per-level view of a rank plan.  interp_needed / prop_needed: the foreign
 * cones this rank reads for interpolation / propagation (dist.cpp:179-237,
 * deduplicated per (rank, cone) like CommLevelStats); halo_cones: their union
 * (what the exchange moves in); sent_cones: blocks this rank sends. */
typedef struct ifgf_dist_level {
  size_t owned_cones, halo_cones, interp_needed, prop_needed, sent_cones;
} ifgf_dist_level;
typedef struct ifgf_dist_info {
  int rank, world, depth;
  size_t point_begin, point_end;      /* owned sorted points */
  ifgf_dist_level levels[IFGF_MAX_LEVELS]; /* index d - 3 */
  size_t block_bytes;                 /* this rank's block storage (owned + halo) */
  size_t device_bytes;                /* all of this rank plan's device memory */
  double compute_seconds;             /* ifgf_run_distributed with IFGF_DIST_RANK_TIMING=1:
                                         this rank's kernels, ranks serialised (load balance) */
} ifgf_dist_info;
int ifgf_dist_plan_info(const ifgf_plan* plan, ifgf_dist_info* info);

/* dist::run_distributed (dist.hpp:90): n_ranks rank plans in THIS process on
 * devices[r] (entries may repeat: several ranks on one GPU), advanced phase
 * by phase, blocks moved rank to rank by device copies; host arrays in/out,
 * output in the caller's order, bitwise equal to ifgf_apply.  info (may be
 * NULL) receives n_ranks entries. */
int ifgf_run_distributed(size_t n, const double* x1, const double* x2, const double* x3,
                         const double* a_re, const double* a_im, int kernel_kind,
                         double wavenumber, const ifgf_params* p, int n_ranks,
                         const int* devices, double* i_re, double* i_im, ifgf_report* rep,
                         ifgf_dist_info* info);

/* ---- oracle side (engine.hpp:117-128), computed on the device ---- */
/* o_* = exact sums at the m listed targets (all points if targets == NULL). */
int ifgf_direct_eval(size_t n, const double* x1, const double* x2, const double* x3,
                     const double* a_re, const double* a_im, int kernel_kind,
                     double wavenumber, const uint32_t* targets, size_t m, int device,
                     double* o_re, double* o_im);
int ifgf_sample_indices(size_t n, size_t m, uint64_t seed, uint32_t* out);
int ifgf_error_at_indices(size_t n, const double* x1, const double* x2, const double* x3,
                          const double* a_re, const double* a_im, const double* i_re,
                          const double* i_im, int kernel_kind, double wavenumber,
                          const uint32_t* idx, size_t m, int device, double* eps);

/* ---- measurement helper: FP64 FMA-pipe peak of the device (TFLOP/s,
 * best of 10 launches of independent DFMA chains over all SMs). ---- */
int ifgf_measure_fp64_peak(int device, double* tflops, double* ms);

/* ---- seeded synthetic inputs; host only ----
 * shape 0: unit sphere (normalised Gaussians); 1: spheroid (1,1,c), area
 * uniform by rejection.  dens 0: complex U(-1,1); 1: real N(0,1), a_im = 0. */
int ifgf_generate(size_t n, int shape, double c, int dens, uint64_t seed, double* x1,
                  double* x2, double* x3, double* a_re, double* a_im);

/* generate_surface (geometry.cpp:57-93, geometry.hpp): 6 n_per_dim^2 points on
 * the cube-face surface of radius a; shape 0 sphere, 1 oblate (z x 0.1),
 * 2 prolate (z x 10) (Shape, geometry.hpp); densities U[0,1) from
 * mt19937_64(seed).  Arrays hold 6 n_per_dim^2 entries. */
int ifgf_generate_surface(int shape, double a, int n_per_dim, uint64_t seed, double* x1,
                          double* x2, double* x3, double* a_re, double* a_im);
/* bench::checksum_hex (bench.cpp:26-41): FNV-1a 64 of re then im, 16 hex
 * digits + NUL into out[17]. */
void ifgf_checksum_hex(const double* re, const double* im, size_t n, char* out);

#ifdef __cplusplus
}
#endif
#endif /* IFGF_B200_H */
