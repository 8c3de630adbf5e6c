/* ifgf_oracle.h -- CPU restatement of the reference IFGF matvec.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA product
 * in paper_2112_15198_b200/ and the "port" CPU baseline; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It is pinned against the unmodified reference (oracle/_ref, built by
 * oracle/Makefile) and against tests/golden/ fixtures generated from it.
 *
 * Plain C11, no FMA contraction (-ffp-contract=off), libm
 * transcendentals.  Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#ifndef IFGF_ORACLE_H
#define IFGF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (same meaning as include/ifgf_b200.h). */
enum { OC_OK = 0, OC_EINVAL = 1, OC_EDOMAIN = 2, OC_ELOGIC = 3, OC_ERUNTIME = 4 };

typedef struct oc_params {
  int depth;          /* 0 = choose (engine.hpp:13) */
  double box_lambda;  /* 0.25 */
  int points_per_box; /* 64 */
  int base_s, base_theta, base_phi; /* 1, 2, 4 */
  int p_s, p_theta, p_phi;          /* 3, 5, 5 */
} oc_params;

void oc_default_params(oc_params* p);
const char* oc_last_error(void);
/* Threads used by oc_apply, oc_problem_build's cone marking and
 * oc_direct_eval (default 1).  Results are bitwise independent of it. */
void oc_set_threads(int threads);
int oc_get_threads(void);

/* ---- seeded synthetic inputs (shared spec with the product generator) ---- */
uint64_t oc_mt64_first(uint64_t seed, int k); /* k-th output of mt19937_64(seed) */
/* shape 0 = sphere (normalised Gaussians), 1 = spheroid (1,1,c) area-uniform by
 * rejection.  dens 0 = complex U(-1,1), 1 = real N(0,1) (a_im = 0). */
int oc_generate(size_t n, int shape, double c, int dens, uint64_t seed, double* x1,
                double* x2, double* x3, double* a_re, double* a_im);

/* ---- scalar building blocks (for KAT tests) ---- */
void oc_sincos_fast(double x, double* s, double* c);
uint64_t oc_morton_encode(uint32_t ix, uint32_t iy, uint32_t iz);
void oc_morton_decode(uint64_t code, uint32_t* ixyz);
int oc_choose_depth(size_t n, double side, double kappa, const oc_params* p);
void oc_cheb_fit(int ps, int pt, int pp, const double* vre, const double* vim, double* cre,
                 double* cim);
void oc_cheb_eval(int ps, int pt, int pp, const double* cre, const double* cim, double ts,
                  double tt, double tp, double* out_re, double* out_im);
/* cone coordinates of x about a box centre of side h (cones.cpp:9-20) */
int oc_cone_coords(const double* center, double h, const double* x, double* s_theta_phi);

/* ---- problem (setup) ---- */
typedef struct oc_problem oc_problem;

int oc_problem_build(size_t n, const double* x1, const double* x2, const double* x3,
                     const double* a_re, const double* a_im, int kind, double wavenumber,
                     const oc_params* p, oc_problem** out);
void oc_problem_free(oc_problem* pr);
int oc_problem_depth(const oc_problem* pr);
void oc_problem_cube(const oc_problem* pr, double* out4);
void oc_problem_sorted(const oc_problem* pr, uint32_t* perm, double* x1, double* x2,
                       double* x3, double* a_re, double* a_im);
/* sizes = {boxes, cones, nbr_entries, cousin_entries} */
void oc_problem_level_sizes(const oc_problem* pr, int d, uint64_t* sizes, double* h);
void oc_problem_level_boxes(const oc_problem* pr, int d, uint64_t* codes, uint32_t* first,
                            uint32_t* count, double* centers3, uint32_t* parent,
                            uint32_t* child_begin);
void oc_problem_level_adjacency(const oc_problem* pr, int d, uint32_t* nbr_off, uint32_t* nbr,
                                uint32_t* cousin_off, uint32_t* cousin);
void oc_problem_level_cones(const oc_problem* pr, int d, uint32_t* cone_box, uint64_t* gamma,
                            uint32_t* box_cone_begin);

/* ---- passes over the sorted problem (engine.hpp:91-110); i_* sorted order,
 *      accumulated (+=); blocks are [cones][P] re and im planes ---- */
int oc_singular_pass(const oc_problem* pr, size_t b, size_t e, double* i_re, double* i_im);
int oc_level_d_pass(const oc_problem* pr, uint32_t qb, uint32_t qe, double* blk_re,
                    double* blk_im);
int oc_propagation_pass(const oc_problem* pr, int d, const double* child_re,
                        const double* child_im, uint32_t qb, uint32_t qe, double* par_re,
                        double* par_im);
int oc_interpolation_pass(const oc_problem* pr, int d, const double* blk_re,
                          const double* blk_im, size_t b, size_t e, double* i_re, double* i_im);

/* ---- operator (engine.cpp:260-325): results in the caller's point order ---- */
typedef struct oc_report {
  double seconds[6]; /* setup, singular, level_d, interpolation, propagation, total */
  int depth;
  size_t peak_live_blocks;
} oc_report;

int oc_apply(size_t n, const double* x1, const double* x2, const double* x3,
             const double* a_re, const double* a_im, int kind, double wavenumber,
             const oc_params* p, double* i_re, double* i_im, oc_report* rep);

/* The same operator depth-first with O(depth) live blocks (C5-sized runs in a
 * few GB); agrees with oc_apply to rounding (cousin sums in another order). */
int oc_apply_lean(size_t n, const double* x1, const double* x2, const double* x3,
                  const double* a_re, const double* a_im, int kind, double wavenumber,
                  const oc_params* p, double* i_re, double* i_im, oc_report* rep);

int oc_direct_eval(size_t n, const double* x1, const double* x2, const double* x3,
                   const double* a_re, const double* a_im, int kind, double wavenumber,
                   const uint32_t* targets, size_t m, double* o_re, double* o_im);
int oc_sample_indices(size_t n, size_t m, uint64_t seed, uint32_t* out);
int oc_error_at_indices(size_t n, const double* x1, const double* x2, const double* x3,
                        const double* a_re, const double* a_im, const double* i_re,
                        const double* i_im, int kind, double wavenumber, const uint32_t* idx,
                        size_t m, double* eps);

/* ---- rank layout and exchange sets (dist.cpp:78-130, 179-237) ---- */
int oc_partition(const oc_problem* pr, int n_ranks, uint32_t* box_begin, uint32_t* point_begin,
                 uint32_t* cone_begin /* (D-2)*(n_ranks+1), level-major */);
/* Number of foreign blocks rank `rank` needs at level d, deduplicated per
 * (rank, cone): kind 0 = interpolation data, 1 = propagation data.  When
 * `cones` is non-NULL the sorted cone ordinals are written there. */
int oc_exchange_set(const oc_problem* pr, int n_ranks, int rank, int d, int kind,
                    uint32_t* cones, size_t* count);

#ifdef __cplusplus
}
#endif
#endif
