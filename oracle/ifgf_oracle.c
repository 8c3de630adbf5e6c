/* ifgf_oracle.c -- plain-C restatement of the reference IFGF matvec.
 *
 * TEST INFRASTRUCTURE ONLY (see ifgf_oracle.h).  Citations are file:line in
 * /root/reference/proj.  Independent data structures (flat arrays, binary
 * search instead of hash maps, a merge sort instead of std::stable_sort), the
 * same arithmetic: every quantity that decides structure (cube, depth, grid
 * indices, box centres, cone coordinates) is computed with the reference's
 * operation order and no FMA contraction, so the octree and the relevant
 * cone sets come out identical, and the sums agree to rounding.
 */
#define _POSIX_C_SOURCE 200809L
#include "ifgf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OC_PI 3.14159265358979323846
#define OC_SMAX 0.57735026918962576451 /* sqrt(3)/3, cones.hpp:24 */
#define OC_MAXLEVEL 21                 /* morton.hpp:15 */
#define OC_MAXORDER 12                 /* interp.hpp:7 */
#define OC_NOCONE 0xffffffffu

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* oc_last_error(void) { return g_err; }

void oc_default_params(oc_params* p) {
  /* engine.hpp:12-19, interp.hpp:11-14 */
  p->depth = 0;
  p->box_lambda = 0.25;
  p->points_per_box = 64;
  p->base_s = 1;
  p->base_theta = 2;
  p->base_phi = 4;
  p->p_s = 3;
  p->p_theta = 5;
  p->p_phi = 5;
}

/* ------------------------------------------------------------ threading
 * oc_set_threads(T): the passes, the relevant-cone marking and the direct
 * sums split their ranges over T pthreads.  Every output slot (a target, a
 * cone, a box's cone list) is still computed by one thread in the serial
 * order, so results are bitwise independent of T. */
static int g_threads = 1;
void oc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int oc_get_threads(void) { return g_threads; }

typedef int (*range_fn)(void* ctx, size_t b, size_t e);
typedef struct {
  range_fn fn;
  void* ctx;
  size_t n, chunk, next;
  int rc;
  char err[256];
  pthread_mutex_t mu;
} par_job;

static void* par_worker(void* arg) {
  par_job* J = (par_job*)arg;
  for (;;) {
    if (__atomic_load_n(&J->rc, __ATOMIC_RELAXED)) break;
    const size_t b = __atomic_fetch_add(&J->next, J->chunk, __ATOMIC_RELAXED);
    if (b >= J->n) break;
    const size_t e = J->n - b > J->chunk ? b + J->chunk : J->n;
    const int rc = J->fn(J->ctx, b, e);
    if (rc) {
      pthread_mutex_lock(&J->mu);
      if (!J->rc) {
        J->rc = rc;
        memcpy(J->err, g_err, sizeof J->err);
      }
      pthread_mutex_unlock(&J->mu);
      break;
    }
  }
  return NULL;
}

/* fn over [0, n) in chunks; returns the first error code (message in g_err) */
static int par_for(size_t n, size_t chunk, range_fn fn, void* ctx) {
  if (!n) return OC_OK;
  if (chunk < 1) chunk = 1;
  int T = g_threads;
  if ((size_t)T > (n + chunk - 1) / chunk) T = (int)((n + chunk - 1) / chunk);
  if (T <= 1) return fn(ctx, 0, n);
  par_job J;
  memset(&J, 0, sizeof J);
  J.fn = fn;
  J.ctx = ctx;
  J.n = n;
  J.chunk = chunk;
  pthread_mutex_init(&J.mu, NULL);
  pthread_t* th = (pthread_t*)malloc((size_t)(T - 1) * sizeof(pthread_t));
  int started = 0;
  for (int t = 0; t < T - 1; ++t)
    if (pthread_create(&th[started], NULL, par_worker, &J) == 0) ++started;
  par_worker(&J);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.mu);
  if (J.rc) memcpy(g_err, J.err, sizeof J.err);
  return J.rc;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------ growable arrays */
typedef struct { uint32_t* v; size_t n, cap; } vu32;
typedef struct { uint64_t* v; size_t n, cap; } vu64;

static void vu32_push(vu32* a, uint32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 64;
    a->v = (uint32_t*)realloc(a->v, a->cap * sizeof(uint32_t));
  }
  a->v[a->n++] = x;
}
static void vu64_push(vu64* a, uint64_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 64;
    a->v = (uint64_t*)realloc(a->v, a->cap * sizeof(uint64_t));
  }
  a->v[a->n++] = x;
}

/* ------------------------------------------------------------- mt19937_64 */
/* Matsumoto-Nishimura 64-bit Mersenne twister (the algorithm std::mt19937_64
 * specifies); used by geometry.cpp:50-53 and engine.cpp:341-352. */
typedef struct { uint64_t mt[312]; int i; } mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g->mt[k] & 0xFFFFFFFF80000000ULL) |
                         (g->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->mt[(k + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[k] = v;
    }
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

uint64_t oc_mt64_first(uint64_t seed, int k) {
  mt64 g;
  mt64_seed(&g, seed);
  uint64_t x = 0;
  for (int i = 0; i < k; ++i) x = mt64_next(&g);
  return x;
}

/* ------------------------------------------------- synthetic inputs */
typedef struct { mt64 g; int have; double spare; } rng_t;

static double u01(rng_t* r) { return (double)(mt64_next(&r->g) >> 11) * 0x1.0p-53; }

static double gauss(rng_t* r) { /* explicit Box-Muller, pairs cached */
  if (r->have) {
    r->have = 0;
    return r->spare;
  }
  const double u1 = u01(r), u2 = u01(r);
  const double rad = sqrt(-2.0 * log(1.0 - u1));
  const double ang = 2.0 * OC_PI * u2;
  r->spare = rad * sin(ang);
  r->have = 1;
  return rad * cos(ang);
}

static void sphere_dir(rng_t* r, double* v) {
  for (;;) {
    const double gx = gauss(r), gy = gauss(r), gz = gauss(r);
    const double nrm = sqrt(gx * gx + gy * gy + gz * gz);
    if (nrm == 0.0) continue;
    const double inv = 1.0 / nrm;
    v[0] = inv * gx;
    v[1] = inv * gy;
    v[2] = inv * gz;
    return;
  }
}

int oc_generate(size_t n, int shape, double c, int dens, uint64_t seed, double* x1,
                double* x2, double* x3, double* a_re, double* a_im) {
  rng_t r;
  mt64_seed(&r.g, seed);
  r.have = 0;
  for (size_t i = 0; i < n; ++i) {
    double u[3];
    if (shape == 0) {
      sphere_dir(&r, u);
      x1[i] = u[0];
      x2[i] = u[1];
      x3[i] = u[2];
    } else {
      for (;;) { /* area element of (x,y,z)->(x,y,cz), normalised to max 1 */
        sphere_dir(&r, u);
        const double p = sqrt(c * c * (u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]);
        const double m = c > 1.0 ? c : 1.0;
        if (u01(&r) < p / m) break;
      }
      x1[i] = u[0];
      x2[i] = u[1];
      x3[i] = c * u[2];
    }
  }
  r.have = 0;
  for (size_t i = 0; i < n; ++i) {
    if (dens == 0) {
      a_re[i] = 2.0 * u01(&r) - 1.0;
      a_im[i] = 2.0 * u01(&r) - 1.0;
    } else {
      a_re[i] = gauss(&r);
      a_im[i] = 0.0;
    }
  }
  return OC_OK;
}

/* ---------------------------------------------------------------- kernels */
/* simd_kernels.hpp:14-42: Cody-Waite reduction by pi/2 + minimax polys. */
void oc_sincos_fast(double x, double* s, double* c) {
  const double q = nearbyint(x * 0.63661977236758134308);
  double r = x - q * 1.57079632673412561417e+00;
  r -= q * 6.07710050650619224932e-11;
  r -= q * 2.02226624879595063154e-21;
  const double r2 = r * r;
  double ps = 1.58962301576546568060e-10;
  ps = ps * r2 + -2.50507477628578072866e-8;
  ps = ps * r2 + 2.75573136213857245213e-6;
  ps = ps * r2 + -1.98412698295895385996e-4;
  ps = ps * r2 + 8.33333333332211858878e-3;
  ps = ps * r2 + -1.66666666666666307295e-1;
  const double sp = r + r * r2 * ps;
  double pc = -1.13585365213876817300e-11;
  pc = pc * r2 + 2.08757008419747316778e-9;
  pc = pc * r2 + -2.75573141792967388112e-7;
  pc = pc * r2 + 2.48015872888517179954e-5;
  pc = pc * r2 + -1.38888888888730564116e-3;
  pc = pc * r2 + 4.16666666666665929218e-2;
  const double cp = 1.0 - 0.5 * r2 + r2 * r2 * pc;
  const int64_t qi = (int64_t)q;
  const double ss = (qi & 1) ? cp : sp, cc = (qi & 1) ? sp : cp;
  *s = (qi & 2) ? -ss : ss;
  *c = ((qi + 1) & 2) ? -cc : cc;
}

/* kernels_scalar.cpp:12-30 (libm cos/sin) */
static void green_sum(const double* x1, const double* x2, const double* x3, const double* ar,
                      const double* ai, size_t i0, size_t i1, size_t skip, double tx,
                      double ty, double tz, double kappa, double* ore, double* oim) {
  const double q4 = 1.0 / (4.0 * OC_PI);
  double sr = 0.0, si = 0.0;
  for (size_t m = i0; m < i1; ++m) {
    if (m == skip) continue;
    const double dx = tx - x1[m], dy = ty - x2[m], dz = tz - x3[m];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double inv = q4 / r, kr = kappa * r;
    const double gr = cos(kr) * inv, gi = sin(kr) * inv;
    sr += ar[m] * gr - ai[m] * gi;
    si += ar[m] * gi + ai[m] * gr;
  }
  *ore = sr;
  *oim = si;
}

/* kernels_scalar.cpp:32-52 */
static void factored_sum(const double* x1, const double* x2, const double* x3,
                         const double* ar, const double* ai, size_t i0, size_t i1,
                         const double* t, const double* c, double kappa, double* ore,
                         double* oim) {
  const double cx = t[0] - c[0], cy = t[1] - c[1], cz = t[2] - c[2];
  const double rc = sqrt(cx * cx + cy * cy + cz * cz);
  double sr = 0.0, si = 0.0;
  for (size_t m = i0; m < i1; ++m) {
    const double dx = t[0] - x1[m], dy = t[1] - x2[m], dz = t[2] - x3[m];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double ratio = rc / r, ph = kappa * (r - rc);
    const double gr = cos(ph) * ratio, gi = sin(ph) * ratio;
    sr += ar[m] * gr - ai[m] * gi;
    si += ar[m] * gi + ai[m] * gr;
  }
  *ore = sr;
  *oim = si;
}

/* ------------------------------------------------------------------ morton */
/* morton.cpp:13-51: bit k of x/y/z lands at 3k/3k+1/3k+2. */
uint64_t oc_morton_encode(uint32_t ix, uint32_t iy, uint32_t iz) {
  uint64_t c = 0;
  for (int b = 0; b < 21; ++b) {
    c |= (uint64_t)((ix >> b) & 1u) << (3 * b);
    c |= (uint64_t)((iy >> b) & 1u) << (3 * b + 1);
    c |= (uint64_t)((iz >> b) & 1u) << (3 * b + 2);
  }
  return c;
}

void oc_morton_decode(uint64_t code, uint32_t* k) {
  k[0] = k[1] = k[2] = 0;
  for (int b = 0; b < 21; ++b) {
    k[0] |= (uint32_t)((code >> (3 * b)) & 1u) << b;
    k[1] |= (uint32_t)((code >> (3 * b + 1)) & 1u) << b;
    k[2] |= (uint32_t)((code >> (3 * b + 2)) & 1u) << b;
  }
}

/* engine.cpp:55-72 */
int oc_choose_depth(size_t n, double side, double kappa, const oc_params* p) {
  int d;
  if (p->depth > 0) {
    d = p->depth;
  } else if (kappa > 0.0) {
    const double lambda = 2.0 * OC_PI / kappa;
    const double ratio = side / (p->box_lambda * lambda);
    d = 1 + (int)floor(log2(ratio > 1.0 ? ratio : 1.0) + 1e-4);
  } else {
    const double boxes = (double)n / (double)(p->points_per_box > 1 ? p->points_per_box : 1);
    d = 1 + (int)ceil(0.5 * log2(boxes > 1.0 ? boxes : 1.0) - 1e-9);
  }
  if (d < 3) d = 3;
  if (d > OC_MAXLEVEL) d = OC_MAXLEVEL;
  return d;
}

/* ------------------------------------------------------------------ interp */
static double cheb_node(int j, int p) { /* interp.hpp:29-31 */
  return cos(OC_PI * (2.0 * j + 1.0) / (2.0 * p));
}

/* interp.cpp:19-34 transform matrices, built on demand */
static void transform_1d(int p, double* m) {
  for (int k = 0; k < p; ++k) {
    const double w = (k == 0 ? 1.0 : 2.0) / p;
    for (int j = 0; j < p; ++j) m[k * p + j] = w * cos(k * OC_PI * (2.0 * j + 1.0) / (2.0 * p));
  }
}

/* one separable pass: along the axis of length p and stride `stride` */
static void fit_axis(const double* m, int p, int stride, int total, const double* in,
                     double* out) {
  for (int base = 0; base < total; ++base) {
    if ((base / stride) % p != 0) continue; /* base = start of a pencil */
    for (int k = 0; k < p; ++k) {
      double acc = 0.0;
      for (int j = 0; j < p; ++j) acc += m[k * p + j] * in[base + j * stride];
      out[base + k * stride] = acc;
    }
  }
}

/* interp.cpp:68-91: phi (stride 1), theta (stride pp), s (stride pt*pp) */
void oc_cheb_fit(int ps, int pt, int pp, const double* vre, const double* vim, double* cre,
                 double* cim) {
  double ms[OC_MAXORDER * OC_MAXORDER], mt[OC_MAXORDER * OC_MAXORDER],
      mp[OC_MAXORDER * OC_MAXORDER];
  double t1[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER], t2[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  transform_1d(ps, ms);
  transform_1d(pt, mt);
  transform_1d(pp, mp);
  const int total = ps * pt * pp;
  for (int part = 0; part < 2; ++part) {
    const double* in = part ? vim : vre;
    double* out = part ? cim : cre;
    fit_axis(mp, pp, 1, total, in, t1);
    fit_axis(mt, pt, pp, total, t1, t2);
    fit_axis(ms, ps, pt * pp, total, t2, out);
  }
}

static double clenshaw(const double* c, int n, double t) { /* interp.cpp:40-50 */
  if (n == 1) return c[0];
  double b1 = c[n - 1], b2 = 0.0;
  const double t2 = 2.0 * t;
  for (int k = n - 2; k >= 1; --k) {
    const double b = c[k] + t2 * b1 - b2;
    b2 = b1;
    b1 = b;
  }
  return c[0] + t * b1 - b2;
}

/* interp.cpp:93-108: nested Clenshaw phi -> theta -> s */
void oc_cheb_eval(int ps, int pt, int pp, const double* cre, const double* cim, double ts,
                  double tt, double tp, double* ore, double* oim) {
  double row_re[OC_MAXORDER], row_im[OC_MAXORDER], col_re[OC_MAXORDER], col_im[OC_MAXORDER];
  for (int ks = 0; ks < ps; ++ks) {
    for (int kt = 0; kt < pt; ++kt) {
      const int base = (ks * pt + kt) * pp;
      row_re[kt] = clenshaw(cre + base, pp, tp);
      row_im[kt] = clenshaw(cim + base, pp, tp);
    }
    col_re[ks] = clenshaw(row_re, pt, tt);
    col_im[ks] = clenshaw(row_im, pt, tt);
  }
  *ore = clenshaw(col_re, ps, ts);
  *oim = clenshaw(col_im, ps, ts);
}

/* ------------------------------------------------------------------- cones */
typedef struct {
  int n[3];
  double w[3], inv_w[3];
} cgeom;

static cgeom level_geom(const oc_params* p, int depth, int d) { /* cones.hpp:26-33 */
  cgeom g;
  const int f = 1 << (depth - d);
  g.n[0] = p->base_s * f;
  g.n[1] = p->base_theta * f;
  g.n[2] = p->base_phi * f;
  g.w[0] = OC_SMAX / g.n[0];
  g.w[1] = OC_PI / g.n[1];
  g.w[2] = 2.0 * OC_PI / g.n[2];
  for (int i = 0; i < 3; ++i) g.inv_w[i] = 1.0 / g.w[i];
  return g;
}

int oc_cone_coords(const double* c, double h, const double* x, double* stp) {
  /* cones.cpp:9-20 */
  const double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  if (r == 0.0) return fail(OC_EDOMAIN, "cone_coords: point at box center");
  double ct = dz / r;
  if (ct < -1.0) ct = -1.0;
  if (ct > 1.0) ct = 1.0;
  stp[0] = sqrt(3.0) * h / (2.0 * r);
  stp[1] = acos(ct);
  double phi = atan2(dy, dx);
  if (phi < 0.0) phi += 2.0 * OC_PI;
  if (phi >= 2.0 * OC_PI) phi = 0.0;
  stp[2] = phi;
  return OC_OK;
}

static uint64_t gamma_pack(const int* idx, const int* n) { /* cones.cpp:22-24 */
  return ((uint64_t)idx[0] * (uint64_t)n[1] + (uint64_t)idx[1]) * (uint64_t)n[2] + (uint64_t)idx[2];
}

static void gamma_unpack(uint64_t g, const int* n, int* idx) { /* cones.cpp:26-32 */
  idx[2] = (int)(g % (uint64_t)n[2]);
  g /= (uint64_t)n[2];
  idx[1] = (int)(g % (uint64_t)n[1]);
  idx[0] = (int)(g / (uint64_t)n[1]);
}

/* setup-side segment lookup, cones.cpp:52-65 (divides by the widths) */
static int cone_of_point(const cgeom* g, const double* c, double h, const double* x,
                         uint64_t* gamma) {
  double stp[3];
  const int rc = oc_cone_coords(c, h, x, stp);
  if (rc) return rc;
  if (stp[0] > OC_SMAX * (1.0 + 1e-9))
    return fail(OC_EDOMAIN, "cone_of_point: point inside the neighbor zone (s > s_max)");
  int idx[3];
  for (int k = 0; k < 3; ++k) {
    int v = (int)(stp[k] / g->w[k]);
    idx[k] = v < g->n[k] - 1 ? v : g->n[k] - 1;
  }
  *gamma = gamma_pack(idx, g->n);
  return OC_OK;
}

/* apply-side locate, engine.cpp:29-51 (multiplies by inverse widths) */
static int locate_cone(const cgeom* g, double rad, const double* c, const double* x,
                       uint64_t* gamma, double* t3) {
  const double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  if (r == 0.0) return fail(OC_EDOMAIN, "cone_coords: point at box center");
  const double s = rad / r;
  if (s > OC_SMAX * (1.0 + 1e-9))
    return fail(OC_EDOMAIN, "cone_of_point: point inside the neighbor zone (s > s_max)");
  double ct = dz / r;
  if (ct < -1.0) ct = -1.0;
  if (ct > 1.0) ct = 1.0;
  const double theta = acos(ct);
  double phi = atan2(dy, dx);
  if (phi < 0.0) phi += 2.0 * OC_PI;
  if (phi >= 2.0 * OC_PI) phi = 0.0;
  const double f[3] = {s * g->inv_w[0], theta * g->inv_w[1], phi * g->inv_w[2]};
  int idx[3];
  for (int k = 0; k < 3; ++k) {
    int v = (int)f[k];
    idx[k] = v < g->n[k] - 1 ? v : g->n[k] - 1;
    t3[k] = 2.0 * (f[k] - idx[k]) - 1.0;
  }
  *gamma = gamma_pack(idx, g->n);
  return OC_OK;
}

/* cones.cpp:67-88: phi fastest */
static void interp_nodes(const oc_params* p, const cgeom* g, uint64_t gamma, const double* c,
                         double h, double* out3) {
  int idx[3];
  gamma_unpack(gamma, g->n, idx);
  const double slo = idx[0] * g->w[0], shi = (idx[0] + 1) * g->w[0];
  const double tlo = idx[1] * g->w[1], thi = (idx[1] + 1) * g->w[1];
  const double plo = idx[2] * g->w[2], phi_ = (idx[2] + 1) * g->w[2];
  const double sm = 0.5 * (slo + shi), sh = 0.5 * (shi - slo);
  const double tm = 0.5 * (tlo + thi), th = 0.5 * (thi - tlo);
  const double fm = 0.5 * (plo + phi_), fh = 0.5 * (phi_ - plo);
  const double rad = sqrt(3.0) * h / 2.0;
  size_t m = 0;
  for (int js = 0; js < p->p_s; ++js) {
    const double s = sm + sh * cheb_node(js, p->p_s);
    const double r = rad / s;
    for (int jt = 0; jt < p->p_theta; ++jt) {
      const double t = tm + th * cheb_node(jt, p->p_theta);
      const double st = sin(t), ct = cos(t);
      for (int jp = 0; jp < p->p_phi; ++jp) {
        const double f = fm + fh * cheb_node(jp, p->p_phi);
        out3[3 * m] = c[0] + r * st * cos(f);
        out3[3 * m + 1] = c[1] + r * st * sin(f);
        out3[3 * m + 2] = c[2] + r * ct;
        ++m;
      }
    }
  }
}

/* ------------------------------------------------------------------- tree */
typedef struct {
  size_t nb;
  double h;
  uint64_t* code;
  uint32_t *first, *count, *parent, *child_begin;
  double* ctr; /* 3 per box */
  vu32 nbr, cous;
  uint32_t *nbr_off, *cous_off;
  /* cones (d >= 3) */
  cgeom g;
  size_t nc;
  uint32_t* cone_box;
  uint64_t* cone_gamma;
  uint32_t* box_cone;
} oc_level;

struct oc_problem {
  size_t n;
  double kappa;
  oc_params p;
  double cube[4]; /* origin xyz, side */
  int depth;
  uint32_t* perm;
  double *x1, *x2, *x3, *ar, *ai;
  oc_level lv[OC_MAXLEVEL + 1]; /* 1-based */
};

static uint32_t lookup_code(const oc_level* L, uint64_t code) {
  size_t lo = 0, hi = L->nb;
  while (lo < hi) {
    const size_t mid = (lo + hi) / 2;
    if (L->code[mid] < code) lo = mid + 1;
    else hi = mid;
  }
  return (lo < L->nb && L->code[lo] == code) ? (uint32_t)lo : OC_NOCONE;
}

/* octree.cpp:157-167 */
static uint32_t box_of_sorted_point(const oc_level* L, size_t i) {
  size_t lo = 0, hi = L->nb;
  while (hi - lo > 1) {
    const size_t mid = lo + (hi - lo) / 2;
    if (L->first[mid] <= i) lo = mid;
    else hi = mid;
  }
  return (uint32_t)lo;
}

/* cones.hpp:110-122 */
static uint32_t find_cone(const oc_level* L, uint32_t b, uint64_t gamma) {
  uint32_t lo = L->box_cone[b], hi = L->box_cone[b + 1];
  const uint32_t end = hi;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (L->cone_gamma[mid] < gamma) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && L->cone_gamma[lo] == gamma) ? lo : OC_NOCONE;
}

/* stable merge sort of indices by key (morton.cpp:85-86 uses std::stable_sort) */
static void msort(uint32_t* idx, uint32_t* tmp, const uint64_t* key, size_t n) {
  if (n < 2) return;
  const size_t h = n / 2;
  msort(idx, tmp, key, h);
  msort(idx + h, tmp, key, n - h);
  size_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = (key[idx[j]] < key[idx[i]]) ? idx[j++] : idx[i++];
  while (i < h) tmp[k++] = idx[i++];
  while (j < n) tmp[k++] = idx[j++];
  memcpy(idx, tmp, n * sizeof(uint32_t));
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

static void box_center(const double* cube, const uint32_t* k, double h, double* c) {
  /* octree.cpp:10-14 */
  c[0] = cube[0] + (k[0] + 0.5) * h;
  c[1] = cube[1] + (k[1] + 0.5) * h;
  c[2] = cube[2] + (k[2] + 0.5) * h;
}

static int grid_index(const double* cube, int level, const double* x, uint32_t* k) {
  /* morton.cpp:53-68 */
  const uint32_t n = 1u << (level - 1);
  const double h = cube[3] / (double)n;
  for (int c = 0; c < 3; ++c) {
    const double rel = x[c] - cube[c];
    if (rel < 0.0 || rel >= cube[3]) return fail(OC_EDOMAIN, "point outside bounding cube");
    int64_t idx = (int64_t)floor(rel / h);
    if (idx >= (int64_t)n) idx = n - 1;
    k[c] = (uint32_t)idx;
  }
  return OC_OK;
}

static int build_levels(oc_problem* P) {
  const int D = P->depth;
  const size_t n = P->n;
  uint64_t* codes = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (size_t i = 0; i < n; ++i) {
    const double x[3] = {P->x1[i], P->x2[i], P->x3[i]};
    uint32_t k[3];
    if (grid_index(P->cube, D, x, k)) {
      free(codes);
      return OC_EDOMAIN;
    }
    codes[i] = oc_morton_encode(k[0], k[1], k[2]);
  }
  /* level D from runs of equal codes (octree.cpp:38-54) */
  {
    oc_level* L = &P->lv[D];
    size_t nb = 0;
    for (size_t i = 0; i < n; ++i) nb += (i == 0 || codes[i] != codes[i - 1]);
    L->nb = nb;
    L->h = P->cube[3] / (double)(1u << (D - 1));
    L->code = (uint64_t*)malloc(nb * sizeof(uint64_t));
    L->first = (uint32_t*)malloc(nb * sizeof(uint32_t));
    L->count = (uint32_t*)malloc(nb * sizeof(uint32_t));
    L->ctr = (double*)malloc(3 * nb * sizeof(double));
    size_t b = 0;
    for (size_t i = 0; i < n; ++i) {
      if (i == 0 || codes[i] != codes[i - 1]) {
        L->code[b] = codes[i];
        L->first[b] = (uint32_t)i;
        L->count[b] = 0;
        ++b;
      }
      L->count[b - 1]++;
    }
  }
  free(codes);
  /* coarser levels by >> 3 runs (octree.cpp:57-76) */
  for (int d = D - 1; d >= 1; --d) {
    const oc_level* F = &P->lv[d + 1];
    oc_level* L = &P->lv[d];
    size_t nb = 0;
    for (size_t i = 0; i < F->nb; ++i) nb += (i == 0 || (F->code[i] >> 3) != (F->code[i - 1] >> 3));
    L->nb = nb;
    L->h = P->cube[3] / (double)(1u << (d - 1));
    L->code = (uint64_t*)malloc(nb * sizeof(uint64_t));
    L->first = (uint32_t*)malloc(nb * sizeof(uint32_t));
    L->count = (uint32_t*)calloc(nb, sizeof(uint32_t));
    L->ctr = (double*)malloc(3 * nb * sizeof(double));
    size_t b = 0;
    for (size_t i = 0; i < F->nb; ++i) {
      if (i == 0 || (F->code[i] >> 3) != (F->code[i - 1] >> 3)) {
        L->code[b] = F->code[i] >> 3;
        L->first[b] = F->first[i];
        ++b;
      }
      L->count[b - 1] += F->count[i];
    }
  }
  for (int d = 1; d <= D; ++d) {
    oc_level* L = &P->lv[d];
    for (size_t b = 0; b < L->nb; ++b) {
      uint32_t k[3];
      oc_morton_decode(L->code[b], k);
      box_center(P->cube, k, L->h, &L->ctr[3 * b]);
    }
    L->parent = (uint32_t*)calloc(L->nb, sizeof(uint32_t));
    L->child_begin = (uint32_t*)calloc(L->nb + 1, sizeof(uint32_t));
  }
  /* parent links and child ranges (octree.cpp:85-94) */
  for (int d = 2; d <= D; ++d) {
    oc_level* L = &P->lv[d];
    oc_level* U = &P->lv[d - 1];
    for (size_t b = 0; b < L->nb; ++b) {
      L->parent[b] = lookup_code(U, L->code[b] >> 3);
      U->child_begin[L->parent[b] + 1]++;
    }
    for (size_t q = 0; q < U->nb; ++q) U->child_begin[q + 1] += U->child_begin[q];
  }
  /* neighbours incl. self, ordinal-sorted (octree.cpp:97-122) */
  for (int d = 1; d <= D; ++d) {
    oc_level* L = &P->lv[d];
    const int64_t side = (int64_t)1 << (d - 1);
    L->nbr_off = (uint32_t*)calloc(L->nb + 1, sizeof(uint32_t));
    for (size_t b = 0; b < L->nb; ++b) {
      uint32_t k[3], found[27];
      int cnt = 0;
      oc_morton_decode(L->code[b], k);
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int64_t j[3] = {(int64_t)k[0] + dx, (int64_t)k[1] + dy, (int64_t)k[2] + dz};
            if (j[0] < 0 || j[1] < 0 || j[2] < 0 || j[0] >= side || j[1] >= side || j[2] >= side)
              continue;
            const uint32_t o = lookup_code(L, oc_morton_encode((uint32_t)j[0], (uint32_t)j[1], (uint32_t)j[2]));
            if (o != OC_NOCONE) found[cnt++] = o;
          }
      for (int a = 1; a < cnt; ++a) /* insertion sort */
        for (int c = a; c > 0 && found[c - 1] > found[c]; --c) {
          const uint32_t t = found[c];
          found[c] = found[c - 1];
          found[c - 1] = t;
        }
      for (int a = 0; a < cnt; ++a) vu32_push(&L->nbr, found[a]);
      L->nbr_off[b + 1] = (uint32_t)L->nbr.n;
    }
  }
  /* cousins: children of parent-neighbours at Chebyshev distance > 1
   * (octree.cpp:127-147) */
  for (int d = 3; d <= D; ++d) {
    oc_level* L = &P->lv[d];
    const oc_level* U = &P->lv[d - 1];
    L->cous_off = (uint32_t*)calloc(L->nb + 1, sizeof(uint32_t));
    for (size_t b = 0; b < L->nb; ++b) {
      uint32_t k[3];
      oc_morton_decode(L->code[b], k);
      const uint32_t pb = L->parent[b];
      for (uint32_t pi = U->nbr_off[pb]; pi < U->nbr_off[pb + 1]; ++pi) {
        const uint32_t pn = U->nbr.v[pi];
        for (uint32_t c = U->child_begin[pn]; c < U->child_begin[pn + 1]; ++c) {
          uint32_t j[3], dist = 0;
          oc_morton_decode(L->code[c], j);
          for (int a = 0; a < 3; ++a) {
            const uint32_t dd = j[a] > k[a] ? j[a] - k[a] : k[a] - j[a];
            if (dd > dist) dist = dd;
          }
          if (dist > 1) vu32_push(&L->cous, c);
        }
      }
      L->cous_off[b + 1] = (uint32_t)L->cous.n;
    }
  }
  return OC_OK;
}

/* cones.cpp:90-150: top-down d = 3..D, clause 1 (cousin points) and clause 2
 * (nodes of the parent box's relevant cones).  Boxes are independent within a
 * level: chunks of RC_CHUNK boxes run in parallel (oc_set_threads), each
 * writing its boxes' sorted unique gammas into its own list, concatenated in
 * box order afterwards. */
#define RC_CHUNK 64
typedef struct {
  oc_problem* P;
  int d;
  vu64* out;      /* per chunk: the chunk's boxes' gammas, box order */
  uint32_t* cnt;  /* per box: number of relevant cones */
} rc_ctx;

static int rc_chunks(void* vctx, size_t c0, size_t c1) {
  rc_ctx* X = (rc_ctx*)vctx;
  oc_problem* P = X->P;
  const int d = X->d;
  const int np = P->p.p_s * P->p.p_theta * P->p.p_phi;
  oc_level* L = &P->lv[d];
  const oc_level* U = d > 3 ? &P->lv[d - 1] : NULL;
  double* nodes = (double*)malloc(3 * (size_t)np * sizeof(double));
  vu64 gam = {0, 0, 0};
  int rc = OC_OK;
  for (size_t ch = c0; ch < c1 && rc == OC_OK; ++ch) {
    vu64* cg = &X->out[ch];
    const size_t b1 = (ch + 1) * RC_CHUNK < L->nb ? (ch + 1) * RC_CHUNK : L->nb;
    for (size_t b = ch * RC_CHUNK; b < b1 && rc == OC_OK; ++b) {
      gam.n = 0;
      const double* c = &L->ctr[3 * b];
      for (uint32_t ci = L->cous_off[b]; ci < L->cous_off[b + 1] && rc == OC_OK; ++ci) {
        const uint32_t o = L->cous.v[ci];
        for (uint32_t i = L->first[o]; i < L->first[o] + L->count[o]; ++i) {
          const double x[3] = {P->x1[i], P->x2[i], P->x3[i]};
          uint64_t g;
          if ((rc = cone_of_point(&L->g, c, L->h, x, &g))) break;
          vu64_push(&gam, g);
        }
      }
      if (U && rc == OC_OK) {
        const uint32_t pb = L->parent[b];
        for (uint32_t q = U->box_cone[pb]; q < U->box_cone[pb + 1] && rc == OC_OK; ++q) {
          interp_nodes(&P->p, &U->g, U->cone_gamma[q], &U->ctr[3 * pb], U->h, nodes);
          for (int m = 0; m < np; ++m) {
            uint64_t g;
            if ((rc = cone_of_point(&L->g, c, L->h, &nodes[3 * m], &g))) break;
            vu64_push(&gam, g);
          }
        }
      }
      qsort(gam.v, gam.n, sizeof(uint64_t), cmp_u64);
      uint32_t k = 0;
      for (size_t i = 0; i < gam.n; ++i) {
        if (i > 0 && gam.v[i] == gam.v[i - 1]) continue;
        vu64_push(cg, gam.v[i]);
        ++k;
      }
      X->cnt[b] = k;
    }
  }
  free(gam.v);
  free(nodes);
  return rc;
}

static int relevant_cones(oc_problem* P) {
  const int D = P->depth;
  int rc = OC_OK;
  for (int d = 3; d <= D && rc == OC_OK; ++d) {
    oc_level* L = &P->lv[d];
    L->g = level_geom(&P->p, D, d);
    L->box_cone = (uint32_t*)calloc(L->nb + 1, sizeof(uint32_t));
    const size_t nch = (L->nb + RC_CHUNK - 1) / RC_CHUNK;
    rc_ctx X = {P, d, (vu64*)calloc(nch ? nch : 1, sizeof(vu64)),
                (uint32_t*)calloc(L->nb ? L->nb : 1, sizeof(uint32_t))};
    rc = par_for(nch, 1, rc_chunks, &X);
    if (rc == OC_OK) {
      for (size_t b = 0; b < L->nb; ++b) L->box_cone[b + 1] = L->box_cone[b] + X.cnt[b];
      const size_t nc = L->box_cone[L->nb];
      L->nc = nc;
      L->cone_box = (uint32_t*)malloc((nc ? nc : 1) * sizeof(uint32_t));
      L->cone_gamma = (uint64_t*)malloc((nc ? nc : 1) * sizeof(uint64_t));
      size_t o = 0;
      for (size_t ch = 0; ch < nch; ++ch) {
        if (X.out[ch].n) memcpy(L->cone_gamma + o, X.out[ch].v, X.out[ch].n * sizeof(uint64_t));
        o += X.out[ch].n;
      }
      for (size_t b = 0; b < L->nb; ++b)
        for (uint32_t q = L->box_cone[b]; q < L->box_cone[b + 1]; ++q) L->cone_box[q] = (uint32_t)b;
    }
    for (size_t ch = 0; ch < nch; ++ch) free(X.out[ch].v);
    free(X.out);
    free(X.cnt);
  }
  return rc;
}

int oc_problem_build(size_t n, const double* x1, const double* x2, const double* x3,
                     const double* a_re, const double* a_im, int kind, double wavenumber,
                     const oc_params* p, oc_problem** out) {
  /* engine.cpp:74-94 */
  *out = NULL;
  if (n < 1) return fail(OC_EINVAL, "empty point cloud");
  if (p->p_s < 1 || p->p_theta < 1 || p->p_phi < 1 || p->p_s > OC_MAXORDER ||
      p->p_theta > OC_MAXORDER || p->p_phi > OC_MAXORDER)
    return fail(OC_EINVAL, "unsupported interpolation orders");
  oc_problem* P = (oc_problem*)calloc(1, sizeof(oc_problem));
  P->n = n;
  P->p = *p;
  P->kappa = kind == 1 ? 0.0 : wavenumber;
  /* bounding cube, geometry.cpp:95-114 */
  double lo[3] = {x1[0], x2[0], x3[0]}, hi[3] = {x1[0], x2[0], x3[0]};
  for (size_t i = 1; i < n; ++i) {
    const double v[3] = {x1[i], x2[i], x3[i]};
    for (int c = 0; c < 3; ++c) {
      if (v[c] < lo[c]) lo[c] = v[c];
      if (v[c] > hi[c]) hi[c] = v[c];
    }
  }
  double ext = hi[0] - lo[0];
  if (hi[1] - lo[1] > ext) ext = hi[1] - lo[1];
  if (hi[2] - lo[2] > ext) ext = hi[2] - lo[2];
  double side = (1.0 + 1e-6) * ext;
  if (side < 1e-9) side = 1e-9;
  for (int c = 0; c < 3; ++c) P->cube[c] = 0.5 * (lo[c] + hi[c]) - 0.5 * side;
  P->cube[3] = side;
  P->depth = oc_choose_depth(n, side, P->kappa, p);
  /* Morton sort (morton.cpp:70-95) */
  uint64_t* codes = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (size_t i = 0; i < n; ++i) {
    const double x[3] = {x1[i], x2[i], x3[i]};
    uint32_t k[3];
    const int rc = grid_index(P->cube, P->depth, x, k);
    if (rc) {
      free(codes);
      oc_problem_free(P);
      return rc;
    }
    codes[i] = oc_morton_encode(k[0], k[1], k[2]);
  }
  P->perm = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* tmp = (uint32_t*)malloc(n * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) P->perm[i] = (uint32_t)i;
  msort(P->perm, tmp, codes, n);
  free(tmp);
  free(codes);
  P->x1 = (double*)malloc(n * sizeof(double));
  P->x2 = (double*)malloc(n * sizeof(double));
  P->x3 = (double*)malloc(n * sizeof(double));
  P->ar = (double*)malloc(n * sizeof(double));
  P->ai = (double*)malloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    const uint32_t j = P->perm[i];
    P->x1[i] = x1[j];
    P->x2[i] = x2[j];
    P->x3[i] = x3[j];
    P->ar[i] = a_re ? a_re[j] : 0.0;
    P->ai[i] = a_im ? a_im[j] : 0.0;
  }
  int rc = build_levels(P);
  if (!rc) rc = relevant_cones(P);
  if (rc) {
    oc_problem_free(P);
    return rc;
  }
  *out = P;
  return OC_OK;
}

void oc_problem_free(oc_problem* P) {
  if (!P) return;
  for (int d = 1; d <= OC_MAXLEVEL; ++d) {
    oc_level* L = &P->lv[d];
    free(L->code);
    free(L->first);
    free(L->count);
    free(L->parent);
    free(L->child_begin);
    free(L->ctr);
    free(L->nbr.v);
    free(L->cous.v);
    free(L->nbr_off);
    free(L->cous_off);
    free(L->cone_box);
    free(L->cone_gamma);
    free(L->box_cone);
  }
  free(P->perm);
  free(P->x1);
  free(P->x2);
  free(P->x3);
  free(P->ar);
  free(P->ai);
  free(P);
}

int oc_problem_depth(const oc_problem* P) { return P->depth; }
void oc_problem_cube(const oc_problem* P, double* o) { memcpy(o, P->cube, 4 * sizeof(double)); }

void oc_problem_sorted(const oc_problem* P, uint32_t* perm, double* x1, double* x2, double* x3,
                       double* a_re, double* a_im) {
  const size_t n = P->n;
  if (perm) memcpy(perm, P->perm, n * sizeof(uint32_t));
  if (x1) memcpy(x1, P->x1, n * sizeof(double));
  if (x2) memcpy(x2, P->x2, n * sizeof(double));
  if (x3) memcpy(x3, P->x3, n * sizeof(double));
  if (a_re) memcpy(a_re, P->ar, n * sizeof(double));
  if (a_im) memcpy(a_im, P->ai, n * sizeof(double));
}

void oc_problem_level_sizes(const oc_problem* P, int d, uint64_t* s, double* h) {
  const oc_level* L = &P->lv[d];
  s[0] = L->nb;
  s[1] = L->nc;
  s[2] = L->nbr.n;
  s[3] = L->cous.n;
  if (h) *h = L->h;
}

void oc_problem_level_boxes(const oc_problem* P, int d, uint64_t* codes, uint32_t* first,
                            uint32_t* count, double* centers3, uint32_t* parent,
                            uint32_t* child_begin) {
  const oc_level* L = &P->lv[d];
  if (codes) memcpy(codes, L->code, L->nb * sizeof(uint64_t));
  if (first) memcpy(first, L->first, L->nb * sizeof(uint32_t));
  if (count) memcpy(count, L->count, L->nb * sizeof(uint32_t));
  if (centers3) memcpy(centers3, L->ctr, 3 * L->nb * sizeof(double));
  if (parent) memcpy(parent, L->parent, L->nb * sizeof(uint32_t));
  if (child_begin && d < P->depth) memcpy(child_begin, L->child_begin, (L->nb + 1) * sizeof(uint32_t));
}

void oc_problem_level_adjacency(const oc_problem* P, int d, uint32_t* nbr_off, uint32_t* nbr,
                                uint32_t* cousin_off, uint32_t* cousin) {
  const oc_level* L = &P->lv[d];
  if (nbr_off) memcpy(nbr_off, L->nbr_off, (L->nb + 1) * sizeof(uint32_t));
  if (nbr) memcpy(nbr, L->nbr.v, L->nbr.n * sizeof(uint32_t));
  if (d >= 3) {
    if (cousin_off) memcpy(cousin_off, L->cous_off, (L->nb + 1) * sizeof(uint32_t));
    if (cousin) memcpy(cousin, L->cous.v, L->cous.n * sizeof(uint32_t));
  }
}

void oc_problem_level_cones(const oc_problem* P, int d, uint32_t* cone_box, uint64_t* gamma,
                            uint32_t* box_cone_begin) {
  const oc_level* L = &P->lv[d];
  if (cone_box) memcpy(cone_box, L->cone_box, L->nc * sizeof(uint32_t));
  if (gamma) memcpy(gamma, L->cone_gamma, L->nc * sizeof(uint64_t));
  if (box_cone_begin) memcpy(box_cone_begin, L->box_cone, (L->nb + 1) * sizeof(uint32_t));
}

/* ------------------------------------------------------------------ passes */
static int P_total(const oc_problem* P) { return P->p.p_s * P->p.p_theta * P->p.p_phi; }

/* engine.cpp:233-258 */
int oc_singular_pass(const oc_problem* P, size_t b, size_t e, double* i_re, double* i_im) {
  const oc_level* L = &P->lv[P->depth];
  for (size_t i = b; i < e; ++i) {
    const uint32_t bx = box_of_sorted_point(L, i);
    double ar = 0.0, ai = 0.0;
    for (uint32_t k = L->nbr_off[bx]; k < L->nbr_off[bx + 1]; ++k) {
      const uint32_t o = L->nbr.v[k];
      double sr, si;
      green_sum(P->x1, P->x2, P->x3, P->ar, P->ai, L->first[o], L->first[o] + L->count[o], i,
                P->x1[i], P->x2[i], P->x3[i], P->kappa, &sr, &si);
      ar += sr;
      ai += si;
    }
    i_re[i] += ar;
    i_im[i] += ai;
  }
  return OC_OK;
}

/* engine.cpp:107-136 */
int oc_level_d_pass(const oc_problem* P, uint32_t qb, uint32_t qe, double* blk_re,
                    double* blk_im) {
  const int D = P->depth, np = P_total(P);
  const oc_level* L = &P->lv[D];
  double nodes[3 * OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  double vr[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER], vi[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  for (uint32_t q = qb; q < qe; ++q) {
    const uint32_t b = L->cone_box[q];
    interp_nodes(&P->p, &L->g, L->cone_gamma[q], &L->ctr[3 * b], L->h, nodes);
    for (int m = 0; m < np; ++m)
      factored_sum(P->x1, P->x2, P->x3, P->ar, P->ai, L->first[b], L->first[b] + L->count[b],
                   &nodes[3 * m], &L->ctr[3 * b], P->kappa, &vr[m], &vi[m]);
    for (int m = 0; m < np; ++m)
      if (!isfinite(vr[m]) || !isfinite(vi[m]))
        return fail(OC_EINVAL, "cheb_fit: non-finite node value");
    oc_cheb_fit(P->p.p_s, P->p.p_theta, P->p.p_phi, vr, vi, blk_re + (size_t)q * np,
                blk_im + (size_t)q * np);
  }
  return OC_OK;
}

/* engine.cpp:138-189 */
int oc_propagation_pass(const oc_problem* P, int d, const double* cre, const double* cim,
                        uint32_t qb, uint32_t qe, double* pre, double* pim) {
  const int np = P_total(P);
  const oc_level* U = &P->lv[d - 1];
  const oc_level* L = &P->lv[d];
  const double rad = sqrt(3.0) * L->h / 2.0;
  double nodes[3 * OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  double rp[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  double acr[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER], aci[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  for (uint32_t q = qb; q < qe; ++q) {
    const uint32_t pb = U->cone_box[q];
    const double* pc = &U->ctr[3 * pb];
    interp_nodes(&P->p, &U->g, U->cone_gamma[q], pc, U->h, nodes);
    for (int m = 0; m < np; ++m) {
      const double dx = nodes[3 * m] - pc[0], dy = nodes[3 * m + 1] - pc[1],
                   dz = nodes[3 * m + 2] - pc[2];
      rp[m] = sqrt(dx * dx + dy * dy + dz * dz);
      acr[m] = aci[m] = 0.0;
    }
    for (uint32_t cb = U->child_begin[pb]; cb < U->child_begin[pb + 1]; ++cb) {
      const double* cc = &L->ctr[3 * cb];
      for (int m = 0; m < np; ++m) {
        uint64_t g;
        double t[3];
        const int rc = locate_cone(&L->g, rad, cc, &nodes[3 * m], &g, t);
        if (rc) return rc;
        const uint32_t cq = find_cone(L, cb, g);
        if (cq == OC_NOCONE)
          return fail(OC_ELOGIC, "propagation: node not covered by a relevant child cone");
        double vr, vi;
        oc_cheb_eval(P->p.p_s, P->p.p_theta, P->p.p_phi, cre + (size_t)cq * np,
                     cim + (size_t)cq * np, t[0], t[1], t[2], &vr, &vi);
        const double dx = nodes[3 * m] - cc[0], dy = nodes[3 * m + 1] - cc[1],
                     dz = nodes[3 * m + 2] - cc[2];
        const double rc_ = sqrt(dx * dx + dy * dy + dz * dz);
        const double ratio = rp[m] / rc_;
        double sn, cn;
        oc_sincos_fast(P->kappa * (rc_ - rp[m]), &sn, &cn);
        const double tr = ratio * cn, ti = ratio * sn;
        acr[m] += vr * tr - vi * ti;
        aci[m] += vr * ti + vi * tr;
      }
    }
    oc_cheb_fit(P->p.p_s, P->p.p_theta, P->p.p_phi, acr, aci, pre + (size_t)q * np,
                pim + (size_t)q * np);
  }
  return OC_OK;
}

/* engine.cpp:191-231 */
int oc_interpolation_pass(const oc_problem* P, int d, const double* bre, const double* bim,
                          size_t b, size_t e, double* i_re, double* i_im) {
  const int np = P_total(P);
  const oc_level* L = &P->lv[d];
  const double rad = sqrt(3.0) * L->h / 2.0;
  const double q4 = 1.0 / (4.0 * OC_PI);
  for (size_t i = b; i < e; ++i) {
    const double x[3] = {P->x1[i], P->x2[i], P->x3[i]};
    const uint32_t bx = box_of_sorted_point(L, i);
    double ar = 0.0, ai = 0.0;
    for (uint32_t ci = L->cous_off[bx]; ci < L->cous_off[bx + 1]; ++ci) {
      const uint32_t cb = L->cous.v[ci];
      const double* c = &L->ctr[3 * cb];
      uint64_t g;
      double t[3];
      const int rc = locate_cone(&L->g, rad, c, x, &g, t);
      if (rc) return rc;
      const uint32_t q = find_cone(L, cb, g);
      if (q == OC_NOCONE)
        return fail(OC_ELOGIC, "interpolation: cousin point not covered by a relevant cone");
      double vr, vi;
      oc_cheb_eval(P->p.p_s, P->p.p_theta, P->p.p_phi, bre + (size_t)q * np, bim + (size_t)q * np,
                   t[0], t[1], t[2], &vr, &vi);
      const double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double inv = q4 / r;
      double sn, cn;
      oc_sincos_fast(P->kappa * r, &sn, &cn);
      const double gr = cn * inv, gi = sn * inv;
      ar += vr * gr - vi * gi;
      ai += vr * gi + vi * gr;
    }
    i_re[i] += ar;
    i_im[i] += ai;
  }
  return OC_OK;
}

/* Range-parallel drivers of the passes (oc_set_threads); each target / cone
 * is computed by exactly one thread with the serial arithmetic. */
typedef struct {
  const oc_problem* P;
  int d;
  const double *in_re, *in_im;
  double *out_re, *out_im;
} pass_ctx;
static int par_singular(void* v, size_t b, size_t e) {
  pass_ctx* X = (pass_ctx*)v;
  return oc_singular_pass(X->P, b, e, X->out_re, X->out_im);
}
static int par_level_d(void* v, size_t b, size_t e) {
  pass_ctx* X = (pass_ctx*)v;
  return oc_level_d_pass(X->P, (uint32_t)b, (uint32_t)e, X->out_re, X->out_im);
}
static int par_interp(void* v, size_t b, size_t e) {
  pass_ctx* X = (pass_ctx*)v;
  return oc_interpolation_pass(X->P, X->d, X->in_re, X->in_im, b, e, X->out_re, X->out_im);
}
static int par_prop(void* v, size_t b, size_t e) {
  pass_ctx* X = (pass_ctx*)v;
  return oc_propagation_pass(X->P, X->d, X->in_re, X->in_im, (uint32_t)b, (uint32_t)e,
                             X->out_re, X->out_im);
}

/* ------------------------------------------------------------------- apply */
int oc_apply(size_t n, const double* x1, const double* x2, const double* x3,
             const double* a_re, const double* a_im, int kind, double wavenumber,
             const oc_params* p, double* i_re, double* i_im, oc_report* rep) {
  /* engine.cpp:260-325 */
  if (n < 2) return fail(OC_EINVAL, "apply: need at least two points");
  const double t_all = now_s();
  double t0 = now_s();
  oc_problem* P;
  int rc = oc_problem_build(n, x1, x2, x3, a_re, a_im, kind, wavenumber, p, &P);
  if (rc) return rc;
  oc_report r;
  memset(&r, 0, sizeof r);
  r.seconds[0] = now_s() - t0;
  const int D = P->depth, np = P_total(P);
  double* sr = (double*)calloc(n, sizeof(double));
  double* si = (double*)calloc(n, sizeof(double));
  t0 = now_s();
  {
    pass_ctx X = {P, 0, NULL, NULL, sr, si};
    rc = par_for(n, 4096, par_singular, &X);
  }
  r.seconds[1] = now_s() - t0;
  size_t ncur = P->lv[D].nc;
  double* cre = (double*)calloc(ncur * np + 1, sizeof(double));
  double* cim = (double*)calloc(ncur * np + 1, sizeof(double));
  r.peak_live_blocks = ncur;
  t0 = now_s();
  if (!rc) {
    pass_ctx X = {P, D, NULL, NULL, cre, cim};
    rc = par_for(ncur, 32, par_level_d, &X);
  }
  r.seconds[2] = now_s() - t0;
  for (int d = D; d >= 3 && !rc; --d) {
    t0 = now_s();
    {
      pass_ctx X = {P, d, cre, cim, sr, si};
      rc = par_for(n, 4096, par_interp, &X);
    }
    r.seconds[3] += now_s() - t0;
    if (rc || d == 3) break;
    const size_t npar = P->lv[d - 1].nc;
    if (ncur + npar > r.peak_live_blocks) r.peak_live_blocks = ncur + npar;
    double* pre = (double*)calloc(npar * np + 1, sizeof(double));
    double* pim = (double*)calloc(npar * np + 1, sizeof(double));
    t0 = now_s();
    {
      pass_ctx X = {P, d, cre, cim, pre, pim};
      rc = par_for(npar, 32, par_prop, &X);
    }
    r.seconds[4] += now_s() - t0;
    free(cre);
    free(cim);
    cre = pre;
    cim = pim;
    ncur = npar;
  }
  if (!rc)
    for (size_t i = 0; i < n; ++i) {
      i_re[P->perm[i]] = sr[i];
      i_im[P->perm[i]] = si[i];
    }
  free(cre);
  free(cim);
  free(sr);
  free(si);
  r.depth = D;
  oc_problem_free(P);
  r.seconds[5] = now_s() - t_all;
  if (rep) *rep = r;
  return rc;
}

/* ------------------------------------------------------------ lean apply
 * oc_apply_lean: the same matvec as oc_apply with O(depth) live blocks
 * instead of the reference's two full levels (engine.cpp:280-308), so C5
 * (25 M points, ~1.1e8 live blocks = 132 GB in the level-by-level form) runs
 * in a few GB.  Depth-first over the tree: a box's blocks are built from its
 * children's (recursively, children in Morton order: the propagation sums of
 * engine.cpp:138-189 in the reference's per-node child order, the same
 * arithmetic as oc_propagation_pass), then pushed to the targets that see
 * the box as a cousin (cousin relation is symmetric: the interpolation of
 * engine.cpp:191-231 reorganised by source box instead of by target), then
 * dropped once the parent has consumed them.  Level-3 subtrees are split
 * round-robin over the threads, each with its own result accumulators, summed
 * in thread order at the end: deterministic for a given thread count.  Only
 * the order in which a target's cousin contributions are added differs from
 * the level-by-level form (agreement to rounding, tests/test_oracle_cpu.py). */
typedef struct {
  const oc_problem* P;
  double *out_re, *out_im; /* this thread's result accumulators (sorted order) */
  double* nodes;           /* 3 * np scratch */
} lean_ctx;

/* engine.cpp:107-136 for the cones of box b at level D, local indexing */
static int lean_level_d(const oc_problem* P, uint32_t b, double* br, double* bi, double* nodes) {
  const int D = P->depth, np = P_total(P);
  const oc_level* L = &P->lv[D];
  double vr[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER], vi[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
  for (uint32_t q = L->box_cone[b]; q < L->box_cone[b + 1]; ++q) {
    const size_t o = (size_t)(q - L->box_cone[b]) * np;
    interp_nodes(&P->p, &L->g, L->cone_gamma[q], &L->ctr[3 * b], L->h, nodes);
    for (int m = 0; m < np; ++m)
      factored_sum(P->x1, P->x2, P->x3, P->ar, P->ai, L->first[b], L->first[b] + L->count[b],
                   &nodes[3 * m], &L->ctr[3 * b], P->kappa, &vr[m], &vi[m]);
    for (int m = 0; m < np; ++m)
      if (!isfinite(vr[m]) || !isfinite(vi[m])) return fail(OC_EINVAL, "cheb_fit: non-finite node value");
    oc_cheb_fit(P->p.p_s, P->p.p_theta, P->p.p_phi, vr, vi, br + o, bi + o);
  }
  return OC_OK;
}

/* engine.cpp:191-231 pushed from source box b at level d (blocks br/bi of
 * b's cones, local order) to every point of every cousin of b */
static int lean_push(lean_ctx* X, int d, uint32_t b, const double* br, const double* bi) {
  const oc_problem* P = X->P;
  const int np = P_total(P);
  const oc_level* L = &P->lv[d];
  const double rad = sqrt(3.0) * L->h / 2.0;
  const double q4 = 1.0 / (4.0 * OC_PI);
  const double* c = &L->ctr[3 * b];
  for (uint32_t k = L->cous_off[b]; k < L->cous_off[b + 1]; ++k) {
    const uint32_t t = L->cous.v[k];
    for (uint32_t i = L->first[t]; i < L->first[t] + L->count[t]; ++i) {
      const double x[3] = {P->x1[i], P->x2[i], P->x3[i]};
      uint64_t g;
      double tl[3];
      const int rc = locate_cone(&L->g, rad, c, x, &g, tl);
      if (rc) return rc;
      const uint32_t q = find_cone(L, b, g);
      if (q == OC_NOCONE)
        return fail(OC_ELOGIC, "interpolation: cousin point not covered by a relevant cone");
      const size_t o = (size_t)(q - L->box_cone[b]) * np;
      double vr, vi;
      oc_cheb_eval(P->p.p_s, P->p.p_theta, P->p.p_phi, br + o, bi + o, tl[0], tl[1], tl[2], &vr, &vi);
      const double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double inv = q4 / r;
      double sn, cn;
      oc_sincos_fast(P->kappa * r, &sn, &cn);
      const double gr = cn * inv, gi = sn * inv;
      X->out_re[i] += vr * gr - vi * gi;
      X->out_im[i] += vr * gi + vi * gr;
    }
  }
  return OC_OK;
}

/* blocks of box b at level d (local cone order) into *pr/*pi (malloc'd) */
static int lean_box(lean_ctx* X, int d, uint32_t b, double** pr, double** pi) {
  const oc_problem* P = X->P;
  const int D = P->depth, np = P_total(P);
  const oc_level* U = &P->lv[d];
  const size_t nbc = U->box_cone[b + 1] - U->box_cone[b];
  double* br = (double*)calloc(nbc * np + 1, sizeof(double));
  double* bi = (double*)calloc(nbc * np + 1, sizeof(double));
  int rc = OC_OK;
  if (d == D) {
    rc = lean_level_d(P, b, br, bi, X->nodes);
  } else {
    /* children first (their own pushes happen inside), then the propagation
     * of engine.cpp:138-189 restricted to b's cones */
    const uint32_t c0 = U->child_begin[b], c1 = U->child_begin[b + 1];
    double **cr = (double**)calloc(c1 - c0 + 1, sizeof(double*)),
           **ci = (double**)calloc(c1 - c0 + 1, sizeof(double*));
    for (uint32_t cb = c0; cb < c1 && rc == OC_OK; ++cb)
      rc = lean_box(X, d + 1, cb, &cr[cb - c0], &ci[cb - c0]);
    const oc_level* L = &P->lv[d + 1];
    const double rad = sqrt(3.0) * L->h / 2.0;
    double* nodes = X->nodes;
    double rp[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
    double acr[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER], aci[OC_MAXORDER * OC_MAXORDER * OC_MAXORDER];
    const double* pc = &U->ctr[3 * b];
    for (uint32_t q = U->box_cone[b]; q < U->box_cone[b + 1] && rc == OC_OK; ++q) {
      interp_nodes(&P->p, &U->g, U->cone_gamma[q], pc, U->h, nodes);
      for (int m = 0; m < np; ++m) {
        const double dx = nodes[3 * m] - pc[0], dy = nodes[3 * m + 1] - pc[1],
                     dz = nodes[3 * m + 2] - pc[2];
        rp[m] = sqrt(dx * dx + dy * dy + dz * dz);
        acr[m] = aci[m] = 0.0;
      }
      for (uint32_t cb = c0; cb < c1 && rc == OC_OK; ++cb) {
        const double* cc = &L->ctr[3 * cb];
        for (int m = 0; m < np; ++m) {
          uint64_t g;
          double t[3];
          if ((rc = locate_cone(&L->g, rad, cc, &nodes[3 * m], &g, t))) break;
          const uint32_t cq = find_cone(L, cb, g);
          if (cq == OC_NOCONE) {
            rc = fail(OC_ELOGIC, "propagation: node not covered by a relevant child cone");
            break;
          }
          const size_t o = (size_t)(cq - L->box_cone[cb]) * np;
          double vr, vi;
          oc_cheb_eval(P->p.p_s, P->p.p_theta, P->p.p_phi, cr[cb - c0] + o, ci[cb - c0] + o, t[0],
                       t[1], t[2], &vr, &vi);
          const double dx = nodes[3 * m] - cc[0], dy = nodes[3 * m + 1] - cc[1],
                       dz = nodes[3 * m + 2] - cc[2];
          const double rc_ = sqrt(dx * dx + dy * dy + dz * dz);
          const double ratio = rp[m] / rc_;
          double sn, cn;
          oc_sincos_fast(P->kappa * (rc_ - rp[m]), &sn, &cn);
          const double tr = ratio * cn, ti = ratio * sn;
          acr[m] += vr * tr - vi * ti;
          aci[m] += vr * ti + vi * tr;
        }
      }
      const size_t o = (size_t)(q - U->box_cone[b]) * np;
      if (rc == OC_OK) oc_cheb_fit(P->p.p_s, P->p.p_theta, P->p.p_phi, acr, aci, br + o, bi + o);
    }
    for (uint32_t k = 0; k < c1 - c0; ++k) {
      free(cr[k]);
      free(ci[k]);
    }
    free(cr);
    free(ci);
  }
  if (rc == OC_OK) rc = lean_push(X, d, b, br, bi);
  *pr = br;
  *pi = bi;
  return rc;
}

typedef struct {
  const oc_problem* P;
  int T;
  lean_ctx* ctx; /* per thread */
} lean_job;

/* thread t takes level-3 boxes t, t + T, ... (deterministic split) */
static int lean_thread_range(void* v, size_t t0, size_t t1) {
  lean_job* J = (lean_job*)v;
  for (size_t t = t0; t < t1; ++t) {
    lean_ctx* X = &J->ctx[t];
    const oc_level* L3 = &J->P->lv[3];
    for (size_t b = t; b < L3->nb; b += (size_t)J->T) {
      double *br, *bi;
      const int rc = lean_box(X, 3, (uint32_t)b, &br, &bi);
      free(br);
      free(bi);
      if (rc) return rc;
    }
  }
  return OC_OK;
}

int oc_apply_lean(size_t n, const double* x1, const double* x2, const double* x3,
                  const double* a_re, const double* a_im, int kind, double wavenumber,
                  const oc_params* p, double* i_re, double* i_im, oc_report* rep) {
  if (n < 2) return fail(OC_EINVAL, "apply: need at least two points");
  const double t_all = now_s();
  double t0 = now_s();
  oc_problem* P;
  int rc = oc_problem_build(n, x1, x2, x3, a_re, a_im, kind, wavenumber, p, &P);
  if (rc) return rc;
  oc_report r;
  memset(&r, 0, sizeof r);
  r.seconds[0] = now_s() - t0;
  const int np = P_total(P);
  double* sr = (double*)calloc(n, sizeof(double));
  double* si = (double*)calloc(n, sizeof(double));
  t0 = now_s();
  {
    pass_ctx X = {P, 0, NULL, NULL, sr, si};
    rc = par_for(n, 4096, par_singular, &X);
  }
  r.seconds[1] = now_s() - t0;
  const int T = g_threads;
  lean_job J = {P, T, (lean_ctx*)calloc((size_t)T, sizeof(lean_ctx))};
  for (int t = 0; t < T && !rc; ++t) {
    J.ctx[t].P = P;
    J.ctx[t].out_re = (double*)calloc(n, sizeof(double));
    J.ctx[t].out_im = (double*)calloc(n, sizeof(double));
    J.ctx[t].nodes = (double*)malloc(3 * (size_t)np * sizeof(double));
    if (!J.ctx[t].out_re || !J.ctx[t].out_im) rc = fail(OC_ERUNTIME, "lean apply: out of memory");
  }
  t0 = now_s();
  if (!rc) rc = par_for((size_t)T, 1, lean_thread_range, &J);
  r.seconds[4] = now_s() - t0; /* propagation + interpolation, interleaved */
  if (!rc) {
    for (int t = 0; t < T; ++t)
      for (size_t i = 0; i < n; ++i) {
        sr[i] += J.ctx[t].out_re[i];
        si[i] += J.ctx[t].out_im[i];
      }
    for (size_t i = 0; i < n; ++i) {
      i_re[P->perm[i]] = sr[i];
      i_im[P->perm[i]] = si[i];
    }
  }
  for (int t = 0; t < T; ++t) {
    free(J.ctx[t].out_re);
    free(J.ctx[t].out_im);
    free(J.ctx[t].nodes);
  }
  free(J.ctx);
  free(sr);
  free(si);
  r.depth = P->depth;
  oc_problem_free(P);
  r.seconds[5] = now_s() - t_all;
  if (rep) *rep = r;
  return rc;
}

typedef struct {
  size_t n;
  const double *x1, *x2, *x3, *ar, *ai;
  double kappa;
  const uint32_t* targets;
  double *o_re, *o_im;
} direct_ctx;
static int par_direct(void* v, size_t b, size_t e) {
  const direct_ctx* X = (const direct_ctx*)v;
  for (size_t j = b; j < e; ++j) {
    const size_t i = X->targets ? X->targets[j] : j;
    green_sum(X->x1, X->x2, X->x3, X->ar, X->ai, 0, X->n, i, X->x1[i], X->x2[i], X->x3[i],
              X->kappa, &X->o_re[j], &X->o_im[j]);
  }
  return OC_OK;
}

/* engine.cpp:327-339 restricted to a target list (all points when targets == NULL) */
int oc_direct_eval(size_t n, const double* x1, const double* x2, const double* x3,
                   const double* a_re, const double* a_im, int kind, double wavenumber,
                   const uint32_t* targets, size_t m, double* o_re, double* o_im) {
  if (n < 2) return fail(OC_EINVAL, "direct_eval: need at least two points");
  direct_ctx X = {n, x1, x2, x3, a_re, a_im, kind == 1 ? 0.0 : wavenumber, targets, o_re, o_im};
  return par_for(targets ? m : n, 4, par_direct, &X);
}

/* engine.cpp:341-352 */
int oc_sample_indices(size_t n, size_t m, uint64_t seed, uint32_t* out) {
  if (m > n) return fail(OC_EINVAL, "sample_indices: m > n");
  uint32_t* idx = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  mt64 g;
  mt64_seed(&g, seed);
  for (size_t j = 0; j < m; ++j) {
    const size_t k = j + (size_t)(mt64_next(&g) % (uint64_t)(n - j));
    const uint32_t t = idx[j];
    idx[j] = idx[k];
    idx[k] = t;
  }
  memcpy(out, idx, m * sizeof(uint32_t));
  free(idx);
  return OC_OK;
}

/* engine.cpp:354-376 */
int oc_error_at_indices(size_t n, const double* x1, const double* x2, const double* x3,
                        const double* a_re, const double* a_im, const double* i_re,
                        const double* i_im, int kind, double wavenumber, const uint32_t* idx,
                        size_t m, double* eps) {
  double* dr = (double*)malloc((m ? m : 1) * sizeof(double));
  double* di = (double*)malloc((m ? m : 1) * sizeof(double));
  int rc = oc_direct_eval(n, x1, x2, x3, a_re, a_im, kind, wavenumber, idx, m, dr, di);
  if (!rc) {
    double num = 0.0, den = 0.0;
    for (size_t j = 0; j < m; ++j) {
      const double er = dr[j] - i_re[idx[j]], ei = di[j] - i_im[idx[j]];
      num += er * er + ei * ei;
      den += dr[j] * dr[j] + di[j] * di[j];
    }
    if (den == 0.0) rc = fail(OC_EDOMAIN, "estimate_error: zero reference norm");
    else *eps = sqrt(num / den);
  }
  free(dr);
  free(di);
  return rc;
}

/* ---------------------------------------------------------------- partition */
int oc_partition(const oc_problem* P, int R, uint32_t* box_begin, uint32_t* point_begin,
                 uint32_t* cone_begin) {
  /* dist.cpp:78-130 */
  if (R < 1) return fail(OC_EINVAL, "partition: need at least one rank");
  const oc_level* L = &P->lv[P->depth];
  const size_t nb = L->nb;
  if ((size_t)R > nb)
    return fail(OC_EINVAL, "partition: more ranks than relevant finest-level boxes");
  const size_t npts = (size_t)L->first[nb - 1] + L->count[nb - 1];
  box_begin[0] = point_begin[0] = 0;
  uint32_t b = 0;
  for (int r = 0; r < R - 1; ++r) {
    const double target = (double)npts * (r + 1) / R;
    const uint32_t max_end = (uint32_t)nb - (uint32_t)(R - 1 - r);
    uint32_t e = b + 1;
    while (e < max_end && (double)(L->first[e - 1] + L->count[e - 1]) < target) ++e;
    box_begin[r + 1] = e;
    point_begin[r + 1] = L->first[e - 1] + L->count[e - 1];
    b = e;
  }
  box_begin[R] = (uint32_t)nb;
  point_begin[R] = (uint32_t)npts;
  for (int d = 3; d <= P->depth; ++d) {
    uint32_t* cb = cone_begin + (size_t)(d - 3) * (R + 1);
    const size_t nc = P->lv[d].nc, base = nc / R, extra = nc % R;
    cb[0] = 0;
    for (int r = 0; r < R; ++r) cb[r + 1] = cb[r] + (uint32_t)(base + ((size_t)r < extra ? 1 : 0));
  }
  return OC_OK;
}

static int owner_of(const uint32_t* begin, int R, uint32_t v) {
  int lo = 0, hi = R; /* last r with begin[r] <= v */
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (begin[mid] <= v) lo = mid;
    else hi = mid;
  }
  return lo;
}

/* dist.cpp:179-201 (kind 0) and dist.cpp:206-237 (kind 1) */
int oc_exchange_set(const oc_problem* P, int R, int rank, int d, int kind, uint32_t* cones,
                    size_t* count) {
  const int D = P->depth;
  uint32_t* bb = (uint32_t*)malloc((R + 1) * sizeof(uint32_t));
  uint32_t* pb_ = (uint32_t*)malloc((R + 1) * sizeof(uint32_t));
  uint32_t* cb = (uint32_t*)malloc((size_t)(D - 2) * (R + 1) * sizeof(uint32_t));
  int rc = oc_partition(P, R, bb, pb_, cb);
  const oc_level* L = &P->lv[d];
  unsigned char* seen = (unsigned char*)calloc(L->nc + 1, 1);
  const uint32_t* own = cb + (size_t)(d - 3) * (R + 1);
  if (!rc && kind == 0) {
    for (uint32_t i = pb_[rank]; i < pb_[rank + 1] && !rc; ++i) {
      const double x[3] = {P->x1[i], P->x2[i], P->x3[i]};
      const uint32_t b = box_of_sorted_point(L, i);
      for (uint32_t ci = L->cous_off[b]; ci < L->cous_off[b + 1]; ++ci) {
        const uint32_t c = L->cous.v[ci];
        uint64_t g;
        if ((rc = cone_of_point(&L->g, &L->ctr[3 * c], L->h, x, &g))) break;
        const uint32_t q = find_cone(L, c, g);
        if (q == OC_NOCONE) {
          rc = fail(OC_ELOGIC, "communicate: cousin cone not relevant");
          break;
        }
        if (owner_of(own, R, q) != rank) seen[q] = 1;
      }
    }
  } else if (!rc && kind == 1 && d > 3) {
    const oc_level* U = &P->lv[d - 1];
    const uint32_t* pown = cb + (size_t)(d - 4) * (R + 1);
    const int np = P_total(P);
    double* nodes = (double*)malloc(3 * (size_t)np * sizeof(double));
    for (uint32_t q = pown[rank]; q < pown[rank + 1] && !rc; ++q) {
      const uint32_t pbx = U->cone_box[q];
      interp_nodes(&P->p, &U->g, U->cone_gamma[q], &U->ctr[3 * pbx], U->h, nodes);
      for (uint32_t c = U->child_begin[pbx]; c < U->child_begin[pbx + 1] && !rc; ++c)
        for (int m = 0; m < np; ++m) {
          uint64_t g;
          if ((rc = cone_of_point(&L->g, &L->ctr[3 * c], L->h, &nodes[3 * m], &g))) break;
          const uint32_t cq = find_cone(L, c, g);
          if (cq == OC_NOCONE) {
            rc = fail(OC_ELOGIC, "communicate: child cone not relevant");
            break;
          }
          if (owner_of(own, R, cq) != rank) seen[cq] = 1;
        }
    }
    free(nodes);
  }
  size_t k = 0;
  for (size_t q = 0; q < L->nc; ++q)
    if (seen[q]) {
      if (cones) cones[k] = (uint32_t)q;
      ++k;
    }
  *count = k;
  free(seen);
  free(bb);
  free(pb_);
  free(cb);
  return rc;
}
