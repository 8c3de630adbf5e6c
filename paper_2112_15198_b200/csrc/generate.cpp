// generate.cpp -- seeded synthetic point clouds for the BASELINE configs
// (DESIGN.md "Inputs").  Host-only harness code: std::mt19937_64 stream,
// 53-bit uniforms as in geometry.cpp:50-53, explicit Box-Muller normals
// (std::normal_distribution is implementation-defined), positions first then
// densities from the same stream.
#include <cmath>
#include <random>

#include "../../include/ifgf_b200.h"

namespace {

struct Stream {
  std::mt19937_64 g;
  bool have = false;
  double spare = 0.0;
  explicit Stream(uint64_t seed) : g(seed) {}
  double u01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = u01(), u2 = u01();
    const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
    const double ang = 2.0 * 3.14159265358979323846 * u2;
    spare = rad * std::sin(ang);
    have = true;
    return rad * std::cos(ang);
  }
  void direction(double* v) {
    for (;;) {
      const double gx = normal(), gy = normal(), gz = normal();
      const double nrm = std::sqrt(gx * gx + gy * gy + gz * gz);
      if (nrm == 0.0) continue;
      const double inv = 1.0 / nrm;
      v[0] = inv * gx;
      v[1] = inv * gy;
      v[2] = inv * gz;
      return;
    }
  }
};

}  // namespace

extern "C" int ifgf_generate(size_t n, int shape, double c, int dens, uint64_t seed, double* x1,
                             double* x2, double* x3, double* a_re, double* a_im) {
  if (shape != 0 && shape != 1) return IFGF_EINVAL;
  if (shape == 1 && !(c > 0.0)) return IFGF_EINVAL;
  Stream st(seed);
  for (size_t i = 0; i < n; ++i) {
    double u[3];
    if (shape == 0) {
      st.direction(u);
      x1[i] = u[0];
      x2[i] = u[1];
      x3[i] = u[2];
      continue;
    }
    // spheroid (1,1,c): accept with the area element of (x,y,z)->(x,y,cz)
    // normalised to its maximum, sqrt(c^2 (ux^2+uy^2) + uz^2) / max(c, 1)
    const double m = c > 1.0 ? c : 1.0;
    for (;;) {
      st.direction(u);
      const double p = std::sqrt(c * c * (u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]);
      if (st.u01() < p / m) break;
    }
    x1[i] = u[0];
    x2[i] = u[1];
    x3[i] = c * u[2];
  }
  st.have = false;
  for (size_t i = 0; i < n; ++i) {
    if (dens == 0) {
      a_re[i] = 2.0 * st.u01() - 1.0;
      a_im[i] = 2.0 * st.u01() - 1.0;
    } else {
      a_re[i] = st.normal();
      a_im[i] = 0.0;
    }
  }
  return IFGF_OK;
}

// generate_surface (geometry.cpp:57-93): the reference's cube-face surfaces,
// n_per_dim^2 cell centres per face projected to the radius-a sphere, z scaled
// by the shape (axis_scale, geometry.cpp:40-47); densities U[0,1) re then im
// per point from mt19937_64(seed) (geometry.cpp:87-91).  Same operation order
// as the reference (no contraction: this file is compiled without -ffp-contract).
extern "C" int ifgf_generate_surface(int shape, double a, int n_per_dim, uint64_t seed,
                                     double* x1, double* x2, double* x3, double* a_re,
                                     double* a_im) {
  if (!(a > 0.0) || n_per_dim < 2 || shape < 0 || shape > 2) return IFGF_EINVAL;
  const int n = n_per_dim;
  const double zs = shape == 0 ? 1.0 : (shape == 1 ? 0.1 : 10.0);
  size_t m = 0;
  for (int face = 0; face < 6; ++face) {
    const int axis = face / 2;
    const double sign = (face % 2 == 0) ? 1.0 : -1.0;
    for (int i = 0; i < n; ++i) {
      const double u = -1.0 + (2.0 * i + 1.0) / n;
      for (int j = 0; j < n; ++j) {
        const double v = -1.0 + (2.0 * j + 1.0) / n;
        double p[3];
        p[axis] = sign;
        p[(axis + 1) % 3] = u;
        p[(axis + 2) % 3] = v;
        const double inv = 1.0 / std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
        x1[m] = a * p[0] * inv;
        x2[m] = a * p[1] * inv;
        x3[m] = zs * a * p[2] * inv;
        ++m;
      }
    }
  }
  std::mt19937_64 g(seed);
  for (size_t i = 0; i < m; ++i) {
    a_re[i] = static_cast<double>(g() >> 11) * 0x1.0p-53;
    a_im[i] = static_cast<double>(g() >> 11) * 0x1.0p-53;
  }
  return IFGF_OK;
}

// bench::checksum_hex (bench.cpp:26-41): 64-bit FNV-1a over the bytes of re
// then im; out receives 16 hex digits and a NUL.
extern "C" void ifgf_checksum_hex(const double* re, const double* im, size_t n, char* out) {
  uint64_t h = 1469598103934665603ull;
  const auto mix = [&h](const double* v, size_t count) {
    const auto* p = reinterpret_cast<const unsigned char*>(v);
    for (size_t i = 0; i < count * sizeof(double); ++i) {
      h ^= p[i];
      h *= 1099511628211ull;
    }
  };
  mix(re, n);
  mix(im, n);
  static const char* hex = "0123456789abcdef";
  for (int i = 0; i < 16; ++i) out[i] = hex[(h >> (60 - 4 * i)) & 15u];
  out[16] = '\0';
}
