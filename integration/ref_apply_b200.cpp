// ref_apply_b200.cpp -- the translation unit a maintainer adds to the
// reference: ifgf::apply (engine.hpp:112-114,
// engine.cpp:260-325) re-exported on top of the C ABI of libifgf_b200.so, so
// the reference's own callers (tests/acceptance.cpp, the CLI) run the GPU
// matvec unmodified.  Exceptions are rethrown with the reference's classes
// (engine.cpp:261, kernel.hpp:30, engine.cpp:170-173, ...).
//
// oracle/Makefile (target `accept`) links it in front of the reference's
// objects, whose own `apply` is weakened, into oracle/_ref/ifgf_acceptance_b200
// (tests/test_gpu_acceptance.py runs it on the B200).
#include <stdexcept>

#include "ifgf/engine.hpp"
#include "ifgf_b200.h"

namespace ifgf {
namespace {
[[noreturn]] void rethrow(int rc) {
  const char* m = ifgf_last_error();
  switch (rc) {
    case IFGF_EINVAL:  throw std::invalid_argument(m);
    case IFGF_EDOMAIN: throw std::domain_error(m);
    case IFGF_ELOGIC:  throw std::logic_error(m);
    default:           throw std::runtime_error(m);
  }
}
}  // namespace

ApplyReport apply(PointCloud& pc, const KernelConfig& cfg, const EngineParams& p) {
  ifgf_params q;
  ifgf_default_params(&q);
  q.depth = p.depth;
  q.box_lambda = p.box_lambda;
  q.points_per_box = p.points_per_box;
  q.base_s = p.base_s;
  q.base_theta = p.base_theta;
  q.base_phi = p.base_phi;
  q.p_s = p.orders.p_s;
  q.p_theta = p.orders.p_theta;
  q.p_phi = p.orders.p_phi;
  ifgf_report r{};
  const int rc = ifgf_apply(pc.size(), pc.x1.data(), pc.x2.data(), pc.x3.data(),
                            pc.a_re.data(), pc.a_im.data(),
                            cfg.kind == KernelKind::Laplace ? IFGF_LAPLACE : IFGF_HELMHOLTZ,
                            cfg.wavenumber, &q, pc.i_re.data(), pc.i_im.data(), &r);
  if (rc) rethrow(rc);
  ApplyReport rep;
  rep.seconds = {r.setup, r.singular, r.level_d, r.interpolation, r.propagation, r.total};
  rep.depth = r.depth;
  rep.n = r.n;
  rep.h_level_d = r.h_level_d;
  for (int i = 0; i < r.n_levels; ++i) rep.levels.push_back({3 + i, r.level_boxes[i], r.level_cones[i]});
  rep.peak_live_blocks = r.peak_live_blocks;
  rep.simd_variant = "sm_100a";
  return rep;
}
}  // namespace ifgf
