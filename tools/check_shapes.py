"""AUTO / DMMA / ROWS K3 on shapes outside the BASELINE configs: agreement and
the sampled error against direct sums.

usage: python tools/check_shapes.py
"""
import sys, os, math, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2112_15198_b200 as ifgf
from paper_2112_15198_b200.points import generate_surface
# cube-face surface grids (sphere and prolate shapes of the reference's generator),
# a spheroid and a Laplace sphere from the seeded generator
for shape, n, kappa, c in ((-1, 320, 16 * math.pi, 1.0), (-2, 360, 20 * math.pi, 1.0),
                           (1, 800000, 24 * math.pi, 0.5), (0, 300000, 0.0, 1.0)):
    if shape < 0:
        pc = generate_surface(-shape - 1, 1.0, n, 5)
        n = len(pc.x1)
        rng = np.random.default_rng(3)
        pc.a_re[:] = rng.uniform(-1, 1, n)
        pc.a_im[:] = rng.uniform(-1, 1, n)
    else:
        pc = ifgf.generate(n, shape, c, 0, 5)
    kind = ifgf.KernelKind.Laplace if kappa == 0.0 else ifgf.KernelKind.Helmholtz
    cfg = ifgf.KernelConfig(kind, kappa)
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams())
    out = {}
    for name, k in (("rows", plan.PROP_ROWS), ("auto", plan.PROP_AUTO), ("dmma", plan.PROP_DMMA)):
        plan.set_prop_kernel(k)
        plan.apply(pc.a_re, pc.a_im)  # builds the kernel's tables
        ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
        out[name] = (ir.copy(), ii.copy(), rep.seconds.propagation)
    ref = out["rows"]
    def rd(a): return math.sqrt(np.sum((a[0]-ref[0])**2 + (a[1]-ref[1])**2) / np.sum(ref[0]**2 + ref[1]**2))
    idx = np.arange(0, n, n // 500)[:500].astype(np.uint32)
    q = pc.copy(); q.i_re[:] = out["auto"][0]; q.i_im[:] = out["auto"][1]
    d = pc.copy(); ifgf.direct_eval(d, cfg, targets=idx)
    err = math.sqrt(np.sum((q.i_re[idx]-d.i_re[idx])**2 + (q.i_im[idx]-d.i_im[idx])**2) / np.sum(d.i_re[idx]**2 + d.i_im[idx]**2))
    print(f"shape {shape} N={n} depth {plan.depth}: prop ms rows {ref[2]*1e3:.2f} auto {out['auto'][2]*1e3:.2f} dmma {out['dmma'][2]*1e3:.2f}; "
          f"rel diff auto {rd(out['auto']):.2e} dmma {rd(out['dmma']):.2e}; eps vs direct {err:.3e}", flush=True)
    plan.close()
