import sys, os; sys.path.insert(0, '/root/repo')
import paper_2112_15198_b200 as ifgf
c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams())
plan.set_serial(True)
ref = None
for name, kind in [("node", 0), ("tiles", 1), ("dmma", 2)]:
    plan.set_prop_kernel(kind)
    for _ in range(3): ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
    import numpy as np
    if ref is None: ref = (ir, ii)
    err = np.sqrt(np.sum((ir-ref[0])**2+(ii-ref[1])**2)/np.sum(ref[0]**2+ref[1]**2))
    print(f"{name}: prop {rep.seconds.propagation*1e3:.2f} ms interp {rep.seconds.interpolation*1e3:.2f} total {rep.seconds.total*1e3:.1f} rel-diff {err:.2e}")
