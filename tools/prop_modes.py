"""Time the K3 propagation kernels on one config (serial stage timing) and
check they agree.

usage: python tools/prop_modes.py C2 [node dmma rows fly]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

KINDS = {"node": 0, "dmma": 2, "rows": 3, "fly": 4, "auto": 7}
c = ifgf.configs.CONFIGS[sys.argv[1]]
modes = sys.argv[2:] or list(KINDS)
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
plan.set_serial(True)
ref = None
for name in modes:
    plan.set_prop_kernel(KINDS[name])
    best = None
    for _ in range(3):
        ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
        best = rep if best is None or rep.seconds.propagation < best.seconds.propagation else best
    if ref is None:
        ref = (ir, ii)
    err = np.sqrt(np.sum((ir - ref[0]) ** 2 + (ii - ref[1]) ** 2) / np.sum(ref[0] ** 2 + ref[1] ** 2))
    print(f"{name}: prop {best.seconds.propagation * 1e3:.2f} ms interp "
          f"{best.seconds.interpolation * 1e3:.2f} total {best.seconds.total * 1e3:.1f} "
          f"rel-diff {err:.2e}", flush=True)
