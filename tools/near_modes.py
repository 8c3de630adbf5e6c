"""Time the K1 near-field kernels on one config (serial stage timing) and
check they agree.

usage: python tools/near_modes.py C2 [point box]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200.work import count_work  # noqa: E402

KINDS = {"point": 0, "box": 1}
c = ifgf.configs.CONFIGS[sys.argv[1]]
modes = sys.argv[2:] or list(KINDS)
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
plan.set_serial(True)
pairs = count_work(plan).near_pairs
ref = None
for name in modes:
    plan.set_near_kernel(KINDS[name])
    best = None
    for _ in range(4):
        ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
        best = rep if best is None or rep.seconds.singular < best.seconds.singular else best
    if ref is None:
        ref = (ir, ii)
    err = np.sqrt(np.sum((ir - ref[0]) ** 2 + (ii - ref[1]) ** 2) / np.sum(ref[0] ** 2 + ref[1] ** 2))
    t = best.seconds.singular
    print(f"{name}: near {t * 1e3:.3f} ms  {pairs * 57 / t / 1e12:.2f} TF/s (57 flop/pair) "
          f"total {best.seconds.total * 1e3:.1f} ms rel-diff {err:.2e}", flush=True)
