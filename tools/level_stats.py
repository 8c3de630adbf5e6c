"""Per-level structure of a plan: boxes, cones, distinct cone segments
(gamma), cones per gamma (the reuse the K3 tiles exploit) and points per box.

usage: python tools/level_stats.py C2
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
print(f"{c.label}: depth {plan.depth}")
for d in range(3, plan.depth + 1):
    L = plan.level(d)
    ng = len(np.unique(L.cone_gamma)) if len(L.cone_gamma) else 0
    nc = len(L.cone_gamma)
    print(f"d={d}: boxes {len(L.count):8d}  pts/box {np.mean(L.count):8.1f}  cones {nc:9d}  "
          f"gammas {ng:8d}  cones/gamma {nc / max(ng, 1):7.2f}  cousins/box "
          f"{len(L.cousin) / max(len(L.count), 1):6.1f}")
