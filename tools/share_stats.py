"""Per parent level: cones, distinct gammas, gamma sharing inside groups of
consecutive parent boxes, children per box (how much a tile's row data could
be reused if cones sharing a gamma were processed together).

usage: python tools/share_stats.py C2
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
D = plan.depth
for d in range(D - 1, 2, -1):
    S = plan.level(d)
    cb, cg = S.cone_box.astype(np.int64), S.cone_gamma.astype(np.int64)
    nch = np.diff(S.child_begin.astype(np.int64))
    line = f"parent d={d}: boxes {len(S.codes)} cones {len(cb)} distinct gamma {len(np.unique(cg))}" \
           f" children/box {nch.mean():.2f} cones/box {len(cb) / len(S.codes):.0f}"
    for gb in (1, 8, 32, 128):
        key = (cb // gb) * (1 << 32) + cg
        u = len(np.unique(key))
        line += f" | gb={gb}: cones/key {len(cb) / u:.2f}"
    print(line, flush=True)
