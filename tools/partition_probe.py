import math, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2112_15198_b200 as ifgf
from paper_2112_15198_b200.dist import simulate
for (n, shape, c, kap, R) in [(400000, 1, 0.25, 2*math.pi*16, 4), (400000, 1, 0.25, 2*math.pi*16, 8), (400000, 0, 1.0, 2*math.pi*16, 8)]:
    pc = ifgf.generate(n, shape, c, 0, 43)
    cfg = ifgf.KernelConfig(ifgf.KernelKind.Helmholtz, kap)
    for mode in (0, 1):
        plans = [ifgf.Plan.from_cloud(pc, cfg) for _ in range(R)]
        res = []
        for _ in range(3):
            secs = []
            simulate(plans, pc.a_re, pc.a_im, partition=mode, rank_seconds=secs)
            res.append(secs)
        best = min(res, key=lambda s: max(s))
        print(n, shape, R, mode, "max/mean %.3f" % (max(best) / (sum(best) / R)), ["%.1f" % (1e3 * x) for x in best], flush=True)
        for p in plans: p.close()
