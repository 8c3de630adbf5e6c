"""One plan + one apply with a chosen K3 kernel (for ncu captures).

usage: python tools/prop_one.py C2 rows
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

KINDS = {"node": 0, "tiles": 1, "dmma": 2, "rows": 3, "fly": 4, "stream": 5, "pipe": 6}
c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
plan.set_serial(True)
plan.set_prop_kernel(KINDS[sys.argv[2] if len(sys.argv) > 2 else "node"])
ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
print(f"prop {rep.seconds.propagation * 1e3:.2f} ms")
