"""One serial apply of a config with the K3 kernel given (for ncu captures).

usage: python tools/prop_one_mode.py C2 dmma [applies]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

KINDS = {"dmma": 2, "rows": 3, "fly": 4}
c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
plan = ifgf.Plan.from_cloud(pc, ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa),
                            ifgf.EngineParams(depth=c.depth))
plan.set_serial(True)
plan.set_prop_kernel(KINDS[sys.argv[2]])
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    plan.apply(pc.a_re, pc.a_im)
print("ok")
