"""Serial per-stage times of the apply at a config (best of k applies) and
the agreement with a reference run saved by the same tool.

usage: python tools/stage_times.py C2 [k] [--save ref.npz | --cmp ref.npz]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200.work import count_work  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
k = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
plan = ifgf.Plan.from_cloud(pc, ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa),
                            ifgf.EngineParams(depth=c.depth))
print(f"{sys.argv[1]}: setup {plan.info.setup_seconds * 1e3:.2f} ms")
plan.set_serial(True)
best = {}
for _ in range(k):
    ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
    for st in ("singular", "level_d", "propagation", "interpolation", "total"):
        v = getattr(rep.seconds, st)
        best[st] = min(best.get(st, 1e9), v)
w = count_work(plan).as_dict()["flops"]
for st, key in (("singular", "near"), ("level_d", "level_d"), ("propagation", "propagation"),
                ("interpolation", "interpolation")):
    print(f"  {st:14s} {best[st] * 1e3:8.3f} ms  {w[key] / best[st] / 1e12:6.2f} TF/s")
print(f"  {'total':14s} {best['total'] * 1e3:8.3f} ms")
if "--save" in sys.argv:
    np.savez(sys.argv[sys.argv.index("--save") + 1], ir=ir, ii=ii)
if "--cmp" in sys.argv:
    r = np.load(sys.argv[sys.argv.index("--cmp") + 1])
    d = np.sqrt(np.sum((ir - r["ir"]) ** 2 + (ii - r["ii"]) ** 2) / np.sum(r["ir"] ** 2 + r["ii"] ** 2))
    print(f"  rel-diff vs saved: {d:.3e}")
