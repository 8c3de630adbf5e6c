"""Small cases over every product kernel for compute-sanitizer runs
(memcheck, racecheck, synccheck): setup, K1 (box and point forms), K2, K3
(ROWS + FLY default, DMMA, NODE), K4, the pass-level API with block
pack/unpack, and an in-process rank group (halo exchange) -- each checked
against the default apply.

usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200.dist import run_distributed  # noqa: E402


def rel(a, b):
    return float(np.sqrt(np.sum((a[0] - b[0]) ** 2 + (a[1] - b[1]) ** 2) /
                         np.sum(b[0] ** 2 + b[1] ** 2)))


n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
for shape, c, kind, kappa in ((0, 1.0, 0, 2 * math.pi * 3.0), (1, 0.25, 0, 2 * math.pi * 4.0),
                              (0, 1.0, 1, 0.0)):
    pc = ifgf.generate(n, shape, c, 1 if kind else 0, 31 + shape)
    cfg = ifgf.KernelConfig(ifgf.KernelKind(kind), kappa)
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams())
    base = plan.apply(pc.a_re, pc.a_im)[:2]
    worst = 0.0
    for k in (plan.PROP_DMMA, plan.PROP_NODE, plan.PROP_FLY):
        plan.set_prop_kernel(k)
        worst = max(worst, rel(plan.apply(pc.a_re, pc.a_im)[:2], base))
    plan.set_prop_kernel(plan.PROP_ROWS)
    plan.set_near_kernel(plan.NEAR_POINT)
    worst = max(worst, rel(plan.apply(pc.a_re, pc.a_im)[:2], base))
    plan.set_near_kernel(plan.NEAR_BOX)
    # pass-level API with a block round trip through pack/unpack
    plan.set_density(pc.a_re, pc.a_im)
    plan.zero_result()
    plan.singular_pass()
    plan.level_d_pass()
    for d in range(plan.depth, 2, -1):
        if d > 3:
            plan.propagation_pass(d)
        plan.interpolation_pass(d)
    s_re, s_im = plan.read_result()
    worst = max(worst, rel((s_re, s_im), base))
    q = pc.copy()
    run_distributed(q, cfg, ifgf.EngineParams(), 3)
    worst = max(worst, rel((q.i_re, q.i_im), base))
    plan.close()
    print(f"shape {shape} kind {kind}: kernels agree to {worst:.2e}", flush=True)
    assert worst < 1e-12
print("SANITIZE CASE OK")
