"""Per-level K3/K4 times through the pass API (each pass synchronous), with
the K3 kernel given per level (tiles -> rows, else fly).

usage: python tools/level_times.py C2 [kernel]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

KINDS = {"node": 0, "dmma": 2, "rows": 3, "fly": 4, "auto": 7}
c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
if len(sys.argv) > 2:
    plan.set_prop_kernel(KINDS[sys.argv[2]])
D = plan.depth
plan.set_density(pc.a_re, pc.a_im)
for rep in range(2):
    plan.zero_result()
    plan.level_d_pass()
    out = []
    for d in range(D, 2, -1):
        if d > 3:
            t0 = time.perf_counter()
            plan.propagation_pass(d)
            t1 = time.perf_counter()
        t2 = time.perf_counter()
        plan.interpolation_pass(d)
        t3 = time.perf_counter()
        nc = plan.n_cones(d - 1) if d > 3 else 0
        out.append(f"d={d:2d}: K3 {1e3 * (t1 - t0) if d > 3 else 0:8.2f} ms ({nc:9d} parent cones)"
                   f"  K4 {1e3 * (t3 - t2):8.2f} ms")
if True:
    print("\n".join(out))
