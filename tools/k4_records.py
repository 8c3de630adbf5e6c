"""K4 from the plan's locate records against the locate-per-pair K4: bitwise
agreement, per-level K4 times, setup times with and without records.

usage: python tools/k4_records.py C2
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
for k in range(3):
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
    print(f"setup {plan.info.setup_seconds * 1e3:.2f} ms, device bytes {plan.info.device_bytes / 2**30:.2f} GiB")
    if k < 2:
        plan.close()
res = {}
for rec in (1, 0, 1):
    plan.set_k4_records(bool(rec))
    for rep in range(2):
        r, i, report = plan.apply(pc.a_re, pc.a_im)
    res[rec] = (r.copy(), i.copy())
    print(f"records={rec}: apply {report.seconds.total * 1e3:.2f} ms")
    D = plan.depth
    plan.set_density(pc.a_re, pc.a_im)
    plan.zero_result()
    plan.level_d_pass()
    out = []
    for d in range(D, 2, -1):
        if d > 3:
            plan.propagation_pass(d)
        t2 = time.perf_counter()
        plan.interpolation_pass(d)
        out.append(f"{1e3 * (time.perf_counter() - t2):.2f}")
    print(f"  K4 per level d={D}..3 (ms): " + " ".join(out))
same = np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
print("bitwise equal:", same)
if not same:
    d = np.hypot(res[0][0] - res[1][0], res[0][1] - res[1][1])
    print("  max abs diff", d.max(), "rel l2",
          np.sqrt((d**2).sum() / (res[0][0]**2 + res[0][1]**2).sum()))
plan.close()
