"""Per-config stage times next to the algorithmic work (work.py) of each stage:
TF/s and fraction of the FP64 peak for C1-C5, plus the per-level K3 work.

usage: python tools/config_work.py C3 [C4 ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200 import work  # noqa: E402

PEAK = 37.1  # TF/s, measured FP64 peak

for name in sys.argv[1:]:
    c = ifgf.configs.CONFIGS[name]
    pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
    cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
    plan.set_serial(True)
    for _ in range(2):
        _, _, rep = plan.apply(pc.a_re, pc.a_im)
    s = rep.seconds
    wc = work.count_work(plan)
    fl = wc.flops
    print(f"{name}: N={c.n} depth {plan.depth} apply {s.total * 1e3:.1f} ms", flush=True)
    for stage, t in (("near", s.singular), ("level_d", s.level_d),
                     ("propagation", s.propagation), ("interpolation", s.interpolation)):
        tf = fl[stage] / t / 1e12
        print(f"  {stage:14s} {t * 1e3:9.1f} ms  {fl[stage] / 1e9:9.1f} GFLOP  {tf:6.2f} TF/s "
              f"({tf / PEAK:5.1%})")
    for d in sorted(wc.prop_evals):
        U = plan.level(d - 1)
        print(f"  K3 d={d:2d}: evals {wc.prop_evals[d]:12d} parent cones {wc.prop_fits[d]:9d} "
              f"parent boxes {len(U.count):8d}")
    plan.close()
