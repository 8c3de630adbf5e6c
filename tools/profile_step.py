"""One plan build + a few applies of a BASELINE config (for ncu captures and
quick stage timings).

usage: python tools/profile_step.py C1 [applies] [--serial] [--setups K]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
setups = int(sys.argv[sys.argv.index("--setups") + 1]) if "--setups" in sys.argv else 1
c = ifgf.configs.CONFIGS[name]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
for k in range(setups):
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
    print(f"{name}: setup {plan.info.setup_seconds * 1e3:.1f} ms (depth {plan.depth})")
    if k < setups - 1:
        plan.close()
if "--serial" in sys.argv:
    plan.set_serial(True)
for _ in range(reps):
    i_re, i_im, rep = plan.apply(pc.a_re, pc.a_im)
    print(f"{name}: apply {rep.seconds.total * 1e3:.2f} ms (near {rep.seconds.singular * 1e3:.2f},"
          f" levelD {rep.seconds.level_d * 1e3:.2f}, interp {rep.seconds.interpolation * 1e3:.2f},"
          f" prop {rep.seconds.propagation * 1e3:.2f})")
plan.close()
