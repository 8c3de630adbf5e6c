"""One plan build + a few applies of a BASELINE config (for ncu captures).

usage: python tools/profile_step.py C1 [applies] [--serial]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
c = ifgf.configs.CONFIGS[name]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
with ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth)) as plan:
    if "--serial" in sys.argv:
        plan.set_serial(True)
    for _ in range(reps):
        i_re, i_im, rep = plan.apply(pc.a_re, pc.a_im)
    print(f"{name}: depth {rep.depth} apply {rep.seconds.total * 1e3:.2f} ms "
          f"(near {rep.seconds.singular * 1e3:.2f}, levelD {rep.seconds.level_d * 1e3:.2f}, "
          f"interp {rep.seconds.interpolation * 1e3:.2f}, prop {rep.seconds.propagation * 1e3:.2f}) "
          f"setup {plan.info.setup_seconds * 1e3:.1f} ms")
