"""One plan + two serial applies of a config with the selected near-field
kernel (ncu target for k_near_box / k_singular).

usage: python tools/near_one.py C2 [point|box]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
kind = {"point": 0, "box": 1}[sys.argv[2] if len(sys.argv) > 2 else "box"]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
plan = ifgf.Plan.from_cloud(pc, ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa),
                            ifgf.EngineParams(depth=c.depth))
plan.set_serial(True)
plan.set_near_kernel(kind)
for _ in range(2):
    ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
print(f"near {rep.seconds.singular * 1e3:.3f} ms")
