import sys; sys.path.insert(0, '/root/repo')
import paper_2112_15198_b200 as ifgf
c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
plan = ifgf.Plan.from_cloud(pc, ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa), ifgf.EngineParams())
plan.set_serial(True); plan.set_prop_kernel(2)
ir, ii, rep = plan.apply(pc.a_re, pc.a_im)
print("prop", rep.seconds.propagation)
