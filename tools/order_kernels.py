import math, sys
sys.path.insert(0, '/root/repo')
import paper_2112_15198_b200 as ifgf
for orders in [(5,7,7),(4,6,6)]:
    pc = ifgf.generate(3456, 0, 1.0, 0, 14)
    cfg = ifgf.KernelConfig(ifgf.KernelKind.Helmholtz, 2*math.pi*2.0)
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(orders=ifgf.InterpOrders(*orders)))
    for k in range(7):
        plan.set_prop_kernel(k)
        try:
            plan.apply(pc.a_re, pc.a_im); print(orders, k, "ok", flush=True)
        except Exception as e:
            print(orders, k, "FAIL", e, flush=True)
            plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(orders=ifgf.InterpOrders(*orders)))
