"""Host-side breakdown of one bench step (plan build, apply, destroy) at a
config, with device syncs between the parts.

usage: python tools/step_breakdown.py C2 [reps]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
kcfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
params = ifgf.EngineParams(depth=c.depth)
dev = torch.device("cuda", 0)
X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
out = [torch.empty(c.n, dtype=torch.float64, device=dev) for _ in range(2)]
s = torch.cuda.Stream(device=dev)
sh = s.cuda_stream
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = ifgf.Plan.from_device(X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), c.n, kcfg,
                                 params, stream=sh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                            out[1].data_ptr(), stream=sh)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    plan.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"build {1e3 * (t1 - t0):7.2f} ms"
          f"  apply {1e3 * (t2 - t1):7.2f} ms (report total {rep.seconds.total * 1e3:.2f})"
          f"  destroy {1e3 * (t3 - t2):6.2f} ms  step {1e3 * (t3 - t0):7.2f} ms", flush=True)
