"""Plan create / apply / destroy in a loop: free device memory and the K4
record count per iteration (no growth, records kept every time).

usage: python tools/plan_churn.py [C2] [iterations]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402  (device memory query only)

import paper_2112_15198_b200 as ifgf  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 25
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
for it in range(iters):
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
    plan.apply(pc.a_re, pc.a_im)
    pairs = plan.info.k4_record_pairs
    plan.close()
    if it % 6 == 0 or it == iters - 1:
        free, _ = torch.cuda.mem_get_info()
        print(it, "free GiB", round(free / 2**30, 2), "record pairs", pairs, flush=True)
