"""Bench-step spread probe: the bench's step (plan build from device
coordinates + apply + destroy) K times, CUDA-event time per step and per part.
Variants: plain; with the bench's NVML clock sampler running; with host syncs
between the parts (as tools/step_breakdown.py does).

usage: python tools/step_spread.py C2 [K]
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2112_15198_b200 as ifgf  # noqa: E402
from bench import ClockSampler  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
kcfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
params = ifgf.EngineParams(depth=c.depth)
dev = torch.device("cuda", 0)
X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
out = [torch.empty(c.n, dtype=torch.float64, device=dev) for _ in range(2)]
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
s = torch.cuda.Stream(device=dev)
sh = s.cuda_stream


def run(label, sampler=False, syncs=False):
    rows = []
    ctx = ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    for i in range(K):
        with torch.cuda.stream(s):
            flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s)
        plan = ifgf.Plan.from_device(X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), c.n,
                                     kcfg, params, stream=sh)
        ev[1].record(s)
        if syncs:
            torch.cuda.synchronize()
        rep = plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                                out[1].data_ptr(), stream=sh)
        ev[2].record(s)
        if syncs:
            torch.cuda.synchronize()
        plan.close()
        ev[3].record(s)
        torch.cuda.synchronize()
        rows.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]),
                     ev[2].elapsed_time(ev[3]), ev[0].elapsed_time(ev[3]),
                     rep.seconds.total * 1e3])
    if ctx:
        ctx.__exit__()
    print(label)
    for r in rows:
        print("  build %7.2f  apply %7.2f  destroy %6.2f  step %7.2f  (apply host %7.2f)" % tuple(r))
    print("  median", [round(statistics.median(r[k] for r in rows[1:]), 2) for k in range(5)],
          "max step", round(max(r[3] for r in rows[1:]), 2), flush=True)


run("plain")
run("sampler", sampler=True)
run("syncs", syncs=True)
run("plain again")
