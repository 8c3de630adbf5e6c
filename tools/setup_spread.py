"""Setup spread probe: K plan builds of a config back to back (as in a bench
step), host wall and CUDA-event device time per build, with and without the
bench's NVML clock sampler running.  IFGF_SETUP_TRACE=2 prints per-phase
host/GPU marks for every build.

usage: python tools/setup_spread.py C2 [K]
"""
import os
import statistics
import sys
import time

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
X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3)]
s = torch.cuda.Stream(device=dev)


def run(label, sampler):
    host, gpu = [], []
    ctx = ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    for _ in range(K):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        plan = ifgf.Plan.from_device(X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), c.n,
                                     kcfg, params, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        host.append((time.perf_counter() - t0) * 1e3)
        gpu.append(e0.elapsed_time(e1))
        plan.close()
    if ctx:
        ctx.__exit__()
    print(f"{label}: host ms {['%.1f' % v for v in host]}\n   gpu ms {['%.1f' % v for v in gpu]}"
          f"\n   median host {statistics.median(host):.2f} gpu {statistics.median(gpu):.2f}",
          flush=True)


run("warm", False)
run("no sampler", False)
run("sampler", True)
run("no sampler", False)
