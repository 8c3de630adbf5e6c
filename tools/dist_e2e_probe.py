"""Host-timed breakdown of the multi-GPU e2e step at world 1 (the N>1 path of
bench.py on one GPU): H2D of the inputs, rank plan create, apply, close, D2H.

usage: python tools/dist_e2e_probe.py C2 [steps]
"""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200.dist import Comm, DistPlan, share_comm_id  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1)
c = ifgf.configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
kcfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
params = ifgf.EngineParams(depth=c.depth)
comm = Comm(share_comm_id(Comm.unique_id), 0, 1, 0)
X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
out = [torch.empty(c.n, dtype=torch.float64, device=dev) for _ in range(2)]
host = [torch.from_numpy(a).pin_memory() for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
hout = [torch.empty(c.n, dtype=torch.float64).pin_memory() for _ in range(2)]
s = torch.cuda.Stream(device=dev)
sh = s.cuda_stream
for i in range(steps):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    with torch.cuda.stream(s):
        for d_, h_ in zip(X, host):
            d_.copy_(h_, non_blocking=True)
    s.synchronize()
    t.append(time.perf_counter())
    plan = DistPlan(comm, X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), c.n, kcfg, params,
                    stream=sh)
    t.append(time.perf_counter())
    plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(), out[1].data_ptr(),
                      stream=sh)
    t.append(time.perf_counter())
    plan.close()
    t.append(time.perf_counter())
    with torch.cuda.stream(s):
        hout[0].copy_(out[0], non_blocking=True)
        hout[1].copy_(out[1], non_blocking=True)
    s.synchronize()
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"step {i}: h2d {d[0]:6.2f}  create {d[1]:7.2f}  apply {d[2]:7.2f}  close {d[3]:6.2f}  "
          f"d2h {d[4]:6.2f}  total {1e3 * (t[-1] - t[0]):7.2f} ms", flush=True)
comm.close()
dist.destroy_process_group()
