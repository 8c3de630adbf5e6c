"""Per-call timing of the end-to-end C-ABI apply (ifgf_apply from pinned host
buffers) at a config: wall time, the report's setup / total, and the stage
times.

usage: python tools/e2e_probe.py C2 [calls]
"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200 import _lib  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
params = ifgf.EngineParams(depth=c.depth)
host = [torch.from_numpy(a).pin_memory().numpy() for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
hout = [torch.empty(c.n, dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
rep = _lib.CReport()
for i in range(calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = _lib.lib.ifgf_apply(c.n, *[_lib.ptr(h) for h in host], int(c.kind), float(c.kappa),
                             C.byref(params.c()), _lib.ptr(hout[0]), _lib.ptr(hout[1]),
                             C.byref(rep))
    t = time.perf_counter() - t0
    ifgf.engine.check(rc)
    print(f"call {i}: wall {t * 1e3:7.2f} ms  setup {rep.setup * 1e3:6.2f}  total "
          f"{rep.total * 1e3:7.2f}  near {rep.singular * 1e3:5.2f} lvd {rep.level_d * 1e3:5.2f} "
          f"prop {rep.propagation * 1e3:6.2f} interp {rep.interpolation * 1e3:6.2f}", flush=True)
