"""Load balance of the rank layouts (IFGF_PARTITION_COUNT, the reference's,
vs IFGF_PARTITION_WORK, the paper's proposed work-balanced extension): the
in-process rank group (ifgf_run_distributed) with IFGF_DIST_RANK_TIMING=1,
each rank's kernels timed alone; prints max/mean per layout.

usage: IFGF_DIST_RANK_TIMING=1 python tools/partition_probe.py C4 8
"""
import os
import sys

os.environ.setdefault("IFGF_DIST_RANK_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402
from paper_2112_15198_b200.dist import run_distributed  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
for name, mode in (("COUNT", 0), ("WORK", 1)):
    best = None
    for _ in range(2):
        q = pc.copy()
        _, infos = run_distributed(q, cfg, ifgf.EngineParams(depth=c.depth, partition=mode), R)
        secs = [i.compute_seconds for i in infos]
        best = secs if best is None or max(secs) < max(best) else best
    mean = sum(best) / len(best)
    print(f"{c.name} R={R} {name}: rank ms {[round(1e3 * v, 1) for v in best]} "
          f"max/mean {max(best) / mean:.3f}  sum {1e3 * sum(best):.1f} ms", flush=True)
