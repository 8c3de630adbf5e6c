"""Run one BASELINE config end to end on the GPU: setup + apply through the
public API, per-pass times, and the relative error against direct sums at
the config's sampled targets (error_at_indices, the reference's metric).

usage: python tools/config_run.py C3 [C4 ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

for name in sys.argv[1:]:
    c = ifgf.configs.CONFIGS[name]
    pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
    cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
    t0 = time.perf_counter()
    plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
    plan.set_serial(True)
    for _ in range(2):
        i_re, i_im, rep = plan.apply(pc.a_re, pc.a_im)
    t1 = time.perf_counter()
    pc.i_re[:], pc.i_im[:] = i_re, i_im
    idx = ifgf.sample_indices(c.n, 1000, c.seed + 1)
    err = ifgf.error_at_indices(pc, cfg, idx)
    s = rep.seconds
    print(f"{name}: N={c.n} depth {plan.depth} setup {plan.info.setup_seconds * 1e3:.1f} ms  "
          f"apply {s.total * 1e3:.1f} ms (near {s.singular * 1e3:.1f}, levelD "
          f"{s.level_d * 1e3:.1f}, interp {s.interpolation * 1e3:.1f}, prop "
          f"{s.propagation * 1e3:.1f})  rel err {err:.3e}  wall {t1 - t0:.1f} s", flush=True)
    plan.close()
