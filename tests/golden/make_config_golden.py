"""Generate tests/golden/config_<C>.npz from the UNMODIFIED reference library
at full BASELINE config sizes (C1 = configs[0], C2 = configs[1], the bench
workload).

Run here (where /root/reference exists and oracle/_ref is built):
    make -C oracle ref && python tests/golden/make_config_golden.py C1 C2

Inputs come from the seeded generator, which the tests
regenerate bit for bit, so a fixture stores only the reference's apply()
output at 4,000 seeded sample targets, exact direct sums at the config's
1,000 error targets (sample_indices(N, 1000, seed + 1)), the reference's
sampled error and the depth.  C2 takes the reference ~4 minutes.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

from bindings import COracle, Params, RefOracle  # noqa: E402

from paper_2112_15198_b200 import configs  # noqa: E402


def main(names):
    ref = RefOracle()
    oc = COracle()
    for name in names:
        c = configs.CONFIGS[name]
        x1, x2, x3, ar, ai = oc.generate(c.n, c.shape, c.c, c.dens, c.seed)
        p = Params(depth=c.depth, threads=os.cpu_count() or 8)
        t0 = time.time()
        ir, ii, rep = ref.apply(x1, x2, x3, ar, ai, c.kind, c.kappa, p)
        t_apply = time.time() - t0
        err_idx = ref.sample_indices(c.n, 1000, c.seed + 1)
        eps = ref.error_at_indices(x1, x2, x3, ar, ai, ir, ii, c.kind, c.kappa, err_idx)
        dre, dim = oc.direct(x1, x2, x3, ar, ai, c.kind, c.kappa, err_idx)  # pinned to the reference
        idx = ref.sample_indices(c.n, 4000, 7919 + c.seed)
        np.savez_compressed(
            os.path.join(HERE, f"config_{name}.npz"), config=name, n=c.n, depth=rep["depth"],
            idx=np.asarray(idx, np.uint64), i_re=ir[idx], i_im=ii[idx],
            err_idx=np.asarray(err_idx, np.uint64), direct_re=dre, direct_im=dim, eps=eps,
            norm2=float(np.sum(ir * ir + ii * ii)), ref_seconds=t_apply)
        print(f"{name}: depth {rep['depth']} eps {eps:.4e} apply {t_apply:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1"])
