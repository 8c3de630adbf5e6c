"""Generate tests/golden/config_<C>.npz at full BASELINE config sizes.

Run here (where /root/reference exists and oracle/_ref is built):
    make -C oracle ref && python tests/golden/make_config_golden.py C1 C2
    python tests/golden/make_config_golden.py --checker oracle --threads 16 C5

Checker: the UNMODIFIED reference library (oracle/_ref, default) or our C
restatement (oracle/liboracle.so) where the reference cannot run: C5 needs
~4 h of single-threaded reference setup and ~150 GB for its two live block
levels, so C5 is pinned against the oracle's
depth-first form (--checker lean: multi-threaded setup, O(depth) live
blocks), which agrees with the reference's whole output to ~1e-15 at C1/C2
(tests/test_oracle_cpu.py) and whose level-by-level form is pinned to the
reference at C1-C4.

Inputs come from the seeded generator, which the tests
regenerate bit for bit, so a fixture stores, from the checker's apply():
  * the signed bucket sketch of the WHOLE output vector (tests/ifgf_sketch.py),
  * the output at 4,000 seeded sample targets and the whole output's squared norm,
  * exact direct sums at the config's 1,000 error targets
    (sample_indices(N, 1000, seed + 1)) and the checker's sampled error,
  * the depth and the checker's wall time.
"""
import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from bindings import COracle, Params, RefOracle  # noqa: E402

import ifgf_sketch  # noqa: E402


def load_configs():
    # configs.py is plain Python; load it without importing the product
    # package (which would map libifgf_b200.so into this checker process)
    import importlib.util
    path = os.path.join(ROOT, "paper_2112_15198_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("ifgf_configs", path)
    m = importlib.util.module_from_spec(spec)
    sys.modules["ifgf_configs"] = m
    spec.loader.exec_module(m)
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["C1"])
    ap.add_argument("--checker", choices=["reference", "oracle", "lean"], default="reference")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--out", default=HERE)
    a = ap.parse_args()
    configs = load_configs()
    oc = COracle()
    chk = RefOracle() if a.checker == "reference" else oc
    for name in a.names:
        c = configs.CONFIGS[name]
        x1, x2, x3, ar, ai = oc.generate(c.n, c.shape, c.c, c.dens, c.seed)
        p = Params(depth=c.depth, threads=a.threads)
        t0 = time.time()
        if a.checker == "lean":  # depth-first oracle: O(depth) live blocks (C5 in a few GB)
            ir, ii, rep = oc.apply_lean(x1, x2, x3, ar, ai, c.kind, c.kappa, p)
        else:
            ir, ii, rep = chk.apply(x1, x2, x3, ar, ai, c.kind, c.kappa, p)
        t_apply = time.time() - t0
        err_idx = oc.sample_indices(c.n, 1000, c.seed + 1)
        # exact sums by the oracle's direct_eval (pinned to the reference's)
        dre, dim = oc.direct(x1, x2, x3, ar, ai, c.kind, c.kappa, err_idx, threads=a.threads)
        e_re, e_im = ir[err_idx], ii[err_idx]
        eps = float(np.sqrt(np.sum((dre - e_re) ** 2 + (dim - e_im) ** 2) /
                            np.sum(dre ** 2 + dim ** 2)))
        idx = oc.sample_indices(c.n, 4000, 7919 + c.seed)
        s_re, s_im, s_q = ifgf_sketch.sketch(ir, ii)
        np.savez_compressed(
            os.path.join(a.out, f"config_{name}.npz"), config=name, n=c.n, depth=rep["depth"],
            checker=a.checker, threads=a.threads,
            idx=np.asarray(idx, np.uint64), i_re=ir[idx], i_im=ii[idx],
            err_idx=np.asarray(err_idx, np.uint64), direct_re=dre, direct_im=dim, eps=eps,
            norm2=float(np.sum(ir * ir + ii * ii)), ref_seconds=t_apply,
            sketch_re=s_re, sketch_im=s_im, sketch_q=s_q, sketch_seed=ifgf_sketch.SEED)
        print(f"{name}: checker {a.checker} depth {rep['depth']} eps {eps:.4e} "
              f"apply {t_apply:.1f} s peak_live_blocks {rep.get('peak_live_blocks')}", flush=True)


if __name__ == "__main__":
    main()
