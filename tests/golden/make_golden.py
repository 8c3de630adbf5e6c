"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists and oracle/_ref is built):
    make -C oracle ref && python tests/golden/make_golden.py

Each fixture holds the seeded inputs, the reference's apply() output in the
caller's order, its Problem structure per level (box codes/first/count,
cousin CSR, relevant cone lists), the permutation, exact direct sums at a
seeded sample of targets and the reference's sampled error.  Tests check the
C oracle against these, and the GPU path against the oracle.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

from bindings import COracle, Params, RefOracle  # noqa: E402

# name, n, shape, c, kind, kappa, dens, seed, orders, depth
CASES = [
    ("helm_sphere_3k", 3000, 0, 1.0, 0, 2 * math.pi * 1.5, 0, 101, (3, 5, 5), 0),
    ("laplace_sphere_4k", 4000, 0, 1.0, 1, 0.0, 1, 102, (3, 5, 5), 0),
    ("helm_oblate_4k", 4000, 1, 0.25, 0, 2 * math.pi * 2.0, 0, 103, (3, 5, 5), 0),
    ("helm_sphere_577", 2000, 0, 1.0, 0, 2 * math.pi * 2.0, 0, 104, (5, 7, 7), 0),
    ("helm_sphere_pinned_d5", 2500, 0, 1.0, 0, 2 * math.pi * 1.0, 0, 105, (3, 5, 5), 5),
    ("two_body_laplace", 2, 0, 1.0, 1, 0.0, 0, 0, (3, 5, 5), 0),
]


def main():
    ref = RefOracle()
    oc = COracle()
    for name, n, shape, c, kind, kappa, dens, seed, orders, depth in CASES:
        if name == "two_body_laplace":
            # test_engine.cpp:50-61: x = (0,0,0), (1,0,0); a = (1,0), (0,0)
            x1, x2, x3 = np.array([0.0, 1.0]), np.zeros(2), np.zeros(2)
            ar, ai = np.array([1.0, 0.0]), np.zeros(2)
        else:
            x1, x2, x3, ar, ai = oc.generate(n, shape, c, dens, seed)
        p = Params(depth=depth, p_s=orders[0], p_theta=orders[1], p_phi=orders[2], threads=8)
        ir, ii, rep = ref.apply(x1, x2, x3, ar, ai, kind, kappa, p)
        out = dict(x1=x1, x2=x2, x3=x3, a_re=ar, a_im=ai, i_re=ir, i_im=ii,
                   kind=kind, kappa=kappa, orders=np.array(orders), depth_param=depth,
                   depth=rep["depth"], peak_live_blocks=rep["peak_live_blocks"])
        prob = ref.problem(x1, x2, x3, ar, ai, kind, kappa, p)
        perm, _ = prob.sorted()
        out["perm"] = perm
        out["cube"] = prob.cube()
        for d in range(1, prob.depth + 1):
            L = prob.level(d)
            out[f"L{d}_codes"] = L.codes
            out[f"L{d}_first"] = L.first
            out[f"L{d}_count"] = L.count
            out[f"L{d}_nbr_off"] = L.nbr_off
            out[f"L{d}_nbr"] = L.nbr
            if d >= 3:
                out[f"L{d}_cousin_off"] = L.cousin_off
                out[f"L{d}_cousin"] = L.cousin
                out[f"L{d}_cone_box"] = L.cone_box
                out[f"L{d}_cone_gamma"] = L.cone_gamma
                out[f"L{d}_box_cone_begin"] = L.box_cone_begin
        m = min(200, n)
        idx = ref.sample_indices(n, m, 7)
        dre, dim = ref.direct(x1, x2, x3, ar, ai, kind, kappa)
        out["sample_idx"] = idx
        out["direct_re"] = dre[idx]
        out["direct_im"] = dim[idx]
        if n > 2:
            out["eps_sample"] = ref.error_at_indices(x1, x2, x3, ar, ai, ir, ii, kind, kappa, idx)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: N={n} depth={rep['depth']} -> {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
