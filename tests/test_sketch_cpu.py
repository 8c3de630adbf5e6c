"""The whole-output sketch used by the full-size parity tests (CPU)."""
import glob
import os

import numpy as np

import ifgf_sketch

HERE = os.path.dirname(os.path.abspath(__file__))


def test_sketch_is_linear_and_estimates_l2():
    rng = np.random.default_rng(3)
    n = 200_000
    a_re, a_im = rng.standard_normal(n), rng.standard_normal(n)
    b_re, b_im = rng.standard_normal(n) * 1e-6, rng.standard_normal(n) * 1e-6
    sa = ifgf_sketch.sketch(a_re, a_im)
    sb = ifgf_sketch.sketch(b_re, b_im)
    sab = ifgf_sketch.sketch(a_re + b_re, a_im + b_im)
    assert np.allclose(sab[0], sa[0] + sb[0], rtol=0, atol=1e-9)
    assert np.allclose(sab[1], sa[1] + sb[1], rtol=0, atol=1e-9)
    # CountSketch: ||S x|| ~ ||x|| (relative spread ~ 1/sqrt(K))
    true = np.sqrt(np.sum(b_re ** 2 + b_im ** 2) / np.sum(a_re ** 2 + a_im ** 2))
    est, _, _ = ifgf_sketch.compare(sab, sa)
    assert 0.9 * true < est < 1.1 * true


def test_sketch_flags_a_localised_error():
    rng = np.random.default_rng(5)
    n = 1_572_864
    re, im = rng.standard_normal(n), rng.standard_normal(n)
    want = ifgf_sketch.sketch(re, im)
    bad_re = re.copy()
    bad_re[[17, 900_001]] *= 1.0 + 1e-3  # two targets off by 1e-3 relative
    rel, worst, qrel = ifgf_sketch.compare(ifgf_sketch.sketch(bad_re, im), want)
    assert rel < 1e-5          # invisible to a global norm bar of ~1e-5 ...
    assert worst > 1e-6        # ... but far above the 1e-9 per-bucket bar
    assert qrel > 1e-7


def test_signs_are_fixed():
    s = ifgf_sketch.signs(8)
    assert set(np.unique(s)) <= {-1.0, 1.0}
    # pinned: the fixtures depend on this exact sign sequence
    assert s.tolist() == [-1.0, 1.0, 1.0, 1.0, -1.0, 1.0, 1.0, 1.0]
    assert abs(ifgf_sketch.signs(1_000_000).mean()) < 5e-3


def test_fixtures_carry_a_sketch():
    for path in sorted(glob.glob(os.path.join(HERE, "golden", "config_*.npz"))):
        g = np.load(path)
        assert "sketch_re" in g.files, path
        k = len(g["sketch_re"])
        assert k == min(ifgf_sketch.K_DEFAULT, int(g["n"]))
        assert np.all(g["sketch_q"] > 0)
        # the bucket norms add up to the whole output's squared norm
        assert abs(g["sketch_q"].sum() - float(g["norm2"])) <= 1e-10 * float(g["norm2"])
