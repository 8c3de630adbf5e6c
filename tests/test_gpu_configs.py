"""Parity at full BASELINE config sizes against the unmodified reference:
C1 (configs[0]) and C2 (configs[1], the bench workload).

tests/golden/config_<C>.npz (tests/golden/make_config_golden.py) holds the
reference's apply() output at 4,000 seeded targets, the squared norm of its
whole output, exact direct sums at the config's 1,000 error targets and its
sampled error.  The inputs are regenerated bit for bit by the product's
generator.  Bars: sampled outputs relative l2 <= 1e-10 (north_star), whole
output norm within 1e-10, sampled error within 1.01x of the reference's.
"""
import glob
import os

import numpy as np
import pytest

from bindings import rel_l2

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "config_*.npz")))


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[7:-4] for p in FIXTURES])
def test_full_config_matches_reference(gpu, path):
    g = np.load(path)
    c = gpu.configs.CONFIGS[str(g["config"])]
    pc = gpu.generate(c.n, c.shape, c.c, c.dens, c.seed)
    cfg = gpu.KernelConfig(gpu.KernelKind(c.kind), c.kappa)
    rep = gpu.apply(pc, cfg, gpu.EngineParams(depth=c.depth))
    assert rep.depth == int(g["depth"])
    idx = g["idx"].astype(np.int64)
    assert rel_l2(pc.i_re[idx], pc.i_im[idx], g["i_re"], g["i_im"]) <= 1e-10
    norm2 = float(np.sum(pc.i_re * pc.i_re + pc.i_im * pc.i_im))
    assert abs(norm2 - float(g["norm2"])) <= 1e-10 * float(g["norm2"])
    e = g["err_idx"].astype(np.int64)
    eps = rel_l2(pc.i_re[e], pc.i_im[e], g["direct_re"], g["direct_im"])
    assert eps <= 1.01 * float(g["eps"])
