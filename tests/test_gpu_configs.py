"""Parity at full BASELINE config sizes (C1-C5) against the CPU checkers.

tests/golden/config_<C>.npz (tests/golden/make_config_golden.py) holds, from
the checker's apply() -- the unmodified reference (oracle/_ref) for C1-C4,
our multi-threaded C restatement for C5:
  * the signed bucket sketch of the WHOLE output vector (tests/ifgf_sketch.py),
  * the output at 4,000 seeded targets and the whole output's squared norm,
  * exact direct sums at the config's 1,000 error targets and its error.
The inputs are regenerated bit for bit by the product's generator.

Bars (north_star): whole-output relative l2 <= 1e-10 (sketch estimate), no
bucket off by more than 1e-9 of the rms bucket (catches a flipped cone
segment at a handful of targets), sampled outputs <= 1e-10, error at the
1,000 targets <= 1.01x the checker's.  C1 is also compared element by
element against a live run of the unmodified reference.
"""
import glob
import os

import numpy as np
import pytest

import ifgf_sketch
from bindings import Params, rel_l2

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "config_*.npz")))


def _run(gpu, c):
    pc = gpu.generate(c.n, c.shape, c.c, c.dens, c.seed)
    cfg = gpu.KernelConfig(gpu.KernelKind(c.kind), c.kappa)
    rep = gpu.apply(pc, cfg, gpu.EngineParams(depth=c.depth))
    return pc, rep


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[7:-4] for p in FIXTURES])
def test_full_config_matches_checker(gpu, path):
    g = np.load(path)
    c = gpu.configs.CONFIGS[str(g["config"])]
    pc, rep = _run(gpu, c)
    assert rep.depth == int(g["depth"])
    # whole output: sketch
    assert "sketch_re" in g.files, f"{path}: fixture without a whole-output sketch"
    got = ifgf_sketch.sketch(pc.i_re, pc.i_im)
    rel, worst, qrel = ifgf_sketch.compare(got, (g["sketch_re"], g["sketch_im"], g["sketch_q"]))
    print(f"{g['config']}: checker {g['checker'] if 'checker' in g.files else 'reference'} "
          f"sketch rel-l2 {rel:.3e} worst bucket {worst:.3e} bucket norms {qrel:.3e}")
    assert rel <= 1e-10
    assert worst <= 1e-9
    assert qrel <= 1e-9
    # sampled outputs and the whole output's norm
    idx = g["idx"].astype(np.int64)
    assert rel_l2(pc.i_re[idx], pc.i_im[idx], g["i_re"], g["i_im"]) <= 1e-10
    norm2 = float(np.sum(pc.i_re * pc.i_re + pc.i_im * pc.i_im))
    assert abs(norm2 - float(g["norm2"])) <= 1e-10 * float(g["norm2"])
    # error against exact sums at the config's 1,000 targets
    e = g["err_idx"].astype(np.int64)
    eps = rel_l2(pc.i_re[e], pc.i_im[e], g["direct_re"], g["direct_im"])
    assert eps <= 1.01 * float(g["eps"])


def test_c1_whole_vector_vs_live_reference(gpu, ref, oracle):
    """C1 (BASELINE configs[0]): the full output vector against a live run of
    the unmodified reference on the same inputs, rel l2 <= 1e-10."""
    c = gpu.configs.C1
    pc, rep = _run(gpu, c)
    x1, x2, x3, ar, ai = oracle.generate(c.n, c.shape, c.c, c.dens, c.seed)
    assert np.array_equal(x1, pc.x1) and np.array_equal(ai, pc.a_im)
    ir, ii, r = ref.apply(x1, x2, x3, ar, ai, c.kind, c.kappa,
                          Params(depth=c.depth, threads=os.cpu_count() or 1))
    assert r["depth"] == rep.depth
    err = rel_l2(pc.i_re, pc.i_im, ir, ii)
    print(f"C1 whole vector vs reference: rel-l2 {err:.3e}")
    assert err <= 1e-10
    # pointwise: no target off by more than 1e-9 of the rms output
    rms = np.sqrt(np.mean(ir * ir + ii * ii))
    assert np.max(np.hypot(pc.i_re - ir, pc.i_im - ii)) <= 1e-9 * rms
