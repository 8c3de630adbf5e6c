"""Edge cases of the operator against the CPU checkers: the smallest clouds
(N = 2..301; Laplace depth clamped to 3), all points in one tiny cluster, a very flat
spheroid (highly non-uniform occupancy), coincident points (the reference
returns NaN at the pair: 1/r of the excluded-by-index twin), zero and real
densities, and a Laplace cloud with a complex density."""
import math

import numpy as np
import pytest

from bindings import Params, rel_l2

pytestmark = pytest.mark.gpu


def _cloud(gpu, x, a_re, a_im):
    return gpu.PointCloud(np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                          np.ascontiguousarray(x[:, 2]), np.ascontiguousarray(a_re),
                          np.ascontiguousarray(a_im))


def _check(gpu, oracle, pc, kind, kappa, tol=1e-10):
    cfg = gpu.KernelConfig(gpu.KernelKind(kind), kappa)
    rep = gpu.apply(pc, cfg, gpu.EngineParams())
    w_re, w_im, r = oracle.apply(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, kind, kappa, Params())
    assert rep.depth == r["depth"]
    assert rel_l2(pc.i_re, pc.i_im, w_re, w_im) <= tol
    return rep


@pytest.mark.parametrize("n", [2, 3, 5, 17, 64, 301])
@pytest.mark.parametrize("kind", [0, 1])
def test_smallest_clouds(gpu, oracle, n, kind):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 3))
    rep = _check(gpu, oracle, _cloud(gpu, x, rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)), kind,
                 0.0 if kind else 2 * math.pi)
    if kind == 1:  # points_per_box rule: N <= 64 x 16 -> the minimum depth
        assert rep.depth == 3


def test_one_tiny_cluster(gpu, oracle):
    rng = np.random.default_rng(9)
    x = 1e-3 * rng.standard_normal((3000, 3)) + np.array([0.3, -0.2, 5.0])
    _check(gpu, oracle, _cloud(gpu, x, rng.uniform(-1, 1, 3000), rng.uniform(-1, 1, 3000)), 0,
           2 * math.pi * 40.0)


def test_very_flat_spheroid(gpu, oracle):
    pc = gpu.generate(20000, 1, 0.01, 0, 21)
    _check(gpu, oracle, pc, 0, 2 * math.pi * 5.0)


def test_coincident_points_like_reference(gpu, oracle):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((500, 3))
    x /= np.linalg.norm(x, axis=1)[:, None]
    x[7] = x[3]
    pc = _cloud(gpu, x, rng.uniform(-1, 1, 500), rng.uniform(-1, 1, 500))
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 6.0)
    gpu.apply(pc, cfg, gpu.EngineParams())
    w_re, w_im, _ = oracle.apply(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, 0, 6.0, Params())
    bad = ~np.isfinite(w_re)
    assert np.array_equal(np.nonzero(bad)[0], [3, 7])
    assert np.array_equal(~np.isfinite(pc.i_re), bad)
    ok = ~bad
    assert rel_l2(pc.i_re[ok], pc.i_im[ok], w_re[ok], w_im[ok]) <= 1e-10


def test_zero_density_gives_zero(gpu):
    pc = gpu.generate(5000, 0, 1.0, 0, 4)
    pc.a_re[:] = 0.0
    pc.a_im[:] = 0.0
    gpu.apply(pc, gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 2.0),
              gpu.EngineParams())
    assert np.all(pc.i_re == 0.0) and np.all(pc.i_im == 0.0)


def test_laplace_complex_density(gpu, oracle):
    pc = gpu.generate(8000, 0, 1.0, 0, 6)  # complex U(-1,1) density on the Laplace kernel
    _check(gpu, oracle, pc, 1, 0.0)
