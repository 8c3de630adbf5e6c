"""Known-answer and property tests from the reference's own unit tests, run
on the CUDA path through the C ABI.

* direct_eval two-body I(x2) = a1 e^{i k r}/(4 pi r) (test_engine.cpp:50-61)
* direct_eval commutes with permutations            (test_engine.cpp:63-79)
* Laplace with real densities stays real, exactly   (test_engine.cpp:303-314)
* apply error budgets at (3,5,5) and (5,7,7)        (test_engine.cpp:256-284,
                                                      acceptance.cpp:77-102)
* bitwise run-to-run and plan-to-plan reproducibility
* reference error classes on bad input              (engine.cpp:261, :76-77)
"""
import math

import numpy as np
import pytest

from bindings import rel_l2

pytestmark = pytest.mark.gpu


def _cloud(gpu, x, a_re, a_im=None):
    n = len(x)
    a_im = np.zeros(n) if a_im is None else a_im
    return gpu.PointCloud(np.ascontiguousarray(x[:, 0]), np.ascontiguousarray(x[:, 1]),
                          np.ascontiguousarray(x[:, 2]), np.asarray(a_re, float),
                          np.asarray(a_im, float))


@pytest.mark.parametrize("kappa", [0.0, 3.0])
def test_two_body_direct(gpu, kappa):
    """direct_eval two-body hand computation (test_engine.cpp:50-61)."""
    x = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    pc = _cloud(gpu, x, [1.0, 0.0])
    kind = gpu.KernelKind.Laplace if kappa == 0.0 else gpu.KernelKind.Helmholtz
    gpu.direct_eval(pc, gpu.KernelConfig(kind, kappa))
    want = complex(math.cos(kappa), math.sin(kappa)) / (4 * math.pi)
    assert pc.i_re[0] == 0.0 and pc.i_im[0] == 0.0  # only the zero coefficient radiates to x1
    assert abs(complex(pc.i_re[1], pc.i_im[1]) - want) <= 1e-15 * abs(want)


def test_direct_commutes_with_permutation(gpu):
    """direct_eval commutes with point permutations (test_engine.cpp:63-79)."""
    pc = gpu.generate(512, 0, 1.0, 1, 3)
    pc.a_re[:] = 1.0
    cfg = gpu.KernelConfig(gpu.KernelKind.Laplace, 0.0)
    fwd = pc.copy()
    gpu.direct_eval(fwd, cfg)
    rev = pc.copy()
    for a in (rev.x1, rev.x2, rev.x3):
        a[:] = a[::-1].copy()
    gpu.direct_eval(rev, cfg)
    assert np.allclose(rev.i_re[::-1], fwd.i_re, rtol=1e-12, atol=0)


def test_two_body_apply(gpu):
    """The operator on two points (N >= 2 is the reference's minimum)."""
    x = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    pc = _cloud(gpu, x, [1.0, 0.0])
    rep = gpu.apply(pc, gpu.KernelConfig(gpu.KernelKind.Laplace, 0.0), gpu.EngineParams())
    assert rep.n == 2 and rep.depth >= 3
    assert pc.i_re[0] == 0.0 and pc.i_im[1] == 0.0
    assert abs(pc.i_re[1] - 1 / (4 * math.pi)) <= 1e-3 / (4 * math.pi)  # IFGF accuracy


def test_laplace_stays_real(gpu):
    pc = gpu.generate(20000, 0, 1.0, 1, 7)
    assert not np.any(pc.a_im)
    gpu.apply(pc, gpu.KernelConfig(gpu.KernelKind.Laplace, 0.0), gpu.EngineParams())
    assert np.all(pc.i_im == 0.0)
    assert np.any(pc.i_re != 0.0)


@pytest.mark.parametrize("orders,budget", [((3, 5, 5), 5e-3), ((5, 7, 7), 5e-4)])
def test_error_budget(gpu, orders, budget):
    pc = gpu.generate(20000, 0, 1.0, 0, 3)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 2.0)
    gpu.apply(pc, cfg, gpu.EngineParams(orders=gpu.InterpOrders(*orders)))
    idx = gpu.sample_indices(pc.size(), 200, 4)
    assert gpu.error_at_indices(pc, cfg, idx) <= budget


def test_bitwise_reproducible(gpu):
    pc = gpu.generate(30000, 1, 0.25, 0, 9)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 3.0)
    ep = gpu.EngineParams()
    p1 = gpu.Plan.from_cloud(pc, cfg, ep)
    a = p1.apply(pc.a_re, pc.a_im)
    b = p1.apply(pc.a_re, pc.a_im)
    p2 = gpu.Plan.from_cloud(pc, cfg, ep)
    c = p2.apply(pc.a_re, pc.a_im)
    for r in (b, c):
        assert np.array_equal(a[0], r[0]) and np.array_equal(a[1], r[1])
    p1.close()
    p2.close()


def test_reference_error_classes(gpu):
    one = _cloud(gpu, np.zeros((1, 3)), [1.0])
    with pytest.raises(gpu.InvalidArgument):
        gpu.apply(one, gpu.KernelConfig(gpu.KernelKind.Helmholtz, 1.0), gpu.EngineParams())
    pc = gpu.generate(1000, 0, 1.0, 0, 2)
    with pytest.raises(gpu.InvalidArgument):  # interpolation orders out of range
        gpu.apply(pc, gpu.KernelConfig(gpu.KernelKind.Helmholtz, 1.0),
                  gpu.EngineParams(orders=gpu.InterpOrders(0, 5, 5)))
