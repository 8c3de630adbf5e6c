"""Multi-density apply (ifgf_plan_apply_batch): every
right-hand side equals its own ifgf_plan_apply, and each equals the
reference's apply on the same cloud."""
import math

import numpy as np
import pytest

from bindings import Params, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nrhs", [1, 2, 3, 5])
def test_batch_equals_single_applies(gpu, nrhs):
    pc = gpu.generate(20000, 0, 1.0, 0, 77)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 4.0)
    plan = gpu.Plan.from_cloud(pc, cfg)
    rng = np.random.default_rng(nrhs)
    A_re = rng.uniform(-1, 1, (nrhs, len(pc.x1)))
    A_im = rng.uniform(-1, 1, (nrhs, len(pc.x1)))
    i_re, i_im, rep = plan.apply_batch(A_re, A_im)
    assert i_re.shape == (nrhs, len(pc.x1))
    for r in range(nrhs):
        s_re, s_im, _ = plan.apply(A_re[r], A_im[r])
        assert np.array_equal(i_re[r], s_re) and np.array_equal(i_im[r], s_im), r
    plan.close()


def test_batch_laplace_real_density(gpu):
    pc = gpu.generate(12000, 0, 1.0, 1, 79)
    cfg = gpu.KernelConfig(gpu.KernelKind.Laplace, 0.0)
    plan = gpu.Plan.from_cloud(pc, cfg)
    rng = np.random.default_rng(3)
    A = rng.standard_normal((3, len(pc.x1)))
    i_re, i_im, _ = plan.apply_batch(A)
    for r in range(3):
        s_re, s_im, _ = plan.apply(A[r])
        assert np.array_equal(i_re[r], s_re) and np.all(i_im[r] == 0.0)
    plan.close()


def test_batch_matches_reference(gpu, ref, oracle):
    """Two right-hand sides in one batch, each against the unmodified
    reference's apply on the same cloud."""
    pc = gpu.generate(8000, 0, 1.0, 0, 83)
    k = 2 * math.pi * 3.0
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, k)
    plan = gpu.Plan.from_cloud(pc, cfg)
    rng = np.random.default_rng(5)
    A_re = np.stack([pc.a_re, rng.uniform(-1, 1, len(pc.x1))])
    A_im = np.stack([pc.a_im, rng.uniform(-1, 1, len(pc.x1))])
    i_re, i_im, _ = plan.apply_batch(A_re, A_im)
    for r in range(2):
        w_re, w_im, _ = ref.apply(pc.x1, pc.x2, pc.x3, A_re[r], A_im[r], 0, k, Params(threads=4))
        assert rel_l2(i_re[r], i_im[r], w_re, w_im) <= 1e-10
    plan.close()
