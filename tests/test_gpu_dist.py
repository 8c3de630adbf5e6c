"""Multi-rank path on one B200: R ranks simulated in one process (one plan
per rank, phases advanced rank by rank, blocks moved through the device
pack/unpack of the C ABI).  Mirrors test_dist.cpp:107-123 -- the output is
bitwise identical to the single-GPU apply for every rank count -- and checks
the device-computed exchange sets against the oracle (dist.cpp:179-237)."""
import math

import numpy as np
import pytest

from bindings import Params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case(gpu):
    pc = gpu.generate(6000, 0, 1.0, 0, 41)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 3.0)
    return pc, cfg


def test_exchange_sets_match_oracle(gpu, oracle, case):
    pc, cfg = case
    plan = gpu.Plan.from_cloud(pc, cfg)
    prob = oracle.problem(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, 0, cfg.wavenumber, Params())
    for R in (2, 4, 8):
        bb, pb, cb = plan.partition(R)
        ob, op, oc = prob.partition(R)
        assert np.array_equal(bb, ob) and np.array_equal(pb, op) and np.array_equal(cb, oc)
        for r in range(R):
            for d in range(3, plan.depth + 1):
                for kind in (0, 1):
                    if kind == 1 and d < 4:
                        continue
                    assert np.array_equal(plan.exchange_set(R, r, d, kind),
                                          prob.exchange_set(R, r, d, kind)), (R, r, d, kind)


@pytest.mark.parametrize("R", [1, 2, 4])
def test_simulated_ranks_bitwise_equal_single_gpu(gpu, case, R):
    from paper_2112_15198_b200.dist import simulate
    pc, cfg = case
    single = gpu.Plan.from_cloud(pc, cfg)
    s_re, s_im, _ = single.apply(pc.a_re, pc.a_im)
    plans = [gpu.Plan.from_cloud(pc, cfg) for _ in range(R)]
    i_re, i_im, moved, ex = simulate(plans, pc.a_re, pc.a_im)
    assert np.array_equal(i_re, s_re) and np.array_equal(i_im, s_im)
    assert moved == ex.volume_blocks()
    if R == 1:
        assert moved == 0
