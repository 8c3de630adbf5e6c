"""GPU parity: the CUDA path through the C ABI against the CPU oracle
(oracle/ifgf_oracle.c, pinned to the reference) on identical seeded inputs.

Structure (octree, neighbour/cousin CSR, relevant cone lists) must be
bit-identical; pass outputs and the full operator within relative l2 1e-10
(BASELINE north_star); the sampled error within 1.01x of the oracle's."""
import math

import numpy as np
import pytest

from bindings import Params, rel_l2

pytestmark = pytest.mark.gpu

# (name, n, shape, c, kind, kappa, dens, seed, orders)
CASES = [
    ("helm_sphere", 4000, 0, 1.0, 0, 2 * math.pi * 1.5, 0, 11, (3, 5, 5)),
    ("laplace_sphere", 5000, 0, 1.0, 1, 0.0, 1, 12, (3, 5, 5)),
    ("helm_oblate", 6000, 1, 0.25, 0, 2 * math.pi * 2.0, 0, 13, (3, 5, 5)),
    ("helm_high_order", 3456, 0, 1.0, 0, 2 * math.pi * 2.0, 0, 14, (5, 7, 7)),
    ("helm_mid_order", 3456, 0, 1.0, 0, 2 * math.pi * 2.0, 0, 14, (4, 6, 6)),
    # the other orders the warp GEMM serves (blocks of 30 and 64 coefficients:
    # a short last K chunk, and K chunks that tile the block exactly)
    ("helm_order_333", 3000, 0, 1.0, 0, 2 * math.pi * 1.5, 0, 15, (3, 3, 3)),
    ("laplace_order_444", 3000, 0, 1.0, 1, 0.0, 1, 16, (4, 4, 4)),
]


def _setup(ifgf, oracle, case):
    name, n, shape, c, kind, kappa, dens, seed, orders = case
    pc = ifgf.generate(n, shape, c, dens, seed)
    cfg = ifgf.KernelConfig(ifgf.KernelKind(kind), kappa)
    ep = ifgf.EngineParams(orders=ifgf.InterpOrders(*orders))
    op = Params(p_s=orders[0], p_theta=orders[1], p_phi=orders[2])
    return pc, cfg, ep, op


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def built(request, gpu, oracle):
    pc, cfg, ep, op = _setup(gpu, oracle, request.param)
    plan = gpu.Plan.from_cloud(pc, cfg, ep)
    prob = oracle.problem(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, int(cfg.kind), cfg.wavenumber, op)
    return request.param, pc, cfg, ep, op, plan, prob


def test_structure_identical(built):
    case, pc, cfg, ep, op, plan, prob = built
    assert plan.depth == prob.depth
    assert np.array_equal(plan.cube(), prob.cube())
    perm, _ = prob.sorted()
    assert np.array_equal(plan.perm(), perm)
    for d in range(1, plan.depth + 1):
        g, o = plan.level(d), prob.level(d)
        assert g.h == o.h
        for f in ("codes", "first", "count", "centers", "nbr_off", "nbr"):
            assert np.array_equal(getattr(g, f), getattr(o, f)), (d, f)
        if d >= 2:
            assert np.array_equal(g.parent, o.parent), (d, "parent")
        if d < plan.depth:
            assert np.array_equal(g.child_begin, o.child_begin), (d, "child_begin")
        if d >= 3:
            for f in ("cousin_off", "cousin", "cone_box", "cone_gamma", "box_cone_begin"):
                assert np.array_equal(getattr(g, f), getattr(o, f)), (d, f)


def test_singular_pass(built):
    case, pc, cfg, ep, op, plan, prob = built
    plan.set_density(pc.a_re, pc.a_im)
    plan.zero_result()
    plan.singular_pass()
    g = plan.read_result(sorted_order=True)
    o = prob.singular()
    assert rel_l2(*g, *o) <= 1e-13


def test_level_d_blocks(built):
    case, pc, cfg, ep, op, plan, prob = built
    plan.set_density(pc.a_re, pc.a_im)
    plan.level_d_pass()
    g = plan.read_blocks(plan.depth)
    o = prob.level_d()
    assert rel_l2(g[0], g[1], o[0], o[1]) <= 1e-12


def test_propagation_pass(built):
    case, pc, cfg, ep, op, plan, prob = built
    D = plan.depth
    if D < 4:
        pytest.skip("depth 3 has no propagation")
    cre, cim = prob.level_d()
    plan.write_blocks(D, cre, cim)
    plan.propagation_pass(D)
    g = plan.read_blocks(D - 1)
    o = prob.propagation(D, cre, cim)
    assert rel_l2(g[0], g[1], o[0], o[1]) <= 1e-12


def test_interpolation_pass(built):
    case, pc, cfg, ep, op, plan, prob = built
    D = plan.depth
    cre, cim = prob.level_d()
    plan.write_blocks(D, cre, cim)
    plan.zero_result()
    plan.interpolation_pass(D)
    g = plan.read_result(sorted_order=True)
    o = prob.interpolation(D, cre, cim)
    assert rel_l2(*g, *o) <= 1e-12


def test_interpolation_records_bitwise(built):
    """K4 from the plan's locate records (k_locate_points at setup, blocks staged
    in shared memory where the orders allow it) equals the K4 that locates
    every (point, cousin) pair again, bitwise: whole applies, and pass ranges
    that cut through a two-point work item."""
    case, pc, cfg, ep, op, plan, prob = built
    D, n = plan.depth, pc.size()
    cre, cim = prob.level_d()
    plan.write_blocks(D, cre, cim)
    res = {}
    for rec in (True, False):
        plan.set_k4_records(rec)
        whole = plan.apply(pc.a_re, pc.a_im)[:2]
        plan.write_blocks(D, cre, cim)
        plan.zero_result()
        for b, e in ((0, 1), (1, n // 3 + 1), (n // 3 + 1, n - 1), (n - 1, n)):
            plan.interpolation_pass(D, b, e)
        res[rec] = (whole, plan.read_result(sorted_order=True))
    plan.set_k4_records(True)
    for a, b in zip(res[True], res[False]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    o = prob.interpolation(D, cre, cim)
    assert rel_l2(*res[True][1], *o) <= 1e-12


def test_apply_parity_and_error(built, oracle):
    case, pc, cfg, ep, op, plan, prob = built
    g_re, g_im, rep = plan.apply(pc.a_re, pc.a_im)
    o_re, o_im, orep = oracle.apply(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, int(cfg.kind),
                                    cfg.wavenumber, op)
    assert rep.depth == orep["depth"]
    assert rel_l2(g_re, g_im, o_re, o_im) <= 1e-10
    idx = oracle.sample_indices(pc.size(), 500, 7)
    e_g = oracle.error_at_indices(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, g_re, g_im,
                                  int(cfg.kind), cfg.wavenumber, idx)
    e_o = oracle.error_at_indices(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, o_re, o_im,
                                  int(cfg.kind), cfg.wavenumber, idx)
    assert e_g <= 1.01 * e_o
    # bitwise reproducible run to run (parallel.hpp:17-19 contract)
    g2 = plan.apply(pc.a_re, pc.a_im)
    assert np.array_equal(g_re, g2[0]) and np.array_equal(g_im, g2[1])
    if int(cfg.kind) == 1:
        assert np.all(g_im == 0.0)  # test_engine.cpp:303-314


def test_one_shot_apply_matches_plan(built, gpu):
    case, pc, cfg, ep, op, plan, prob = built
    q = pc.copy()
    rep = gpu.apply(q, cfg, ep)
    g = plan.apply(pc.a_re, pc.a_im)
    assert np.array_equal(q.i_re, g[0]) and np.array_equal(q.i_im, g[1])
    assert rep.n == pc.size() and rep.depth == plan.depth
    assert [l.cones for l in rep.levels] == [plan.n_cones(d) for d in range(3, plan.depth + 1)]


def test_direct_eval(built, gpu, oracle):
    case, pc, cfg, ep, op, plan, prob = built
    idx = oracle.sample_indices(pc.size(), 300, 3)
    q = pc.copy()
    gpu.direct_eval(q, cfg, targets=idx)
    o = oracle.direct(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, int(cfg.kind), cfg.wavenumber, idx)
    assert rel_l2(q.i_re[idx], q.i_im[idx], *o) <= 1e-13


def test_propagation_kernels_agree(built):
    """The K3 implementations (per-node locate, the FP64 tensor-core warp GEMM
    on every level, register-blocked node rows from the tiles and grouped on
    the fly, and the default per-level choice between warp GEMM and rows)
    compute the same operator up to rounding; removed kernels are refused."""
    case, pc, cfg, ep, op, plan, prob = built
    res = []
    kinds = (plan.PROP_NODE, plan.PROP_DMMA, plan.PROP_ROWS, plan.PROP_FLY, plan.PROP_AUTO)
    for kind in kinds:
        plan.set_prop_kernel(kind)
        res.append(plan.apply(pc.a_re, pc.a_im)[:2])
    plan.set_prop_kernel(plan.PROP_AUTO)
    for r in res[1:]:
        assert rel_l2(r[0], r[1], res[0][0], res[0][1]) <= 1e-13
    for removed in (1, 5, 6):
        with pytest.raises(Exception):
            plan.set_prop_kernel(removed)
