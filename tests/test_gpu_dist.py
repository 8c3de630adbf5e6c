"""Multi-GPU engine (csrc/dist.cu) on one B200: R rank plans in one process
(ifgf_run_distributed, the analogue of dist::run_distributed), each with its
own partitioned block storage (owned cones + halo), blocks moved rank to rank
by the device pack + copies that NCCL send/recv replaces across processes.
Mirrors test_dist.cpp:107-123 -- the output is bitwise identical to the
single-GPU apply for every rank count -- and pins the per-rank exchange sets
against the oracle and the reference's CommStats counters
(dist.cpp:179-237, 253-272)."""
import math

import numpy as np
import pytest

from bindings import Params, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case(gpu):
    pc = gpu.generate(6000, 0, 1.0, 0, 41)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 3.0)
    return pc, cfg


def _single(gpu, pc, cfg, p=None):
    plan = gpu.Plan.from_cloud(pc, cfg, p or gpu.EngineParams())
    out = plan.apply(pc.a_re, pc.a_im)
    plan.close()
    return out


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


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_rank_group_bitwise_equal_single_gpu(gpu, case, R):
    from paper_2112_15198_b200.dist import run_distributed
    pc, cfg = case
    s_re, s_im, _ = _single(gpu, pc, cfg)
    q = pc.copy()
    rep, infos = run_distributed(q, cfg, gpu.EngineParams(), R)
    assert np.array_equal(q.i_re, s_re) and np.array_equal(q.i_im, s_im)
    assert [i.rank for i in infos] == list(range(R))
    # the ranks' point intervals tile [0, N); owned cones tile every level
    assert infos[0].point_begin == 0 and infos[-1].point_end == len(pc.x1)
    for a, b in zip(infos, infos[1:]):
        assert a.point_end == b.point_begin
    for k, lv in enumerate(infos[0].levels):
        assert sum(i.levels[k]["owned_cones"] for i in infos) == rep.levels[k].cones
        # what one rank sends is what the others receive
        assert sum(i.levels[k]["sent_cones"] for i in infos) == \
            sum(i.levels[k]["halo_cones"] for i in infos)
    if R == 1:
        assert all(lv["halo_cones"] == 0 for lv in infos[0].levels)


@pytest.mark.parametrize("R", [2, 3])
def test_rank_group_bitwise_equal_with_warp_gemm(gpu, case, R, monkeypatch):
    """With the warp GEMM taken at every level that has the precomputed
    geometry (thresholds lifted), rank plans -- whose units cover only their
    cone intervals -- still reproduce the single-GPU blocks bitwise: a cone's
    result does not depend on the unit it is batched into."""
    from paper_2112_15198_b200.dist import run_distributed
    monkeypatch.setenv("IFGF_G4_MIN_SHARE", "0")
    monkeypatch.setenv("IFGF_G4_MIN_CONES", "0")
    pc, cfg = case
    s_re, s_im, _ = _single(gpu, pc, cfg)
    q = pc.copy()
    run_distributed(q, cfg, gpu.EngineParams(), R)
    assert np.array_equal(q.i_re, s_re) and np.array_equal(q.i_im, s_im)
    monkeypatch.delenv("IFGF_G4_MIN_SHARE")
    monkeypatch.delenv("IFGF_G4_MIN_CONES")
    r_re, r_im, _ = _single(gpu, pc, cfg)
    assert rel_l2(s_re, s_im, r_re, r_im) <= 1e-13


def test_rank_group_counters_match_reference(gpu, ref, case):
    """Per level, the ranks' interpolation / propagation fetch counts equal the
    reference's window counters (dist.cpp:253-272) at R = 4."""
    from paper_2112_15198_b200.dist import run_distributed
    pc, cfg = case
    R = 4
    _, infos = run_distributed(pc.copy(), cfg, gpu.EngineParams(), R)
    _, _, comm = ref.run_distributed(pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im, 0, cfg.wavenumber,
                                     Params(threads=4), R)
    for k, row in enumerate(comm):
        assert sum(i.levels[k]["interp_needed"] for i in infos) == int(row[0])
        assert sum(i.levels[k]["prop_needed"] for i in infos) == int(row[1])


def test_rank_storage_shrinks_with_ranks(gpu):
    """Block storage is partitioned: per rank it falls ~1/R (owned + halo),
    while a single-GPU plan holds every level's blocks."""
    from paper_2112_15198_b200.dist import run_distributed
    pc = gpu.generate(40000, 0, 1.0, 0, 53)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 6.0)
    per = {}
    for R in (1, 2, 4, 8):
        q = pc.copy()
        _, infos = run_distributed(q, cfg, gpu.EngineParams(), R)
        per[R] = max(i.block_bytes for i in infos)
    assert per[2] < 0.62 * per[1]
    assert per[4] < 0.36 * per[1]
    assert per[8] < 0.22 * per[1]


@pytest.mark.parametrize("R", [2, 4, 8])
def test_work_partition_layout_and_bitwise(gpu, R):
    """IFGF_PARTITION_WORK (contiguous intervals balanced by evaluation work,
    the paper's proposed extension) on a non-uniform spheroid: a valid layout
    that differs from the reference's count-balanced one, and the rank group
    result is still bitwise the single-GPU apply."""
    from paper_2112_15198_b200.dist import run_distributed
    pc = gpu.generate(40000, 1, 0.25, 0, 43)  # oblate spheroid (1,1,0.25)
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, 2 * math.pi * 6.0)
    single = gpu.Plan.from_cloud(pc, cfg)
    s_re, s_im, _ = single.apply(pc.a_re, pc.a_im)
    bb0, pb0, cb0 = single.partition(R)
    single.set_partition(gpu.Plan.PARTITION_WORK)
    bb, pb, cb = single.partition(R)
    info = single.info
    assert bb[0] == 0 and bb[-1] == info.boxes[single.depth] and np.all(np.diff(bb) >= 1)
    assert pb[0] == 0 and pb[-1] == len(pc.x1) and np.all(np.diff(pb.astype(np.int64)) > 0)
    for d in range(3, single.depth + 1):
        row = cb[d - 3]
        assert row[0] == 0 and row[-1] == info.cones[d] and np.all(np.diff(row.astype(np.int64)) >= 0)
    assert not (np.array_equal(bb, bb0) and np.array_equal(cb, cb0))
    q = pc.copy()
    _, infos = run_distributed(q, cfg, gpu.EngineParams(partition=gpu.Plan.PARTITION_WORK), R)
    assert np.array_equal(q.i_re, s_re) and np.array_equal(q.i_im, s_im)
    assert [i.point_begin for i in infos] + [infos[-1].point_end] == [int(v) for v in pb]


def test_rank_group_laplace_and_deeper_tree(gpu):
    from paper_2112_15198_b200.dist import run_distributed
    pc = gpu.generate(20000, 0, 1.0, 1, 71)
    cfg = gpu.KernelConfig(gpu.KernelKind.Laplace, 0.0)
    s_re, s_im, _ = _single(gpu, pc, cfg)
    q = pc.copy()
    run_distributed(q, cfg, gpu.EngineParams(), 3)
    assert np.array_equal(q.i_re, s_re) and np.array_equal(q.i_im, s_im)


def test_nccl_rank_plan_world1(gpu, case):
    """The multi-process entry points on one GPU: an NCCL communicator of one
    rank (libnccl loaded on first use), a rank plan and its apply through the
    C ABI (device pointers), bitwise equal to the single-GPU apply.  (Two
    ranks need two GPUs: NCCL refuses two ranks on one device; the in-process
    group above covers the multi-rank data path.)"""
    import torch

    from paper_2112_15198_b200.dist import Comm, DistPlan
    pc, cfg = case
    s_re, s_im, _ = _single(gpu, pc, cfg)
    comm = Comm(Comm.unique_id(), 0, 1, 0)
    dev = torch.device("cuda", 0)
    X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
    out = [torch.empty(len(pc.x1), dtype=torch.float64, device=dev) for _ in range(2)]
    plan = DistPlan(comm, X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), len(pc.x1), cfg)
    for _ in range(2):  # plan reuse
        plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(), out[1].data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(out[0].cpu().numpy(), s_re)
        assert np.array_equal(out[1].cpu().numpy(), s_im)
    ri = plan.info()
    assert ri.world == 1 and ri.point_begin == 0 and ri.point_end == len(pc.x1)
    plan.close()
    comm.close()
