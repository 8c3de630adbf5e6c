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


@pytest.mark.parametrize("R", [2, 4, 8])
def test_work_partition_layout_and_bitwise(gpu, R):
    """IFGF_PARTITION_WORK (contiguous intervals balanced by evaluation work,
    the paper's proposed extension) on a non-uniform spheroid: a valid layout
    (monotone, covering, whole boxes, point cuts on box boundaries) that
    differs from the reference's count-balanced one, and the distributed
    result is still bitwise the single-GPU apply."""
    from paper_2112_15198_b200.dist import simulate
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
    plans = [gpu.Plan.from_cloud(pc, cfg) for _ in range(R)]
    i_re, i_im, moved, ex = simulate(plans, pc.a_re, pc.a_im, partition=gpu.Plan.PARTITION_WORK)
    assert np.array_equal(i_re, s_re) and np.array_equal(i_im, s_im)
    assert moved == ex.volume_blocks()


def _dplan_worker(rank, world, port, args, out, partition=0):
    import os

    import torch
    import torch.distributed as dist

    import paper_2112_15198_b200 as ifgf
    from paper_2112_15198_b200.dist import DistributedPlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, shape, c, dens, seed, kappa = args
    pc = ifgf.generate(n, shape, c, dens, seed)
    cfg = ifgf.KernelConfig(ifgf.KernelKind.Helmholtz, kappa)
    dp = DistributedPlan(pc.x1, pc.x2, pc.x3, cfg, partition=partition)
    i_re, i_im = dp.apply(pc.a_re, pc.a_im)
    vol = dp.ex.volume_blocks()
    dp.close()
    out.put((rank, i_re, i_im, vol))
    dist.destroy_process_group()


@pytest.mark.parametrize("partition", [0, 1])
def test_distributed_plan_two_ranks_one_gpu(gpu, partition):
    """The whole DistributedPlan path (rank layout, per-rank exchange sets and
    the all-to-all that pairs them, per-level block exchange, result gather)
    on real kernels: two processes share the GPU, blocks travel through gloo
    (host staging; NCCL moves device buffers on a multi-GPU box).  Ranks only
    wait on each other at the host exchanges, never inside kernels.  The
    result equals the single-GPU apply bitwise."""
    import socket

    import torch.multiprocessing as mp
    args = (6000, 0, 1.0, 0, 61, 2 * math.pi * 2.0)
    pc = gpu.generate(*args[:5])
    cfg = gpu.KernelConfig(gpu.KernelKind.Helmholtz, args[5])
    plan = gpu.Plan.from_cloud(pc, cfg, gpu.EngineParams())
    ref = plan.apply(pc.a_re, pc.a_im)
    plan.close()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dplan_worker, args=(r, 2, port, args, q, partition))
          for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, i_re, i_im, vol in res:
        assert vol > 0
        assert np.array_equal(i_re, ref[0]) and np.array_equal(i_im, ref[1]), rank
