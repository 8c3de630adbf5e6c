"""Multi-rank host logic on the CPU: rank layout and exchange lists against
the oracle / reference (dist.cpp:78-237), the halo / send-list pairing the
C++ engine (csrc/dist.cu) relies on, and the launcher side of the
multi-process path (communicator id broadcast, max-over-ranks timing) over a
real torch.distributed gloo group of world size 2."""
import math
import os
import socket

import numpy as np
import pytest

from bindings import Params


def _problem(oracle, n=6000, seed=41, kappa=2 * math.pi * 3.0):
    x1, x2, x3, ar, ai = oracle.generate(n, 0, 1.0, 0, seed)
    return oracle.problem(x1, x2, x3, ar, ai, 0, kappa, Params())


def _layout_and_plan(prob, R):
    from paper_2112_15198_b200.dist import Layout, build_exchange_plan
    bb, pb, cb = prob.partition(R)
    lay = Layout(R, bb, pb, cb)
    ex = build_exchange_plan(lay, prob.depth, lambda r, d, k: prob.exchange_set(R, r, d, k))
    return lay, ex


@pytest.mark.parametrize("R", [2, 4, 8])
def test_exchange_lists_consistent(oracle, R):
    prob = _problem(oracle)
    lay, ex = _layout_and_plan(prob, R)
    for (d, kind), recv in ex.recv.items():
        for r in range(R):
            for p in range(R):
                a = recv[r][p]
                assert p != r or len(a) == 0
                if len(a):
                    assert np.all(np.diff(a.astype(np.int64)) > 0)  # sorted, deduplicated
                    qb, qe = lay.cones(d, p)
                    assert np.all((a >= qb) & (a < qe))               # owned by p
                assert np.array_equal(ex.send[(d, kind)][p][r], a)
    # point intervals tile [0, N) (dist.cpp:90-116)
    assert lay.point_begin[0] == 0 and lay.point_begin[-1] == prob.n
    assert np.all(np.diff(lay.point_begin.astype(np.int64)) > 0)


def test_exchange_volume_matches_reference_counters(oracle, ref):
    x1, x2, x3, ar, ai = oracle.generate(6000, 0, 1.0, 0, 41)
    k = 2 * math.pi * 3.0
    prob = oracle.problem(x1, x2, x3, ar, ai, 0, k, Params())
    lay, ex = _layout_and_plan(prob, 8)
    _, _, comm = ref.run_distributed(x1, x2, x3, ar, ai, 0, k, Params(threads=4), 8)
    for d in range(3, prob.depth + 1):
        got = sum(len(a) for row in ex.recv[(d, 0)] for a in row)
        assert got == int(comm[d - 3][0])
        if d > 3:
            got = sum(len(a) for row in ex.recv[(d, 1)] for a in row)
            assert got == int(comm[d - 3][1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _boot_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2112_15198_b200.dist import max_over_ranks, share_comm_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0's id (a stand-in for ifgf_comm_unique_id's 128 NCCL bytes)
    made = []

    def make():
        made.append(1)
        return bytes(range(128))

    cid = share_comm_id(make)
    slowest = max_over_ranks(0.5 + rank)
    out.put((rank, cid, len(made), slowest))
    dist.destroy_process_group()


def test_rank_bootstrap_over_gloo_world2():
    """The launcher side of the multi-GPU path (bench.py --gpus N): rank 0
    alone makes the communicator id and every rank receives the same bytes;
    step times reduce to the slowest rank's."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_boot_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] == bytes(range(128)) for r in res)
    assert [r[2] for r in res] == [1, 0]      # only rank 0 made the id
    assert all(r[3] == 1.5 for r in res)      # max over ranks


def test_send_lists_pair_with_halos(oracle):
    """The request protocol of csrc/dist.cu on host data: rank r's halo at a
    level is the union of its two exchange sets, sorted; the owner p's send
    list for r is the slice of r's halo owned by p (contiguous, since owner
    intervals are), so sends and receives pair up one to one."""
    prob = _problem(oracle, n=5000, seed=47)
    R = 3
    lay, ex = _layout_and_plan(prob, R)
    for d in range(3, prob.depth + 1):
        for r in range(R):
            parts = [np.concatenate(ex.recv[(d, k)][r]) for k in (0, 1) if (d, k) in ex.recv]
            halo = np.unique(np.concatenate(parts)) if parts else np.zeros(0, np.uint32)
            owner = lay.cone_owner(d, halo) if len(halo) else np.zeros(0, np.int64)
            assert np.all(np.diff(owner) >= 0)  # owner runs are contiguous in the halo
            qb, qe = lay.cones(d, r)
            below = int(np.sum(halo < qb))
            assert np.all(halo[below:] >= qe)   # [halo below | owned | halo above]
            for p in range(R):
                mine = halo[owner == p]
                assert p != r or len(mine) == 0
                pb, pe = lay.cones(d, p)
                assert np.all((mine >= pb) & (mine < pe))
