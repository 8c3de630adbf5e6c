"""Multi-rank host logic of paper_2112_15198_b200.dist on the CPU: rank
layout and exchange lists against the oracle / reference (dist.cpp:78-237),
and the block exchange protocol over a real torch.distributed gloo group of
world size 2 (the NCCL path on B200 runs the same code)."""
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


class FakeStore:
    """Level block storage on the CPU: owned cones hold f(d, q, k), the rest NaN."""

    def __init__(self, torch, ncones, depth, lay, rank, bd=8):
        self.torch, self.block_doubles = torch, bd
        self.lv = {}
        for d in range(3, depth + 1):
            t = torch.full((ncones[d], bd), float("nan"), dtype=torch.float64)
            qb, qe = lay.cones(d, rank)
            q = torch.arange(qb, qe, dtype=torch.float64)[:, None]
            t[qb:qe] = d * 1e7 + q * 16 + torch.arange(bd, dtype=torch.float64)[None, :]
            self.lv[d] = t

    def pack(self, d, idx, buf):
        buf.copy_(self.lv[d].index_select(0, idx.long()).reshape(-1))

    def unpack(self, d, idx, buf):
        self.lv[d].index_copy_(0, idx.long(), buf.reshape(len(idx), -1))


def _worker(rank, world, port, depth, ncones, lay, ex, out):
    import torch
    import torch.distributed as dist

    from paper_2112_15198_b200.dist import INTERP, PROP, TorchExchanger
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = FakeStore(torch, ncones, depth, lay, rank)
    x = TorchExchanger(store, ex, rank, torch.device("cpu"))
    moved = 0
    # the reference's phase order (dist.cpp:292-327)
    if depth > 3:
        moved += x.exchange(depth, PROP)
    for d in range(depth, 2, -1):
        moved += x.exchange(d, INTERP)
        if d > 4:
            moved += x.exchange(d - 1, PROP)
    ok = True
    for d in range(3, depth + 1):
        need = set()
        for kind in (INTERP, PROP):
            if (d, kind) in ex.recv:
                for p in range(world):
                    need.update(int(q) for q in ex.recv[(d, kind)][rank][p])
        t = store.lv[d]
        for q in need:
            want = d * 1e7 + q * 16 + np.arange(store.block_doubles)
            ok &= bool(np.array_equal(t[q].numpy(), want))
        qb, qe = lay.cones(d, rank)
        valid = set(np.nonzero(~np.isnan(t[:, 0].numpy()))[0].tolist())
        ok &= valid == set(range(qb, qe)) | need  # nothing else arrived
    out.put((rank, ok, moved))
    dist.destroy_process_group()


def test_block_exchange_over_gloo_world2(oracle):
    import torch.multiprocessing as mp
    prob = _problem(oracle, n=5000, seed=43)
    lay, ex = _layout_and_plan(prob, 2)
    ncones = {d: prob.n_cones(d) for d in range(3, prob.depth + 1)}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, prob.depth, ncones, lay, ex, q))
          for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    total = sum(len(a) for lists in ex.recv.values() for row in lists for a in row)
    assert sum(m for _, _, m in res) == total


def _plan_worker(rank, world, port, lay, depth, needs, out):
    import torch.distributed as dist

    from paper_2112_15198_b200.dist import build_exchange_plan_rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = build_exchange_plan_rank(lay, depth, rank, lambda d, k: needs[rank][(d, k)])
    out.put((rank, {k: ([a.tolist() for a in ex.recv[k][rank]],
                        [a.tolist() for a in ex.send[k][rank]]) for k in ex.recv}))
    dist.destroy_process_group()


def test_rank_local_exchange_plan_over_gloo(oracle):
    """build_exchange_plan_rank (own needs + all-to-all) gives every rank the
    same rows as the full plan computed from everyone's needs."""
    import torch.multiprocessing as mp
    prob = _problem(oracle, n=5000, seed=47)
    R = 2
    lay, ex = _layout_and_plan(prob, R)
    needs = [{k: np.concatenate(ex.recv[k][r]).astype(np.uint32) for k in ex.recv}
             for r in range(R)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_plan_worker, args=(r, R, port, lay, prob.depth, needs, q))
          for r in range(R)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(R):
        for k in ex.recv:
            recv, send = res[r][k]
            assert recv == [a.tolist() for a in ex.recv[k][r]]
            assert send == [a.tolist() for a in ex.send[k][r]]
