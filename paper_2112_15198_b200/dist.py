"""Multi-GPU IFGF matvec: the reference's rank algorithm (dist.cpp:241-361,
the paper's "IFGF Method" in MPI form) with real exchanges.

* Layout (dist.cpp:78-130): points in contiguous Morton intervals of level-D
  boxes balanced by population; each level's cones in equal-count intervals
  of the (box, gamma) order -- boxes at fine levels, cone segments at coarse
  levels.  Every rank builds the same plan (setup is cheap on the GPU), so
  every rank can compute every other rank's needs locally.
* Exchange sets (dist.cpp:179-237): per level d, the deduplicated foreign
  cones a rank needs for interpolation (its points' cousin cones) and for
  propagation (child cones hit by its parent cones' nodes), computed on the
  device by ifgf_plan_exchange_set.
* Transport: blocks are packed on the device (ifgf_plan_pack_blocks), moved
  with torch.distributed batched P2P (NCCL over NVLink on B200; gloo in the
  CPU tests) and unpacked into the receiving rank's level storage at their
  global cone ordinal -- the analogue of Window::get (dist.cpp:154-173).

Phase order follows dist.cpp:273-342: near field and level-D seeding on owned
work, then per level: interpolation data in; propagation of owned parent
cones (after the propagation data of that level arrived); interpolation of
owned points.  Each kernel computes its work items independently, so the
distributed result is bitwise equal to the single-GPU apply (tested).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INTERP, PROP = 0, 1


@dataclass
class Layout:
    """RankLayout (dist.hpp:13-21)."""
    n_ranks: int
    box_begin: np.ndarray
    point_begin: np.ndarray
    cone_begin: np.ndarray  # [level d-3][rank + 1]

    def points(self, r):
        return int(self.point_begin[r]), int(self.point_begin[r + 1])

    def cones(self, d, r):
        cb = self.cone_begin[d - 3]
        return int(cb[r]), int(cb[r + 1])

    def cone_owner(self, d, q):
        return np.searchsorted(self.cone_begin[d - 3], q, side="right") - 1


@dataclass
class ExchangePlan:
    """Per level and kind: recv[r][p] = cones rank r receives from owner p;
    send[r][p] = cones rank r sends to p (= recv[p][r])."""
    depth: int
    n_ranks: int
    recv: dict = field(default_factory=dict)  # (d, kind) -> [r][p] -> np.ndarray
    send: dict = field(default_factory=dict)

    def volume_blocks(self):
        return sum(len(a) for lists in self.recv.values() for row in lists for a in row)


def build_exchange_plan(layout: Layout, depth: int, need) -> ExchangePlan:
    """need(r, d, kind) -> sorted foreign cone ordinals rank r needs."""
    R = layout.n_ranks
    ex = ExchangePlan(depth, R)
    for d in range(3, depth + 1):
        for kind in (INTERP, PROP):
            if kind == PROP and d < 4:
                continue
            recv = [[np.zeros(0, np.uint32) for _ in range(R)] for _ in range(R)]
            for r in range(R):
                cones = np.asarray(need(r, d, kind), dtype=np.uint32)
                if len(cones):
                    owner = layout.cone_owner(d, cones)
                    for p in range(R):
                        sel = cones[owner == p]
                        if p == r and len(sel):
                            raise AssertionError("a rank never fetches its own cones")
                        recv[r][p] = sel
            ex.recv[(d, kind)] = recv
            ex.send[(d, kind)] = [[recv[p][r] for p in range(R)] for r in range(R)]
    return ex


def build_exchange_plan_rank(layout: Layout, depth: int, rank: int, need_self, group=None,
                             device=None) -> ExchangePlan:
    """This rank's rows of the exchange plan without computing anyone else's
    needs: the rank computes its own foreign-cone sets (need_self(d, kind)),
    tells every owner which of its cones it needs (one all-to-all of counts and
    one of indices per level and kind) and learns what it must send.  Only
    row `rank` of recv/send is filled."""
    import torch
    import torch.distributed as dist
    R = layout.n_ranks
    dev = device if device is not None else torch.device("cpu")
    ex = ExchangePlan(depth, R)
    empty = np.zeros(0, np.uint32)
    for d in range(3, depth + 1):
        for kind in (INTERP, PROP):
            if kind == PROP and d < 4:
                continue
            cones = np.asarray(need_self(d, kind), dtype=np.uint32)
            owner = layout.cone_owner(d, cones) if len(cones) else np.zeros(0, np.int64)
            mine = [cones[owner == p] for p in range(R)]
            if len(mine[rank]):
                raise AssertionError("a rank never fetches its own cones")
            cnt = torch.tensor([len(a) for a in mine], dtype=torch.int64, device=dev)
            cnt_in = torch.empty_like(cnt)
            dist.all_to_all_single(cnt_in, cnt, group=group)
            sizes_out, sizes_in = cnt.tolist(), cnt_in.tolist()
            flat = torch.as_tensor(np.concatenate(mine).astype(np.int64) if len(cones) else
                                   np.zeros(0, np.int64), device=dev)
            got = torch.empty(sum(sizes_in), dtype=torch.int64, device=dev)
            dist.all_to_all_single(got, flat, sizes_in, sizes_out, group=group)
            got = got.cpu().numpy().astype(np.uint32)
            off = np.concatenate([[0], np.cumsum(sizes_in)])
            recv = [[empty] * R for _ in range(R)]
            send = [[empty] * R for _ in range(R)]
            recv[rank] = mine
            send[rank] = [got[off[p]:off[p + 1]] for p in range(R)]
            ex.recv[(d, kind)] = recv
            ex.send[(d, kind)] = send
    return ex


class TorchExchanger:
    """Moves blocks between ranks with torch.distributed batched P2P.

    `store` provides block_doubles (2 * Pst), pack(d, idx_tensor, buf) and
    unpack(d, idx_tensor, buf) over tensors on `device`.  With a backend that
    moves host tensors only (gloo) the packed buffers are staged through host
    memory (`wire` = cpu); with NCCL they travel device to device."""

    def __init__(self, store, ex: ExchangePlan, rank: int, device, group=None, wire=None):
        import torch
        self.torch = torch
        self.store, self.ex, self.rank, self.device, self.group = store, ex, rank, device, group
        self.wire = wire if wire is not None else device
        self._idx = {}
        for key in ex.recv:
            for p in range(ex.n_ranks):
                for role, lists in (("send", ex.send[key][rank]), ("recv", ex.recv[key][rank])):
                    a = lists[p]
                    if len(a):
                        self._idx[(key, role, p)] = torch.as_tensor(a.astype(np.int32),
                                                                    device=device)

    def exchange(self, d, kind):
        torch = self.torch
        import torch.distributed as dist
        key = (d, kind)
        if key not in self.ex.recv:
            return 0
        bd = self.store.block_doubles
        ops, recv_bufs = [], []
        for p in range(self.ex.n_ranks):
            if p == self.rank:
                continue
            si = self._idx.get((key, "send", p))
            if si is not None:
                buf = torch.empty(len(si) * bd, dtype=torch.float64, device=self.device)
                self.store.pack(d, si, buf)
                if self.wire != self.device:
                    torch.cuda.synchronize()
                    buf = buf.to(self.wire)
                ops.append(dist.P2POp(dist.isend, buf, p, group=self.group))
            ri = self._idx.get((key, "recv", p))
            if ri is not None:
                buf = torch.empty(len(ri) * bd, dtype=torch.float64, device=self.wire)
                recv_bufs.append((ri, buf))
                ops.append(dist.P2POp(dist.irecv, buf, p, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        moved = 0
        for ri, buf in recv_bufs:
            self.store.unpack(d, ri, buf.to(self.device))
            moved += len(ri)
        return moved


class PlanStore:
    """Block store over an ifgf Plan's level storage (device pointers)."""

    def __init__(self, plan, stream=0):
        from . import _lib
        self.plan = plan
        self.block_doubles = 2 * int(_lib.lib.ifgf_plan_block_stride(plan._h))
        self.stream = stream

    def pack(self, d, idx, buf):
        self.plan.pack_blocks(d, idx.data_ptr(), idx.numel(), buf.data_ptr(), self.stream)

    def unpack(self, d, idx, buf):
        self.plan.unpack_blocks(d, idx.data_ptr(), idx.numel(), buf.data_ptr(), self.stream)


def rank_layout(plan, n_ranks) -> Layout:
    bb, pb, cb = plan.partition(n_ranks)
    return Layout(n_ranks, bb, pb, cb)


def run_rank_share(plan, layout: Layout, rank: int, a_re, a_im, exchange):
    """This rank's part of the distributed apply, in the reference's phase
    order (dist.cpp:273-342).  `exchange(d, kind)` moves the blocks of that
    level/kind in (and out).  Returns (i_re, i_im) of the rank's sorted point
    interval."""
    D = plan.depth
    pb, pe = layout.points(rank)
    plan.set_density(a_re, a_im)
    plan.zero_result()
    plan.singular_pass(pb, pe)
    qb, qe = layout.cones(D, rank)
    plan.level_d_pass(qb, qe)
    if D > 3:
        exchange(D, PROP)
    for d in range(D, 2, -1):
        exchange(d, INTERP)
        if d > 3:
            qb, qe = layout.cones(d - 1, rank)
            plan.propagation_pass(d, qb, qe)
            if d > 4:
                exchange(d - 1, PROP)
        plan.interpolation_pass(d, pb, pe)
    i_re, i_im = plan.read_result(sorted_order=True)
    return i_re[pb:pe], i_im[pb:pe]


class DistributedPlan:
    """One plan per rank (this process's GPU); apply() returns the full
    result in the caller's order on every rank.  Every rank builds the same
    plan (setup is cheap on the GPU); each rank computes only its own
    exchange sets and learns its send sets with one all-to-all per level and
    kind (build_exchange_plan_rank)."""

    def __init__(self, x1, x2, x3, cfg, params=None, group=None, partition: int = 0):
        import torch
        import torch.distributed as dist

        from .engine import EngineParams, Plan
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.device("cuda", torch.cuda.current_device())
        # NCCL moves device tensors; gloo (CPU tests, shared-GPU checks) host ones
        self.wire = self.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
        p = params or EngineParams()
        p.device = torch.cuda.current_device()
        self.plan = Plan(x1, x2, x3, cfg, p)
        self.plan.set_partition(partition)
        self.layout = rank_layout(self.plan, self.world)
        self.ex = build_exchange_plan_rank(
            self.layout, self.plan.depth, self.rank,
            lambda d, kind: self.plan.exchange_set(self.world, self.rank, d, kind),
            group=group, device=self.wire)
        self.store = PlanStore(self.plan)
        self.xch = TorchExchanger(self.store, self.ex, self.rank, self.device, group,
                                  wire=self.wire)
        self.perm = self.plan.perm()

    def apply(self, a_re, a_im=None):
        torch = self.torch
        a_im = np.zeros_like(a_re) if a_im is None else a_im
        part = run_rank_share(self.plan, self.layout, self.rank, a_re, a_im, self.xch.exchange)
        n = self.plan.n
        m = int(np.max(np.diff(self.layout.point_begin)))
        mine = torch.zeros((2, m), dtype=torch.float64, device=self.wire)
        mine[0, :len(part[0])] = torch.as_tensor(part[0], device=self.wire)
        mine[1, :len(part[1])] = torch.as_tensor(part[1], device=self.wire)
        pieces = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(pieces, mine, group=self.group)
        s_re, s_im = np.zeros(n), np.zeros(n)
        for r in range(self.world):
            b, e = self.layout.points(r)
            pr = pieces[r].cpu().numpy()
            s_re[b:e] = pr[0, :e - b]
            s_im[b:e] = pr[1, :e - b]
        i_re, i_im = np.zeros(n), np.zeros(n)
        i_re[self.perm] = s_re
        i_im[self.perm] = s_im
        return i_re, i_im

    def close(self):
        self.plan.close()


def simulate(plans, a_re, a_im, partition: int = 0, rank_seconds=None):
    """R ranks in one process (one plan each, all on the same GPU), blocks
    moved plan to plan through pack/unpack -- the reference's in-process rank
    simulation (dist.cpp) on real kernels.  Ranks advance phase by phase, so
    no kernel ever waits on another rank's kernel.  Returns the full result
    in the caller's order and the number of blocks moved.  `partition`:
    Plan.PARTITION_COUNT (the reference's layout) or Plan.PARTITION_WORK.
    `rank_seconds` (a list): filled with each rank's compute time (its passes,
    synchronised one by one -- exchanges excluded), the load-balance measure."""
    import torch

    R = len(plans)
    for p in plans:
        p.set_partition(partition)
    layout = rank_layout(plans[0], R)
    ex = build_exchange_plan(layout, plans[0].depth,
                             lambda r, d, kind: plans[0].exchange_set(R, r, d, kind))
    stores = [PlanStore(p) for p in plans]
    bd = stores[0].block_doubles
    dev = torch.device("cuda", torch.cuda.current_device())
    moved = [0]

    def exchange_all(d, kind):
        key = (d, kind)
        if key not in ex.recv:
            return
        for r in range(R):
            for p in range(R):
                a = ex.recv[key][r][p]
                if not len(a):
                    continue
                idx = torch.as_tensor(a.astype(np.int32), device=dev)
                buf = torch.empty(len(a) * bd, dtype=torch.float64, device=dev)
                stores[p].pack(d, idx, buf)
                torch.cuda.synchronize()
                stores[r].unpack(d, idx, buf)
                torch.cuda.synchronize()
                moved[0] += len(a)

    secs = [0.0] * R

    def run(r, fn, *args):
        if rank_seconds is None:
            return fn(*args)
        import time
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(*args)
        torch.cuda.synchronize()
        secs[r] += time.perf_counter() - t0

    D = plans[0].depth
    for r in range(R):
        pb, pe = layout.points(r)
        plans[r].set_density(a_re, a_im)
        plans[r].zero_result()
        run(r, plans[r].singular_pass, pb, pe)
        run(r, plans[r].level_d_pass, *layout.cones(D, r))
    if D > 3:
        exchange_all(D, PROP)
    for d in range(D, 2, -1):
        exchange_all(d, INTERP)
        if d > 3:
            for r in range(R):
                run(r, plans[r].propagation_pass, d, *layout.cones(d - 1, r))
            if d > 4:
                exchange_all(d - 1, PROP)
        for r in range(R):
            run(r, plans[r].interpolation_pass, d, *layout.points(r))
    if rank_seconds is not None:
        rank_seconds[:] = secs
    n = plans[0].n
    s_re, s_im = np.zeros(n), np.zeros(n)
    for r in range(R):
        b, e = layout.points(r)
        g_re, g_im = plans[r].read_result(sorted_order=True)
        s_re[b:e], s_im[b:e] = g_re[b:e], g_im[b:e]
    perm = plans[0].perm()
    i_re, i_im = np.zeros(n), np.zeros(n)
    i_re[perm], i_im[perm] = s_re, s_im
    return i_re, i_im, moved[0], ex
