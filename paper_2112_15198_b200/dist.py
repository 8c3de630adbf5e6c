"""Multi-GPU IFGF matvec: the reference's rank algorithm (dist.cpp:241-361,
the paper's "IFGF Method" in MPI form) on the C++ engine of libifgf_b200.so
(csrc/dist.cu, include/ifgf_b200.h "multi-GPU").

* Layout (dist.cpp:78-130): points in contiguous Morton intervals of level-D
  boxes balanced by population; each level's cones in equal-count intervals
  of the (box, gamma) order -- boxes at fine levels, cone segments at coarse
  levels.  The structure is built on every rank; the interpolant blocks are
  partitioned: a rank stores its owned cones plus its halo (the foreign cones
  its points and parent cones read, dist.cpp:179-237).
* Transport: per level, the owners pack the requested blocks on the device
  and one NCCL group of send/recv moves them (one process per GPU,
  Comm/DistPlan); in-process rank groups (run_distributed, the analogue of
  dist::run_distributed) move them with device copies.

This module is the host-side mirror: ctypes wrappers over the C ABI, plus the
rank layout and exchange lists as host data (Layout, build_exchange_plan)
that the CLI's CommStats and the CPU tests use.
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




def rank_layout(plan, n_ranks) -> Layout:
    bb, pb, cb = plan.partition(n_ranks)
    return Layout(n_ranks, bb, pb, cb)


# ---------------------------------------------------------------- C ABI mirror
def _engine():
    from . import _lib, engine
    return _lib, engine


@dataclass
class RankInfo:
    """ifgf_dist_info: one rank's share of a multi-GPU plan."""
    rank: int
    world: int
    point_begin: int
    point_end: int
    levels: list  # per d = 3..D: dict(owned_cones, halo_cones, interp_needed, prop_needed, sent_cones)
    block_bytes: int
    device_bytes: int
    compute_seconds: float = 0.0  # with IFGF_DIST_RANK_TIMING=1 (run_distributed)

    @classmethod
    def from_c(cls, c, depth):
        lv = [{f: int(getattr(c.levels[d - 3], f)) for f in
               ("owned_cones", "halo_cones", "interp_needed", "prop_needed", "sent_cones")}
              | {"d": d} for d in range(3, depth + 1)]
        return cls(c.rank, c.world, int(c.point_begin), int(c.point_end), lv,
                   int(c.block_bytes), int(c.device_bytes), float(c.compute_seconds))


def run_distributed(pc, cfg, p=None, n_ranks: int = 2, devices=None):
    """dist::run_distributed (dist.hpp:90) on the GPU: n_ranks rank plans in
    this process (devices[r], default all on p.device), blocks exchanged
    rank to rank.  Fills pc.i_re / pc.i_im (caller's order, bitwise equal to
    apply()) and returns (ApplyReport, [RankInfo])."""
    import ctypes as C
    _lib, engine = _engine()
    p = p or engine.EngineParams()
    devs = None
    if devices is not None:
        devs = (C.c_int * n_ranks)(*[int(v) for v in devices])
    rep = _lib.CReport()
    infos = (_lib.CDistInfo * n_ranks)()
    a_im = pc.a_im
    engine.check(_lib.lib.ifgf_run_distributed(
        pc.size(), _lib.ptr(pc.x1), _lib.ptr(pc.x2), _lib.ptr(pc.x3), _lib.ptr(pc.a_re),
        _lib.ptr(a_im), int(cfg.kind), float(cfg.wavenumber), C.byref(p.c()), n_ranks, devs,
        _lib.ptr(pc.i_re), _lib.ptr(pc.i_im), C.byref(rep), C.cast(infos, C.c_void_p)))
    r = engine.ApplyReport.from_c(rep)
    return r, [RankInfo.from_c(infos[k], r.depth) for k in range(n_ranks)]


class Comm:
    """A rank's handle of a multi-process group (ifgf_comm): one process per
    GPU, NCCL over NVLink/NVSwitch.  Rank 0 makes the id (unique_id()), the
    launcher broadcasts it (share_comm_id below), every rank constructs."""

    def __init__(self, comm_id: bytes, rank: int, world: int, device: int):
        import ctypes as C
        _lib, engine = _engine()
        self._lib = _lib
        self.rank, self.world, self.device = rank, world, device
        buf = C.create_string_buffer(bytes(comm_id), _lib.COMM_ID_BYTES)
        h = C.c_void_p()
        engine.check(_lib.lib.ifgf_comm_create(buf, rank, world, device, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        _lib, engine = _engine()
        buf = C.create_string_buffer(_lib.COMM_ID_BYTES)
        engine.check(_lib.lib.ifgf_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lib.ifgf_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class DistPlan:
    """One rank's plan of a multi-process group (collective create / apply)."""

    def __init__(self, comm: Comm, x1_ptr: int, x2_ptr: int, x3_ptr: int, n: int, cfg, p=None,
                 stream: int = 0):
        import ctypes as C
        _lib, engine = _engine()
        self._lib, self._engine = _lib, engine
        p = p or engine.EngineParams()
        h = C.c_void_p()
        engine.check(_lib.lib.ifgf_dist_plan_create_device(
            comm._h, C.c_void_p(x1_ptr), C.c_void_p(x2_ptr), C.c_void_p(x3_ptr), n,
            int(cfg.kind), float(cfg.wavenumber), C.byref(p.c()), C.c_void_p(stream),
            C.byref(h)))
        self._h = h
        self.n = n
        self.comm = comm

    def apply_device(self, a_re_ptr: int, a_im_ptr, i_re_ptr: int, i_im_ptr: int,
                     stream: int = 0):
        import ctypes as C
        rep = self._lib.CReport()
        self._engine.check(self._lib.lib.ifgf_dist_plan_apply_device(
            self._h, C.c_void_p(a_re_ptr), C.c_void_p(a_im_ptr) if a_im_ptr else None,
            C.c_void_p(i_re_ptr), C.c_void_p(i_im_ptr), C.c_void_p(stream), C.byref(rep)))
        return self._engine.ApplyReport.from_c(rep)

    def info(self) -> RankInfo:
        import ctypes as C
        c = self._lib.CDistInfo()
        self._engine.check(self._lib.lib.ifgf_dist_plan_info(self._h, C.byref(c)))
        return RankInfo.from_c(c, c.depth)

    def plan_info(self):
        import ctypes as C
        c = self._lib.CPlanInfo()
        self._engine.check(self._lib.lib.ifgf_plan_get_info(self._h, C.byref(c)))
        return c

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lib.ifgf_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def share_comm_id(make_id, group=None) -> bytes:
    """The launcher side of Comm: rank 0 calls make_id() (Comm.unique_id),
    every rank of the torch.distributed group receives the same bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def max_over_ranks(value: float, group=None, device=None) -> float:
    """The slowest rank's time (bench timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
