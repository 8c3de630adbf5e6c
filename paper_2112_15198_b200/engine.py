"""Host-side mirror of the reference operator interface (include/ifgf/*.hpp in
/root/reference/proj), backed by libifgf_b200.so.

Names, argument meaning and error behaviour follow the reference:

  KernelKind / KernelConfig          kernel.hpp:13-25
  InterpOrders                       interp.hpp:11-25
  EngineParams                       engine.hpp:12-19  (`threads` kept, `device` added)
  PointCloud                         geometry.hpp:14-27
  StageSeconds / LevelInfo /
  ApplyReport                        engine.hpp:23-42
  choose_depth                       engine.hpp:21
  apply                              engine.hpp:112-114
  Plan (Problem::build + passes)     engine.hpp:46-110
  direct_eval / sample_indices /
  error_at_indices / estimate_error  engine.hpp:117-128

Exceptions map the reference's classes: InvalidArgument (std::invalid_argument),
DomainError (std::domain_error), LogicError (std::logic_error),
IFGFRuntimeError (std::runtime_error: CUDA / no device).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib, ptr


class IFGFError(Exception):
    code = -1


class InvalidArgument(IFGFError, ValueError):
    code = _lib.IFGF_EINVAL


class DomainError(IFGFError, ValueError):
    code = _lib.IFGF_EDOMAIN


class LogicError(IFGFError, RuntimeError):
    code = _lib.IFGF_ELOGIC


class IFGFRuntimeError(IFGFError, RuntimeError):
    code = _lib.IFGF_ERUNTIME


_ERR = {_lib.IFGF_EINVAL: InvalidArgument, _lib.IFGF_EDOMAIN: DomainError,
        _lib.IFGF_ELOGIC: LogicError, _lib.IFGF_ERUNTIME: IFGFRuntimeError}


def check(rc: int):
    if rc != 0:
        raise _ERR.get(rc, IFGFRuntimeError)(_lib.last_error())


class KernelKind(enum.IntEnum):
    Helmholtz = 0
    Laplace = 1


@dataclass
class KernelConfig:
    kind: KernelKind = KernelKind.Helmholtz
    wavenumber: float = 0.0

    def kappa(self) -> float:
        return 0.0 if self.kind == KernelKind.Laplace else float(self.wavenumber)

    def wavelength(self) -> float:
        k = self.kappa()
        return 2.0 * math.pi / k if k > 0.0 else 0.0


@dataclass
class InterpOrders:
    p_s: int = 3
    p_theta: int = 5
    p_phi: int = 5

    def total(self) -> int:
        return self.p_s * self.p_theta * self.p_phi

    def valid(self) -> bool:
        return all(1 <= p <= 12 for p in (self.p_s, self.p_theta, self.p_phi))


@dataclass
class EngineParams:
    depth: int = 0
    box_lambda: float = 0.25
    points_per_box: int = 64
    base_s: int = 1
    base_theta: int = 2
    base_phi: int = 4
    orders: InterpOrders = field(default_factory=InterpOrders)
    threads: int = 1  # accepted for API parity; the GPU ignores it
    device: int = 0
    partition: int = 0  # rank layout of multi-GPU plans (Plan.PARTITION_COUNT / _WORK)

    def c(self) -> _lib.CParams:
        o = self.orders
        return _lib.CParams(self.depth, self.box_lambda, self.points_per_box, self.base_s,
                            self.base_theta, self.base_phi, o.p_s, o.p_theta, o.p_phi,
                            self.device, self.partition)


@dataclass
class PointCloud:
    """SoA cloud (geometry.hpp:14-27): coordinates, densities, results."""
    x1: np.ndarray
    x2: np.ndarray
    x3: np.ndarray
    a_re: np.ndarray
    a_im: np.ndarray
    i_re: np.ndarray = None
    i_im: np.ndarray = None

    def __post_init__(self):
        for k in ("x1", "x2", "x3", "a_re", "a_im"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k), dtype=np.float64))
        n = self.size()
        if self.i_re is None:
            self.i_re = np.zeros(n)
        if self.i_im is None:
            self.i_im = np.zeros(n)

    def size(self) -> int:
        return len(self.x1)

    def copy(self) -> "PointCloud":
        return PointCloud(self.x1.copy(), self.x2.copy(), self.x3.copy(), self.a_re.copy(),
                          self.a_im.copy(), self.i_re.copy(), self.i_im.copy())


@dataclass
class StageSeconds:
    setup: float = 0.0
    singular: float = 0.0
    level_d: float = 0.0
    interpolation: float = 0.0
    propagation: float = 0.0
    total: float = 0.0


@dataclass
class LevelInfo:
    d: int
    boxes: int
    cones: int


@dataclass
class ApplyReport:
    seconds: StageSeconds
    depth: int
    n: int
    h_level_d: float
    levels: list
    peak_live_blocks: int
    simd_variant: str = "sm_100a"
    gpu_launches: int = 0

    @classmethod
    def from_c(cls, r: _lib.CReport) -> "ApplyReport":
        lv = [LevelInfo(3 + i, int(r.level_boxes[i]), int(r.level_cones[i]))
              for i in range(r.n_levels)]
        return cls(StageSeconds(r.setup, r.singular, r.level_d, r.interpolation, r.propagation,
                                r.total), r.depth, int(r.n), r.h_level_d, lv,
                   int(r.peak_live_blocks), "sm_100a", int(r.gpu_launches))


def default_params() -> EngineParams:
    return EngineParams()


def choose_depth(n: int, cube_side: float, kappa: float, p: EngineParams) -> int:
    out = C.c_int()
    check(lib.ifgf_choose_depth(n, cube_side, kappa, C.byref(p.c()), C.byref(out)))
    return out.value


def device_ok() -> bool:
    return bool(lib.ifgf_device_ok())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def apply(pc: PointCloud, cfg: KernelConfig, p: EngineParams | None = None) -> ApplyReport:
    """ifgf::apply (engine.cpp:260-325): rebuild, apply, results into
    pc.i_re / pc.i_im in the caller's order."""
    p = p or EngineParams()
    n = pc.size()
    rep = _lib.CReport()
    i_re, i_im = np.zeros(n), np.zeros(n)
    check(lib.ifgf_apply(n, ptr(pc.x1), ptr(pc.x2), ptr(pc.x3), ptr(pc.a_re), ptr(pc.a_im),
                         int(cfg.kind), float(cfg.wavenumber), C.byref(p.c()), ptr(i_re),
                         ptr(i_im), C.byref(rep)))
    pc.i_re, pc.i_im = i_re, i_im
    return ApplyReport.from_c(rep)


@dataclass
class LevelStructure:
    d: int
    h: float
    codes: np.ndarray
    first: np.ndarray
    count: np.ndarray
    centers: np.ndarray
    parent: np.ndarray
    child_begin: np.ndarray | None
    nbr_off: np.ndarray
    nbr: np.ndarray
    cousin_off: np.ndarray | None
    cousin: np.ndarray | None
    cone_box: np.ndarray | None
    cone_gamma: np.ndarray | None
    box_cone_begin: np.ndarray | None


class Plan:
    """Problem::build on the device + the operator and its passes.

    The plan owns the Morton-sorted cloud, the octree, the relevant cone
    sets and the block storage; apply() can be called repeatedly with new
    densities (the reference rebuilds per call, engine.cpp:267)."""

    def __init__(self, x1, x2, x3, cfg: KernelConfig, p: EngineParams | None = None):
        self.p = p or EngineParams()
        self.cfg = cfg
        x1, x2, x3 = _f64(x1), _f64(x2), _f64(x3)
        self.n = len(x1)
        h = C.c_void_p()
        check(lib.ifgf_plan_create(ptr(x1), ptr(x2), ptr(x3), self.n, int(cfg.kind),
                                   float(cfg.wavenumber), C.byref(self.p.c()), C.byref(h)))
        self._h = h
        self.info = self._info()

    @classmethod
    def from_cloud(cls, pc: PointCloud, cfg: KernelConfig, p: EngineParams | None = None):
        return cls(pc.x1, pc.x2, pc.x3, cfg, p)

    @classmethod
    def from_device(cls, x1_ptr: int, x2_ptr: int, x3_ptr: int, n: int, cfg: KernelConfig,
                    p: EngineParams | None = None, stream: int = 0):
        self = cls.__new__(cls)
        self.p = p or EngineParams()
        self.cfg = cfg
        self.n = n
        h = C.c_void_p()
        check(lib.ifgf_plan_create_device(C.c_void_p(x1_ptr), C.c_void_p(x2_ptr),
                                          C.c_void_p(x3_ptr), n, int(cfg.kind),
                                          float(cfg.wavenumber), C.byref(self.p.c()),
                                          C.c_void_p(stream), C.byref(h)))
        self._h = h
        self.info = self._info()
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib.ifgf_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_serial(self, on: bool = True):
        """Run all apply kernels on one stream (exclusive per-pass timings)."""
        check(lib.ifgf_plan_set_option(self._h, 1, 1 if on else 0))

    PROP_NODE, PROP_DMMA, PROP_ROWS, PROP_FLY, PROP_AUTO = 0, 2, 3, 4, 7

    NEAR_POINT, NEAR_BOX = 0, 1

    def set_option(self, option: int, value: int):
        """IFGF_OPT_* (include/ifgf_b200.h): 1 serial streams, 2 propagation
        kernel (PROP_NODE, PROP_DMMA, PROP_ROWS, PROP_FLY, PROP_AUTO default), 3 near-field kernel (NEAR_POINT, NEAR_BOX default),
        4 rank layout (PARTITION_COUNT default, PARTITION_WORK), 5 K4 reads the
        plan's locate records (default 1; 0 locates every pair again)."""
        check(lib.ifgf_plan_set_option(self._h, option, value))

    def set_k4_records(self, on: bool = True):
        """K4 from the plan's stored locate records (default, when the plan
        keeps them) or with a fresh locate per (point, cousin) pair; the
        results are bitwise equal."""
        self.set_option(5, 1 if on else 0)

    def set_prop_kernel(self, kind: int):
        self.set_option(2, kind)

    def set_near_kernel(self, kind: int):
        self.set_option(3, kind)

    PARTITION_COUNT, PARTITION_WORK = 0, 1

    def set_partition(self, mode: int):
        """Rank layout of partition()/exchange_set(): PARTITION_COUNT (the
        reference's, dist.cpp:90-128) or PARTITION_WORK (balanced by
        evaluation work)."""
        self.set_option(4, mode)

    def _info(self) -> _lib.CPlanInfo:
        info = _lib.CPlanInfo()
        check(lib.ifgf_plan_get_info(self._h, C.byref(info)))
        return info

    @property
    def depth(self) -> int:
        return self.info.depth

    @property
    def P(self) -> int:
        return self.info.P

    def cube(self):
        i = self.info
        return np.array([i.cube_origin[0], i.cube_origin[1], i.cube_origin[2], i.cube_side])

    def n_cones(self, d: int) -> int:
        return int(self.info.cones[d])

    def n_boxes(self, d: int) -> int:
        return int(self.info.boxes[d])

    # -- operator
    def apply(self, a_re, a_im=None):
        n = self.n
        a_re = _f64(a_re)
        a_im = None if a_im is None else _f64(a_im)
        i_re, i_im = np.zeros(n), np.zeros(n)
        rep = _lib.CReport()
        check(lib.ifgf_plan_apply(self._h, ptr(a_re), ptr(a_im), ptr(i_re), ptr(i_im),
                                  C.byref(rep)))
        return i_re, i_im, ApplyReport.from_c(rep)

    def apply_batch(self, a_re, a_im=None):
        """nrhs densities at once (rows of a [nrhs, n] array); returns
        (i_re, i_im) of shape [nrhs, n] and the report (ifgf_plan_apply_batch)."""
        a_re = np.ascontiguousarray(np.atleast_2d(a_re), dtype=np.float64)
        nrhs, n = a_re.shape
        if n != self.n:
            raise InvalidArgument("apply_batch: densities of the wrong length")
        a_im = None if a_im is None else np.ascontiguousarray(np.atleast_2d(a_im),
                                                               dtype=np.float64)
        i_re, i_im = np.zeros((nrhs, n)), np.zeros((nrhs, n))
        rep = _lib.CReport()
        check(lib.ifgf_plan_apply_batch(self._h, nrhs, ptr(a_re), ptr(a_im), ptr(i_re),
                                        ptr(i_im), C.byref(rep)))
        return i_re, i_im, ApplyReport.from_c(rep)

    def apply_batch_device(self, nrhs: int, a_re_ptr: int, a_im_ptr: int | None, i_re_ptr: int,
                           i_im_ptr: int, stream: int = 0) -> ApplyReport:
        rep = _lib.CReport()
        check(lib.ifgf_plan_apply_batch_device(self._h, nrhs, C.c_void_p(a_re_ptr),
                                               C.c_void_p(a_im_ptr) if a_im_ptr else None,
                                               C.c_void_p(i_re_ptr), C.c_void_p(i_im_ptr),
                                               C.c_void_p(stream), C.byref(rep)))
        return ApplyReport.from_c(rep)

    def apply_device(self, a_re_ptr: int, a_im_ptr: int | None, i_re_ptr: int, i_im_ptr: int,
                     stream: int = 0) -> ApplyReport:
        """Device pointers (e.g. torch tensor.data_ptr()), ordered on `stream`."""
        rep = _lib.CReport()
        check(lib.ifgf_plan_apply_device(self._h, C.c_void_p(a_re_ptr),
                                         C.c_void_p(a_im_ptr) if a_im_ptr else None,
                                         C.c_void_p(i_re_ptr), C.c_void_p(i_im_ptr),
                                         C.c_void_p(stream), C.byref(rep)))
        return ApplyReport.from_c(rep)

    # -- structure
    def perm(self) -> np.ndarray:
        out = np.zeros(self.n, np.uint32)
        check(lib.ifgf_plan_export_perm(self._h, ptr(out)))
        return out

    def level(self, d: int) -> LevelStructure:
        i = self.info
        nb = int(i.boxes[d])
        nn = int(i.nbr_entries[d])
        D = i.depth
        codes = np.zeros(nb, np.uint64)
        first = np.zeros(nb, np.uint32)
        count = np.zeros(nb, np.uint32)
        ctr = np.zeros(3 * nb)
        parent = np.zeros(nb, np.uint32)
        child = np.zeros(nb + 1, np.uint32) if d < D else None
        nbr_off = np.zeros(nb + 1, np.uint32)
        nbr = np.zeros(max(nn, 1), np.uint32)
        coff = cous = cb = cg = bcb = None
        if d >= 3:
            nc = int(i.cones[d])
            ncs = int(i.cousin_entries[d])
            coff = np.zeros(nb + 1, np.uint32)
            cous = np.zeros(max(ncs, 1), np.uint32)
            cb = np.zeros(max(nc, 1), np.uint32)
            cg = np.zeros(max(nc, 1), np.uint64)
            bcb = np.zeros(nb + 1, np.uint32)
        check(lib.ifgf_plan_export_level(self._h, d, ptr(codes), ptr(first), ptr(count),
                                         ptr(ctr), ptr(parent), ptr(child), ptr(nbr_off),
                                         ptr(nbr), ptr(coff), ptr(cous), ptr(cb), ptr(cg),
                                         ptr(bcb)))
        if d >= 3:
            cous, cb, cg = cous[:int(i.cousin_entries[d])], cb[:int(i.cones[d])], cg[:int(i.cones[d])]
        return LevelStructure(d, float(i.h[d]), codes, first, count, ctr.reshape(-1, 3), parent,
                              child, nbr_off, nbr[:nn], coff, cous, cb, cg, bcb)

    # -- passes (engine.hpp:91-110) on plan-owned device state
    def set_density(self, a_re, a_im=None):
        a_re = _f64(a_re)
        a_im = None if a_im is None else _f64(a_im)
        check(lib.ifgf_plan_set_density(self._h, ptr(a_re), ptr(a_im)))

    def zero_result(self):
        check(lib.ifgf_plan_zero_result(self._h))

    def singular_pass(self, b=0, e=None):
        check(lib.ifgf_plan_singular_pass(self._h, b, self.n if e is None else e))

    def level_d_pass(self, qb=0, qe=None):
        qe = self.n_cones(self.depth) if qe is None else qe
        check(lib.ifgf_plan_level_d_pass(self._h, qb, qe))

    def propagation_pass(self, d, qb=0, qe=None):
        qe = self.n_cones(d - 1) if qe is None else qe
        check(lib.ifgf_plan_propagation_pass(self._h, d, qb, qe))

    def interpolation_pass(self, d, b=0, e=None):
        check(lib.ifgf_plan_interpolation_pass(self._h, d, b, self.n if e is None else e))

    def read_blocks(self, d):
        cnt = self.n_cones(d) * self.P
        re, im = np.zeros(cnt + 1), np.zeros(cnt + 1)
        check(lib.ifgf_plan_read_blocks(self._h, d, ptr(re), ptr(im)))
        return re[:cnt].reshape(-1, self.P), im[:cnt].reshape(-1, self.P)

    def write_blocks(self, d, re, im):
        re, im = _f64(re).ravel(), _f64(im).ravel()
        if re.size != self.n_cones(d) * self.P or im.size != re.size:
            raise InvalidArgument("block array size mismatch")
        check(lib.ifgf_plan_write_blocks(self._h, d, ptr(re), ptr(im)))

    def read_result(self, sorted_order=False):
        i_re, i_im = np.zeros(self.n), np.zeros(self.n)
        check(lib.ifgf_plan_read_result(self._h, 1 if sorted_order else 0, ptr(i_re), ptr(i_im)))
        return i_re, i_im

    # -- ranks (dist.cpp:78-237)
    def partition(self, n_ranks: int):
        D = self.depth
        bb = np.zeros(n_ranks + 1, np.uint32)
        pb = np.zeros(n_ranks + 1, np.uint32)
        cb = np.zeros((D - 2) * (n_ranks + 1), np.uint32)
        check(lib.ifgf_plan_partition(self._h, n_ranks, ptr(bb), ptr(pb), ptr(cb)))
        return bb, pb, cb.reshape(D - 2, n_ranks + 1)

    def exchange_set(self, n_ranks: int, rank: int, d: int, kind: int) -> np.ndarray:
        cnt = C.c_size_t()
        check(lib.ifgf_plan_exchange_set(self._h, n_ranks, rank, d, kind, None, C.byref(cnt)))
        out = np.zeros(max(cnt.value, 1), np.uint32)
        check(lib.ifgf_plan_exchange_set(self._h, n_ranks, rank, d, kind, ptr(out),
                                         C.byref(cnt)))
        return out[:cnt.value]

    def pack_blocks(self, d, cones_dev_ptr, m, buf_dev_ptr, stream=0):
        check(lib.ifgf_plan_pack_blocks(self._h, d, C.c_void_p(cones_dev_ptr), m,
                                        C.c_void_p(buf_dev_ptr), C.c_void_p(stream)))

    def unpack_blocks(self, d, cones_dev_ptr, m, buf_dev_ptr, stream=0):
        check(lib.ifgf_plan_unpack_blocks(self._h, d, C.c_void_p(cones_dev_ptr), m,
                                          C.c_void_p(buf_dev_ptr), C.c_void_p(stream)))


def direct_eval(pc: PointCloud, cfg: KernelConfig, threads: int = 1, device: int = 0,
                targets=None):
    """ifgf::direct_eval (engine.cpp:327-339) on the device; with `targets`
    only those result slots are written."""
    n = pc.size()
    tg = None if targets is None else np.ascontiguousarray(targets, np.uint32)
    m = n if tg is None else len(tg)
    o_re, o_im = np.zeros(max(m, 1)), np.zeros(max(m, 1))
    check(lib.ifgf_direct_eval(n, ptr(pc.x1), ptr(pc.x2), ptr(pc.x3), ptr(pc.a_re),
                               ptr(pc.a_im), int(cfg.kind), float(cfg.wavenumber), ptr(tg), m,
                               device, ptr(o_re), ptr(o_im)))
    if tg is None:
        pc.i_re, pc.i_im = o_re[:n], o_im[:n]
    else:
        pc.i_re[tg] = o_re[:m]
        pc.i_im[tg] = o_im[:m]


def sample_indices(n: int, m: int, seed: int) -> np.ndarray:
    out = np.zeros(max(m, 1), np.uint32)
    check(lib.ifgf_sample_indices(n, m, seed, ptr(out)))
    return out[:m]


def error_at_indices(pc: PointCloud, cfg: KernelConfig, idx, threads: int = 1,
                     device: int = 0) -> float:
    idx = np.ascontiguousarray(idx, np.uint32)
    eps = C.c_double()
    check(lib.ifgf_error_at_indices(pc.size(), ptr(pc.x1), ptr(pc.x2), ptr(pc.x3), ptr(pc.a_re),
                                    ptr(pc.a_im), ptr(pc.i_re), ptr(pc.i_im), int(cfg.kind),
                                    float(cfg.wavenumber), ptr(idx), len(idx), device,
                                    C.byref(eps)))
    return eps.value


def estimate_error(pc: PointCloud, cfg: KernelConfig, m: int, seed: int, threads: int = 1,
                   device: int = 0) -> float:
    return error_at_indices(pc, cfg, sample_indices(pc.size(), m, seed), threads, device)


def generate(n: int, shape: int = 0, c: float = 1.0, dens: int = 0, seed: int = 1) -> PointCloud:
    """Seeded synthetic cloud: shape 0 unit sphere,
    1 spheroid (1,1,c); dens 0 complex U(-1,1), 1 real N(0,1)."""
    arrs = [np.zeros(n) for _ in range(5)]
    check(lib.ifgf_generate(n, shape, c, dens, seed, *(ptr(a) for a in arrs)))
    return PointCloud(*arrs)
