"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``COracle`` -- oracle/liboracle.so, our plain-C restatement (ifgf_oracle.c).
* ``RefOracle`` -- oracle/_ref/libifgf_ref.so, the unmodified reference
  library compiled from /root/reference by oracle/Makefile plus ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.  The product (paper_2112_15198_b200) never does.
Both classes expose the same methods so tests can run one check against
either checker.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libifgf_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


@dataclass
class Params:
    """Mirror of ifgf::EngineParams (engine.hpp:12-19)."""
    depth: int = 0
    box_lambda: float = 0.25
    points_per_box: int = 64
    base_s: int = 1
    base_theta: int = 2
    base_phi: int = 4
    p_s: int = 3
    p_theta: int = 5
    p_phi: int = 5
    threads: int = 1

    def ip(self):
        return (C.c_int * 9)(self.depth, self.points_per_box, self.base_s, self.base_theta,
                             self.base_phi, self.p_s, self.p_theta, self.p_phi, self.threads)

    @property
    def P(self):
        return self.p_s * self.p_theta * self.p_phi


class _OcParams(C.Structure):
    _fields_ = [("depth", C.c_int), ("box_lambda", C.c_double), ("points_per_box", C.c_int),
                ("base_s", C.c_int), ("base_theta", C.c_int), ("base_phi", C.c_int),
                ("p_s", C.c_int), ("p_theta", C.c_int), ("p_phi", C.c_int)]

    @classmethod
    def of(cls, p: Params):
        return cls(p.depth, p.box_lambda, p.points_per_box, p.base_s, p.base_theta,
                   p.base_phi, p.p_s, p.p_theta, p.p_phi)


class _OcReport(C.Structure):
    _fields_ = [("seconds", C.c_double * 6), ("depth", C.c_int),
                ("peak_live_blocks", C.c_size_t)]


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


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


class _Problem:
    """Sorted problem + structure + passes, common to both checkers."""

    def __init__(self, lib, handle, n, prefix, P):
        self._lib, self._h, self.n, self._p, self.P = lib, handle, n, prefix, P

    def __del__(self):
        try:
            getattr(self._lib, self._p + "problem_free")(self._h)
        except Exception:
            pass

    def _f(self, name):
        return getattr(self._lib, self._p + name)

    @property
    def depth(self):
        return self._f("problem_depth")(self._h)

    def cube(self):
        o = np.zeros(4)
        self._f("problem_cube")(self._h, o)
        return o

    def sorted(self):
        n = self.n
        perm = np.zeros(n, np.uint32)
        arrs = [np.zeros(n) for _ in range(5)]
        self._f("problem_sorted")(self._h, perm, *arrs)
        return perm, arrs

    def level(self, d) -> LevelStructure:
        s = np.zeros(5, np.uint64)
        h = C.c_double(0.0)
        if self._p == "oc_":
            self._f("problem_level_sizes")(self._h, d, s, C.byref(h))
            hval = h.value
        else:
            self._f("problem_level_sizes")(self._h, d, s)
            hval = s[4:5].view(np.float64)[0]
        nb, nc, nn, ncs = (int(v) for v in s[:4])
        codes = np.zeros(nb, np.uint64)
        first = np.zeros(nb, np.uint32)
        count = np.zeros(nb, np.uint32)
        ctr = np.zeros(3 * nb)
        parent = np.zeros(nb, np.uint32)
        D = self.depth
        child = np.zeros(nb + 1, np.uint32) if d < D else None
        self._f("problem_level_boxes")(self._h, d, codes, first, count, ctr, parent,
                                       None if child is None else child.ctypes.data_as(C.c_void_p))
        nbr_off = np.zeros(nb + 1, np.uint32)
        nbr = np.zeros(max(nn, 1), np.uint32)
        coff = np.zeros(nb + 1, np.uint32)
        cous = np.zeros(max(ncs, 1), np.uint32)
        self._f("problem_level_adjacency")(self._h, d, nbr_off, nbr, coff, cous)
        cone_box = cone_gamma = bcb = None
        if d >= 3:
            cone_box = np.zeros(max(nc, 1), np.uint32)
            cone_gamma = np.zeros(max(nc, 1), np.uint64)
            bcb = np.zeros(nb + 1, np.uint32)
            self._f("problem_level_cones")(self._h, d, cone_box, cone_gamma, bcb)
            cone_box, cone_gamma = cone_box[:nc], cone_gamma[:nc]
        return LevelStructure(d, hval, codes, first, count, ctr.reshape(-1, 3), parent, child,
                              nbr_off, nbr[:nn], coff if d >= 3 else None,
                              cous[:ncs] if d >= 3 else None, cone_box, cone_gamma, bcb)

    def n_cones(self, d):
        s = np.zeros(5, np.uint64)
        if self._p == "oc_":
            self._f("problem_level_sizes")(self._h, d, s, None)
        else:
            self._f("problem_level_sizes")(self._h, d, s)
        return int(s[1])


class _Checker:
    prefix = ""

    def _check(self, rc):
        if rc != 0:
            raise CheckerError(rc, self.last_error())

    def last_error(self):
        return getattr(self.lib, self.prefix + "last_error")().decode()


class COracle(_Checker):
    """Our C restatement (oracle/ifgf_oracle.c)."""
    prefix = "oc_"
    kind = "port"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.oc_last_error.restype = C.c_char_p
        L.oc_mt64_first.restype = C.c_uint64
        L.oc_mt64_first.argtypes = [C.c_uint64, C.c_int]
        L.oc_generate.argtypes = [C.c_size_t, C.c_int, C.c_double, C.c_int, C.c_uint64] + [_dp] * 5
        L.oc_sincos_fast.argtypes = [C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.oc_morton_encode.restype = C.c_uint64
        L.oc_morton_encode.argtypes = [C.c_uint32] * 3
        L.oc_morton_decode.argtypes = [C.c_uint64, _u32p]
        L.oc_choose_depth.argtypes = [C.c_size_t, C.c_double, C.c_double, C.POINTER(_OcParams)]
        L.oc_cheb_fit.argtypes = [C.c_int] * 3 + [_dp] * 4
        L.oc_cheb_eval.argtypes = [C.c_int] * 3 + [_dp] * 2 + [C.c_double] * 3 + [
            C.POINTER(C.c_double)] * 2
        L.oc_cone_coords.argtypes = [_dp, C.c_double, _dp, _dp]
        L.oc_problem_build.argtypes = [C.c_size_t] + [_dp] * 5 + [
            C.c_int, C.c_double, C.POINTER(_OcParams), C.POINTER(C.c_void_p)]
        L.oc_problem_free.argtypes = [C.c_void_p]
        L.oc_problem_depth.argtypes = [C.c_void_p]
        L.oc_problem_cube.argtypes = [C.c_void_p, _dp]
        L.oc_problem_sorted.argtypes = [C.c_void_p, _u32p] + [_dp] * 5
        L.oc_problem_level_sizes.argtypes = [C.c_void_p, C.c_int, _u64p, C.c_void_p]
        L.oc_problem_level_boxes.argtypes = [C.c_void_p, C.c_int, _u64p, _u32p, _u32p, _dp, _u32p,
                                             C.c_void_p]
        L.oc_problem_level_adjacency.argtypes = [C.c_void_p, C.c_int] + [_u32p] * 4
        L.oc_problem_level_cones.argtypes = [C.c_void_p, C.c_int, _u32p, _u64p, _u32p]
        L.oc_singular_pass.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, _dp, _dp]
        L.oc_level_d_pass.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, _dp, _dp]
        L.oc_propagation_pass.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_uint32, C.c_uint32,
                                          _dp, _dp]
        L.oc_interpolation_pass.argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_size_t,
                                            C.c_size_t, _dp, _dp]
        L.oc_apply.argtypes = [C.c_size_t] + [_dp] * 5 + [C.c_int, C.c_double,
                                                           C.POINTER(_OcParams), _dp, _dp,
                                                           C.POINTER(_OcReport)]
        L.oc_apply_lean.argtypes = L.oc_apply.argtypes
        L.oc_direct_eval.argtypes = [C.c_size_t] + [_dp] * 5 + [C.c_int, C.c_double, C.c_void_p,
                                                                 C.c_size_t, _dp, _dp]
        L.oc_sample_indices.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, _u32p]
        L.oc_error_at_indices.argtypes = [C.c_size_t] + [_dp] * 7 + [
            C.c_int, C.c_double, _u32p, C.c_size_t, C.POINTER(C.c_double)]
        L.oc_partition.argtypes = [C.c_void_p, C.c_int, _u32p, _u32p, _u32p]
        L.oc_set_threads.argtypes = [C.c_int]
        L.oc_exchange_set.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                      C.POINTER(C.c_size_t)]

    # -- inputs
    def generate(self, n, shape=0, c=1.0, dens=0, seed=1):
        arrs = [np.zeros(n) for _ in range(5)]
        self._check(self.lib.oc_generate(n, shape, c, dens, seed, *arrs))
        return arrs

    def mt64(self, seed, k):
        return self.lib.oc_mt64_first(seed, k)

    def sincos_fast(self, x):
        s, c = C.c_double(), C.c_double()
        self.lib.oc_sincos_fast(x, C.byref(s), C.byref(c))
        return s.value, c.value

    def choose_depth(self, n, side, kappa, p: Params):
        return self.lib.oc_choose_depth(n, side, kappa, C.byref(_OcParams.of(p)))

    def cheb_fit(self, ps, pt, pp, vre, vim):
        cre, cim = np.zeros(ps * pt * pp), np.zeros(ps * pt * pp)
        self.lib.oc_cheb_fit(ps, pt, pp, _c(vre), _c(vim), cre, cim)
        return cre, cim

    def cheb_eval(self, ps, pt, pp, cre, cim, ts, tt, tp):
        r, i = C.c_double(), C.c_double()
        self.lib.oc_cheb_eval(ps, pt, pp, _c(cre), _c(cim), ts, tt, tp, C.byref(r), C.byref(i))
        return complex(r.value, i.value)

    # -- operator
    def apply(self, x1, x2, x3, ar, ai, kind, k, p: Params):
        n = len(x1)
        ir, ii = np.zeros(n), np.zeros(n)
        rep = _OcReport()
        self.lib.oc_set_threads(max(1, p.threads))
        self._check(self.lib.oc_apply(n, _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind, k,
                                      C.byref(_OcParams.of(p)), ir, ii, C.byref(rep)))
        return ir, ii, {"seconds": list(rep.seconds), "depth": rep.depth,
                        "peak_live_blocks": rep.peak_live_blocks}

    def apply_lean(self, x1, x2, x3, ar, ai, kind, k, p: Params):
        """oc_apply_lean: depth-first, O(depth) live blocks (C5 in a few GB)."""
        n = len(x1)
        ir, ii = np.zeros(n), np.zeros(n)
        rep = _OcReport()
        self.lib.oc_set_threads(max(1, p.threads))
        self._check(self.lib.oc_apply_lean(n, _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind, k,
                                           C.byref(_OcParams.of(p)), ir, ii, C.byref(rep)))
        return ir, ii, {"seconds": list(rep.seconds), "depth": rep.depth,
                        "peak_live_blocks": rep.peak_live_blocks}

    def direct(self, x1, x2, x3, ar, ai, kind, k, targets=None, threads=1):
        n = len(x1)
        m = n if targets is None else len(targets)
        self.lib.oc_set_threads(max(1, threads))
        o_re, o_im = np.zeros(m), np.zeros(m)
        tp = None if targets is None else _c(targets, np.uint32)
        self._check(self.lib.oc_direct_eval(
            n, _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind, k,
            None if tp is None else tp.ctypes.data_as(C.c_void_p), m, o_re, o_im))
        return o_re, o_im

    def sample_indices(self, n, m, seed):
        out = np.zeros(m, np.uint32)
        self._check(self.lib.oc_sample_indices(n, m, seed, out))
        return out

    def error_at_indices(self, x1, x2, x3, ar, ai, ir, ii, kind, k, idx):
        e = C.c_double()
        self._check(self.lib.oc_error_at_indices(len(x1), _c(x1), _c(x2), _c(x3), _c(ar), _c(ai),
                                                 _c(ir), _c(ii), kind, k,
                                                 _c(idx, np.uint32), len(idx), C.byref(e)))
        return e.value

    # -- problem
    def problem(self, x1, x2, x3, ar, ai, kind, k, p: Params):
        h = C.c_void_p()
        self._check(self.lib.oc_problem_build(len(x1), _c(x1), _c(x2), _c(x3), _c(ar), _c(ai),
                                              kind, k, C.byref(_OcParams.of(p)), C.byref(h)))
        return _OcProblem(self, h, len(x1), p)


class _OcProblem(_Problem):
    def __init__(self, chk, h, n, p):
        super().__init__(chk.lib, h, n, "oc_", p.P)
        self._chk = chk

    def singular(self):
        ir, ii = np.zeros(self.n), np.zeros(self.n)
        self._chk._check(self._lib.oc_singular_pass(self._h, 0, self.n, ir, ii))
        return ir, ii

    def level_d(self):
        nc = self.n_cones(self.depth)
        br, bi = np.zeros(nc * self.P + 1), np.zeros(nc * self.P + 1)
        self._chk._check(self._lib.oc_level_d_pass(self._h, 0, nc, br, bi))
        return br[:-1].reshape(nc, self.P), bi[:-1].reshape(nc, self.P)

    def propagation(self, d, cre, cim):
        npar = self.n_cones(d - 1)
        pr, pi = np.zeros(npar * self.P + 1), np.zeros(npar * self.P + 1)
        self._chk._check(self._lib.oc_propagation_pass(self._h, d, _c(cre).ravel(),
                                                       _c(cim).ravel(), 0, npar, pr, pi))
        return pr[:-1].reshape(npar, self.P), pi[:-1].reshape(npar, self.P)

    def interpolation(self, d, bre, bim):
        ir, ii = np.zeros(self.n), np.zeros(self.n)
        self._chk._check(self._lib.oc_interpolation_pass(self._h, d, _c(bre).ravel(),
                                                         _c(bim).ravel(), 0, self.n, ir, ii))
        return ir, ii

    def partition(self, R):
        D = self.depth
        bb, pb = np.zeros(R + 1, np.uint32), np.zeros(R + 1, np.uint32)
        cb = np.zeros((D - 2) * (R + 1), np.uint32)
        self._chk._check(self._lib.oc_partition(self._h, R, bb, pb, cb))
        return bb, pb, cb.reshape(D - 2, R + 1)

    def exchange_set(self, R, rank, d, kind):
        cnt = C.c_size_t()
        self._chk._check(self._lib.oc_exchange_set(self._h, R, rank, d, kind, None,
                                                   C.byref(cnt)))
        out = np.zeros(max(cnt.value, 1), np.uint32)
        self._chk._check(self._lib.oc_exchange_set(self._h, R, rank, d, kind,
                                                   out.ctypes.data_as(C.c_void_p),
                                                   C.byref(cnt)))
        return out[:cnt.value]


class RefOracle(_Checker):
    """The unmodified reference library (oracle/_ref/libifgf_ref.so)."""
    prefix = "ref_"
    kind = "reference"

    def __init__(self, path=REF_SO, simd="avx2"):
        self.path = path
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        os.environ.setdefault("IFGF_SIMD", simd)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_simd_variant.restype = C.c_char_p
        L.ref_choose_depth.argtypes = [C.c_size_t, C.c_double, C.c_double, C.c_void_p,
                                       C.c_double, C.POINTER(C.c_int)]
        L.ref_apply.argtypes = [C.c_size_t] + [_dp] * 5 + [
            C.c_int, C.c_double, C.c_void_p, C.c_double, _dp, _dp, _dp,
            C.POINTER(C.c_int), C.POINTER(C.c_size_t)]
        L.ref_run_distributed.argtypes = [C.c_size_t] + [_dp] * 5 + [
            C.c_int, C.c_double, C.c_void_p, C.c_double, C.c_int, _dp, _dp, _u64p,
            C.POINTER(C.c_int)]
        L.ref_generate_surface.argtypes = [C.c_int, C.c_double, C.c_int, C.c_uint64] + [_dp] * 5
        L.ref_checksum_hex.argtypes = [_dp, _dp, C.c_size_t, C.c_char_p]
        L.ref_checksum_hex.restype = None
        L.ref_write_points_binary.argtypes = [C.c_char_p, C.c_size_t] + [_dp] * 5
        L.ref_direct_eval.argtypes = [C.c_size_t] + [_dp] * 5 + [C.c_int, C.c_double, C.c_int,
                                                                  _dp, _dp]
        L.ref_sample_indices.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, _u32p]
        L.ref_error_at_indices.argtypes = [C.c_size_t] + [_dp] * 7 + [
            C.c_int, C.c_double, _u32p, C.c_size_t, C.c_int, C.POINTER(C.c_double)]
        L.ref_problem_build.restype = C.c_void_p
        L.ref_problem_build.argtypes = [C.c_size_t] + [_dp] * 5 + [C.c_int, C.c_double,
                                                                    C.c_void_p, C.c_double]
        L.ref_problem_free.argtypes = [C.c_void_p]
        L.ref_problem_depth.argtypes = [C.c_void_p]
        L.ref_problem_cube.argtypes = [C.c_void_p, _dp]
        L.ref_problem_sorted.argtypes = [C.c_void_p, _u32p] + [_dp] * 5
        L.ref_problem_level_sizes.argtypes = [C.c_void_p, C.c_int, _u64p]
        L.ref_problem_level_boxes.argtypes = [C.c_void_p, C.c_int, _u64p, _u32p, _u32p, _dp,
                                              _u32p, C.c_void_p]
        L.ref_problem_level_adjacency.argtypes = [C.c_void_p, C.c_int] + [_u32p] * 4
        L.ref_problem_level_cones.argtypes = [C.c_void_p, C.c_int, _u32p, _u64p, _u32p]
        L.ref_problem_singular.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_int, _dp, _dp]
        L.ref_problem_level_d.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.ref_problem_propagation.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_problem_interpolation.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_problem_partition.argtypes = [C.c_void_p, C.c_int, _u32p, _u32p, _u32p]
        L.ref_bench_open.restype = C.c_void_p
        L.ref_bench_open.argtypes = [C.c_void_p]
        L.ref_bench_close.argtypes = [C.c_void_p]
        L.ref_bench_slice.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp]

    def variant(self):
        return self.lib.ref_simd_variant().decode()

    def choose_depth(self, n, side, kappa, p: Params):
        out = C.c_int()
        self._check(self.lib.ref_choose_depth(n, side, kappa, p.ip(), p.box_lambda,
                                              C.byref(out)))
        return out.value

    def apply(self, x1, x2, x3, ar, ai, kind, k, p: Params):
        n = len(x1)
        ir, ii = np.zeros(n), np.zeros(n)
        secs = np.zeros(6)
        depth, peak = C.c_int(), C.c_size_t()
        self._check(self.lib.ref_apply(n, _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind, k,
                                       p.ip(), p.box_lambda, ir, ii, secs, C.byref(depth),
                                       C.byref(peak)))
        return ir, ii, {"seconds": secs.tolist(), "depth": depth.value,
                        "peak_live_blocks": peak.value}

    def run_distributed(self, x1, x2, x3, ar, ai, kind, k, p: Params, ranks):
        n = len(x1)
        ir, ii = np.zeros(n), np.zeros(n)
        comm = np.zeros(7 * 22, np.uint64)
        nl = C.c_int()
        self._check(self.lib.ref_run_distributed(n, _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind,
                                                 k, p.ip(), p.box_lambda, ranks, ir, ii, comm,
                                                 C.byref(nl)))
        return ir, ii, comm[:7 * nl.value].reshape(nl.value, 7)

    def direct(self, x1, x2, x3, ar, ai, kind, k, threads=0):
        n = len(x1)
        o_re, o_im = np.zeros(n), np.zeros(n)
        self._check(self.lib.ref_direct_eval(n, _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind, k,
                                             threads, o_re, o_im))
        return o_re, o_im

    def sample_indices(self, n, m, seed):
        out = np.zeros(m, np.uint32)
        self._check(self.lib.ref_sample_indices(n, m, seed, out))
        return out

    # harness: geometry.cpp:57-93, 147-226; bench.cpp:26-41
    def generate_surface(self, shape, a, npd, seed):
        m = 6 * npd * npd
        arrs = [np.zeros(m) for _ in range(5)]
        self._check(self.lib.ref_generate_surface(shape, C.c_double(a), npd, C.c_uint64(seed),
                                                  *arrs))
        return arrs

    def checksum_hex(self, re, im):
        out = C.create_string_buffer(17)
        self.lib.ref_checksum_hex(_c(re), _c(im), C.c_size_t(len(re)), out)
        return out.value.decode()

    def write_points_binary(self, path, x1, x2, x3, ar, ai):
        self._check(self.lib.ref_write_points_binary(str(path).encode(), C.c_size_t(len(x1)),
                                                     _c(x1), _c(x2), _c(x3), _c(ar), _c(ai)))

    def read_points(self, path):
        """The reference's read_points, run out of process (oracle/_ref/
        ref_read_points): its iostream CSV parsing crashes inside this
        process.  Returns the five arrays, or raises RuntimeError(what)."""
        import subprocess
        exe = os.path.join(os.path.dirname(self.path), "ref_read_points")
        out = subprocess.run([exe, str(path)], capture_output=True, text=True).stdout
        if out.startswith("error: "):
            raise RuntimeError(out[7:].strip())
        lines = out.splitlines()
        n = int(lines[0])
        a = np.array([[float(v) for v in ln.split()] for ln in lines[1:1 + n]]).reshape(n, 5)
        return [a[:, k].copy() for k in range(5)]

    def error_at_indices(self, x1, x2, x3, ar, ai, ir, ii, kind, k, idx, threads=0):
        e = C.c_double()
        self._check(self.lib.ref_error_at_indices(len(x1), _c(x1), _c(x2), _c(x3), _c(ar),
                                                  _c(ai), _c(ir), _c(ii), kind, k,
                                                  _c(idx, np.uint32), len(idx), threads,
                                                  C.byref(e)))
        return e.value

    def problem(self, x1, x2, x3, ar, ai, kind, k, p: Params):
        h = self.lib.ref_problem_build(len(x1), _c(x1), _c(x2), _c(x3), _c(ar), _c(ai), kind, k,
                                       p.ip(), p.box_lambda)
        if not h:
            raise CheckerError(-1, self.last_error())
        return _RefProblem(self, h, len(x1), p)


class _RefProblem(_Problem):
    def __init__(self, chk, h, n, p):
        super().__init__(chk.lib, C.c_void_p(h), n, "ref_", p.P)
        self._chk = chk
        self._threads = p.threads

    def bench(self):
        """Handle for bench.py's reference leg: the stock passes of apply()
        on this Problem in S slices (oracle/ref_shim.cpp ref_bench_slice)."""
        return _RefBench(self)

    def singular(self):
        ir, ii = np.zeros(self.n), np.zeros(self.n)
        self._chk._check(self._lib.ref_problem_singular(self._h, 0, self.n, self._threads, ir, ii))
        return ir, ii

    def level_d(self):
        nc = self.n_cones(self.depth)
        br, bi = np.zeros(nc * self.P + 1), np.zeros(nc * self.P + 1)
        self._chk._check(self._lib.ref_problem_level_d(self._h, self._threads, br, bi))
        return br[:-1].reshape(nc, self.P), bi[:-1].reshape(nc, self.P)

    def propagation(self, d, cre, cim):
        npar = self.n_cones(d - 1)
        pr, pi = np.zeros(npar * self.P + 1), np.zeros(npar * self.P + 1)
        self._chk._check(self._lib.ref_problem_propagation(
            self._h, d, self._threads, _c(cre).ravel(), _c(cim).ravel(), pr, pi))
        return pr[:-1].reshape(npar, self.P), pi[:-1].reshape(npar, self.P)

    def interpolation(self, d, bre, bim):
        ir, ii = np.zeros(self.n), np.zeros(self.n)
        self._chk._check(self._lib.ref_problem_interpolation(
            self._h, d, self._threads, _c(bre).ravel(), _c(bim).ravel(), ir, ii))
        return ir, ii

    def partition(self, R):
        D = self.depth
        bb, pb = np.zeros(R + 1, np.uint32), np.zeros(R + 1, np.uint32)
        cb = np.zeros((D - 2) * (R + 1), np.uint32)
        self._chk._check(self._lib.ref_problem_partition(self._h, R, bb, pb, cb))
        return bb, pb, cb.reshape(D - 2, R + 1)


class _RefBench:
    def __init__(self, prob):
        self._prob = prob  # keeps the Problem alive
        self._lib = prob._lib
        h = self._lib.ref_bench_open(prob._h)
        if not h:
            raise CheckerError(-1, prob._chk.last_error())
        self._h = C.c_void_p(h)

    def slice(self, threads, k, S):
        """Slice k of S of every pass; returns {singular, level_d, interpolation,
        propagation} seconds."""
        secs = np.zeros(4)
        self._prob._chk._check(self._lib.ref_bench_slice(self._h, threads, k, S, secs))
        return dict(zip(("singular", "level_d", "interpolation", "propagation"), secs.tolist()))

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.ref_bench_close(self._h)
            self._h = None


def rel_l2(got_re, got_im, want_re, want_im):
    num = np.sum((got_re - want_re) ** 2 + (got_im - want_im) ** 2)
    den = np.sum(want_re ** 2 + want_im ** 2)
    return float(np.sqrt(num / den))
