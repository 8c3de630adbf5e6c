"""`python -m paper_2112_15198_b200 {run,verify,scale}` -- the reference's
harness CLI (tools/ifgf.cpp) on the B200 operator: same options, the JSON
report of schema version 1 (`run`), the pass/FAIL line and exit code
(`verify`), the CSV sweep (`scale`).  `--ranks R` runs the reference's rank
algorithm (dist.cpp:241-361) with R ranks simulated on the GPU
(dist.simulate); `--threads` is accepted and ignored (kernel launches replace
the host thread pool).
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

from . import dist
from .engine import (EngineParams, InterpOrders, KernelConfig, KernelKind, Plan, apply,
                     error_at_indices, estimate_error, sample_indices)
from .points import (checksum_hex, diameter, generate_surface, read_points, shape_diameter,
                     shape_from_string)


class ValidationError(Exception):
    pass


def _ints(s: str):
    return [int(v) for v in s.split(",") if v != ""]


def add_common(p: argparse.ArgumentParser) -> None:
    """add_common (tools/ifgf.cpp:45-66)."""
    p.add_argument("--shape", default="sphere", choices=["sphere", "oblate", "prolate"])
    p.add_argument("--size-lambda", type=float, default=4.0, dest="size_lambda")
    p.add_argument("--n", type=int, default=20000)
    p.add_argument("--kernel", default="helmholtz", choices=["helmholtz", "laplace"])
    p.add_argument("--depth", type=int, default=0)
    p.add_argument("--box-lambda", type=float, default=0.25, dest="box_lambda")
    p.add_argument("--p", type=_ints, default=[])
    p.add_argument("--cones", type=_ints, default=[])
    p.add_argument("--ranks", type=int, default=1)
    p.add_argument("--threads", type=int, default=0)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--input", default="")
    p.add_argument("--output", default="")
    p.add_argument("--m", type=int, default=1000)


class Built:
    def __init__(self):
        self.pc = None
        self.cfg = None
        self.params = None
        self.diameter = 0.0
        self.n_requested = 0


def _lround(x: float) -> int:  # std::lround: halves away from zero
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def build_case(o, n_override: int = 0, size_override: float = 0.0) -> Built:
    """build_case (tools/ifgf.cpp:76-122)."""
    b = Built()
    kind = KernelKind.Laplace if o.kernel == "laplace" else KernelKind.Helmholtz
    n_req = n_override or o.n
    size_lambda = size_override if size_override > 0.0 else o.size_lambda
    b.n_requested = n_req
    if o.input:
        b.pc = read_points(o.input)
        b.diameter = diameter(b.pc)
    else:
        shape = shape_from_string(o.shape)
        k = max(2, _lround(math.sqrt(n_req / 6.0)))
        b.pc = generate_surface(shape, 1.0, k, o.seed)
        b.diameter = shape_diameter(shape, 1.0)
    wavenumber = 0.0
    if kind == KernelKind.Helmholtz:
        if size_lambda <= 0.0:
            raise ValidationError("--size-lambda must be positive for helmholtz")
        wavenumber = 2.0 * math.pi * size_lambda / b.diameter
    else:
        b.pc.a_im[:] = 0.0  # a real kernel with real data keeps the output real
    b.cfg = KernelConfig(kind, wavenumber)
    orders = InterpOrders()
    if o.p:
        if len(o.p) != 3:
            raise ValidationError("--p needs three values")
        orders = InterpOrders(*o.p)
    params = EngineParams(depth=o.depth, box_lambda=o.box_lambda, orders=orders)
    if o.cones:
        if len(o.cones) != 3:
            raise ValidationError("--cones needs three values")
        params.base_s, params.base_theta, params.base_phi = o.cones
    b.params = params
    return b


class CommStats:
    """dist::CommStats (dist.hpp) from the exchange sets of a simulated run:
    per level the fetched blocks (what the reference's window counts), the
    largest number of ranks fetching one block, the blocks owned, and the
    largest per-rank cache (interpolation + propagation fetches of the level,
    dist.cpp:302-306)."""

    def __init__(self, ex, plan, R):
        self.levels = []
        D = plan.depth
        for d in range(3, D + 1):
            row = {"d": d}
            per_rank = {}
            for kind, name in ((dist.INTERP, "interp"), (dist.PROP, "prop")):
                sets = []
                rec = ex.recv.get((d, kind))
                for r in range(R):
                    if rec is None:
                        sets.append(np.zeros(0, np.uint32))
                    else:
                        parts = [np.asarray(a) for a in rec[r] if len(a)]
                        sets.append(np.concatenate(parts) if parts else np.zeros(0, np.uint32))
                per_rank[name] = sets
                allc = np.concatenate(sets) if sets else np.zeros(0, np.uint32)
                row[f"{name}_fetched"] = int(len(allc))
                row[f"max_{name}_fanout"] = int(np.bincount(allc).max()) if len(allc) else 0
            row["owned_blocks"] = plan.n_cones(d)
            row["peak_rank_cache_blocks"] = int(max(
                len(per_rank["interp"][r]) + (len(per_rank["prop"][r]) if d > 3 else 0)
                for r in range(R)))
            self.levels.append(row)

    def total_fetched(self) -> int:
        return sum(l["interp_fetched"] + l["prop_fetched"] for l in self.levels)


def _evaluate(b: Built, ranks: int):
    """ifgf::apply, or run_distributed with `ranks` simulated ranks; fills
    b.pc.i_re/i_im and returns (report dict, CommStats or None)."""
    if ranks <= 1:
        rep = apply(b.pc, b.cfg, b.params)
        s = rep.seconds
        return {"seconds": {"setup": s.setup, "singular": s.singular, "level_d_eval": s.level_d,
                            "interpolation": s.interpolation, "propagation": s.propagation,
                            "total": s.total},
                "n": rep.n, "depth": rep.depth, "h_level_d": rep.h_level_d,
                "levels": [{"d": l.d, "boxes": l.boxes, "cones": l.cones} for l in rep.levels],
                "peak_live_blocks": rep.peak_live_blocks}, None
    # the result from the C++ rank group (ifgf_run_distributed); the
    # reference's CommStats from the device exchange sets of one plan
    drep, _ = dist.run_distributed(b.pc, b.cfg, b.params, ranks)
    plan = Plan.from_cloud(b.pc, b.cfg, b.params)
    try:
        ex = dist.build_exchange_plan(dist.rank_layout(plan, ranks), plan.depth,
                                      lambda r, d, kind: plan.exchange_set(ranks, r, d, kind))
        comm = CommStats(ex, plan, ranks)
        D = plan.depth
        s = drep.seconds
        rep = {"seconds": {"setup": s.setup, "singular": 0.0, "level_d_eval": 0.0,
                           "interpolation": 0.0, "propagation": 0.0, "total": s.total},
               "n": b.pc.size(), "depth": D, "h_level_d": plan.info.h[D],
               "levels": [{"d": d, "boxes": plan.n_boxes(d), "cones": plan.n_cones(d)}
                          for d in range(3, D + 1)],
               "peak_live_blocks": int(max(plan.n_cones(d) + (plan.n_cones(d - 1) if d > 3 else 0)
                                           for d in range(3, D + 1)))}
        return rep, comm
    finally:
        plan.close()


def report_json(o, b: Built, rep, comm, eps: float, m_used: int) -> dict:
    """report_json (tools/ifgf.cpp:140-181), schema version 1."""
    lam = b.cfg.wavelength()
    cfg = {"shape": o.shape if not o.input else "file:" + o.input, "kernel": o.kernel,
           "wavenumber": b.cfg.wavenumber, "size_lambda": o.size_lambda,
           "n_requested": b.n_requested, "seed": o.seed, "depth": o.depth,
           "box_lambda": o.box_lambda,
           "p": [b.params.orders.p_s, b.params.orders.p_theta, b.params.orders.p_phi],
           "cones": [b.params.base_s, b.params.base_theta, b.params.base_phi],
           "ranks": o.ranks, "threads": 1, "m": o.m}
    j = {"schema_version": 1, "config": cfg, "n": rep["n"], "depth": rep["depth"],
         "diameter_lambda": b.diameter / lam if lam > 0.0 else 0.0,
         "h_level_d_lambda": rep["h_level_d"] / lam if lam > 0.0 else 0.0,
         "stage_seconds": rep["seconds"],
         "epsilon": {"m": m_used, "seed": o.seed, "value": eps},
         "levels": rep["levels"], "peak_live_blocks": rep["peak_live_blocks"]}
    if comm is not None:
        j["comm"] = {"levels": comm.levels, "total_fetched": comm.total_fetched()}
    j["simd_variant"] = "sm_100a"
    j["result_checksum"] = checksum_hex(b.pc.i_re, b.pc.i_im)
    j["imag_max_abs"] = float(np.max(np.abs(b.pc.i_im))) if b.pc.size() else 0.0
    return j


def emit(output: str, text: str) -> None:
    if not output:
        sys.stdout.write(text)
    else:
        with open(output, "w") as f:
            f.write(text)


def cmd_run(o) -> int:
    b = build_case(o)
    rep, comm = _evaluate(b, o.ranks)
    m_used = min(o.m * max(1, o.ranks), b.pc.size())
    eps = estimate_error(b.pc, b.cfg, m_used, o.seed + 1)
    emit(o.output, json.dumps(report_json(o, b, rep, comm, eps, m_used), indent=2) + "\n")
    return 0


def cmd_verify(o) -> int:
    b = build_case(o)
    if o.verify == "full" and b.pc.size() > 5000:
        raise ValidationError("--verify full is limited to N <= 5000")
    _evaluate(b, o.ranks)
    if o.verify == "full":
        eps = error_at_indices(b.pc, b.cfg, np.arange(b.pc.size(), dtype=np.uint32))
    elif o.ranks > 1:
        # m points drawn on each rank from its own interval (dist.cpp:363-373)
        with Plan.from_cloud(b.pc, b.cfg, b.params) as plan:
            layout = dist.rank_layout(plan, o.ranks)
            perm = plan.perm()
        idx = []
        for r in range(o.ranks):
            begin, end = layout.points(r)
            count = end - begin
            local = sample_indices(count, min(o.m, count), o.seed + 1 + r)
            idx.extend(int(perm[begin + int(i)]) for i in local)
        eps = error_at_indices(b.pc, b.cfg, np.asarray(idx, np.uint32))
    else:
        eps = estimate_error(b.pc, b.cfg, min(o.m, b.pc.size()), o.seed + 1)
    ok = eps <= o.threshold
    print(f"epsilon {eps:.6e} threshold {o.threshold:.6e} : {'pass' if ok else 'FAIL'}")
    return 0 if ok else 1


def cmd_scale(o) -> int:
    lines = ["n,size_lambda,depth,t_seconds,t_per_nlog2n,peak_live_blocks,relevant_cones,"
             "blocks_fetched_total,fetched_per_nlog2n"]
    n0 = o.ns[0]
    for n in o.ns:
        size = o.size_lambda * math.sqrt(n / n0)  # fixed points per box
        b = build_case(o, n, size)
        rep, comm = _evaluate(b, o.ranks)
        fetched = comm.total_fetched() if comm is not None else 0
        cones = sum(l["cones"] for l in rep["levels"])
        nlogn = rep["n"] * math.log2(rep["n"])
        t = rep["seconds"]["total"]
        lines.append(f"{rep['n']},{size:g},{rep['depth']},{t:g},{t / nlogn:g},"
                     f"{rep['peak_live_blocks']},{cones},{fetched},{fetched / nlogn:g}")
    emit(o.output, "\n".join(lines) + "\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ifgf", description="IFGF operator evaluation benchmark")
    sub = ap.add_subparsers(dest="cmd", required=True)
    run = sub.add_parser("run", help="single evaluation with a JSON report")
    add_common(run)
    ver = sub.add_parser("verify", help="compare against the direct oracle")
    add_common(ver)
    ver.add_argument("--verify", default="subsample", choices=["full", "subsample"])
    ver.add_argument("--threshold", type=float, default=5e-3)
    sc = sub.add_parser("scale", help="complexity sweep, CSV output")
    add_common(sc)
    sc.add_argument("--ns", type=_ints, required=True)
    o = ap.parse_args(argv)
    try:
        if o.cmd == "run":
            return cmd_run(o)
        if o.cmd == "verify":
            return cmd_verify(o)
        return cmd_scale(o)
    except Exception as e:  # the reference prints "error: <what>" and exits 2
        sys.stderr.write(f"error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
