"""Structural work counts and algorithmic FLOPs of one IFGF matvec.

Counts are properties of the octree and cone sets (identical for the oracle
and the GPU).  FLOP weights follow SURVEY.md §8(d) (FP64, sqrt = div = 1,
sincos = 36, FMA = 2):

  near-field pair (green_sum)                 57
  level-D node x source pair (factored_sum)   58
  interpolant evaluation  4 (P + ps pt + ps)  372 at (3,5,5)
    + centred factor (interpolation)          +57  -> 429
    + transfer factor (propagation)           +58  -> 430
  Chebyshev fit  2 * 2 * P (pp + pt + ps)     3,900 at (3,5,5)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

W_NEAR = 57
W_LEVELD = 58


def w_eval(ps, pt, pp):
    return 4 * (ps * pt * pp + ps * pt + ps)


def w_fit(ps, pt, pp):
    return 4 * ps * pt * pp * (ps + pt + pp)


@dataclass
class WorkCounts:
    n: int
    depth: int
    P: int
    orders: tuple
    near_pairs: int = 0
    leveld_pairs: int = 0
    leveld_fits: int = 0
    prop_evals: dict = field(default_factory=dict)    # d -> evals of K3(d)
    prop_fits: dict = field(default_factory=dict)     # d -> parent cones (level d-1)
    interp_evals: dict = field(default_factory=dict)  # d -> evals of K4(d)

    @property
    def flops(self) -> dict:
        ps, pt, pp = self.orders
        we, wf = w_eval(ps, pt, pp), w_fit(ps, pt, pp)
        return {
            "near": W_NEAR * self.near_pairs,
            "level_d": W_LEVELD * self.leveld_pairs + wf * self.leveld_fits,
            "propagation": sum((we + 58) * v for v in self.prop_evals.values())
            + wf * sum(self.prop_fits.values()),
            "interpolation": sum((we + 57) * v for v in self.interp_evals.values()),
        }

    @property
    def total_flops(self) -> int:
        return sum(self.flops.values())

    def as_dict(self):
        return {"near_pairs": self.near_pairs, "leveld_pairs": self.leveld_pairs,
                "leveld_fits": self.leveld_fits,
                "prop_evals": int(sum(self.prop_evals.values())),
                "prop_fits": int(sum(self.prop_fits.values())),
                "interp_evals": int(sum(self.interp_evals.values())),
                "flops": {k: int(v) for k, v in self.flops.items()},
                "total_flops": int(self.total_flops)}


def count_work(plan) -> WorkCounts:
    D, Pn = plan.depth, plan.P
    info = plan.info
    wc = WorkCounts(plan.n, D, Pn, (info.p_s, info.p_theta, info.p_phi))
    levels = {d: plan.level(d) for d in range(max(2, 3 - 1), D + 1)}
    # near field: every target against all points of its neighbour boxes, minus self
    L = levels[D]
    cnt = L.count.astype(np.int64)
    nb_deg = np.diff(L.nbr_off.astype(np.int64))
    nb_pts = np.add.reduceat(cnt[L.nbr], L.nbr_off[:-1].astype(np.int64)) if len(L.nbr) else 0
    nb_pts = np.where(nb_deg > 0, nb_pts, 0)
    wc.near_pairs = int(np.sum(cnt * nb_pts) - plan.n)
    # level-D seeding
    wc.leveld_fits = int(len(L.cone_box))
    wc.leveld_pairs = int(Pn * np.sum(cnt[L.cone_box]))
    for d in range(3, D + 1):
        Ld = levels[d]
        ncous = np.diff(Ld.cousin_off.astype(np.int64))
        wc.interp_evals[d] = int(np.sum(Ld.count.astype(np.int64) * ncous))
        if d > 3:
            U = levels[d - 1]
            nchild = np.diff(U.child_begin.astype(np.int64))
            wc.prop_evals[d] = int(Pn * np.sum(nchild[U.cone_box]))
            wc.prop_fits[d] = int(len(U.cone_box))
    return wc
