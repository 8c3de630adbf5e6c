"""Warp-GEMM unit composition: MMA column-octant work of cutting strategies
against the ideal (every cone only its own children), per parent level.

usage: python tools/unit_stats.py C2
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_15198_b200 as ifgf  # noqa: E402

c = ifgf.configs.CONFIGS[sys.argv[1]]
pc = ifgf.generate(c.n, c.shape, c.c, c.dens, c.seed)
cfg = ifgf.KernelConfig(ifgf.KernelKind(c.kind), c.kappa)
plan = ifgf.Plan.from_cloud(pc, cfg, ifgf.EngineParams(depth=c.depth))
POPC = np.array([bin(i).count("1") for i in range(256)])


def cost_units(masks, cuts):
    """cuts: unit start indices (sorted, first 0); cost = cols * popc(union)."""
    tot = 0
    ends = list(cuts[1:]) + [len(masks)]
    for a, b in zip(cuts, ends):
        u = np.bitwise_or.reduce(masks[a:b])
        tot += (8 if b - a <= 8 else 16) * POPC[u]
    return tot


for d in range(plan.depth, 4, -1):
    U, L = plan.level(d - 1), plan.level(d)
    cb = U.child_begin.astype(np.int64)
    oct_ = (L.codes.astype(np.int64) & 7)
    bmask = np.zeros(len(cb) - 1, dtype=np.int64)
    np.bitwise_or.at(bmask, np.repeat(np.arange(len(cb) - 1), np.diff(cb)), 1 << oct_)
    gam = U.cone_gamma.astype(np.int64)
    msk = bmask[U.cone_box.astype(np.int64)]
    order = np.lexsort((np.arange(len(gam)), msk, gam))
    gam, msk = gam[order], msk[order]
    ideal = POPC[msk].sum()
    starts = np.flatnonzero(np.r_[True, gam[1:] != gam[:-1]])
    ends = np.r_[starts[1:], len(gam)]
    c0 = c1 = c2 = ct = 0
    nu0 = nu1 = 0
    for a, b in zip(starts, ends):
        m = msk[a:b]
        n = b - a
        # S0: every 16
        cuts = list(range(0, n, 16))
        c0 += cost_units(m, cuts)
        nu0 += len(cuts)
        # S0 with a column tile's MMAs skipped for octants none of its 8 cones
        # has (the kernel's predicate): every tile pays only its own union
        for t in range(0, n, 8):
            ct += 8 * POPC[np.bitwise_or.reduce(m[t:t + 8])]
        # S1: new unit at a mask change once the unit holds >= 8 cones
        cuts, size = [0], 0
        for i in range(n):
            if size == 16 or (size >= 8 and i > 0 and m[i] != m[i - 1]):
                cuts.append(i)
                size = 0
            size += 1
        c1 += cost_units(m, cuts)
        nu1 += len(cuts)
        # S2: dynamic programme over contiguous cuts (units of 1..16)
        best = [0] + [1 << 60] * n
        for i in range(1, n + 1):
            u = 0
            for k in range(1, min(16, i) + 1):
                u |= int(m[i - k])
                cst = best[i - k] + (8 if k <= 8 else 16) * POPC[u]
                if cst < best[i]:
                    best[i] = cst
        c2 += best[n]
    # S5: masks re-ranked by a greedy similarity chain over the level's mask
    # histogram (next = unvisited mask with the smallest union growth), then
    # every 16 / optimal contiguous cuts
    hist = np.bincount(msk, minlength=256)
    present = [int(x) for x in np.flatnonzero(hist)]
    cur = int(np.argmax(hist))
    chain, left = [cur], set(present) - {cur}
    while left:
        nxt = min(left, key=lambda x: (POPC[x | cur] - min(POPC[x], POPC[cur]), POPC[x ^ cur], -hist[x]))
        chain.append(nxt)
        left.remove(nxt)
        cur = nxt
    rank = np.zeros(256, dtype=np.int64)
    rank[chain] = np.arange(len(chain))
    o5 = np.lexsort((np.arange(len(gam)), rank[msk], gam))
    g5, m5 = gam[o5], msk[o5]
    c5 = c6 = 0
    for a, b in zip(starts, ends):
        m = m5[a:b]
        n = b - a
        c5 += cost_units(m, list(range(0, n, 16)))
        best = [0] + [1 << 60] * n
        for i in range(1, n + 1):
            u = 0
            for k in range(1, min(16, i) + 1):
                u |= int(m[i - k])
                cst = best[i - k] + (8 if k <= 8 else 16) * POPC[u]
                if cst < best[i]:
                    best[i] = cst
        c6 += best[n]
    print(f"   similarity-chain mask order: every 16 {c5 / ideal:.3f}, optimal contiguous {c6 / ideal:.3f} ({len(present)} masks)")
    # S4: no mask key -- cones of a gamma in box (Morton) order, every 16
    o4 = np.lexsort((np.arange(len(gam)), U.cone_gamma.astype(np.int64)))
    g4, m4 = U.cone_gamma.astype(np.int64)[o4], bmask[U.cone_box.astype(np.int64)][o4]
    s4 = np.flatnonzero(np.r_[True, g4[1:] != g4[:-1]])
    e4 = np.r_[s4[1:], len(g4)]
    c4 = 0
    for a, b in zip(s4, e4):
        c4 += cost_units(m4[a:b], list(range(0, b - a, 16)))
    print(f"   Morton order within gamma, every 16: {c4 / ideal:.3f}")
    print(f"   every 16, MMAs per column tile's own octants: {ct / ideal:.3f}")
    print(f"d={d}: cones {len(gam)} gammas {len(starts)} ideal {ideal}  every-16 {c0 / ideal:.3f} ({nu0} units)  "
          f"cut-at-mask>=8 {c1 / ideal:.3f} ({nu1} units)  optimal contiguous {c2 / ideal:.3f}", flush=True)
