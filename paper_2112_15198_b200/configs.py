"""BASELINE.json configurations C1-C5 as seeded synthetic workloads.

The reference measures on no public dataset; BASELINE.json names seeded
synthetic clouds, regenerated here by ifgf_generate:
config Ck uses mt19937_64(seed=k), positions first, then densities; the
error sample is sample_indices(N, 1000, seed=k+1) (tools/ifgf.cpp:202).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    shape: int        # 0 sphere, 1 spheroid (1,1,c)
    c: float          # spheroid z semi-axis
    kind: int         # 0 Helmholtz, 1 Laplace
    kappa: float
    dens: int         # 0 complex U(-1,1), 1 real N(0,1)
    seed: int
    depth: int = 0    # 0 = choose_depth rule
    note: str = ""

    @property
    def label(self):
        return f"{self.name}: N={self.n:,} {'oblate' if self.shape else 'sphere'} " \
               f"{'Laplace' if self.kind else f'kappa={self.kappa / math.pi:g}pi'}"


C1 = Config("C1", 98_304, 0, 1.0, 0, 8 * math.pi, 0, 1,
            note="unit sphere, 8 wavelengths across the diameter")
C2 = Config("C2", 1_572_864, 0, 1.0, 0, 32 * math.pi, 0, 2,
            note="unit sphere, 32 wavelengths")
C3 = Config("C3", 6_291_456, 0, 1.0, 1, 0.0, 1, 3,
            note="Laplace, real N(0,1) density, depth from the points_per_box=64 rule (D=10)")
C4 = Config("C4", 6_291_456, 1, 0.25, 0, 128 * math.pi, 0, 4,
            note="oblate spheroid (1,1,0.25), area-uniform by rejection")
C5 = Config("C5", 25_165_824, 0, 1.0, 0, 256 * math.pi, 0, 5,
            note="unit sphere, 256 wavelengths")

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}


def weak(G: int) -> Config:
    """Weak-scaling companion: N = 3,145,728 G at C1's points-per-lambda^2."""
    n = 3_145_728 * G
    return Config(f"W{G}", n, 0, 1.0, 0, 8 * math.pi * math.sqrt(n / 98_304), 0, 10 + G)


def scaled(cfg: Config, n: int) -> Config:
    """Same surface and points-per-wavelength density as cfg with n points
    (kappa scales with sqrt(n)); used for bounded CPU samples."""
    k = cfg.kappa * math.sqrt(n / cfg.n)
    return Config(f"{cfg.name}@{n}", n, cfg.shape, cfg.c, cfg.kind, k, cfg.dens, cfg.seed,
                  cfg.depth, f"{cfg.name} density sample")
