"""Whole-output sketch of an IFGF result vector (test infrastructure).

A full-size output (C2: 1.57 M complex values, C5: 25 M) is too large to
commit, so the fixtures store a signed bucket sketch of the WHOLE vector
instead of a sample of it:

    bucket(i) = floor(i * K / N)            (K contiguous buckets of the
                                             caller's original point order)
    s_i       = +-1 from splitmix64(i + seed * 0x9E3779B97F4A7C15)
    S_b(I)    = sum over bucket b of s_i * I_i          (complex)
    Q_b(I)    = sum over bucket b of |I_i|^2

The signed sums are a CountSketch: E ||S(x)||^2 = ||x||^2 for every vector
x, so ||S(I_gpu) - S(I_ref)|| / ||S(I_ref)|| estimates the relative l2
difference of the whole outputs (north_star bar 1e-10).  A localised error
(one flipped cone segment changing a few targets by ~1e-3 relative) moves
its bucket's signed sum by ~1e-3 / sqrt(bucket size) relative, so the
per-bucket bound below catches it even where the global estimate would not.
"""
from __future__ import annotations

import numpy as np

K_DEFAULT = 16384
SEED = 20240531
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def signs(n: int, seed: int = SEED, chunk: int = 1 << 22) -> np.ndarray:
    out = np.empty(n, np.float64)
    with np.errstate(over="ignore"):
        off = np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
    for a in range(0, n, chunk):
        i = np.arange(a, min(n, a + chunk), dtype=np.uint64)
        with np.errstate(over="ignore"):
            h = _splitmix64(i + off)
        out[a:a + len(i)] = 1.0 - 2.0 * (h >> np.uint64(63)).astype(np.float64)
    return out


def buckets(n: int, k: int) -> np.ndarray:
    return (np.arange(n, dtype=np.int64) * k) // n


def sketch(i_re: np.ndarray, i_im: np.ndarray, k: int = K_DEFAULT, seed: int = SEED):
    """(S_re, S_im, Q) of the whole output vector, each of length k."""
    n = len(i_re)
    k = min(k, n)
    s = signs(n, seed)
    b = buckets(n, k)
    s_re = np.bincount(b, weights=s * i_re, minlength=k)
    s_im = np.bincount(b, weights=s * i_im, minlength=k)
    q = np.bincount(b, weights=i_re * i_re + i_im * i_im, minlength=k)
    return s_re, s_im, q


def compare(got, want):
    """(global relative l2 estimate, worst per-bucket deviation relative to
    the rms bucket magnitude, worst relative bucket-norm deviation)."""
    g_re, g_im, g_q = got
    w_re, w_im, w_q = want
    dre, dim = g_re - w_re, g_im - w_im
    den = float(np.sum(w_re * w_re + w_im * w_im))
    rel = float(np.sqrt(np.sum(dre * dre + dim * dim) / den))
    rms = np.sqrt(den / len(w_re))
    worst = float(np.max(np.hypot(dre, dim)) / rms)
    qrel = float(np.max(np.abs(g_q - w_q) / np.maximum(w_q, 1e-300)))
    return rel, worst, qrel
