"""Point-cloud harness of the reference (geometry.cpp / geometry.hpp,
bench.cpp): the cube-face surface generator, the IFGF v1 binary and CSV point
formats, the diameter estimate and the result checksum.  Host-side harness
code around the operator -- the formats are what `ifgf run --input` reads.
"""
from __future__ import annotations

import ctypes as C
import math
import struct

import numpy as np

from ._lib import lib, ptr
from .engine import InvalidArgument, PointCloud, check

# Shape (geometry.hpp) and shape_from_string / shape_diameter (geometry.cpp:14-36)
SHAPES = {"sphere": 0, "oblate": 1, "prolate": 2}
_MAGIC = b"IFGF"
_VERSION = 1


def shape_from_string(name: str) -> int:
    if name not in SHAPES:
        raise InvalidArgument(f"unknown shape: {name}")
    return SHAPES[name]


def shape_diameter(shape: int, a: float = 1.0) -> float:
    """geometry.cpp:28-36: 2a for the sphere and the oblate spheroid (z x 0.1),
    20a for the prolate one (z x 10)."""
    return (2.0, 2.0, 20.0)[shape] * a


def generate_surface(shape: int, a: float, n_per_dim: int, seed: int) -> PointCloud:
    """generate_surface (geometry.cpp:57-93), bitwise: 6 n_per_dim^2 points."""
    m = 6 * n_per_dim * n_per_dim if n_per_dim >= 2 else 0
    arrs = [np.zeros(max(m, 1)) for _ in range(5)]
    check(lib.ifgf_generate_surface(int(shape), float(a), int(n_per_dim), int(seed),
                                    *(ptr(x) for x in arrs)))
    return PointCloud(*(x[:m] for x in arrs))


def diameter(pc: PointCloud) -> float:
    """geometry.cpp:116-140: exact max pairwise distance for N <= 10,000, else
    the bounding-box diagonal."""
    n = pc.size()
    if n == 0:
        raise InvalidArgument("diameter: empty cloud")
    if n <= 10000:
        best = 0.0
        for i in range(n - 1):  # row by row: O(N) memory
            dx = pc.x1[i] - pc.x1[i + 1:]
            dy = pc.x2[i] - pc.x2[i + 1:]
            dz = pc.x3[i] - pc.x3[i + 1:]
            best = max(best, float(np.max(dx * dx + dy * dy + dz * dz)))
        return math.sqrt(best)
    ex = pc.x1.max() - pc.x1.min()
    ey = pc.x2.max() - pc.x2.min()
    ez = pc.x3.max() - pc.x3.min()
    return math.sqrt(ex * ex + ey * ey + ez * ez)


def checksum_hex(re: np.ndarray, im: np.ndarray) -> str:
    """bench::checksum_hex (bench.cpp:26-41): FNV-1a 64 over the bytes."""
    re = np.ascontiguousarray(re, np.float64)
    im = np.ascontiguousarray(im, np.float64)
    if len(re) != len(im):
        raise InvalidArgument("checksum_hex: re and im differ in length")
    out = C.create_string_buffer(17)
    lib.ifgf_checksum_hex(ptr(re), ptr(im), len(re), out)
    return out.value.decode()


def write_points_binary(path: str, pc: PointCloud) -> None:
    """geometry.cpp:147-163: 'IFGF', u32 version 1, u64 n, n xyz triples,
    n (a_re, a_im) pairs, little endian."""
    n = pc.size()
    xyz = np.stack([pc.x1, pc.x2, pc.x3], axis=1).astype("<f8")
    ab = np.stack([pc.a_re, pc.a_im], axis=1).astype("<f8")
    with open(path, "wb") as f:
        f.write(_MAGIC + struct.pack("<IQ", _VERSION, n))
        f.write(xyz.tobytes())
        f.write(ab.tobytes())


def read_points_binary(path: str) -> PointCloud:
    """geometry.cpp:165-192, with the reference's error classes and messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError("cannot open: " + str(path)) from None
    with f:
        head = f.read(16)
        if len(head) < 16 or head[:4] != _MAGIC:
            raise RuntimeError("not an IFGF point file: " + str(path))
        version, n = struct.unpack("<IQ", head[4:])
        if version != _VERSION:
            raise RuntimeError("unsupported point file version")
        xyz = np.frombuffer(f.read(24 * n), "<f8")
        ab = np.frombuffer(f.read(16 * n), "<f8")
    if len(xyz) != 3 * n or len(ab) != 2 * n:
        raise RuntimeError("truncated point file: " + str(path))
    xyz = xyz.reshape(n, 3)
    ab = ab.reshape(n, 2)
    return PointCloud(xyz[:, 0], xyz[:, 1], xyz[:, 2], ab[:, 0], ab[:, 1])


def _parse_csv_line(line: str):
    # `ss >> v0 >> c >> v1 >> c ...` (geometry.cpp:205-208): five numbers, each
    # pair separated by one non-space character, whitespace allowed around
    parts = []
    rest = line.strip()
    for k in range(5):
        j = 0
        while j < len(rest) and (rest[j].isdigit() or rest[j] in "+-.eEinfaINFA"):
            j += 1
        tok = rest[:j]
        try:
            parts.append(float(tok))
        except ValueError:
            return None
        rest = rest[j:].lstrip()
        if k < 4:
            if not rest:
                return None
            rest = rest[1:].lstrip()
    return parts


def read_points_csv(path: str) -> PointCloud:
    """geometry.cpp:194-216: x1,x2,x3,a_re,a_im per line, optional header,
    blank lines skipped."""
    try:
        f = open(path, "r")
    except OSError:
        raise RuntimeError("cannot open: " + str(path)) from None
    rows = []
    first = True
    with f:
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            v = _parse_csv_line(line)
            if v is None:
                if first:
                    first = False
                    continue
                raise RuntimeError("bad CSV line: " + line)
            first = False
            rows.append(v)
    if not rows:
        raise RuntimeError("empty CSV point file: " + str(path))
    a = np.asarray(rows, np.float64)
    return PointCloud(a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4])


def read_points(path: str) -> PointCloud:
    """geometry.cpp:218-226: binary when the file starts with 'IFGF', else CSV."""
    try:
        with open(path, "rb") as f:
            magic = f.read(4)
    except OSError:
        raise RuntimeError("cannot open: " + str(path)) from None
    return read_points_binary(path) if magic == _MAGIC else read_points_csv(path)
