"""Point sets and covariance kernels of the reference (geometry.cpp:20-168),
host side.  These only produce the synthetic inputs for construction; the
kernel evaluation itself runs on the device inside ``build_tlr``.

* ``generate_points`` — cell-centred Grid2D / Grid3D lattices truncated to the
  first N points in (ix, iy[, iz]) loop order (geometry.cpp:32-58), and the
  RandomBall3D rejection sampler driven by tlr::Rng (geometry.cpp:60-74).
* ``kd_order`` — recursive split along the widest bounding-box axis with the
  reference's tie-break by original index and its left-child size
  ``tile * (bit_ceil(ceil(m / tile)) / 2)`` (geometry.cpp:84-128).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GRID2D, GRID3D, BALL3D = 0, 1, 2
EXPONENTIAL, SQUARED_EXPONENTIAL = 0, 1


@dataclass
class PointSet:
    dim: int
    coords: np.ndarray     # (N, dim), original point order
    ordering: np.ndarray   # matrix index -> original point index

    def size(self):
        return len(self.ordering)

    def matrix_order(self) -> np.ndarray:
        """Coordinates in matrix order, (N, dim)."""
        return self.coords[self.ordering]


@dataclass
class KernelSpec:
    kind: int = EXPONENTIAL
    correlation_length: float = 0.1
    nugget: float = 0.0


def _grid_side(n, dim):
    s = 1
    while s ** dim < n:
        s += 1
    return s


def generate_points(kind: int, n: int, seed: int = 0) -> PointSet:
    if n < 1:
        raise ValueError("generate_points: n must be >= 1")
    if kind == GRID2D:
        s = _grid_side(n, 2)
        ix, iy = np.meshgrid(np.arange(s), np.arange(s), indexing="ij")
        pts = np.stack([(ix.ravel() + 0.5) / s, (iy.ravel() + 0.5) / s], 1)[:n]
        return PointSet(2, pts, np.arange(n))
    if kind == GRID3D:
        s = _grid_side(n, 3)
        ix, iy, iz = np.meshgrid(np.arange(s), np.arange(s), np.arange(s), indexing="ij")
        pts = np.stack([(ix.ravel() + 0.5) / s, (iy.ravel() + 0.5) / s,
                        (iz.ravel() + 0.5) / s], 1)[:n]
        return PointSet(3, pts, np.arange(n))
    if kind == BALL3D:
        from .mt64 import Mt64
        from .util import mix64
        rng = Mt64(mix64(seed ^ 0xBA11))
        out = []
        while len(out) < n:
            u = rng.uniforms(3 * 4096).reshape(-1, 3) * 2.0 - 1.0
            ok = (u * u).sum(1) <= 1.0
            out.extend(u[ok].tolist())
        return PointSet(3, np.asarray(out[:n]), np.arange(n))
    raise ValueError("generate_points: unsupported kind")


def kd_order(ps: PointSet, tile: int) -> PointSet:
    n = ps.size()
    if tile < 1 or tile > n:
        raise ValueError("kd_order: tile size out of range")
    ordv = ps.ordering.copy()
    stack = [(0, n)]
    while stack:
        lo, hi = stack.pop()
        m = hi - lo
        if m <= tile:
            continue
        seg = ordv[lo:hi]
        c = ps.coords[seg]
        ext = c.max(0) - c.min(0)
        d = int(np.argmax(ext))  # first widest axis (strict > in geometry.cpp:101)
        key = np.lexsort((seg, c[:, d]))  # by coordinate, ties by original index
        ordv[lo:hi] = seg[key]
        clusters = (m + tile - 1) // tile
        left = tile * ((1 << (clusters - 1).bit_length()) // 2)
        stack.append((lo + left, hi))
        stack.append((lo, lo + left))
    return PointSet(ps.dim, ps.coords, ordv)
