"""Host-side pixel domains and grain maps (mirror of polygrain/geometry.py).

A regular grid keeps only its resolution M: the device regenerates the
coordinate of pixel p with the reference's expression
-1 + (k - 1/2)/M, row-major with the first axis slowest (geometry.py:59-71).
``points`` is materialised lazily on the host only when a caller asks for it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TIE_RTOL = 1e-12  # geometry.py:19


def grid_axis(m: int) -> np.ndarray:
    return -1.0 + (np.arange(1, 2 * int(m) + 1) - 0.5) / int(m)


class PixelGrid:
    """A point list in [-1,1]^dim: regular (resolution M) or unstructured."""

    def __init__(self, points=None, resolution: int | None = None, dim: int = 2):
        self.resolution = None if resolution is None else int(resolution)
        self._points = None
        if points is not None:
            pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
            if pts.ndim != 2 or pts.shape[1] not in (2, 3):
                raise ValueError(f"points must have shape (n, 2) or (n, 3), got {pts.shape}")
            if pts.shape[0] == 0:
                raise ValueError("a grid needs at least one point")
            if not np.all(np.isfinite(pts)):
                raise ValueError("grid points must be finite")
            if np.any(np.abs(pts) >= 1.0):
                raise ValueError("grid points must lie strictly inside [-1,1]^2")
            pts.setflags(write=False)
            self._points = pts
            dim = pts.shape[1]
        elif self.resolution is None:
            raise ValueError("need points or a resolution")
        if self.resolution is not None and self.resolution < 1:
            raise ValueError("resolution must be a positive integer")
        self.dim = int(dim)
        n = (2 * self.resolution) ** self.dim if self.resolution is not None else pts.shape[0]
        if self._points is not None and self.resolution is not None and self._points.shape[0] != n:
            raise ValueError(
                f"regular grid with M={self.resolution} requires {n} points, got {self._points.shape[0]}")
        self._n = n

    @property
    def points(self) -> np.ndarray:
        if self._points is None:
            c = grid_axis(self.resolution)
            if self.dim == 2:
                pts = np.column_stack([np.repeat(c, c.size), np.tile(c, c.size)])
            else:
                n = c.size
                pts = np.column_stack([np.repeat(c, n * n), np.tile(np.repeat(c, n), n),
                                       np.tile(c, n * n)])
            pts.setflags(write=False)
            self._points = pts
        return self._points

    def __len__(self) -> int:
        return self._n


def make_grid(m: int, dim: int = 2) -> PixelGrid:
    """Regular (2M)^dim grid (geometry.py:59-71; dim 3 is the extension)."""
    m = int(m)
    if m < 1:
        raise ValueError("grid resolution M must be >= 1")
    return PixelGrid(resolution=m, dim=dim)


@dataclass(frozen=True)
class GrainMap:
    """Labels in {1..N} over a grid (geometry.py:74-107)."""

    grid: object
    labels: np.ndarray
    n_grains: int

    def __post_init__(self):
        lab = np.ascontiguousarray(np.asarray(self.labels, dtype=np.int64))
        if lab.ndim != 1:
            raise ValueError("labels must be one-dimensional")
        if lab.shape[0] != len(self.grid):
            raise ValueError(
                f"labels length {lab.shape[0]} != number of grid points {len(self.grid)}")
        n = int(self.n_grains)
        if n <= 1:
            raise ValueError("a grain map needs at least two grains")
        if lab.size and (lab.min() < 1 or lab.max() > n):
            raise ValueError(f"labels must lie in 1..{n}")
        lab.setflags(write=False)
        object.__setattr__(self, "labels", lab)
        object.__setattr__(self, "n_grains", n)

    def __len__(self) -> int:
        return len(self.grid)

    def grain_sizes(self) -> np.ndarray:
        return np.bincount(self.labels - 1, minlength=self.n_grains)


def accuracy_and_error(grain_map, assigned) -> tuple[float, float]:
    """(acc, err) with acc + err == 1 exactly (geometry.py:251-262)."""
    assigned = np.asarray(assigned)
    if assigned.shape != grain_map.labels.shape:
        raise ValueError(
            f"label array length {assigned.shape} != grain map length {grain_map.labels.shape}")
    acc = float(np.count_nonzero(assigned == grain_map.labels)) / len(grain_map)
    return acc, 1.0 - acc
