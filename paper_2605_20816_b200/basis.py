"""Host-side basis descriptors (mirror of polygrain/basis.py).

Only descriptors live here: the K x P design matrix of the reference
(``assemble_design_matrix``, basis.py:183-193) is never materialised — the
device regenerates eta(x) from the grid coordinates inside every kernel.
``DesignMatrix`` therefore carries ``basis`` and ``grid`` but no ``values``.

Ordering (basis.py:1-13,42-48): graded-lex, a1 descending, e.g. d = 2:
(0,0), (1,0), (0,1), (2,0), (1,1), (0,2).  The 3-D extension (SURVEY.md
Appendix B) orders by total degree, then a1 descending, then a2 descending.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ORDERING_CONVENTION = "graded-lex-a1-desc"
MONOMIAL = "monomial"
LEGENDRE = "legendre"
BASIS_KINDS = (MONOMIAL, LEGENDRE)
GAUGE_FREE = "free"
GAUGE_LAST_ZERO = "last-column-zero"


def feature_count(degree: int, dim: int = 2) -> int:
    """K = C(d + dim, dim); (d+1)(d+2)/2 in 2-D (basis.py:37-39)."""
    return math.comb(int(degree) + dim, dim)


def graded_lex_indices(degree: int, dim: int = 2) -> tuple:
    out = []
    for total in range(degree + 1):
        for a1 in range(total, -1, -1):
            if dim == 2:
                out.append((a1, total - a1))
            else:
                for a2 in range(total - a1, -1, -1):
                    out.append((a1, a2, total - a1 - a2))
    return tuple(out)


@dataclass(frozen=True)
class MultiIndexSet:
    degree: int
    dim: int = 2
    indices: tuple = field(default=(), compare=False)

    @classmethod
    def for_degree(cls, degree: int, dim: int = 2) -> "MultiIndexSet":
        if degree < 0:
            raise ValueError("degree must be non-negative")
        return cls(degree=int(degree), dim=dim, indices=graded_lex_indices(int(degree), dim))

    def __len__(self) -> int:
        return feature_count(self.degree, self.dim)

    def position(self, alpha) -> int:
        """Row of a multi-index (basis.py:73-79 for 2-D)."""
        alpha = tuple(int(a) for a in alpha)
        if len(alpha) != self.dim or min(alpha) < 0 or sum(alpha) > self.degree:
            raise ValueError(f"multi-index {alpha} not in the degree-{self.degree} set")
        return self.indices.index(alpha)


@dataclass(frozen=True)
class DesignBasis:
    kind: str
    index_set: MultiIndexSet

    @classmethod
    def make(cls, kind: str, degree: int, dim: int = 2) -> "DesignBasis":
        return cls(kind=kind, index_set=MultiIndexSet.for_degree(degree, dim))

    def __post_init__(self):
        if self.kind not in BASIS_KINDS:
            raise ValueError(f"unknown basis kind {self.kind!r}; expected one of {BASIS_KINDS}")

    @property
    def degree(self) -> int:
        return self.index_set.degree

    @property
    def dim(self) -> int:
        return self.index_set.dim

    @property
    def dimension(self) -> int:
        return len(self.index_set)

    def evaluate(self, points) -> np.ndarray:
        """The (K, n) features of ``points`` on the host (basis.py:105-117), for the
        small-problem diagnostics only (hessian_block); the hot path regenerates
        eta(x) on the device and never forms this matrix."""
        pts = np.asarray(points, dtype=np.float64)
        d = self.degree
        tabs = []
        for j in range(pts.shape[1]):
            t = pts[:, j]
            u = np.empty((d + 1,) + t.shape)
            u[0] = 1.0
            if d >= 1:
                u[1] = t
            for m in range(1, d):  # (m+1) P_{m+1} = (2m+1) t P_m - m P_{m-1}, or powers
                u[m + 1] = ((2 * m + 1) * t * u[m] - m * u[m - 1]) / (m + 1) if self.kind == LEGENDRE \
                    else u[m] * t
            tabs.append(u)
        return np.asarray([np.prod([tabs[j][a[j]] for j in range(len(a))], axis=0)
                           for a in self.index_set.indices])


@dataclass(frozen=True)
class DesignMatrix:
    """Lazy design: column j would be eta(x_j); the device regenerates it."""

    basis: DesignBasis
    grid: object

    @property
    def n_points(self) -> int:
        return len(self.grid)

    @property
    def values(self):
        raise AttributeError(
            "paper_2605_20816_b200 never materialises the K x P design matrix; "
            "features are generated on the device from design.grid")


def assemble_design_matrix(basis: DesignBasis, grid) -> DesignMatrix:
    """Replacement of basis.assemble_design_matrix (basis.py:183-193): O(1)."""
    return DesignMatrix(basis=basis, grid=grid)


@dataclass(frozen=True)
class ParamMatrix:
    """theta (K, N), column i = grain i (basis.py:287-327)."""

    values: np.ndarray
    basis: DesignBasis
    gauge: str = GAUGE_FREE

    def __post_init__(self):
        vals = np.ascontiguousarray(np.asarray(self.values, dtype=np.float64))
        if vals.ndim != 2:
            raise ValueError("parameter matrix must be two-dimensional")
        if vals.shape[0] != self.basis.dimension:
            raise ValueError(
                f"parameter rows {vals.shape[0]} != basis dimension {self.basis.dimension}")
        if vals.shape[1] < 2:
            raise ValueError("need at least two grains")
        if self.gauge not in (GAUGE_FREE, GAUGE_LAST_ZERO):
            raise ValueError(f"unknown gauge {self.gauge!r}")
        if self.gauge == GAUGE_LAST_ZERO and np.any(vals[:, -1] != 0.0):
            raise ValueError("gauge 'last-column-zero' requires an exactly zero final column")
        vals.setflags(write=False)
        object.__setattr__(self, "values", vals)

    @property
    def n_grains(self) -> int:
        return self.values.shape[1]

    @property
    def degree(self) -> int:
        return self.basis.degree

    def with_values(self, values, gauge: str | None = None) -> "ParamMatrix":
        return ParamMatrix(values=values, basis=self.basis,
                           gauge=self.gauge if gauge is None else gauge)
