"""Moment-based initial coefficients (the reference's heuristics.py), with the
per-grain moments computed on the device.

The step before the hot path: per grain the pixel count,
centroid and central second-moment matrix (heuristics.py:46-73) give a power
diagram (degree 1: seeds = centroids, weights = area ratios) or an anisotropic
power diagram (degree >= 2: anisotropy = inverse second moments,
heuristics.py:76-92), whose monomial coefficients (conversions.py:52-96) are
zero-padded to the fit degree, mapped to the fit basis (conversions.py:156-167)
and re-gauged so the last column is zero (heuristics.py:95-125).

On a regular grid (make_grid) the moments are exact integer sums computed by
the CUDA kernel behind ``pgx_label_moments`` (the coordinates are odd
integers / 2M), so the second moments carry no cancellation error; other
point sets use a NumPy bincount.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np

from . import _lib
from .basis import GAUGE_LAST_ZERO, LEGENDRE, MONOMIAL, DesignBasis, MultiIndexSet, ParamMatrix

DEGENERATE_EIG = 1e-10  # heuristics.py:19-23
RIDGE_SCALE = 1e-6


@dataclass(frozen=True)
class MomentSummary:
    """heuristics.MomentSummary (heuristics.py:26-43)."""

    counts: np.ndarray
    centroids: np.ndarray
    second_moments: np.ndarray
    empty: np.ndarray
    degenerate: np.ndarray

    @property
    def n_grains(self) -> int:
        return self.counts.shape[0]


def _sym2x2_eigvals(b: np.ndarray) -> np.ndarray:
    """Ascending eigenvalues of symmetric 2x2 matrices (geometry.py:186-198)."""
    a, off, c = b[..., 0, 0], 0.5 * (b[..., 0, 1] + b[..., 1, 0]), b[..., 1, 1]
    half_tr = 0.5 * (a + c)
    disc = np.sqrt(0.25 * (a - c) ** 2 + off * off)
    return np.stack([half_tr - disc, half_tr + disc], axis=-1)


def label_moment_sums(grid, labels0: np.ndarray, n_grains: int, problem=None) -> np.ndarray | None:
    """(N, 6) int64 sums of {1, a1, a2, a1^2, a1 a2, a2^2} per grain with
    a = 2M x, on the device (regular 2-D grids); None for other point sets.
    With ``problem`` (a Problem holding these labels) the sums come from its
    device-resident labels: no upload, no allocation."""
    from .objective import _grid_spec

    dim, res, _ = _grid_spec(grid)  # res > 0 only for make_grid's regular grid
    if dim != 2 or not res:
        return None
    if problem is not None:
        return problem.label_moments()
    labels0 = np.ascontiguousarray(labels0, dtype=np.int64)
    if labels0.shape[0] != 4 * int(res) ** 2:
        return None
    lib = _lib.load()
    out = np.zeros((n_grains, 6), dtype=np.int64)
    st = lib.pgx_label_moments(int(res), labels0.shape[0], labels0.ctypes.data, int(n_grains),
                               out.ctypes.data)
    if st != _lib.PGX_OK:
        msg = lib.pgx_label_moments_error().decode()
        raise ValueError(msg) if st == _lib.PGX_ERR_INVALID_ARGUMENT else RuntimeError(msg)
    return out


def moments(grain_map, problem=None) -> MomentSummary:
    """Pixel counts, centroids and central second-moment matrices per grain
    (heuristics.py:46-73)."""
    n = int(grain_map.n_grains)
    lab0 = np.asarray(grain_map.labels, dtype=np.int64) - 1
    sums = label_moment_sums(grain_map.grid, lab0, n, problem)
    if sums is not None:
        m2 = int(round(math.sqrt(lab0.shape[0])))  # 2M
        counts = sums[:, 0].copy()
        empty = counts == 0
        safe = np.where(empty, 1, counts)
        centroids = np.column_stack([sums[:, 1] / (safe * m2), sums[:, 2] / (safe * m2)])
        # central moments from exact integers: (n S_ab - S_a S_b) / (n^2 (2M)^2)
        b = np.zeros((n, 2, 2))
        for i in np.nonzero(~empty)[0]:
            c, s1, s2, s11, s12, s22 = (int(v) for v in sums[i])
            den = c * c * m2 * m2
            b[i, 0, 0] = (c * s11 - s1 * s1) / den
            b[i, 0, 1] = b[i, 1, 0] = (c * s12 - s1 * s2) / den
            b[i, 1, 1] = (c * s22 - s2 * s2) / den
    else:  # a point list: the reference's bincount form
        pts = np.asarray(grain_map.grid.points, dtype=np.float64)
        x1, x2 = pts[:, 0], pts[:, 1]
        counts = np.bincount(lab0, minlength=n)
        empty = counts == 0
        safe = np.where(empty, 1, counts).astype(np.float64)
        centroids = np.column_stack([np.bincount(lab0, weights=x1, minlength=n) / safe,
                                     np.bincount(lab0, weights=x2, minlength=n) / safe])
        q = [np.bincount(lab0, weights=w, minlength=n) / safe for w in (x1 * x1, x1 * x2, x2 * x2)]
        b = np.empty((n, 2, 2))
        b[:, 0, 0] = q[0] - centroids[:, 0] ** 2
        b[:, 0, 1] = b[:, 1, 0] = q[1] - centroids[:, 0] * centroids[:, 1]
        b[:, 1, 1] = q[2] - centroids[:, 1] ** 2
    centroids[empty] = 0.0
    b[empty] = 0.0
    degenerate = (_sym2x2_eigvals(b)[:, 0] < DEGENERATE_EIG) | empty
    return MomentSummary(counts=counts, centroids=centroids, second_moments=b, empty=empty,
                         degenerate=degenerate)


def _invert_spread(summary: MomentSummary) -> np.ndarray:
    """Anisotropy guesses B^{-1}, ridge-regularising degenerate spreads (heuristics.py:76-92)."""
    b = summary.second_moments.copy()
    b[summary.empty] = np.eye(2)
    for i in np.nonzero(summary.degenerate & ~summary.empty)[0]:
        tr = b[i, 0, 0] + b[i, 1, 1]
        ridge = RIDGE_SCALE * (tr / 2.0 if tr > 0 else 1.0)
        b[i, 0, 0] += ridge
        b[i, 1, 1] += ridge
    det = b[:, 0, 0] * b[:, 1, 1] - b[:, 0, 1] * b[:, 1, 0]
    inv = np.empty_like(b)
    inv[:, 0, 0] = b[:, 1, 1] / det
    inv[:, 0, 1] = -b[:, 0, 1] / det
    inv[:, 1, 0] = -b[:, 1, 0] / det
    inv[:, 1, 1] = b[:, 0, 0] / det
    inv[summary.empty] = np.eye(2)
    return inv


@lru_cache(maxsize=None)
def _legendre_monomial_rows(degree: int) -> tuple:
    """Exact monomial coefficients of P_0..P_d ((m+1) P_{m+1} = (2m+1) t P_m - m P_{m-1})."""
    rows = [(Fraction(1),)]
    if degree >= 1:
        rows.append((Fraction(0), Fraction(1)))
    for m in range(1, degree):
        nxt = [Fraction(0)] * (m + 2)
        for j, c in enumerate(rows[m]):
            nxt[j + 1] += (2 * m + 1) * c
        for j, c in enumerate(rows[m - 1]):
            nxt[j] -= m * c
        rows.append(tuple(c / (m + 1) for c in nxt))
    return tuple(rows[: degree + 1])


@lru_cache(maxsize=None)
def monomial_to_legendre(degree: int) -> np.ndarray:
    """T with theta_leg = T theta_mono for equal costs (conversions.py:156-167,
    basis.py:196-267): with eta_leg = B eta_mono (B lower triangular in the
    graded-lex order), theta_mono = B^T theta_leg, so T = (B^T)^{-1}; inverted
    exactly over the rationals, rounded once."""
    idx = MultiIndexSet.for_degree(degree).indices
    k = len(idx)
    pos = {a: i for i, a in enumerate(idx)}
    uni = _legendre_monomial_rows(degree)
    bm = [[Fraction(0)] * k for _ in range(k)]
    for r, (a1, a2) in enumerate(idx):
        for b1, c1 in enumerate(uni[a1]):
            for b2, c2 in enumerate(uni[a2]):
                if c1 and c2:
                    bm[r][pos[(b1, b2)]] = c1 * c2
    inv = [[Fraction(0)] * k for _ in range(k)]  # B^{-1} by forward substitution
    for col in range(k):
        for r in range(k):
            s = Fraction(int(r == col))
            for j in range(r):
                if bm[r][j]:
                    s -= bm[r][j] * inv[j][col]
            inv[r][col] = s / bm[r][r]
    t = np.array([[float(inv[j][i]) for j in range(k)] for i in range(k)])  # (B^{-1})^T
    t.setflags(write=False)
    return t


def _monomial_theta(summary: MomentSummary, degree: int, n_pixels: int) -> np.ndarray:
    """Degree-1 (power diagram) or degree-2 (anisotropic) monomial coefficients
    of the moment guess (pd_to_theta / apd_to_theta, conversions.py:52-96)."""
    n = summary.n_grains
    area = np.where(summary.empty, 0.0, summary.counts / (n_pixels * np.pi))
    y1, y2 = summary.centroids[:, 0], summary.centroids[:, 1]
    idx = MultiIndexSet.for_degree(1 if degree == 1 else 2)
    theta = np.zeros((len(idx), n))
    if degree == 1:
        theta[idx.position((1, 0))] = -2.0 * y1
        theta[idx.position((0, 1))] = -2.0 * y2
        theta[idx.position((0, 0))] = y1 * y1 + y2 * y2 - area
        return theta
    mats = _invert_spread(summary)
    det = mats[:, 0, 0] * mats[:, 1, 1] - mats[:, 0, 1] * mats[:, 1, 0]
    w = np.where(summary.empty, 0.0, np.sqrt(np.maximum(det, 0.0)) * area)
    a11, a12, a22 = mats[:, 0, 0], 0.5 * (mats[:, 0, 1] + mats[:, 1, 0]), mats[:, 1, 1]
    theta[idx.position((2, 0))] = a11
    theta[idx.position((1, 1))] = 2.0 * a12
    theta[idx.position((0, 2))] = a22
    theta[idx.position((1, 0))] = -2.0 * (a11 * y1 + a12 * y2)
    theta[idx.position((0, 1))] = -2.0 * (a12 * y1 + a22 * y2)
    theta[idx.position((0, 0))] = y1 * (a11 * y1 + a12 * y2) + y2 * (a12 * y1 + a22 * y2) - w
    return theta


def heuristic_theta(grain_map, degree: int, kind: str = LEGENDRE, *, problem=None) -> ParamMatrix:
    """Moment-based initial coefficients for a degree-d fit, gauge-fixed
    (heuristics.py:95-125)."""
    if degree < 1:
        raise ValueError("heuristic initialisation needs degree >= 1")
    if kind not in (LEGENDRE, MONOMIAL):
        raise ValueError(f"unknown basis kind {kind!r}")
    summary = moments(grain_map, problem)
    mono = _monomial_theta(summary, degree, len(grain_map.labels))
    padded = np.zeros((math.comb(degree + 2, 2), summary.n_grains))  # zero_pad (basis.py:330-344)
    padded[: mono.shape[0]] = mono
    vals = monomial_to_legendre(degree) @ padded if kind == LEGENDRE else padded
    vals = vals - vals[:, -1][:, None]
    return ParamMatrix(values=vals, basis=DesignBasis.make(kind, degree), gauge=GAUGE_LAST_ZERO)
