"""NumPy fp64 restatement of the polygrain hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates
(reference = ``/root/reference/pkg/src/polygrain``).  Nothing in the product
package imports this module.

Extensions (not in the reference):
  * ``dim == 3`` grids and 3-D total-degree bases (ordering: total degree
    ascending, then a1 descending, then a2 descending);
  * ``lam`` (lambda) penalty  Phi_lam = Phi - lam/2 * ||theta[:, :N-1]||_F^2,
    grad[:, :N-1] -= lam * theta[:, :N-1]; ``lam == 0`` is the reference.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from typing import NamedTuple

import numpy as np

__all__ = [
    "TIE_RTOL", "CHUNK_SIZE", "LEGENDRE", "MONOMIAL",
    "grid_axis", "grid_points", "multi_indices", "feature_count",
    "legendre_table", "power_table", "design_values",
    "argmin_labels", "top2_margin",
    "OracleResult", "evaluate_objective", "evaluate_problem",
    "hard_assign_points", "label_moments",
]

# geometry.py:19 — tie tolerance of the arg-min, relative to (1 + |min|)
TIE_RTOL = 1e-12
# objective.py:30 — pixel chunk of the streamed evaluation
CHUNK_SIZE = 8192
LEGENDRE = "legendre"
MONOMIAL = "monomial"


# --------------------------------------------------------------------------- grid
def grid_axis(m: int) -> np.ndarray:
    """Pixel-centre coordinates of one axis: -1 + (k - 1/2)/M, k = 1..2M
    (geometry.py:68)."""
    m = int(m)
    if m < 1:
        raise ValueError("grid resolution M must be >= 1")
    return -1.0 + (np.arange(1, 2 * m + 1) - 0.5) / m


def grid_points(m: int, dim: int = 2) -> np.ndarray:
    """Regular grid, row-major with the first axis slowest (geometry.py:69-70:
    ``x1 = repeat``, ``x2 = tile``).  ``dim == 3`` is the Appendix-B extension:
    row-major in (k1, k2, k3)."""
    c = grid_axis(m)
    if dim == 2:
        return np.column_stack([np.repeat(c, c.size), np.tile(c, c.size)])
    if dim == 3:
        n = c.size
        return np.column_stack([
            np.repeat(c, n * n),
            np.tile(np.repeat(c, n), n),
            np.tile(c, n * n),
        ])
    raise ValueError("dim must be 2 or 3")


# -------------------------------------------------------------------------- basis
def feature_count(degree: int, dim: int = 2) -> int:
    """K = C(d+dim, dim); dim 2 gives (d+1)(d+2)/2 (basis.py:37-39)."""
    return math.comb(degree + dim, dim)


def multi_indices(degree: int, dim: int = 2) -> tuple:
    """Graded-lex, a1 descending (basis.py:42-48); for dim 3 ties in a1 are
    broken by a2 descending."""
    out = []
    for total in range(degree + 1):
        if dim == 2:
            for a1 in range(total, -1, -1):
                out.append((a1, total - a1))
        else:
            for a1 in range(total, -1, -1):
                for a2 in range(total - a1, -1, -1):
                    out.append((a1, a2, total - a1 - a2))
    return tuple(out)


def legendre_table(degree: int, t: np.ndarray) -> np.ndarray:
    """P_0..P_d by (m+1)P_{m+1} = (2m+1) t P_m - m P_{m-1} (basis.py:128-142)."""
    t = np.asarray(t, dtype=np.float64)
    out = np.empty((degree + 1,) + t.shape)
    out[0] = 1.0
    if degree >= 1:
        out[1] = t
    for m in range(1, degree):
        out[m + 1] = ((2 * m + 1) * t * out[m] - m * out[m - 1]) / (m + 1)
    return out


def power_table(degree: int, t: np.ndarray) -> np.ndarray:
    """1, t, t^2, ... by repeated multiplication (basis.py:120-125)."""
    t = np.asarray(t, dtype=np.float64)
    out = np.empty((degree + 1,) + t.shape)
    out[0] = 1.0
    for k in range(1, degree + 1):
        out[k] = out[k - 1] * t
    return out


def design_values(kind: str, degree: int, points: np.ndarray) -> np.ndarray:
    """Feature matrix (K, n): row alpha = prod_j u[a_j](x_j) (basis.py:105-117)."""
    points = np.asarray(points, dtype=np.float64)
    dim = points.shape[1]
    table = legendre_table if kind == LEGENDRE else power_table
    u = [table(degree, points[:, j]) for j in range(dim)]
    rows = []
    for alpha in multi_indices(degree, dim):
        r = u[0][alpha[0]] * u[1][alpha[1]]
        if dim == 3:
            r = r * u[2][alpha[2]]
        rows.append(r)
    return np.asarray(rows)


# ------------------------------------------------------------------------ arg-min
def argmin_labels(costs: np.ndarray) -> np.ndarray:
    """1-based smallest index with cost <= min + TIE_RTOL (1 + |min|)
    (geometry.py:201-210)."""
    m = costs.min(axis=0)
    thr = m + TIE_RTOL * (1.0 + np.abs(m))
    return np.argmax(costs <= thr, axis=0).astype(np.int64) + 1


def top2_margin(costs: np.ndarray) -> np.ndarray:
    """Second-smallest minus smallest cost per column (extension: the
    north_star's ambiguity measure)."""
    if costs.shape[0] < 2:
        return np.full(costs.shape[1], np.inf)
    part = np.partition(costs, 1, axis=0)
    return part[1] - part[0]


# ---------------------------------------------------------------------- objective
class OracleResult(NamedTuple):
    """Mirror of objective.EvalResult (objective.py:90-94) plus counters."""

    phi: float
    grad: np.ndarray | None
    err: float | None
    e0: float | None
    n_correct: int | None


def _chunk_stats(theta, d, g0, eps, want_grad, want_assign):
    # objective.py:97-120, one chunk of pixels (columns of d)
    c = theta.T @ d
    cols = np.arange(c.shape[1])
    m = c.min(axis=0)
    z = (m[None, :] - c) / eps
    e = np.exp(z)
    s = e.sum(axis=0)
    lse_sum = float(z[g0, cols].sum() - np.log(s).sum())
    gacc = None
    if want_grad:
        r = -(e / s[None, :])
        r[g0, cols] += 1.0
        gacc = d @ r.T
    ncorrect = 0
    e0_sum = 0.0
    if want_assign:
        ncorrect = int(np.count_nonzero(argmin_labels(c) - 1 == g0))
        e0_sum = float((c[g0, cols] - m).sum())
    return lse_sum, gacc, ncorrect, e0_sum


def _combine(a, b):
    # objective.py:123-126
    return (a[0] + b[0], None if a[1] is None else a[1] + b[1], a[2] + b[2], a[3] + b[3])


def _reduce(parts):
    # objective.py:146-158: fixed pairwise tree over chunk partials
    while len(parts) > 1:
        parts = [_combine(parts[i], parts[i + 1]) if i + 1 < len(parts) else parts[i]
                 for i in range(0, len(parts), 2)]
    return parts[0]


def _finish(total, n, eps, theta, want_grad, want_assign, lam):
    # objective.py:160-165 (+ lambda extension)
    lse_sum, gacc, ncorrect, e0_sum = total
    phi = lse_sum / n
    grad = -gacc / (eps * n) if want_grad else None
    if lam:
        free = theta[:, :-1]
        phi -= 0.5 * lam * float((free * free).sum())
        if grad is not None:
            grad[:, :-1] -= lam * free
    err = 1.0 - float(ncorrect) / n if want_assign else None
    e0 = e0_sum / n if want_assign else None
    return OracleResult(phi, grad, err, e0, ncorrect if want_assign else None)


def evaluate_objective(theta_values, design_values_, labels0, eps, *, want_grad=True,
                       want_assign=False, threads=1, chunk_size=CHUNK_SIZE,
                       lam=0.0) -> OracleResult:
    """Restatement of objective.evaluate_objective (objective.py:129-165)."""
    theta = np.asarray(theta_values, dtype=np.float64)
    design = np.asarray(design_values_, dtype=np.float64)
    labels0 = np.asarray(labels0)
    n = design.shape[1]
    slices = [slice(lo, min(lo + chunk_size, n)) for lo in range(0, n, chunk_size)]

    def stats(sl):
        return _chunk_stats(theta, design[:, sl], labels0[sl], eps, want_grad, want_assign)

    if threads > 1 and len(slices) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            total = _reduce(list(pool.map(stats, slices)))
    else:
        total = stats(slices[0])
        for sl in slices[1:]:
            total = _combine(total, stats(sl))
    return _finish(total, n, eps, theta, want_grad, want_assign, lam)


def evaluate_problem(theta_values, kind, degree, points, labels0, eps, *, want_grad=True,
                     want_assign=False, threads=1, chunk_size=CHUNK_SIZE, lam=0.0,
                     max_points=None) -> OracleResult:
    """Same as ``evaluate_objective`` but the design chunk is generated on the fly
    from the points (the (K, P) design of basis.py:183-193 is never held whole),
    so c3..c5-sized point sets fit in host memory.  ``max_points`` evaluates only
    a prefix (bounded CPU-baseline samples); the normalisation then uses the
    prefix size."""
    theta = np.asarray(theta_values, dtype=np.float64)
    points = np.asarray(points, dtype=np.float64)
    labels0 = np.asarray(labels0)
    n = points.shape[0] if max_points is None else min(points.shape[0], int(max_points))
    slices = [slice(lo, min(lo + chunk_size, n)) for lo in range(0, n, chunk_size)]

    def stats(sl):
        d = design_values(kind, degree, points[sl])
        return _chunk_stats(theta, d, labels0[sl], eps, want_grad, want_assign)

    if threads > 1 and len(slices) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            total = _reduce(list(pool.map(stats, slices)))
    else:
        total = stats(slices[0])
        for sl in slices[1:]:
            total = _combine(total, stats(sl))
    return _finish(total, n, eps, theta, want_grad, want_assign, lam)


def hard_assign_points(theta_values, kind, degree, points, chunk_size=CHUNK_SIZE,
                       with_margin=False):
    """objective.hard_assign (objective.py:70-77) without the whole N x P cost
    matrix: the arg-min is column-independent, so chunking is exact."""
    theta = np.asarray(theta_values, dtype=np.float64)
    points = np.asarray(points, dtype=np.float64)
    n = points.shape[0]
    labels = np.empty(n, dtype=np.int64)
    margin = np.empty(n) if with_margin else None
    for lo in range(0, n, chunk_size):
        hi = min(lo + chunk_size, n)
        c = theta.T @ design_values(kind, degree, points[lo:hi])
        labels[lo:hi] = argmin_labels(c)
        if with_margin:
            margin[lo:hi] = top2_margin(c)
    return (labels, margin) if with_margin else labels


def label_moments(kind, degree, points, labels0, n_grains):
    """M_i = sum_{x in G_i} eta(x) (K, N) — the theta = 0 closed form of the
    gradient is -(M - sum_x eta(x)/N)/(eps P)."""
    d = design_values(kind, degree, points)
    out = np.zeros((d.shape[0], n_grains))
    for k in range(d.shape[0]):
        out[k] = np.bincount(labels0, weights=d[k], minlength=n_grains)
    return out
