"""Seeded synthetic workloads c1..c5 of BASELINE.json.

The paper's EBSD maps are proprietary and absent; these seeded
synthetic grain maps with the configs' shapes stand in for them.  Label maps
are the tie-tolerant arg-min of a generator cost (geometry.py:201-248): a
power / anisotropic power diagram written as a degree-1/2 monomial polynomial
(conversions.py:52-96 form) or a random degree-d Legendre diagram, then the
label noise of Appendix B.  The arg-min runs on the GPU (``labeler="gpu"``,
pgx_assign in exact mode) or, for small grids, chunked on the host.

All randomness is ``numpy.random.default_rng(seed)``; draw order is the
order of the code below.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .basis import LEGENDRE, MONOMIAL, graded_lex_indices
from .geometry import PixelGrid, grid_axis, make_grid


@dataclass
class Workload:
    name: str
    dim: int
    M: int
    n_grains: int
    kind: str
    degree: int
    eps: float
    lam: float
    labels0: np.ndarray          # int64, 0-based
    theta_bench: np.ndarray      # (K, N) theta the throughput is measured at
    theta_dtype: str
    grid: PixelGrid
    description: str
    n_nonempty: int = 0

    @property
    def n_points(self) -> int:
        return len(self.grid)

    @property
    def K(self) -> int:
        return math.comb(self.degree + self.dim, self.dim)

    @property
    def logits(self) -> int:
        return self.n_points * self.n_grains


# ------------------------------------------------------------------ helpers
def _host_tables(kind, degree, t):
    out = np.empty((degree + 1,) + t.shape)
    out[0] = 1.0
    if degree >= 1:
        out[1] = t
    for m in range(1, degree):
        out[m + 1] = (((2 * m + 1) * t * out[m] - m * out[m - 1]) / (m + 1)
                      if kind == LEGENDRE else out[m] * t)
    return out


def host_assign(theta, kind, degree, dim, M, chunk=8192, rows=None):
    """Chunked host arg-min (input preparation for small grids only; the
    product path is pgx_assign).  ``rows`` limits it to a pixel prefix."""
    theta = np.asarray(theta, dtype=np.float64)
    c = grid_axis(M)
    side = c.size
    n = side ** dim if rows is None else int(rows)
    idx = graded_lex_indices(degree, dim)
    out = np.empty(n, dtype=np.int64)
    for lo in range(0, n, chunk):
        p = np.arange(lo, min(n, lo + chunk))
        if dim == 2:
            xs = [c[p // side], c[p % side]]
        else:
            xs = [c[p // (side * side)], c[(p // side) % side], c[p % side]]
        us = [_host_tables(kind, degree, x) for x in xs]
        d = np.asarray([np.prod([us[j][a[j]] for j in range(dim)], axis=0) for a in idx])
        cost = theta.T @ d
        m = cost.min(axis=0)
        out[lo:lo + len(p)] = np.argmax(cost <= m + 1e-12 * (1.0 + np.abs(m)), axis=0)
    return out


def gpu_assign(theta, kind, degree, dim, M):
    from .objective import Problem

    grid = make_grid(M, dim)
    prob = Problem(grid, kind, degree, theta.shape[1], None, precision="exact")
    try:
        return prob.assign(np.asarray(theta, dtype=np.float64)) - 1
    finally:
        prob.close()


def _assign(theta, kind, degree, dim, M, labeler):
    if labeler == "gpu":
        return gpu_assign(theta, kind, degree, dim, M)
    return host_assign(theta, kind, degree, dim, M)


def _pd_theta(seeds, weights):
    # |x - y|^2 - w minus the grain-independent |x|^2 (degree-1 monomial, 2-D)
    th = np.empty((3, seeds.shape[0]))
    th[0] = (seeds ** 2).sum(axis=1) - weights
    th[1] = -2.0 * seeds[:, 0]
    th[2] = -2.0 * seeds[:, 1]
    return th


def _apd_theta(seeds, weights, mats):
    """(x-y)^T A (x-y) - w as a degree-2 monomial theta (any dim)."""
    n, dim = seeds.shape
    idx = graded_lex_indices(2, dim)
    pos = {a: k for k, a in enumerate(idx)}
    ay = np.einsum("nij,nj->ni", mats, seeds)
    th = np.zeros((len(idx), n))
    zero = (0,) * dim
    th[pos[zero]] = (seeds * ay).sum(axis=1) - weights
    for j in range(dim):
        e = [0] * dim
        e[j] = 1
        th[pos[tuple(e)]] = -2.0 * ay[:, j]
        e[j] = 2
        th[pos[tuple(e)]] = mats[:, j, j]
        for l in range(j + 1, dim):
            e = [0] * dim
            e[j] = e[l] = 1
            th[pos[tuple(e)]] = mats[:, j, l] + mats[:, l, j]
    return th


def _grid_neighbour_pairs(labels, side, dim):
    """Pairs of 4- (6-) neighbouring pixels with differing labels."""
    lab = labels.reshape((side,) * dim)
    pairs = []
    for ax in range(dim):
        a = np.take(lab, np.arange(side - 1), axis=ax)
        b = np.take(lab, np.arange(1, side), axis=ax)
        pairs.append((a.ravel(), b.ravel()))
    return pairs


def _noise_neighbour_grain(rng, labels, side, frac, n_grains):
    """Appendix B (c2): relabel frac of all pixels to a random grain adjacent
    (4-neighbour edge) to the pixel's grain."""
    adj = [set() for _ in range(n_grains)]
    for a, b in _grid_neighbour_pairs(labels, side, 2):
        diff = a != b
        for u, v in zip(a[diff].tolist(), b[diff].tolist()):
            adj[u].add(v)
            adj[v].add(u)
    nbrs = [sorted(s) for s in adj]
    n = labels.size
    pick = rng.choice(n, size=int(round(frac * n)), replace=False)
    out = labels.copy()
    u = rng.random(pick.size)
    for j, p in enumerate(pick.tolist()):
        nb = nbrs[labels[p]]
        if nb:
            out[p] = nb[int(u[j] * len(nb))]
    return out


def _noise_boundary(rng, labels, side, frac):
    """Appendix B (c3/c5): round(frac P) pixels chosen uniformly among pixels
    with a differing 4-neighbour, each relabelled to a differing neighbour's label."""
    lab = labels.reshape(side, side)
    nb = np.full((4,) + lab.shape, -1, dtype=np.int64)
    nb[0, 1:, :] = lab[:-1, :]
    nb[1, :-1, :] = lab[1:, :]
    nb[2, :, 1:] = lab[:, :-1]
    nb[3, :, :-1] = lab[:, 1:]
    diff = (nb >= 0) & (nb != lab[None])
    boundary = np.flatnonzero(diff.any(axis=0).ravel())
    k = min(boundary.size, int(round(frac * labels.size)))
    pick = rng.choice(boundary, size=k, replace=False)
    out = labels.copy()
    d = diff.reshape(4, -1)[:, pick]
    v = nb.reshape(4, -1)[:, pick]
    u = rng.random(k)
    for j in range(k):
        choices = v[d[:, j], j]
        out[pick[j]] = choices[int(u[j] * choices.size)]
    return out


def _log_uniform(rng, lo, hi, size):
    return np.exp(rng.uniform(math.log(lo), math.log(hi), size))


def _rotation2(phi):
    c, s = np.cos(phi), np.sin(phi)
    return np.stack([np.stack([c, -s], -1), np.stack([s, c], -1)], -2)


def _haar3(rng, n):
    q, r = np.linalg.qr(rng.normal(size=(n, 3, 3)))
    return q * np.sign(np.diagonal(r, axis1=1, axis2=2))[:, None, :]


def _bench_theta(rng, K, N, dtype):
    th = 0.01 * rng.normal(size=(K, N))
    return th.astype(np.float32) if dtype == "f32" else th


# ------------------------------------------------------------------ configs
def c1(labeler="host", seed=1):
    rng = np.random.default_rng(seed)
    M, N = 64, 20
    seeds = rng.uniform(-1.0, 1.0, (N, 2))
    labels = _assign(_pd_theta(seeds, np.zeros(N)), MONOMIAL, 1, 2, M, labeler)
    th = _bench_theta(rng, 3, N, "f64")
    return Workload("c1", 2, M, N, LEGENDRE, 1, 0.05, 1e-4, labels, th, "f64", make_grid(M),
                    "2D 128x128, Voronoi N=20, Legendre d=1 (K=3), eps=0.05, lam=1e-4",
                    int(np.unique(labels).size))


def c2(labeler="host", seed=2):
    rng = np.random.default_rng(seed)
    M, N = 256, 200
    seeds = rng.uniform(-1.0, 1.0, (N, 2))
    weights = rng.normal(0.0, 0.01, N)
    phi = rng.uniform(0.0, math.pi, N)
    s = _log_uniform(rng, 0.5, 2.0, (N, 2))
    R = _rotation2(phi)
    A = np.einsum("nij,nj,nkj->nik", R, s, R)
    labels = _assign(_apd_theta(seeds, weights, A), MONOMIAL, 2, 2, M, labeler)
    labels = _noise_neighbour_grain(rng, labels, 2 * M, 0.02, N)
    th = _bench_theta(rng, 6, N, "f32")
    return Workload("c2", 2, M, N, LEGENDRE, 2, 0.02, 1e-4, labels, th, "f32", make_grid(M),
                    "2D 512x512, APD N=200 + 2% neighbour-grain noise, Legendre d=2 (K=6), "
                    "eps=0.02, lam=1e-4, fp32 theta", int(np.unique(labels).size))


def c3(labeler="gpu", seed=3):
    rng = np.random.default_rng(seed)
    M, N, d = 512, 1000, 4
    theta_true = rng.normal(size=(15, N))
    labels = _assign(theta_true, LEGENDRE, d, 2, M, labeler)
    labels = _noise_boundary(rng, labels, 2 * M, 0.01)
    th = _bench_theta(rng, 15, N, "f64")
    return Workload("c3", 2, M, N, LEGENDRE, d, 0.01, 1e-5, labels, th, "f64", make_grid(M),
                    "2D 1024x1024, degree-4 polynomial diagram N=1000 + 1% boundary noise, "
                    "Legendre d=4 (K=15), eps=0.01, lam=1e-5", int(np.unique(labels).size))


def c4(labeler="gpu", seed=4):
    rng = np.random.default_rng(seed)
    M, N = 64, 2000
    seeds = rng.uniform(-1.0, 1.0, (N, 3))
    weights = rng.normal(0.0, 0.01, N)
    R = _haar3(rng, N)
    s = _log_uniform(rng, 0.5, 2.0, (N, 3))
    A = np.einsum("nij,nj,nkj->nik", R, s, R)
    labels = _assign(_apd_theta(seeds, weights, A), MONOMIAL, 2, 3, M, labeler)
    th = _bench_theta(rng, 10, N, "f64")
    return Workload("c4", 3, M, N, LEGENDRE, 2, 0.02, 1e-4, labels, th, "f64", make_grid(M, 3),
                    "3D 128^3, APD N=2000 (Haar rotations), 3-D Legendre d=2 (K=10), "
                    "eps=0.02, lam=1e-4", int(np.unique(labels).size))


def c5(labeler="gpu", seed=5):
    rng = np.random.default_rng(seed)
    M, N, d = 1024, 4096, 8
    theta_true = rng.normal(size=(45, N))
    labels = _assign(theta_true, LEGENDRE, d, 2, M, labeler)
    labels = _noise_boundary(rng, labels, 2 * M, 0.01)
    th = _bench_theta(rng, 45, N, "f64")
    return Workload("c5", 2, M, N, LEGENDRE, d, 0.005, 1e-5, labels, th, "f64", make_grid(M),
                    "2D 2048x2048, degree-8 polynomial diagram N=4096 + 1% boundary noise, "
                    "Legendre d=8 (K=45), eps=0.005, lam=1e-5", int(np.unique(labels).size))


def paper140(labeler="host", seed=14):
    """The shape of the paper's own reconstruction experiment (Fig. 4:
    |Omega| = 19,600 = 140 x 140 pixels, N = 50 cells, 2nd-degree fit, eps = 0.01) on a
    seeded synthetic anisotropic power diagram; a side that is not a multiple of 128."""
    rng = np.random.default_rng(seed)
    M, N = 70, 50
    seeds = rng.uniform(-1.0, 1.0, (N, 2))
    weights = rng.normal(0.0, 0.01, N)
    s = _log_uniform(rng, 0.5, 2.0, (N, 2))
    R = _rotation2(rng.uniform(0.0, math.pi, N))
    A = np.einsum("nij,nj,nkj->nik", R, s, R)
    labels = _assign(_apd_theta(seeds, weights, A), MONOMIAL, 2, 2, M, labeler)
    th = _bench_theta(rng, 6, N, "f64")
    return Workload("paper140", 2, M, N, LEGENDRE, 2, 0.01, 0.0, labels, th, "f64", make_grid(M),
                    "2D 140x140 (|Omega| = 19,600), anisotropic power diagram N=50, Legendre d=2 "
                    "(K=6), eps=0.01 (the paper's reconstruction experiment shape)",
                    int(np.unique(labels).size))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5, "paper140": paper140}


def make(name: str, labeler: str | None = None) -> Workload:
    fn = CONFIGS[name]
    return fn() if labeler is None else fn(labeler=labeler)
