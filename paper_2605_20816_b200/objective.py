"""Drop-in objective / gradient / assignment surface backed by libpgx.so.

Mirrors polygrain/objective.py: ``evaluate_objective`` (objective.py:129-165),
``objective`` (:168-178), ``gradient`` (:181-198), ``hard_assign`` (:70-77),
``energy_zero``/``energy_eps`` (:220-231).  Every number is computed by the
sm_100a kernels behind the C ABI (include/pgx.h); there is no CPU fallback.

The functions accept this package's descriptors *and* the reference's own
objects (duck-typed: ``theta.values``, ``theta.basis.kind/.degree``,
``design.basis``, ``design.grid.points/.resolution``, ``grain_map.labels``),
so a polygrain user can route calls here unchanged.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from typing import NamedTuple

import numpy as np

from . import _lib
from .basis import GAUGE_LAST_ZERO, LEGENDRE, MONOMIAL

CHUNK_SIZE = 8192  # accepted for signature parity (objective.py:30); unused on the GPU
DEFAULT_PRECISION = os.environ.get("PGX_PRECISION", "tc")


class EvalResult(NamedTuple):
    """objective.EvalResult (objective.py:90-94)."""

    phi: float
    grad: np.ndarray | None
    err: float | None
    e0: float | None


class EvalStats(NamedTuple):
    phi: float
    err: float
    e0: float
    n_points: int
    n_correct: int
    n_ambiguous: int
    n_nonfinite: int
    n_rescanned: int = 0
    flags: int = 0


def _basis_key(basis):
    kind = getattr(basis, "kind")
    degree = int(getattr(basis, "degree"))
    dim = int(getattr(basis, "dim", 2))
    return kind, degree, dim


def _grid_spec(grid):
    """(dim, resolution, points-or-None) for this package's or the reference's grid."""
    res = getattr(grid, "resolution", None)
    dim = getattr(grid, "dim", None)
    if res is not None:
        res = int(res)
        pts = getattr(grid, "_points", None)
        if dim is None:  # reference PixelGrid: points are materialised; dim is 2
            pts = np.asarray(grid.points)
            dim = pts.shape[1]
        if pts is not None and pts.shape[0] <= 1 << 22:
            # a regular grid is regenerated on the device: make sure the points
            # really are make_grid's (geometry.py:68-70)
            c = -1.0 + (np.arange(1, 2 * res + 1) - 0.5) / res
            ok = (np.array_equal(pts[:, 0], np.repeat(c, pts.shape[0] // c.size))
                  and np.array_equal(pts[:, -1], np.tile(c, pts.shape[0] // c.size)))
            if not ok:
                return dim, 0, np.ascontiguousarray(pts, dtype=np.float64)
        return int(dim), res, None
    pts = np.ascontiguousarray(np.asarray(grid.points, dtype=np.float64))
    return pts.shape[1], 0, pts


class Problem:
    """A device-resident problem: grid/points + basis + labels (pgx_problem_create).

    Created once per fit (labels are fixed, optimizer.py:205-207); every
    evaluation then only moves theta down and (Phi, grad, err, e0) back.
    """

    def __init__(self, grid, basis_kind: str, degree: int, n_grains: int, labels0=None, *,
                 precision: str | None = None, device: int = 0, stream: int | None = None,
                 dim: int | None = None, design=None):
        lib = _lib.load()
        if design is not None:  # explicit (K, P) design matrix (objective.py:129-132 form)
            self._init_design(lib, design, n_grains, labels0, device, stream)
            return
        gdim, res, pts = _grid_spec(grid)
        if dim is not None and dim != gdim:
            raise ValueError(f"grid dimension {gdim} != requested {dim}")
        self.dim = gdim
        self.resolution = res
        self.n_points = len(grid) if pts is None else pts.shape[0]
        self.n_grains = int(n_grains)
        self.basis_kind = basis_kind
        self.degree = int(degree)
        self.K = math.comb(self.degree + gdim, gdim)
        self.precision = precision or DEFAULT_PRECISION
        if self.precision not in _lib.PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}")
        if basis_kind not in (LEGENDRE, MONOMIAL):
            raise ValueError(f"unknown basis kind {basis_kind!r}")
        self._labels = None
        if labels0 is not None:
            self._labels = np.ascontiguousarray(np.asarray(labels0, dtype=np.int64))
            if self._labels.shape != (self.n_points,):
                raise ValueError(
                    f"labels length {self._labels.shape[0]} != number of grid points {self.n_points}")
        self._points = pts
        desc = _lib.PgxDesc()
        desc.dim = gdim
        desc.basis_kind = _lib.PGX_BASIS_LEGENDRE if basis_kind == LEGENDRE else _lib.PGX_BASIS_MONOMIAL
        desc.degree = self.degree
        desc.n_grains = self.n_grains
        desc.n_points = self.n_points
        desc.resolution = res
        desc.precision = _lib.PRECISIONS[self.precision]
        desc.points = _lib.as_ptr(pts)
        desc.labels0 = _lib.as_ptr(self._labels)
        desc.mem = _lib.PGX_MEM_HOST
        desc.device = int(device)
        desc.stream = stream or 0
        handle = ctypes.c_void_p()
        _lib.check(lib.pgx_problem_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._lib = lib
        self._h = handle
        self._lock = threading.Lock()
        self._stats = _lib.PgxStats()
        self._spec = (grid, basis_kind, degree, self._labels, int(device), stream, gdim)
        self._exact = None

    def _init_design(self, lib, design, n_grains, labels0, device, stream):
        d = np.ascontiguousarray(np.asarray(design, dtype=np.float64))
        if d.ndim != 2:
            raise ValueError("design_values must be a (K, P) matrix")
        self.dim, self.resolution, self.degree, self.basis_kind = 0, 0, -1, None
        self.K, self.n_points = d.shape
        self.n_grains = int(n_grains)
        self.precision = "exact"
        self._labels = None
        if labels0 is not None:
            self._labels = np.ascontiguousarray(np.asarray(labels0, dtype=np.int64))
            if self._labels.shape != (self.n_points,):
                raise ValueError(
                    f"labels length {self._labels.shape[0]} != number of design columns {self.n_points}")
        self._points = None
        self._design = d
        desc = _lib.PgxDesc()
        desc.n_grains = self.n_grains
        desc.n_points = self.n_points
        desc.precision = _lib.PGX_PREC_EXACT
        desc.labels0 = _lib.as_ptr(self._labels)
        desc.mem = _lib.PGX_MEM_HOST
        desc.device = int(device)
        desc.stream = stream or 0
        desc.design = d.ctypes.data
        desc.design_k = self.K
        handle = ctypes.c_void_p()
        _lib.check(lib.pgx_problem_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._lib = lib
        self._h = handle
        self._lock = threading.Lock()
        self._stats = _lib.PgxStats()
        self._spec = None
        self._exact = None

    # ------------------------------------------------------------------ basics
    @property
    def handle(self):
        return self._h

    def close(self):
        for st in list(self.__dict__.get("_fit_states", {}).values()):  # cached optimiser states
            st.close()
        self.__dict__.pop("_fit_states", None)
        if getattr(self, "_exact", None) is not None:
            self._exact.close()
            self._exact = None
        if getattr(self, "_h", None):
            self._lib.pgx_problem_destroy(self._h)
            self._h = None

    # fp32 / fp16-split logits carry ~2^-22 relative error; beyond this bound
    # on |h''| = |theta^T eta| / (eps ln 2) the error would reach 2^-6 in the
    # exponent: the library then flags the result (pgx.h PGX_STAT_RANGE) and,
    # for host buffers, re-evaluates it on the exact kernels itself
    FAST_RANGE = _lib.PGX_FAST_RANGE

    def _exact_problem(self) -> "Problem":
        if self._exact is None:
            grid, kind, degree, labels, device, stream, dim = self._spec
            self._exact = Problem(grid, kind, degree, self.n_grains, labels, precision="exact",
                                  device=device, stream=stream, dim=dim)
        return self._exact

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int):
        _lib.check(self._lib.pgx_set_stream(self._h, stream))

    @property
    def kernel_path(self) -> str:
        """'general', 'grid_fp64' or 'grid_tc' (pgx_problem_path)."""
        return _lib.PATH_NAMES[int(self._lib.pgx_problem_path(self._h))]

    def eval_kernels(self, theta, eps: float, **kw):
        """eval() with kernel-level profiling: (result, stats, [kernel names])."""
        self.set_profiling(True)
        try:
            res, st = self.eval(theta, eps, **kw)
            names = [n for n, _ in self.profile()]
        finally:
            self.set_profiling(False)
        return res, st, names

    def device_bytes(self) -> int:
        """Bytes of device memory the handle holds (pgx_problem_bytes)."""
        return int(self._lib.pgx_problem_bytes(self._h))

    def label_moments(self) -> np.ndarray:
        """(N, 6) exact int64 sums of {1, a1, a2, a1^2, a1 a2, a2^2} per grain over
        the problem's resident labels (pgx_problem_label_moments; regular 2-D
        grids; heuristics.py:46-73 is the bincount form)."""
        out = np.zeros((self.n_grains, 6), dtype=np.int64)
        with self._lock:
            _lib.check(self._lib.pgx_problem_label_moments(self._h, 0, out.ctypes.data))
        return out

    def last_launch_count(self) -> int:
        return int(self._lib.pgx_last_launch_count(self._h))

    def synchronize(self):
        _lib.check(self._lib.pgx_synchronize(self._h))

    def set_profiling(self, enable: bool = True):
        _lib.check(self._lib.pgx_set_profiling(self._h, 1 if enable else 0))

    def profile(self) -> list:
        """[(kernel name, ms)] of the last call (CUDA events on the problem's stream)."""
        n = self._lib.pgx_profile_count(self._h)
        return [(self._lib.pgx_profile_name(self._h, i).decode(),
                 float(self._lib.pgx_profile_ms(self._h, i))) for i in range(n)]

    def _theta(self, theta):
        t = np.asarray(theta)
        if t.shape != (self.K, self.n_grains):
            raise ValueError(f"theta shape {t.shape} != (K={self.K}, N={self.n_grains})")
        if t.dtype == np.float32:
            return np.ascontiguousarray(t), _lib.PGX_THETA_F32
        return np.ascontiguousarray(t, dtype=np.float64), 0

    # ------------------------------------------------------------------ calls
    def eval(self, theta, eps: float, *, lam: float = 0.0, want_grad: bool = True,
             want_assign: bool = False) -> tuple[EvalResult, EvalStats]:
        """One fused evaluation with host buffers (copies inside the call)."""
        t, tflag = self._theta(theta)
        flags = tflag | (_lib.PGX_WANT_GRAD if want_grad else 0) | (
            _lib.PGX_WANT_ASSIGN if want_assign else 0)
        grad = np.empty((self.K, self.n_grains)) if want_grad else None
        with self._lock:
            st = self._stats
            _lib.check(self._lib.pgx_eval(self._h, t.ctypes.data, float(eps), float(lam), flags,
                                          _lib.as_ptr(grad), ctypes.addressof(st)))
            stats = EvalStats(st.phi, st.err, st.e0, st.n_points, st.n_correct, st.n_ambiguous,
                              st.n_nonfinite, int(st.n_rescanned), int(st.flags))
        res = EvalResult(phi=stats.phi, grad=grad,
                         err=stats.err if want_assign else None,
                         e0=stats.e0 if want_assign else None)
        return res, stats

    def eval_device(self, theta_ptr: int, eps: float, lam: float, flags: int, grad_ptr: int,
                    stats_ptr: int) -> None:
        """Asynchronous evaluation on device pointers (PGX_DEVICE_PTRS)."""
        _lib.check(self._lib.pgx_eval(self._h, theta_ptr, float(eps), float(lam),
                                      int(flags) | _lib.PGX_DEVICE_PTRS, grad_ptr, stats_ptr))

    def assign_device(self, theta_ptr: int, flags: int, labels_ptr: int, margin_ptr: int = 0,
                      stats_ptr: int = 0) -> None:
        """Asynchronous hard assignment on device pointers (int64 labels, 1-based)."""
        _lib.check(self._lib.pgx_assign(self._h, theta_ptr, int(flags) | _lib.PGX_DEVICE_PTRS,
                                        labels_ptr, margin_ptr or None, stats_ptr or None))

    def soft_assign(self, theta, eps: float) -> np.ndarray:
        """Dense (N, P) softmax memberships (objective.py:80-87), pgx_soft_assign."""
        if not eps > 0:
            raise ValueError("eps must be positive")
        t, tflag = self._theta(theta)
        prob = np.empty((self.n_grains, self.n_points))
        with self._lock:
            _lib.check(self._lib.pgx_soft_assign(self._h, t.ctypes.data, float(eps), tflag,
                                                 prob.ctypes.data))
        return prob

    def assign(self, theta, *, with_margin: bool = False):
        """Tie-tolerant hard assignment (1-based labels) without the N x P costs."""
        t, tflag = self._theta(theta)  # (tc problems: the sweep's ASSIGN variant; else the exact fp64 kernels)
        labels = np.empty(self.n_points, dtype=np.int64)
        margin = np.empty(self.n_points, dtype=np.float32) if with_margin else None
        with self._lock:
            st = self._stats
            _lib.check(self._lib.pgx_assign(self._h, t.ctypes.data, tflag, labels.ctypes.data,
                                            _lib.as_ptr(margin), ctypes.addressof(st)))
            n_amb = int(st.n_ambiguous)
        return (labels, margin, n_amb) if with_margin else labels


# ---------------------------------------------------------------- problem cache
_CACHE: list = []
_CACHE_MAX = 4
_CACHE_LOCK = threading.Lock()


def problem_for(design, labels0, n_grains: int, precision: str | None = None) -> Problem:
    """Problem handle for (design.grid, design.basis, labels0), reused across calls."""
    if isinstance(design, Problem):
        return design
    grid = design.grid
    kind, degree, _ = _basis_key(design.basis)
    prec = precision or DEFAULT_PRECISION
    labels0 = None if labels0 is None else np.asarray(labels0, dtype=np.int64)
    with _CACHE_LOCK:
        for entry in _CACHE:
            g, k, d, n, p, lab, prob = entry
            if g is grid and k == kind and d == degree and n == n_grains and p == prec:
                if (lab is None and labels0 is None) or (
                        lab is not None and labels0 is not None and np.array_equal(lab, labels0)):
                    return prob
        prob = Problem(grid, kind, degree, n_grains, labels0, precision=prec)
        _CACHE.insert(0, (grid, kind, degree, n_grains, prec,
                          None if labels0 is None else labels0.copy(), prob))
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.pop()[-1].close()
        return prob


_DCACHE: list = []


def problem_for_design(design_values, labels0, n_grains: int) -> Problem:
    """Problem handle for an explicit (K, P) design matrix, reused while the
    same matrix and labels come back (the reference's evaluate_objective
    callers pass one design for a whole fit)."""
    d = np.asarray(design_values, dtype=np.float64)
    lab = None if labels0 is None else np.asarray(labels0, dtype=np.int64)
    with _CACHE_LOCK:
        for entry in _DCACHE:
            dd, n, ll, prob = entry
            if n == n_grains and dd.shape == d.shape and np.array_equal(dd, d) and (
                    (ll is None and lab is None) or (ll is not None and lab is not None
                                                     and np.array_equal(ll, lab))):
                return prob
        prob = Problem(None, None, 0, n_grains, lab, design=d)
        _DCACHE.insert(0, (d.copy(), n_grains, None if lab is None else lab.copy(), prob))
        while len(_DCACHE) > _CACHE_MAX:
            _DCACHE.pop()[-1].close()
        return prob


def clear_cache():
    with _CACHE_LOCK:
        while _CACHE:
            _CACHE.pop()[-1].close()
        while _DCACHE:
            _DCACHE.pop()[-1].close()


# ---------------------------------------------------------------- public API
def _check_compatible(theta, design) -> None:
    if _basis_key(theta.basis) != _basis_key(design.basis):
        raise ValueError(
            f"parameter basis ({theta.basis.kind}, d={theta.basis.degree}) does not match "
            f"design basis ({design.basis.kind}, d={design.basis.degree})")


def _check_theta(theta) -> None:
    if not np.all(np.isfinite(theta.values)):
        raise ValueError("parameter matrix contains non-finite entries")


def evaluate_objective(theta_values, design, labels0, eps, *, want_grad: bool = True,
                       want_assign: bool = False, threads: int = 1,
                       chunk_size: int = CHUNK_SIZE, lam: float = 0.0,
                       precision: str | None = None) -> EvalResult:
    """Drop-in for objective.evaluate_objective (objective.py:129-165).

    ``design`` is a DesignMatrix (this package's lazy one or the reference's;
    only ``.basis`` and ``.grid`` are read) or a :class:`Problem`.  ``threads``
    and ``chunk_size`` are accepted for signature parity: the device
    reduction is fixed-order and bit-reproducible regardless.
    """
    theta_values = np.asarray(theta_values)
    if isinstance(design, np.ndarray):  # explicit (K, P) design values (objective.py:129-132)
        prob = problem_for_design(design, labels0, theta_values.shape[1])
    else:
        prob = problem_for(design, labels0, theta_values.shape[1], precision)
    res, _ = prob.eval(theta_values, eps, lam=lam, want_grad=want_grad, want_assign=want_assign)
    return res


def objective(theta, design, grain_map, eps: float) -> float:
    """Mean log-probability of the true labels (objective.py:168-178)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    _check_compatible(theta, design)
    _check_theta(theta)
    return evaluate_objective(theta.values, design, grain_map.labels - 1, eps,
                              want_grad=False).phi


def gradient(theta, design, grain_map, eps: float) -> np.ndarray:
    """Gradient (K, N) with the gauge projection of objective.py:181-198."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    _check_compatible(theta, design)
    _check_theta(theta)
    grad = evaluate_objective(theta.values, design, grain_map.labels - 1, eps,
                              want_grad=True).grad
    if getattr(theta, "gauge", None) == GAUGE_LAST_ZERO:
        grad[:, -1] = 0.0
    return grad


def hard_assign(theta, basis, grid, design=None) -> np.ndarray:
    """Arg-min labels, smallest index on ties (objective.py:70-77), no N x P matrix."""
    if _basis_key(theta.basis) != _basis_key(basis):
        raise ValueError("parameter matrix was built for a different basis")
    _check_theta(theta)
    kind, degree, _ = _basis_key(basis)

    class _D:  # descriptor shim for the cache
        pass

    d = _D()
    d.grid, d.basis = grid, basis
    prob = problem_for(d, None, theta.values.shape[1])
    return prob.assign(theta.values)


class SoftAssignment:
    """objective.SoftAssignment (objective.py:33-51): column x holds (p_i(x))_i."""

    def __init__(self, probabilities, epsilon: float):
        if epsilon <= 0:
            raise ValueError("epsilon must be positive")
        self.probabilities = probabilities
        self.epsilon = epsilon

    def validate(self, tol: float = 1e-12) -> None:
        p = self.probabilities
        if np.any(p <= 0.0) or np.any(p >= 1.0):
            raise ValueError("soft assignment entries must lie strictly in (0, 1)")
        if np.abs(p.sum(axis=0) - 1.0).max() > tol:
            raise ValueError("soft assignment columns must sum to one")


def _problem_of(design, n_grains: int) -> Problem:
    """A label-free problem for a DesignMatrix (lazy or the reference's)."""
    if getattr(design, "grid", None) is not None and getattr(design, "basis", None) is not None:
        return problem_for(design, None, n_grains)
    return problem_for_design(np.asarray(design.values if hasattr(design, "values") else design),
                              None, n_grains)


def soft_assign(theta, design, eps: float) -> SoftAssignment:
    """Softmax memberships at temperature eps (objective.py:80-87), computed on the
    device (pgx_soft_assign): dense (N, P), for small problems like the reference's."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    _check_compatible(theta, design)
    _check_theta(theta)
    return SoftAssignment(_problem_of(design, theta.values.shape[1]).soft_assign(theta.values, eps),
                          epsilon=eps)


def hessian_block(theta, design, grain_map, eps: float, i: int, k: int) -> np.ndarray:
    """The (i, k) block of the Hessian (objective.py:201-217), grain indices
    1-based: -(1/(eps^2 n)) sum_x p_i(x) (1[i==k] - p_k(x)) eta(x) eta(x)^T.
    A small-problem diagnostic: p from the device soft assignment, the K x K
    contraction of the (host) features on the host."""
    n_grains = theta.values.shape[1]
    if not (1 <= i <= n_grains and 1 <= k <= n_grains):
        raise ValueError(f"grain indices must lie in 1..{n_grains}")
    p = soft_assign(theta, design, eps).probabilities
    pi, pk = p[i - 1], p[k - 1]
    w = pi * ((1.0 if i == k else 0.0) - pk)
    try:
        d = np.asarray(design.values)
    except AttributeError:
        d = design.basis.evaluate(np.asarray(design.grid.points))
    return -(d * w[None, :]) @ d.T / (eps * eps * d.shape[1])


def energy_eps(theta, design, grain_map, eps: float) -> float:
    """-eps * Phi (objective.py:220-223)."""
    return -eps * objective(theta, design, grain_map, eps)


def energy_zero(theta, design, grain_map) -> float:
    """mean(h_G - min h) (objective.py:226-231), from the fused kernel's e0."""
    _check_compatible(theta, design)
    _check_theta(theta)
    return evaluate_objective(theta.values, design, grain_map.labels - 1, 1.0,
                              want_grad=False, want_assign=True).e0
