"""The a12 extensions of the fit loop (not in the reference):
plain gradient ascent with Armijo backtracking (``method="ascent"``) and the
geometric eps schedule (``eps_schedule``), on BASELINE config c1 ("100
gradient-ascent iterations").

The checker is an oracle-driven restatement of the same loop: every
evaluation goes through oracle.evaluate_problem (the NumPy restatement of
objective.py:129-165 with the lambda term), so the GPU fit must reproduce its
trajectory.  Neutral settings must reduce to the reference loop bit for bit:
``eps_schedule=(eps, 1.0)`` and ``eps_schedule=None`` give identical L-BFGS
trajectories (optimizer.py:248-318).
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu



@pytest.fixture(scope="module")
def pgb():
    import paper_2605_20816_b200 as m

    m._lib.load()
    return m


WOLFE_C1 = 1e-4       # optimizer.py:29
MAX_LINE_EVALS = 25   # optimizer.py:31


def _c1():
    from paper_2605_20816_b200 import configs

    return configs.c1(labeler="host")


def _oracle_ascent(w, iters, lam, step0, eps_schedule=None):
    """Gradient ascent on u = theta[:, :N-1] (gauge: last column zero,
    optimizer.py:210-221) with Armijo backtracking and a step that doubles
    after each accepted trial; eps_k = max(eps, eps0 r^k), re-evaluated when
    it changes."""
    pts = oracle.grid_points(w.M)
    k, n = w.K, w.n_grains

    def ev(u, eps):
        th = np.zeros((k, n))
        th[:, : n - 1] = u.reshape(k, n - 1)
        r = oracle.evaluate_problem(th, w.kind, w.degree, pts, w.labels0, eps, want_grad=True,
                                    want_assign=True, lam=lam)
        return r.phi, r.grad[:, : n - 1].ravel(), r.err

    def eps_at(it):
        if eps_schedule is None:
            return w.eps
        return max(w.eps, eps_schedule[0] * eps_schedule[1] ** it)

    u = np.zeros(k * (n - 1))
    eps = eps_at(0)
    phi, g, err = ev(u, eps)
    traj, errs, step = [phi], [err], step0
    for it in range(1, iters + 1):
        if eps_at(it) != eps:
            eps = eps_at(it)
            phi, g, err = ev(u, eps)
        gn2 = float(g @ g)
        t = step
        for _ in range(MAX_LINE_EVALS):
            p_t, g_t, e_t = ev(u + t * g, eps)
            if np.isfinite(p_t) and p_t >= phi + WOLFE_C1 * t * gn2:
                break
            t *= 0.5
        else:
            raise AssertionError("oracle loop: no Armijo step")
        u, phi, g, err = u + t * g, p_t, g_t, e_t
        step = 2.0 * t
        traj.append(phi)
        errs.append(err)
    return np.asarray(traj), np.asarray(errs), u


@pytest.mark.parametrize("prec,tol", [("exact", 1e-9), ("tc", 5e-5)])
def test_ascent_c1_matches_oracle_loop(prec, tol):
    import paper_2605_20816_b200 as pgb

    w = _c1()
    iters = 100 if prec == "exact" else 30
    ref_phi, ref_err, ref_u = _oracle_ascent(w, iters, w.lam, 1.0)
    gm = pgb.GrainMap(grid=pgb.make_grid(w.M), labels=w.labels0 + 1, n_grains=w.n_grains)
    rep = pgb.fit(gm, pgb.FitConfig(degree=w.degree, eps=w.eps, lam=w.lam, max_iters=iters,
                                    method="ascent", ascent_step=1.0, precision=prec))
    got = np.asarray(rep.phi_traj)
    assert got.shape == ref_phi.shape and rep.iterations_run == iters
    assert np.abs(got - ref_phi).max() <= tol * (1 + np.abs(ref_phi).max())
    assert np.all(np.diff(got) >= 0)  # Armijo: monotone ascent
    if prec == "exact":
        assert np.abs(np.asarray(rep.err_traj) - ref_err).max() <= 1.5 / len(w.labels0)
        assert np.abs(rep.theta.values[:, :-1].ravel() - ref_u).max() <= 1e-7 * (1 + np.abs(ref_u).max())
    assert rep.gauge_residual == 0.0


def test_eps_schedule_matches_oracle_loop():
    import paper_2605_20816_b200 as pgb

    w = _c1()
    sched = (4 * w.eps, 0.8)  # eps_k = max(0.05, 0.2 * 0.8^k): reaches eps at k = 7
    ref_phi, _, _ = _oracle_ascent(w, 20, w.lam, 1.0, sched)
    gm = pgb.GrainMap(grid=pgb.make_grid(w.M), labels=w.labels0 + 1, n_grains=w.n_grains)
    rep = pgb.fit(gm, pgb.FitConfig(degree=w.degree, eps=w.eps, lam=w.lam, max_iters=20,
                                    method="ascent", eps_schedule=sched, precision="exact"))
    got = np.asarray(rep.phi_traj)
    assert got.shape == ref_phi.shape
    assert np.abs(got - ref_phi).max() <= 1e-9 * (1 + np.abs(ref_phi).max())


@pytest.mark.parametrize("method", ["lbfgs", "ascent"])
def test_neutral_schedule_is_the_constant_eps_loop(method):
    """eps_schedule=(eps, 1.0) never changes eps: the fit is the constant-eps
    one (for lbfgs, the reference loop of optimizer.py:248-318) bit for bit."""
    import paper_2605_20816_b200 as pgb

    w = _c1()
    gm = pgb.GrainMap(grid=pgb.make_grid(w.M), labels=w.labels0 + 1, n_grains=w.n_grains)
    kw = dict(degree=w.degree, eps=w.eps, max_iters=15, method=method, precision="exact")
    a = pgb.fit(gm, pgb.FitConfig(**kw))
    b = pgb.fit(gm, pgb.FitConfig(eps_schedule=(w.eps, 1.0), **kw))
    assert a.phi_traj == b.phi_traj and a.err_traj == b.err_traj
    assert np.array_equal(a.theta.values, b.theta.values)


def test_problem_label_moments_match_standalone():
    """pgx_problem_label_moments (resident int32 labels, stream-ordered) equals
    the stand-alone pgx_label_moments and the oracle's bincount form."""
    import paper_2605_20816_b200 as pgb
    from paper_2605_20816_b200 import configs

    w = configs.c2(labeler="host")
    grid = pgb.make_grid(w.M)
    prob = pgb.Problem(grid, w.kind, w.degree, w.n_grains, w.labels0, precision="fp64")
    a = prob.label_moments()
    b = pgb.heuristics.label_moment_sums(grid, w.labels0, w.n_grains)
    assert a.dtype == np.int64 and np.array_equal(a, b)
    side = 2 * w.M
    p = np.arange(side * side)
    a1, a2 = 2 * (p // side) + 1 - side, 2 * (p % side) + 1 - side
    for q, v in enumerate([np.ones_like(a1), a1, a2, a1 * a1, a1 * a2, a2 * a2]):
        assert np.array_equal(a[:, q], np.bincount(w.labels0, weights=v, minlength=w.n_grains).astype(np.int64))
    assert prob.last_launch_count() == 1
    prob.close()


@pytest.mark.parametrize("cfg,prec", [("c2", "tc"), ("c2", "fp64"), ("c1", "exact")])
def test_workspace_bytes_match_allocation(cfg, prec):
    """pgx_workspace_bytes (the figure a ResourceError reports, basis.py:185-192)
    equals what pgx_problem_create really allocates, coefficient tables included."""
    import ctypes

    import paper_2605_20816_b200 as pgb
    from paper_2605_20816_b200 import _lib, configs

    w = configs.make(cfg, labeler="host")
    prob = pgb.Problem(pgb.make_grid(w.M), w.kind, w.degree, w.n_grains, w.labels0, precision=prec)
    d = _lib.PgxDesc()
    d.dim, d.degree, d.n_grains, d.n_points, d.resolution = 2, w.degree, w.n_grains, len(w.labels0), w.M
    d.basis_kind = _lib.PGX_BASIS_LEGENDRE
    d.precision = _lib.PRECISIONS[prec]
    est = _lib.load().pgx_workspace_bytes(ctypes.byref(d))
    got = prob.device_bytes()
    prob.close()
    assert abs(est - got) <= 0.02 * got + 65536, (est, got)


# ---------------------------------------------------------------- device-resident optimiser state
def test_device_loop_two_loop_matches_numpy(pgb):
    """pgx_lbfgs_direction (the fused two-loop kernel, optimizer.py:253-269)
    against a NumPy two-loop on the same (s, y) history, through a real fit state."""
    from paper_2605_20816_b200 import configs
    from paper_2605_20816_b200.optimizer import _DeviceState

    w = configs.c1(labeler="host")
    prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision="exact")
    dev = _DeviceState(prob, 4, 0.0)
    rng = np.random.default_rng(0)
    theta = np.zeros((w.K, w.n_grains))
    theta[:, :-1] = 0.05 * rng.normal(size=(w.K, w.n_grains - 1))
    n = w.n_grains
    s_hist, y_hist = [], []

    def grad_at(th):
        res, _ = prob.eval(th, w.eps, want_grad=True, want_assign=True)
        return res.phi, res.grad[:, : n - 1].ravel()

    phi, err, e0, gg = dev.start(theta, w.eps)
    p_ref, g = grad_at(theta)
    assert phi == p_ref and gg == pytest.approx(float(g @ g), rel=1e-13)
    u = theta[:, : n - 1].ravel().copy()
    for it in range(7):  # more pairs than the memory: the ring wraps
        slope0, dd, gg, used = dev.direction(0)
        assert used == min(len(s_hist), 4)
        if s_hist:
            q = g.copy()
            alphas = []
            for s_v, y_v in zip(reversed(s_hist[-4:]), reversed(y_hist[-4:])):
                a = (s_v @ q) / (s_v @ y_v)
                q -= a * y_v
                alphas.append(a)
            r = (s_hist[-1] @ y_hist[-1]) / (y_hist[-1] @ y_hist[-1]) * q
            for s_v, y_v, a in zip(s_hist[-4:], y_hist[-4:], reversed(alphas)):
                r += s_v * (a - (y_v @ r) / (s_v @ y_v))
            d = r
        else:
            d = g / (g @ g)
        assert slope0 == pytest.approx(float(g @ d), rel=1e-9)
        assert dd == pytest.approx(float(d @ d), rel=1e-9)
        t = 0.5
        p_t, s_t, e_t, z_t, gg_t, _ = dev.trial(t, w.eps)
        th_t = np.zeros_like(theta)
        th_t[:, : n - 1] = (u + t * d).reshape(w.K, n - 1)
        p_ref, g_t = grad_at(th_t)
        assert p_t == pytest.approx(p_ref, rel=1e-12)
        assert s_t == pytest.approx(float(g_t @ d), rel=1e-8, abs=1e-14)
        gg2, pushed, uu = dev.accept(True)
        s_v, y_v = t * d, g - g_t
        assert pushed == bool(s_v @ y_v > 1e-10 * np.linalg.norm(s_v) * np.linalg.norm(y_v))
        if pushed:
            s_hist.append(s_v)
            y_hist.append(y_v)
        u, g = u + t * d, g_t
        assert np.allclose(dev.theta()[:, : n - 1].ravel(), u, rtol=1e-13, atol=1e-15)
        assert np.all(dev.theta()[:, -1] == 0.0)
    dev.close()
    prob.close()


def test_device_loop_range_fallback(pgb):
    """A theta beyond the fast modes' logit range (theta x 1e8) moves the
    device-resident fit onto the exact kernels instead of returning -inf."""
    from paper_2605_20816_b200 import configs

    w = configs.c1(labeler="host")
    gm = pgb.GrainMap(grid=pgb.make_grid(64), labels=w.labels0 + 1, n_grains=20)
    rng = np.random.default_rng(3)
    vals = 1e8 * rng.normal(size=(3, 20))
    vals[:, -1] = 0.0
    init = pgb.ParamMatrix(vals, pgb.DesignBasis.make("legendre", 1), gauge=pgb.GAUGE_LAST_ZERO)
    cfg = dict(degree=1, eps=0.05, max_iters=3, init=init)
    host = pgb.fit(gm, pgb.FitConfig(**cfg, precision="exact"))
    dev = pgb.fit(gm, pgb.FitConfig(**cfg, precision="tc", device_loop=True))
    assert np.isfinite(dev.phi_traj[0]) and dev.phi_traj[0] == pytest.approx(host.phi_traj[0], rel=1e-12)


def test_device_loop_ascent_and_schedule(pgb):
    """method='ascent' and an eps schedule on the device state follow the host loop."""
    from paper_2605_20816_b200 import configs

    w = configs.c1(labeler="host")
    gm = pgb.GrainMap(grid=pgb.make_grid(64), labels=w.labels0 + 1, n_grains=20)
    for extra in (dict(method="ascent", lam=1e-4), dict(eps_schedule=(0.2, 0.8), lam=1e-4)):
        cfg = dict(degree=1, eps=0.05, max_iters=12, precision="exact", **extra)
        host = pgb.fit(gm, pgb.FitConfig(**cfg))
        dev = pgb.fit(gm, pgb.FitConfig(**cfg, device_loop=True))
        a, b = np.asarray(host.phi_traj), np.asarray(dev.phi_traj)
        assert a.shape == b.shape and host.stop_reason == dev.stop_reason
        assert np.abs(a - b).max() <= 1e-9 * (1 + np.abs(a).max())
        assert host.evaluations == dev.evaluations
