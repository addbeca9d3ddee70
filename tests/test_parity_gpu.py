"""GPU parity: libpgx.so (through the C ABI) against the reference golden
vectors and the CPU oracle, plus size-independent properties at full config
sizes.  Tolerances:

  exact : Phi rel 1e-12, grad 1e-10 x max|grad|, err/e0 exact-ish
  fp64  : Phi 2e-7 (1+|Phi|), grad 2e-6 x max|grad| (fp64 logits; fp32 MUFU exp of
          an exact fp64 argument — MUFU.EX2 itself has a measured ~-5e-8 bias)
  tc    : Phi 1e-6 (1+|Phi|), grad 1e-5 x max|grad| (tcgen05 logits from a 3-product
          fp16 split with fp32 accumulation; near-minimal logits re-evaluated in fp64)
Labels: bit-exact except at pixels whose top-2 cost margin is <= 1e-6 (1+|min|)
(counted and reported; the reference's own tie rule is 1e-12 (1+|min|)).
"""

import math

import numpy as np
import pytest

import golden_lib as gl
import oracle

pytestmark = pytest.mark.gpu

TOL = {"exact": (1e-12, 1e-10), "fp64": (2e-7, 2e-6), "tc": (1e-6, 1e-5)}
FP64_PHI, FP64_GRAD = TOL["fp64"]
PRECISIONS = ["exact", "fp64", "tc"]


@pytest.fixture(scope="module")
def pgb():
    import paper_2605_20816_b200 as m

    m._lib.load()
    return m


def _grid_or_points(pgb, z):
    if "point_index" in z:
        return pgb.PixelGrid(points=gl.points(z))
    return pgb.make_grid(int(z["grid_m"]))


def _expected_path(grid, prec, degree=1, dim=2):
    """Which kernel family a (grid, precision) pair runs (pgx_problem_path): the
    tcgen05 kernels on regular grids with side >= 64, the separable fp64 kernels on
    sides that are a multiple of 128, the exact general kernels everywhere else --
    a "tc" / "fp64" case on a point list or a tiny grid is a test of that fallback."""
    res = getattr(grid, "resolution", None)
    ok_deg = degree <= (8 if dim == 2 else 4)
    if prec == "tc" and res is not None and 2 * res >= 64 and ok_deg:
        return "grid_tc"
    if prec == "fp64" and res is not None and (2 * res) % 128 == 0 and ok_deg:
        return "grid_fp64"
    return "general"


def _assert_grad(z, j, grad, tol):
    if f"grad{j}" in z:
        ref = z[f"grad{j}"]
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(grad - ref).max() <= tol * scale, np.abs(grad - ref).max() / scale
    else:
        s = gl.grad_summary(grad)
        nrm = float(z[f"grad{j}_norm"])
        assert abs(s["norm"] - nrm) <= tol * nrm
        assert np.abs(s["vals"] - z[f"grad{j}_vals"]).max() <= tol * nrm


CASES = ["small_legendre_d2", "small_monomial_d3", "c1_full", "c2_full", "c3_sub", "c5_sub",
         "ties_d2"]


@pytest.mark.parametrize("prec", PRECISIONS)
@pytest.mark.parametrize("name", CASES)
def test_golden_eval_and_assign(pgb, name, prec):
    z = gl.load(name)
    kind, degree, n = str(z["kind"]), int(z["degree"]), int(z["n_grains"])
    eps = float(z["eps"])
    labels0 = np.asarray(z["labels0"], dtype=np.int64)
    grid = _grid_or_points(pgb, z)
    prob = pgb.Problem(grid, kind, degree, n, labels0, precision=prec)
    path = _expected_path(grid, prec, degree)
    assert prob.kernel_path == path
    tphi, tgrad = TOL[prec]
    for j, th in enumerate(gl.thetas(z)):
        res, st, names = prob.eval_kernels(th, eps, want_grad=True, want_assign=True)
        want = {"grid_tc": "tc_pass1", "grid_fp64": "grid_pass1", "general": "general_pass1"}[path]
        assert want in names, (path, names)
        phi_ref = float(z[f"phi{j}"])
        assert abs(res.phi - phi_ref) <= tphi * (1 + abs(phi_ref)), (j, res.phi, phi_ref)
        _assert_grad(z, j, res.grad, tgrad)
        near = set(np.asarray(z[f"near_tie{j}"]).tolist())
        # err may differ only through near-tie pixels
        assert abs(res.err - float(z[f"err{j}"])) * len(labels0) <= len(near) + 1e-9
        assert res.e0 == pytest.approx(float(z[f"e0{j}"]), rel=1e-9, abs=1e-12)
        lab, margin, n_amb = prob.assign(th, with_margin=True)
        ref_lab = np.asarray(z[f"assign{j}"], dtype=np.int64)
        bad = np.flatnonzero(lab != ref_lab)
        assert set(bad.tolist()) <= near, (j, bad[:10])
    prob.close()


@pytest.mark.parametrize("prec", PRECISIONS)
def test_random_shapes_vs_oracle(pgb, prec):
    """Ragged N/P, tiny cases, both bases, 2-D and 3-D, unstructured lists: every
    precision request on a point list runs the exact general kernels (asserted)."""
    rng = np.random.default_rng(77)
    tphi, tgrad = TOL[prec]
    cases = [(2, 1, 2, 1, "legendre"), (2, 3, 3, 1, "monomial"), (2, 2, 7, 37, "legendre"),
             (2, 5, 129, 300, "legendre"), (3, 2, 65, 500, "legendre"),
             (3, 3, 5, 200, "monomial"), (2, 10, 17, 100, "legendre"), (2, 0, 3, 50, "legendre")]
    for dim, d, n, p, kind in cases:
        pts = rng.uniform(-0.99, 0.99, (p, dim))
        k = math.comb(d + dim, dim)
        labels0 = rng.integers(0, n, p)
        th = rng.normal(size=(k, n))
        eps = float(rng.uniform(0.05, 1.0))
        ref = oracle.evaluate_objective(th, oracle.design_values(kind, d, pts), labels0, eps,
                                        want_grad=True, want_assign=True)
        prob = pgb.Problem(pgb.PixelGrid(points=pts), kind, d, n, labels0, precision=prec)
        assert prob.kernel_path == "general"
        res, st = prob.eval(th, eps, want_grad=True, want_assign=True)
        assert abs(res.phi - ref.phi) <= tphi * (1 + abs(ref.phi)), (dim, d, n, p)
        assert np.abs(res.grad - ref.grad).max() <= tgrad * max(np.abs(ref.grad).max(), 1e-300)
        assert res.err == pytest.approx(ref.err, abs=st.n_ambiguous / p + 1e-15)
        lab = prob.assign(th)
        assert np.array_equal(lab, oracle.hard_assign_points(th, kind, d, pts))
        prob.close()


def test_regular_grid_3d_vs_oracle(pgb):
    rng = np.random.default_rng(3)
    m, d, n = 6, 2, 40
    pts = oracle.grid_points(m, 3)
    labels0 = rng.integers(0, n, pts.shape[0])
    th = rng.normal(size=(10, n))
    ref = oracle.evaluate_problem(th, "legendre", d, pts, labels0, 0.1, want_assign=True)
    for prec in PRECISIONS:
        prob = pgb.Problem(pgb.make_grid(m, 3), "legendre", d, n, labels0, precision=prec)
        res, _ = prob.eval(th, 0.1, want_assign=True)
        tphi, tgrad = TOL[prec]
        assert abs(res.phi - ref.phi) <= tphi * (1 + abs(ref.phi))
        assert np.abs(res.grad - ref.grad).max() <= tgrad * np.abs(ref.grad).max()
        prob.close()


def test_lambda_term(pgb):
    z = gl.load("c1_full")
    th = gl.thetas(z)[2]
    lab = np.asarray(z["labels0"], dtype=np.int64)
    ref = oracle.evaluate_problem(th, "legendre", 1, gl.points(z), lab, 0.05, lam=1e-4)
    prob = pgb.Problem(pgb.make_grid(64), "legendre", 1, 20, lab, precision="exact")
    res, _ = prob.eval(th, 0.05, lam=1e-4)
    assert abs(res.phi - ref.phi) <= 1e-12 * (1 + abs(ref.phi))
    assert np.abs(res.grad - ref.grad).max() <= 1e-10 * np.abs(ref.grad).max()


def test_known_answers(pgb):
    # theta = 0 -> Phi = -log N exactly, p = 1/N (test_objective.py:67-74)
    rng = np.random.default_rng(1)
    grid = pgb.make_grid(6)
    labels0 = rng.integers(0, 50, len(grid))
    prob = pgb.Problem(grid, "legendre", 1, 50, labels0, precision="exact")
    res, _ = prob.eval(np.zeros((3, 50)), 1e-2)
    assert res.phi == pytest.approx(-math.log(50.0), abs=1e-12)
    # single pixel, two grains: grad = +-0.5 on the constant (test_objective.py:98-110)
    g1 = pgb.PixelGrid(points=np.array([[0.0, 0.0]]))
    p1 = pgb.Problem(g1, "monomial", 1, 2, np.array([0]), precision="exact")
    r1, _ = p1.eval(np.zeros((3, 2)), 1.0)
    expected = np.zeros((3, 2))
    expected[0, 0], expected[0, 1] = -0.5, 0.5
    assert np.array_equal(r1.grad, expected)
    # log-3 gap: p = 0.75 / 0.25 -> Phi = log 0.75 for label 1
    th = np.zeros((3, 2))
    th[0, 1] = math.log(3.0) * 0.25
    r2, _ = p1.eval(th, 0.25)
    assert r2.phi == pytest.approx(math.log(0.75), abs=1e-15)


def test_tie_semantics(pgb):
    rng = np.random.default_rng(9)
    grid = pgb.make_grid(5)
    basis = pgb.DesignBasis.make("legendre", 2)
    vals = rng.normal(size=(6, 4))
    vals[:, 3] = vals[:, 1]
    lab = pgb.hard_assign(pgb.ParamMatrix(vals, basis), basis, grid)
    assert not np.any(lab == 4)  # duplicated later column never wins
    tie = np.tile(rng.normal(size=(6, 1)), (1, 4))
    assert np.all(pgb.hard_assign(pgb.ParamMatrix(tie, basis), basis, grid) == 1)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size_modes_against_exact(pgb, name):
    """Every BASELINE config at full size: the fast modes (fp64 grid path,
    tcgen05 path) against the reference-faithful exact mode (itself pinned to
    the oracle / golden vectors above), at the bench theta and a N(0,1) theta."""
    from paper_2605_20816_b200 import configs

    w = configs.make(name, labeler="gpu")
    rng = np.random.default_rng(21)
    thetas = [np.asarray(w.theta_bench, dtype=np.float64), rng.normal(size=(w.K, w.n_grains))]
    probs = {m: pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=m)
             for m in ("exact", "fp64", "tc")}
    for th in thetas:
        ref, rs = probs["exact"].eval(th, w.eps, lam=w.lam, want_assign=True)
        for mode in ("fp64", "tc"):
            res, st = probs[mode].eval(th, w.eps, lam=w.lam, want_assign=True)
            tphi, tgrad = TOL[mode]
            assert abs(res.phi - ref.phi) <= tphi * (1 + abs(ref.phi)), (mode, res.phi, ref.phi)
            assert np.abs(res.grad - ref.grad).max() <= tgrad * np.abs(ref.grad).max(), mode
            assert abs(res.err - ref.err) * w.n_points <= rs.n_ambiguous, mode
            assert res.e0 == pytest.approx(ref.e0, rel=1e-9, abs=1e-12), mode
            again, _ = probs[mode].eval(th, w.eps, lam=w.lam, want_assign=True)
            assert again.phi == res.phi and np.array_equal(again.grad, res.grad)  # bit-reproducible
    for p in probs.values():
        p.close()


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
@pytest.mark.parametrize("prec", ["fp64", "tc"])
def test_full_config_properties(pgb, name, prec):
    """Size-independent properties on the full-size configs."""
    from paper_2605_20816_b200 import configs

    w = configs.make(name, labeler="gpu")
    rng = np.random.default_rng(11)
    prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=prec)
    tol_phi, tol_grad = TOL[prec]
    th = rng.normal(size=(w.K, w.n_grains))
    a, _ = prob.eval(th, w.eps, want_assign=True)
    b, _ = prob.eval(th, w.eps, want_assign=True)
    assert a.phi == b.phi and np.array_equal(a.grad, b.grad)  # bit-reproducible
    # gauge invariance (test_objective.py:236-244)
    c = rng.normal(size=(w.K, 1))
    s, _ = prob.eval(th + c, w.eps, want_assign=True)
    assert abs(s.phi - a.phi) <= tol_phi * (1 + abs(a.phi))
    # eps scaling (test_objective.py:246-254)
    e, _ = prob.eval(th / w.eps, 1.0, want_assign=True)
    assert abs(e.phi - a.phi) <= tol_phi * (1 + abs(a.phi))
    # un-projected gradient columns sum to zero
    assert np.abs(a.grad.sum(axis=1)).max() <= tol_grad * np.abs(a.grad).max()
    # separable grid path (fp64 mode) == reference-faithful general path (exact)
    ex = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision="exact")
    x, xs = ex.eval(th, w.eps, want_assign=True)
    assert abs(x.phi - a.phi) <= tol_phi * (1 + abs(x.phi))
    assert np.abs(x.grad - a.grad).max() <= tol_grad * np.abs(x.grad).max()
    assert abs(x.err - a.err) * len(w.labels0) <= xs.n_ambiguous
    assert x.e0 == pytest.approx(a.e0, rel=1e-9)
    ex.close()
    # theta = 0: Phi = -log N, grad = -(M - sum eta / N)/(eps P)
    z, _ = prob.eval(np.zeros((w.K, w.n_grains)), w.eps)
    assert z.phi == pytest.approx(-math.log(w.n_grains), abs=1e-12)
    pts = oracle.grid_points(w.M, w.dim)
    mom = oracle.label_moments(w.kind, w.degree, pts, w.labels0, w.n_grains)
    g0 = -(mom - mom.sum(axis=1, keepdims=True) / w.n_grains) / (w.eps * len(pts))
    assert np.abs(z.grad - g0).max() <= tol_grad * np.abs(g0).max()
    prob.close()


def test_fit_trajectory_matches_reference(pgb):
    z = gl.load("fit_traj")
    grid = pgb.make_grid(6)
    gm = pgb.GrainMap(grid=grid, labels=np.asarray(z["labels"], dtype=np.int64), n_grains=5)
    rep = pgb.fit(gm, pgb.FitConfig(degree=2, max_iters=40, precision="exact"))
    ref = np.asarray(z["phi"])
    got = np.asarray(rep.phi_traj)
    assert rep.stop_reason == str(z["stop"])
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 1e-8 * (1 + np.abs(ref).max())
    assert np.all(np.diff(got) >= 0)
    assert rep.gauge_residual == 0.0


def test_fit_c1_trajectory(pgb):
    from paper_2605_20816_b200 import configs

    z = gl.load("fit_traj")
    w = configs.c1(labeler="host")
    gm = pgb.GrainMap(grid=pgb.make_grid(64), labels=w.labels0 + 1, n_grains=20)
    rep = pgb.fit(gm, pgb.FitConfig(degree=1, eps=0.05, max_iters=25, precision="exact"))
    ref = np.asarray(z["c1_phi"])
    got = np.asarray(rep.phi_traj)
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 1e-7 * (1 + np.abs(ref).max())


@pytest.mark.parametrize("prec", ["exact", "tc"])
def test_fit_device_loop_matches_host_loop(pgb, prec):
    """fit(device_loop=True) keeps u, the gradient and the L-BFGS history on the
    GPU; only dot-product summation order differs from the host loop. Over 25
    iterations that 1-ulp difference is amplified by the line searches: to ~1e-12
    with exact gradients, to ~1e-6 with tc gradients (the tc Φ tolerance)."""
    from paper_2605_20816_b200 import configs

    z = gl.load("fit_traj")
    w = configs.c1(labeler="host")
    gm = pgb.GrainMap(grid=pgb.make_grid(64), labels=w.labels0 + 1, n_grains=20)
    cfg = dict(degree=1, eps=0.05, max_iters=25, precision=prec)
    host = pgb.fit(gm, pgb.FitConfig(**cfg))
    dev = pgb.fit(gm, pgb.FitConfig(**cfg, device_loop=True))
    a, b = np.asarray(host.phi_traj), np.asarray(dev.phi_traj)
    assert a.shape == b.shape and dev.stop_reason == host.stop_reason
    scale = 1 + np.abs(a).max()
    assert np.abs(a[:10] - b[:10]).max() <= 1e-9 * scale  # before the amplification
    tol, ttol = (1e-9, 1e-6) if prec == "exact" else (1e-6, 1e-4)
    assert np.abs(a - b).max() <= tol * scale
    assert np.abs(dev.theta.values - host.theta.values).max() <= ttol * (1 + np.abs(host.theta.values).max())
    assert dev.gauge_residual == 0.0
    if prec == "exact":
        ref = np.asarray(z["c1_phi"])
        assert np.abs(b - ref).max() <= 1e-7 * (1 + np.abs(ref).max())


def test_errors_map_to_reference_exceptions(pgb):
    grid = pgb.make_grid(3)
    basis = pgb.DesignBasis.make("legendre", 1)
    design = pgb.assemble_design_matrix(basis, grid)
    gm = pgb.GrainMap(grid=grid, labels=np.ones(36, dtype=np.int64), n_grains=3)
    th = pgb.ParamMatrix(np.zeros((3, 3)), basis)
    with pytest.raises(ValueError):
        pgb.objective(th, design, gm, 0.0)
    bad = np.zeros((3, 3))
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        pgb.objective(pgb.ParamMatrix(bad, basis), design, gm, 0.1)
    with pytest.raises(ValueError):
        pgb.Problem(grid, "legendre", 1, 3, np.full(36, 5))
    prob = pgb.Problem(grid, "legendre", 1, 3, np.zeros(36, dtype=np.int64))
    with pytest.raises(pgb.NumericalError):
        prob.eval(bad, 0.1)


def test_drop_in_with_reference_style_objects(pgb):
    """objective()/gradient() accept duck-typed reference objects (points materialised)."""
    z = gl.load("small_legendre_d2")
    pts = gl.points(z)

    class G:  # a reference-like PixelGrid: materialised points + resolution
        def __init__(self):
            self.points, self.resolution = pts, 5

        def __len__(self):
            return pts.shape[0]

    class B:
        kind, degree = "legendre", 2

    class D:
        basis, grid = B(), G()

    class T:
        basis, gauge = B(), "free"

        def __init__(self, v):
            self.values = v

    class GM:
        labels = np.asarray(z["labels0"], dtype=np.int64) + 1

    th = gl.thetas(z)[1]
    phi = pgb.objective(T(th), D(), GM(), 0.5)
    assert phi == pytest.approx(float(z["phi1"]), rel=FP64_PHI)
    g = pgb.gradient(T(th), D(), GM(), 0.5)
    assert np.abs(g - z["grad1"]).max() <= 1e-6 * np.abs(z["grad1"]).max()


EDGE = {
    # name: (degree, n_grains, theta scale, eps, label rule)
    "theta_1e8": (2, 12, 1e8, 0.05, "random"),      # no overflow (test_objective.py:52-57)
    "two_grains": (2, 2, 1.0, 0.02, "random"),      # N = 2, the smallest allowed (geometry.py:94-95)
    "one_label": (2, 9, 1.0, 0.02, "single"),       # every pixel in one grain, the rest empty
    "degree0": (0, 33, 1.0, 0.05, "random"),        # K = 1: constant costs, ties everywhere
    "tiny_eps": (3, 40, 1.0, 1e-4, "argmin"),       # |h|/eps ~ 1e4: one dominant grain per pixel
    "n_not_x32": (2, 45, 0.3, 0.02, "argmin"),      # partial 32-grain block
}


@pytest.mark.parametrize("prec", ["fp64", "tc"])
@pytest.mark.parametrize("case", sorted(EDGE))
def test_edge_cases_regular_grid(pgb, case, prec):
    """The grid/tensor-core paths against the fp64 oracle on edge inputs of a
    128 x 128 grid (the smallest side the separable paths take)."""
    d, n, scale, eps, rule = EDGE[case]
    rng = np.random.default_rng(7)
    m = 64
    pts = oracle.grid_points(m)
    k = (d + 1) * (d + 2) // 2
    theta = rng.normal(size=(k, n)) * scale
    if rule == "random":
        labels0 = rng.integers(0, n, len(pts))
    elif rule == "single":
        labels0 = np.full(len(pts), 3, dtype=np.int64)
    else:
        labels0 = oracle.hard_assign_points(theta, "legendre", d, pts) - 1
        flip = rng.random(len(pts)) < 0.05
        labels0[flip] = rng.integers(0, n, int(flip.sum()))
    ref = oracle.evaluate_problem(theta, "legendre", d, pts, labels0, eps, want_grad=True,
                                  want_assign=True)
    prob = pgb.Problem(pgb.make_grid(m), "legendre", d, n, labels0, precision=prec)
    res, st = prob.eval(theta, eps, want_grad=True, want_assign=True)
    tp, tg = TOL[prec]
    assert np.isfinite(res.phi) and np.all(np.isfinite(res.grad))
    assert abs(res.phi - ref.phi) <= tp * (1 + abs(ref.phi)), (res.phi, ref.phi)
    assert np.abs(res.grad - ref.grad).max() <= tg * max(np.abs(ref.grad).max(), 1e-300)
    assert abs(res.err - ref.err) <= st.n_ambiguous / len(pts) + 1e-15
    assert abs(res.e0 - ref.e0) <= tp * (1 + abs(ref.e0))
    labels = prob.assign(theta)
    assert np.array_equal(labels, oracle.hard_assign_points(theta, "legendre", d, pts))
    prob.close()


_PDL_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import configs
w = configs.make("c2", labeler="gpu")
th = np.asarray(w.theta_bench, dtype=np.float64)
out = {{}}
for prec in ("fp64", "tc"):
    pr = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=prec)
    for rep in range(3):  # back-to-back evaluations: the overlap crosses evaluations too
        r, s = pr.eval(th * (1 + 0.01 * rep), w.eps, lam=w.lam, want_assign=True)
        out[f"{{prec}}{{rep}}"] = np.concatenate([[r.phi, r.err, r.e0, s.n_ambiguous], r.grad.ravel()])
    pr.close()
np.savez({path!r}, **out)
"""


def test_pdl_on_off_bitwise(pgb, tmp_path):
    """Programmatic dependent launch (kernels set up while their predecessor
    drains, pgx_launch.cuh) changes no result bit: a child process with
    PGX_PDL=0 gives identical Φ, ∇, err, e0 in both fast modes."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        path = str(tmp_path / f"pdl{flag}.npz")
        env = dict(os.environ, PGX_PDL=flag)
        subprocess.run([sys.executable, "-c", _PDL_CHILD.format(root=root, path=path)], env=env,
                       check=True, timeout=600)
        res[flag] = np.load(path)
    for key in res["0"].files:
        np.testing.assert_array_equal(res["0"][key], res["1"][key], err_msg=key)


@pytest.mark.parametrize("prec", ["fp64", "tc"])
def test_pinned_results_zero_copy_bitwise(pgb, prec):
    """Host results in pinned memory are written by the tail kernel through
    the mapped alias (no D2H copies); pageable results are copied. Both give
    identical bits, also with a host fp32 theta (the e2e bench call)."""
    import torch

    from paper_2605_20816_b200 import _lib, configs

    w = configs.make("c2", labeler="gpu")
    pr = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=prec)
    lib = _lib.load()
    K, N = np.asarray(w.theta_bench).shape
    th = np.ascontiguousarray(np.asarray(w.theta_bench, dtype=np.float32))
    flags = _lib.PGX_WANT_GRAD | _lib.PGX_WANT_ASSIGN | _lib.PGX_THETA_F32
    g_page, s_page = np.zeros((K, N)), np.zeros(_lib.STATS_WORDS)
    _lib.check(lib.pgx_eval(pr.handle, th.ctypes.data, float(w.eps), float(w.lam), flags,
                            g_page.ctypes.data, s_page.ctypes.data))
    th_pin = torch.from_numpy(th).pin_memory()
    g_pin = torch.zeros((K, N), dtype=torch.float64).pin_memory()
    s_pin = torch.zeros(_lib.STATS_WORDS, dtype=torch.float64).pin_memory()
    for _ in range(2):  # repeated calls reuse the mapped aliases
        _lib.check(lib.pgx_eval(pr.handle, th_pin.data_ptr(), float(w.eps), float(w.lam), flags,
                                g_pin.data_ptr(), s_pin.data_ptr()))
        np.testing.assert_array_equal(g_pin.numpy(), g_page)
        np.testing.assert_array_equal(s_pin.numpy(), s_page)
    pr.close()


def test_design_values_form_vs_oracle(pgb):
    """evaluate_objective(theta_values, design_values, labels0, eps) with an
    explicit (K, P) design (objective.py:129-132; the reference's own tests call
    it this way): any features, K not a basis size."""
    rng = np.random.default_rng(5)
    for k, n, p in ((3, 4, 300), (7, 13, 1000), (40, 9, 257), (66, 3, 50)):
        d = rng.normal(size=(k, p))
        th = rng.normal(size=(k, n)) * 0.5
        lab = rng.integers(0, n, p)
        ref = oracle.evaluate_objective(th, d, lab, 0.3, want_grad=True, want_assign=True)
        res = pgb.evaluate_objective(th, d, lab, 0.3, want_grad=True, want_assign=True)
        assert abs(res.phi - ref.phi) <= 1e-12 * (1 + abs(ref.phi))
        assert np.abs(res.grad - ref.grad).max() <= 1e-10 * np.abs(ref.grad).max()
        assert res.err == ref.err and res.e0 == pytest.approx(ref.e0, rel=1e-12, abs=1e-14)


def test_soft_assign_vs_oracle(pgb):
    """soft_assign (objective.py:80-87) on the device: dense (N, P) memberships."""
    rng = np.random.default_rng(6)
    grid = pgb.make_grid(5)
    basis = pgb.DesignBasis.make("legendre", 2)
    design = pgb.assemble_design_matrix(basis, grid)
    th = pgb.ParamMatrix(rng.normal(size=(6, 7)), basis)
    soft = pgb.soft_assign(th, design, 0.2)
    soft.validate()
    c = th.values.T @ oracle.design_values("legendre", 2, oracle.grid_points(5))
    z = np.exp((c.min(axis=0)[None] - c) / 0.2)
    assert np.abs(soft.probabilities - z / z.sum(axis=0)).max() <= 1e-14
    zero = pgb.soft_assign(pgb.ParamMatrix(np.zeros((6, 5)), basis), design, 0.3)
    assert np.all(zero.probabilities == 0.2)
