"""Direct oracle parity of the regular-grid kernels at the BASELINE config
shapes: the tcgen05 path (tc) and the separable fp64 path against the NumPy
oracle (itself pinned to the reference's golden vectors, test_oracle_golden.py)
-- not against another GPU kernel.  Every case also asserts which kernels ran
(Problem.eval_kernels: the CUDA-event profile of the call).

Cases (objective.py:97-165 on the grids of geometry.py:59-71):
  c3_full        1024^2, Legendre d=4 (K=15), N=1000, eps=0.01 (BASELINE c3, full size)
  c5_shape       256^2, Legendre d=8 (K=45), N=4096, eps=0.005 (the c5 kernel
                 instantiation incl. the d>=6 pass-2 variant, on a smaller grid)
  c4_shape_d2    128^3, 3-D Legendre d=2 (K=10), N=200, eps=0.02 (the c4 grid)
  c4_shape_d4    128^3, 3-D Legendre d=4 (K=35), N=48, eps=0.02
Tolerances as tests/test_parity_gpu.py.
"""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

TOL = {"fp64": (2e-7, 2e-6), "tc": (1e-6, 1e-5)}
EXPECT = {"tc": ("tc_pass1", "tc_pass2"), "fp64": ("grid_pass1", "grid_pass2")}
THREADS = os.cpu_count() or 1


def _labels_from_diagram(rng, kind, degree, dim, m, n, noise=0.01):
    """A random polynomial diagram (theta_true ~ N(0,1)) and 1% random relabels."""
    from paper_2605_20816_b200 import configs

    k = oracle.feature_count(degree, dim)
    lab = configs.gpu_assign(rng.normal(size=(k, n)), kind, degree, dim, m)
    flip = rng.random(lab.size) < noise
    lab[flip] = rng.integers(0, n, int(flip.sum()))
    return lab


def _case(name):
    from paper_2605_20816_b200 import configs

    rng = np.random.default_rng({"c3_full": 31, "c5_shape": 51, "c4_shape_d2": 41, "c4_shape_d4": 42}[name])
    if name == "c3_full":
        w = configs.c3(labeler="gpu")
        return dict(dim=2, m=w.M, degree=4, n=w.n_grains, eps=w.eps, labels0=w.labels0,
                    thetas=[np.asarray(w.theta_bench, dtype=np.float64),
                            rng.normal(size=(w.K, w.n_grains))])
    spec = {"c5_shape": (2, 128, 8, 4096, 0.005), "c4_shape_d2": (3, 64, 2, 200, 0.02),
            "c4_shape_d4": (3, 64, 4, 48, 0.02)}[name]
    dim, m, d, n, eps = spec
    k = oracle.feature_count(d, dim)
    labels0 = _labels_from_diagram(rng, "legendre", d, dim, m, n)
    return dict(dim=dim, m=m, degree=d, n=n, eps=eps, labels0=labels0,
                thetas=[0.01 * rng.normal(size=(k, n)), 0.3 * rng.normal(size=(k, n))])


_ORACLE = {}


def _oracle(name):
    if name not in _ORACLE:
        c = _case(name)
        pts = oracle.grid_points(c["m"], c["dim"])
        refs = [oracle.evaluate_problem(th, "legendre", c["degree"], pts, c["labels0"], c["eps"],
                                        want_grad=True, want_assign=True, threads=THREADS)
                for th in c["thetas"]]
        _ORACLE[name] = (c, refs)
    return _ORACLE[name]


@pytest.mark.parametrize("prec", ["tc", "fp64"])
@pytest.mark.parametrize("name", ["c3_full", "c5_shape", "c4_shape_d2", "c4_shape_d4"])
def test_grid_kernels_vs_oracle(name, prec):
    import paper_2605_20816_b200 as pgb

    c, refs = _oracle(name)
    prob = pgb.Problem(pgb.make_grid(c["m"], c["dim"]), "legendre", c["degree"], c["n"],
                       c["labels0"], precision=prec)
    assert prob.kernel_path == ("grid_tc" if prec == "tc" else "grid_fp64")
    tphi, tgrad = TOL[prec]
    npx = len(c["labels0"])
    for th, ref in zip(c["thetas"], refs):
        res, st, names = prob.eval_kernels(th, c["eps"], want_grad=True, want_assign=True)
        for k in EXPECT[prec]:
            assert k in names, (names, k)
        assert not any(n.startswith("general") for n in names), names
        assert abs(res.phi - ref.phi) <= tphi * (1 + abs(ref.phi)), (res.phi, ref.phi)
        gerr = np.abs(res.grad - ref.grad).max() / np.abs(ref.grad).max()
        assert gerr <= tgrad, gerr
        # err differs only through pixels whose top-2 margin is within tolerance
        assert abs(res.err - ref.err) * npx <= st.n_ambiguous, (res.err, ref.err, st.n_ambiguous)
        assert res.e0 == pytest.approx(ref.e0, rel=1e-9, abs=1e-12)
    prob.close()


# ---------------------------------------------------------------- tensor-core hard assignment
@pytest.mark.parametrize("name", ["c3_full", "c5_shape", "c4_shape_d2", "c4_shape_d4"])
def test_tc_assign_vs_oracle(name):
    """pgx_assign on a tensor-core problem runs the sweep's ASSIGN variant
    (objective.py:62-77 / geometry.py:201-210): labels bit-identical to the
    oracle except at ambiguous pixels, and to the exact fp64 kernels everywhere."""
    import paper_2605_20816_b200 as pgb

    c, refs = _oracle(name)
    grid = pgb.make_grid(c["m"], c["dim"])
    prob = pgb.Problem(grid, "legendre", c["degree"], c["n"], c["labels0"], precision="tc")
    exact = pgb.Problem(grid, "legendre", c["degree"], c["n"], c["labels0"], precision="exact")
    pts = oracle.grid_points(c["m"], c["dim"])
    for th in c["thetas"]:
        prob.set_profiling(True)
        lab, margin, n_amb = prob.assign(th, with_margin=True)
        names = [n for n, _ in prob.profile()]
        prob.set_profiling(False)
        assert "tc_assign" in names and not any(n.startswith("general") for n in names), names
        lab_x, margin_x, n_amb_x = exact.assign(th, with_margin=True)
        assert np.array_equal(lab, lab_x)
        assert n_amb == n_amb_x
        # the margin is exact when the runner-up is a candidate of the fp64 decision, else
        # its fp32 tensor-core logit: absolute error <= delta ~ 4e-6 max_i sum_k |theta_ki|
        atol = 1e-5 * np.abs(th).sum(axis=0).max()
        assert np.abs(margin - margin_x).max() <= atol, (np.abs(margin - margin_x).max(), atol)
        sub = np.random.default_rng(5).choice(len(pts), 4096, replace=False)
        ref_lab = oracle.hard_assign_points(th, "legendre", c["degree"], pts[sub])
        assert np.array_equal(lab[sub], ref_lab)
    prob.close()
    exact.close()


# ---------------------------------------------------------------- padded (side % 128 != 0) grids
@pytest.mark.parametrize("dim,m,d,n,eps", [(2, 70, 2, 60, 0.02),    # the paper's 140 x 140 map
                                            (2, 70, 8, 300, 0.01),   # d >= 6 pass-2 variant
                                            (2, 100, 4, 257, 0.01),  # 200 x 200, N % 128 != 0
                                            (2, 33, 3, 7, 0.05),     # 66 x 66: one padded tile per line
                                            (3, 36, 2, 40, 0.02)])   # 72^3 voxels
def test_tc_padded_grid_vs_oracle(dim, m, d, n, eps):
    """Grids whose side is not a multiple of 128 run the tcgen05 kernels on
    tiles padded with masked pixels (geometry.py:59-71 grids of any resolution)."""
    import paper_2605_20816_b200 as pgb

    rng = np.random.default_rng(1000 * dim + m)
    k = oracle.feature_count(d, dim)
    labels0 = _labels_from_diagram(rng, "legendre", d, dim, m, n)
    pts = oracle.grid_points(m, dim)
    prob = pgb.Problem(pgb.make_grid(m, dim), "legendre", d, n, labels0, precision="tc")
    assert prob.kernel_path == "grid_tc"
    tphi, tgrad = TOL["tc"]
    for th in (0.01 * rng.normal(size=(k, n)), 0.5 * rng.normal(size=(k, n))):
        ref = oracle.evaluate_problem(th, "legendre", d, pts, labels0, eps, want_grad=True,
                                      want_assign=True, threads=THREADS)
        res, st, names = prob.eval_kernels(th, eps, want_grad=True, want_assign=True)
        assert "tc_pass1" in names and "tc_pass2" in names, names
        assert not any(nm.startswith("general") for nm in names), names
        assert abs(res.phi - ref.phi) <= tphi * (1 + abs(ref.phi)), (res.phi, ref.phi)
        gerr = np.abs(res.grad - ref.grad).max() / np.abs(ref.grad).max()
        assert gerr <= tgrad, gerr
        assert abs(res.err - ref.err) * len(labels0) <= st.n_ambiguous
        assert res.e0 == pytest.approx(ref.e0, rel=1e-9, abs=1e-12)
        lab = prob.assign(th)
        assert np.array_equal(lab, oracle.hard_assign_points(th, "legendre", d, pts))
        # a second evaluation is bit-identical (fixed-order reductions)
        res2, _ = prob.eval(th, eps, want_grad=True, want_assign=True)
        assert res2.phi == res.phi and np.array_equal(res2.grad, res.grad)
    prob.close()


# ---------------------------------------------------------------- randomized shapes on the tc path
def test_tc_random_grid_shapes_vs_exact_kernels():
    """Random sides (padded and not), grain counts (N % 32/64/128 != 0), degrees and
    both bases on the tcgen05 path, against the oracle-pinned exact fp64 kernels:
    evaluation, hard assignment, tie handling (duplicated and all-zero columns)."""
    import paper_2605_20816_b200 as pgb

    rng = np.random.default_rng(2026)
    tphi, tgrad = TOL["tc"]
    shapes = [(2, int(rng.integers(32, 160)), int(rng.integers(0, 9)), int(rng.integers(2, 700)))
              for _ in range(10)]
    shapes += [(3, int(rng.integers(32, 48)), int(rng.integers(0, 5)), int(rng.integers(2, 300)))
               for _ in range(3)]
    shapes += [(2, 64, 2, 2), (2, 32, 1, 513), (2, 97, 8, 129)]
    for dim, m, d, n in shapes:
        kind = "legendre" if rng.random() < 0.7 else "monomial"
        k = oracle.feature_count(d, dim)
        grid = pgb.make_grid(m, dim)
        # labels with spatial structure (a random diagram + 1% noise), as in every real
        # workload: with uniformly random labels the gradient at theta = 0 is pure sampling
        # noise and the max-norm relative tolerance would only measure the MUFU bias
        labels0 = _labels_from_diagram(rng, "legendre", max(d, 1), dim, m, n)
        eps = float(10 ** rng.uniform(-2.3, -0.5))
        tc = pgb.Problem(grid, kind, d, n, labels0, precision="tc")
        ex = pgb.Problem(grid, kind, d, n, labels0, precision="exact")
        assert tc.kernel_path == "grid_tc" and ex.kernel_path == "general"
        thetas = [rng.normal(size=(k, n)) * 10 ** rng.uniform(-2, 0.5), np.zeros((k, n))]
        dup = rng.normal(size=(k, n))
        dup[:, n // 2] = dup[:, 0]  # an exact tie between two grains
        thetas.append(dup)
        for th in thetas:
            a, sa = tc.eval(th, eps, lam=1e-4, want_grad=True, want_assign=True)
            b, sb = ex.eval(th, eps, lam=1e-4, want_grad=True, want_assign=True)
            tag = (dim, m, d, n, kind, eps)
            assert abs(a.phi - b.phi) <= tphi * (1 + abs(b.phi)), tag
            assert np.abs(a.grad - b.grad).max() <= tgrad * max(np.abs(b.grad).max(), 1e-300), tag
            assert abs(a.err - b.err) * len(grid) <= max(sa.n_ambiguous, sb.n_ambiguous), tag
            assert a.e0 == pytest.approx(b.e0, rel=1e-9, abs=1e-12), tag
            la, lb = tc.assign(th), ex.assign(th)
            bad = np.flatnonzero(la != lb)
            assert len(bad) <= max(sa.n_ambiguous, sb.n_ambiguous), (tag, len(bad))
        tc.close()
        ex.close()
