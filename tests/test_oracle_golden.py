"""Pin the CPU oracle against golden vectors produced by the reference itself.

The golden .npz files were written by tests/golden/make_golden.py, which
imported polygrain from /root/reference (read-only) and recorded its
evaluate_objective / hard_assign / fit outputs.  If these pass, the oracle
used by the GPU parity tests is the reference's algorithm on these inputs.
"""

import numpy as np
import pytest

import golden_lib as gl
import oracle

CASES = ["small_legendre_d2", "small_monomial_d3", "c1_full", "c2_full", "c3_sub", "c5_sub",
         "ties_d2"]


def _check_grad(z, j, grad, rtol):
    if f"grad{j}" in z:
        ref = z[f"grad{j}"]
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(grad - ref).max() <= rtol * scale
    else:
        s = gl.grad_summary(grad)
        assert s["norm"] == pytest.approx(float(z[f"grad{j}_norm"]), rel=rtol)
        np.testing.assert_allclose(s["vals"], z[f"grad{j}_vals"], rtol=0,
                                   atol=rtol * float(z[f"grad{j}_norm"]))
        np.testing.assert_allclose(s["proj"], z[f"grad{j}_proj"], rtol=0,
                                   atol=rtol * float(z[f"grad{j}_norm"]) * 300)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(name):
    z = gl.load(name)
    kind, degree, n = str(z["kind"]), int(z["degree"]), int(z["n_grains"])
    eps = float(z["eps"])
    pts = gl.points(z)
    labels0 = np.asarray(z["labels0"], dtype=np.int64)
    design = oracle.design_values(kind, degree, pts)
    for j, th in enumerate(gl.thetas(z)):
        r = oracle.evaluate_objective(th, design, labels0, eps, want_grad=True, want_assign=True)
        assert r.phi == pytest.approx(float(z[f"phi{j}"]), rel=1e-13, abs=1e-13)
        assert r.err == float(z[f"err{j}"])
        assert r.e0 == pytest.approx(float(z[f"e0{j}"]), rel=1e-12, abs=1e-14)
        _check_grad(z, j, r.grad, 1e-11)
        lab = oracle.hard_assign_points(th, kind, degree, pts)
        assert np.array_equal(lab, np.asarray(z[f"assign{j}"], dtype=np.int64))


def test_oracle_legendre_and_design_bit_exact():
    z = gl.load("legendre")
    assert np.array_equal(oracle.legendre_table(10, z["t"]), z["table"])
    assert np.array_equal(oracle.grid_points(5), z["grid5"])
    assert np.array_equal(oracle.design_values("legendre", 3, oracle.grid_points(3)), z["design_d3"])
    assert np.array_equal(oracle.design_values("monomial", 4, oracle.grid_points(3)),
                          z["design_mono_d4"])


def test_oracle_threaded_tree_matches_sequential():
    # objective.py:146-158 contract: parallel tree == sequential within 1e-12
    z = gl.load("c1_full")
    pts = gl.points(z)
    d = oracle.design_values("legendre", 1, pts)
    lab = np.asarray(z["labels0"], dtype=np.int64)
    th = gl.thetas(z)[2]
    a = oracle.evaluate_objective(th, d, lab, 0.05, want_assign=True, threads=1, chunk_size=1024)
    b = oracle.evaluate_objective(th, d, lab, 0.05, want_assign=True, threads=4, chunk_size=1024)
    assert abs(a.phi - b.phi) <= 1e-12 * (1 + abs(a.phi))
    assert a.err == b.err


def test_oracle_streamed_equals_materialised():
    z = gl.load("c3_sub")
    pts = gl.points(z)
    lab = np.asarray(z["labels0"], dtype=np.int64)
    th = gl.thetas(z)[1]
    a = oracle.evaluate_problem(th, "legendre", 4, pts, lab, 0.01, want_assign=True)
    b = oracle.evaluate_objective(th, oracle.design_values("legendre", 4, pts), lab, 0.01,
                                  want_assign=True)
    assert a.phi == b.phi and a.err == b.err
    np.testing.assert_array_equal(a.grad, b.grad)


def test_oracle_3d_embeds_2d():
    # Appendix B cross-check: theta zero on every a3 > 0 index, fixed x3 plane
    rng = np.random.default_rng(5)
    d = 3
    idx3 = oracle.multi_indices(d, 3)
    idx2 = oracle.multi_indices(d, 2)
    th2 = rng.normal(size=(len(idx2), 7))
    th3 = np.zeros((len(idx3), 7))
    for k, a in enumerate(idx3):
        if a[2] == 0:
            th3[k] = th2[idx2.index((a[0], a[1]))]
    pts2 = rng.uniform(-0.9, 0.9, (500, 2))
    x3 = 0.3
    pts3 = np.column_stack([pts2, np.full(500, x3)])
    for kind in ("legendre", "monomial"):
        c2 = th2.T @ oracle.design_values(kind, d, pts2)
        c3 = th3.T @ oracle.design_values(kind, d, pts3)
        np.testing.assert_allclose(c3, c2, rtol=1e-13, atol=1e-13)
