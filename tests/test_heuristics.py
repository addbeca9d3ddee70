"""Moment heuristic (heuristics.py:46-125) against golden vectors of the
reference (tests/golden/make_golden_heuristic.py).

CPU: the NumPy path (an explicit point list).  GPU: the regular-grid path
whose moments are exact integer sums from the pgx_label_moments kernel."""

import numpy as np
import pytest

import golden_lib as gl

CASES = {"c1": [(1, "legendre"), (2, "legendre"), (3, "monomial")],
         "c2": [(2, "legendre"), (4, "legendre")],
         "deg": [(1, "legendre"), (2, "legendre"), (2, "monomial")]}


def _grain_map(pgb, z, name, regular):
    m = int(z[f"{name}_m"])
    labels = np.asarray(z[f"{name}_labels"], dtype=np.int64) + 1
    grid = pgb.make_grid(m)
    if not regular:
        grid = pgb.PixelGrid(points=np.asarray(grid.points) + 0.0)  # a point list: no resolution
        assert grid.resolution is None
    return pgb.GrainMap(grid=grid, labels=labels, n_grains=int(z[f"{name}_n"]))


def _check(pgb, z, name, gm):
    mom = pgb.moments(gm)
    assert np.array_equal(mom.counts, z[f"{name}_counts"])
    assert np.abs(mom.centroids - z[f"{name}_centroids"]).max() <= 1e-14
    ref_b = z[f"{name}_second"]
    assert np.abs(mom.second_moments - ref_b).max() <= 1e-13 * max(1.0, np.abs(ref_b).max())
    assert np.array_equal(mom.degenerate, z[f"{name}_degenerate"])
    for d, kind in CASES[name]:
        th = pgb.heuristic_theta(gm, d, kind)
        ref = z[f"{name}_theta_{d}_{kind}"]
        assert th.values.shape == ref.shape
        assert np.abs(th.values - ref).max() <= 1e-8 * max(1.0, np.abs(ref).max()), (name, d, kind)
        assert np.all(th.values[:, -1] == 0.0)


@pytest.mark.parametrize("name", sorted(CASES))
def test_heuristic_point_list_cpu(name):
    import paper_2605_20816_b200 as pgb

    _check(pgb, gl.load("heuristic"), name, _grain_map(pgb, gl.load("heuristic"), name, False))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_heuristic_regular_grid_gpu(name):
    import paper_2605_20816_b200 as pgb

    z = gl.load("heuristic")
    gm = _grain_map(pgb, z, name, True)
    sums = pgb.heuristics.label_moment_sums(gm.grid, np.asarray(gm.labels) - 1, gm.n_grains)
    assert sums is not None and sums.dtype == np.int64
    _check(pgb, z, name, gm)


@pytest.mark.gpu
def test_fit_heuristic_init():
    import paper_2605_20816_b200 as pgb

    z = gl.load("heuristic")
    gm = _grain_map(pgb, z, "c1", True)
    rep = pgb.fit(gm, pgb.FitConfig(degree=2, eps=0.05, max_iters=10, init="heuristic",
                                    precision="fp64"))
    zero = pgb.fit(gm, pgb.FitConfig(degree=2, eps=0.05, max_iters=10, precision="fp64"))
    assert np.isfinite(rep.phi_final) and rep.phi_traj[0] > zero.phi_traj[0]
