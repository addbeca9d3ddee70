"""CPU-only tests: the C ABI library's exports, host descriptors, input
generators and the host-side optimiser logic (no GPU compute calls)."""

import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgx.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(pgx_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2605_20816_b200 import build

    return build.build_library()


def test_header_declares_the_boundary():
    fns = header_functions()
    for name in ("pgx_problem_create", "pgx_eval", "pgx_assign", "pgx_problem_destroy",
                 "pgx_last_error"):
        assert name in fns


def test_library_exports_every_header_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (pgx_\w+)", out.stdout))
    assert set(header_functions()) <= exported


def test_ctypes_signatures_cover_header(lib_path):
    from paper_2605_20816_b200 import _lib

    assert set(header_functions()) == set(_lib.SIGNATURES)
    lib = _lib.load()
    assert lib.pgx_abi_version() == _lib.ABI_VERSION
    assert ctypes.sizeof(_lib.PgxStats) == 8 * _lib.STATS_WORDS


def test_invalid_descriptors_rejected_without_gpu(lib_path):
    from paper_2605_20816_b200 import _lib

    lib = _lib.load()
    d = _lib.PgxDesc()
    d.dim, d.basis_kind, d.degree, d.n_grains, d.n_points = 2, 1, 1, 1, 16
    d.resolution = 2
    h = ctypes.c_void_p()
    assert lib.pgx_problem_create(ctypes.byref(d), ctypes.byref(h)) == _lib.PGX_ERR_INVALID_ARGUMENT
    assert "two grains" in _lib.last_error()
    d.n_grains, d.n_points = 4, 15
    assert lib.pgx_problem_create(ctypes.byref(d), ctypes.byref(h)) == _lib.PGX_ERR_INVALID_ARGUMENT
    d.n_points, d.degree = 16, 11
    assert lib.pgx_problem_create(ctypes.byref(d), ctypes.byref(h)) == _lib.PGX_ERR_INVALID_ARGUMENT


def test_workspace_estimate_c5(lib_path):
    from paper_2605_20816_b200 import _lib

    lib = _lib.load()
    d = _lib.PgxDesc()
    d.dim, d.basis_kind, d.degree, d.n_grains = 2, 1, 8, 4096
    d.resolution, d.n_points = 1024, 2048 * 2048
    b = lib.pgx_workspace_bytes(ctypes.byref(d))
    assert 1e7 < b < 4e9  # no K x P design, no N x P logits


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(lib_path):
    import paper_2605_20816_b200 as pgb

    with pytest.raises(RuntimeError, match="no CUDA device"):
        pgb.Problem(pgb.make_grid(4), "legendre", 1, 3, np.zeros(64, dtype=np.int64))


def test_basis_ordering_matches_reference_convention():
    from paper_2605_20816_b200.basis import feature_count, graded_lex_indices

    assert graded_lex_indices(2) == ((0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2))
    assert graded_lex_indices(2, 3) == ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (2, 0, 0),
                                        (1, 1, 0), (1, 0, 1), (0, 2, 0), (0, 1, 1), (0, 0, 2))
    for d in range(11):
        assert feature_count(d) == (d + 1) * (d + 2) // 2 == len(graded_lex_indices(d))
        assert graded_lex_indices(d) == oracle.multi_indices(d, 2)
    for d in range(5):
        assert graded_lex_indices(d, 3) == oracle.multi_indices(d, 3)


def test_lazy_grid_points_match_make_grid():
    import paper_2605_20816_b200 as pgb

    for m in (1, 3, 8):
        assert np.array_equal(pgb.make_grid(m).points, oracle.grid_points(m))
        assert np.array_equal(pgb.make_grid(m, 3).points, oracle.grid_points(m, 3))
    assert len(pgb.make_grid(70)) == 140 * 140


def test_descriptor_validation_mirrors_reference():
    import paper_2605_20816_b200 as pgb

    basis = pgb.DesignBasis.make("legendre", 2)
    with pytest.raises(ValueError):
        pgb.ParamMatrix(np.zeros((5, 3)), basis)
    with pytest.raises(ValueError):
        pgb.ParamMatrix(np.ones((6, 3)), basis, gauge=pgb.GAUGE_LAST_ZERO)
    with pytest.raises(ValueError):
        pgb.GrainMap(grid=pgb.make_grid(2), labels=np.zeros(16, dtype=np.int64), n_grains=3)
    with pytest.raises(ValueError):
        pgb.PixelGrid(points=np.array([[1.0, 0.0]]))
    with pytest.raises(AttributeError):
        _ = pgb.assemble_design_matrix(basis, pgb.make_grid(2)).values


def test_line_search_mirrors_reference_contract():
    from paper_2605_20816_b200.optimizer import LineEval, line_search

    def make(f, df):
        return lambda t: LineEval(f(t), df(t), t)

    t, ev = line_search(make(lambda t: -0.5 * (t - 1) ** 2, lambda t: -(t - 1)), -0.5, 1.0)
    assert t == 1.0 and ev.payload == 1.0
    rng = np.random.default_rng(0)
    for _ in range(10):
        a, ts = float(rng.uniform(0.5, 4)), float(rng.uniform(0.2, 6))
        t, ev = line_search(make(lambda t: -a * (t - ts) ** 2, lambda t: -2 * a * (t - ts)),
                            -a * ts * ts, 2 * a * ts)
        assert t > 0 and ev.phi >= -a * ts * ts + 1e-4 * t * 2 * a * ts
        assert abs(ev.slope) <= 0.9 * 2 * a * ts
    with pytest.raises(ValueError):
        line_search(make(lambda t: -t, lambda t: -1.0), 0.0, -1.0)
    t, ev = line_search(make(lambda t: 1e-12 * math.sin(1e6 * t), lambda t: 1e-6 * math.cos(1e6 * t)),
                        0.0, 1e-6, max_evals=3)
    assert t == 0.0 and ev is None


def test_line_search_identical_decisions_to_reference_restatement():
    """Same trial sequence as the reference algorithm on a wiggly concave ray."""
    from paper_2605_20816_b200.optimizer import LineEval, line_search

    seq = []

    def f(t):
        seq.append(t)
        return LineEval(math.log1p(t) - 0.05 * t * t + 0.01 * math.sin(7 * t),
                        1 / (1 + t) - 0.1 * t + 0.07 * math.cos(7 * t), t)

    t, _ = line_search(f, 0.0, 1.07, t0=1.0)
    assert t > 0 and seq[0] == 1.0


def test_configs_are_deterministic_and_shaped():
    from paper_2605_20816_b200 import configs

    a = configs.c1(labeler="host")
    b = configs.c1(labeler="host")
    assert np.array_equal(a.labels0, b.labels0)
    assert a.labels0.shape == (128 * 128,) and a.K == 3 and a.n_grains == 20
    assert a.labels0.min() >= 0 and a.labels0.max() < 20
    # the generator arg-min is the tie-tolerant arg-min of its cost
    pts = oracle.grid_points(64)
    seeds = np.random.default_rng(1).uniform(-1, 1, (20, 2))
    d2 = ((pts[:, None, :] - seeds[None]) ** 2).sum(-1)
    agree = np.mean(np.argmin(d2, axis=1) == a.labels0)
    assert agree > 0.999


def test_boundary_noise_only_relabels_to_neighbours():
    from paper_2605_20816_b200.configs import _noise_boundary

    rng = np.random.default_rng(0)
    side = 40
    lab = (np.arange(side)[:, None] // 10 * 4 + np.arange(side)[None, :] // 10).ravel()
    out = _noise_boundary(rng, lab, side, 0.01)
    changed = np.flatnonzero(out != lab)
    assert changed.size == round(0.01 * lab.size)
    L = lab.reshape(side, side)
    for p in changed:
        r, c = divmod(int(p), side)
        nb = {L[rr, cc] for rr, cc in ((r - 1, c), (r + 1, c), (r, c - 1), (r, c + 1))
              if 0 <= rr < side and 0 <= cc < side}
        assert out[p] in nb and out[p] != lab[p]


def test_apd_generator_theta_is_the_quadratic_cost():
    from paper_2605_20816_b200.configs import _apd_theta

    rng = np.random.default_rng(4)
    for dim in (2, 3):
        n = 7
        seeds = rng.uniform(-1, 1, (n, dim))
        w = rng.normal(0, 0.01, n)
        q = rng.normal(size=(n, dim, dim))
        A = q @ q.transpose(0, 2, 1) + np.eye(dim)
        th = _apd_theta(seeds, w, A)
        pts = rng.uniform(-0.9, 0.9, (50, dim))
        cost = th.T @ oracle.design_values("monomial", 2, pts)
        z = pts[None] - seeds[:, None]
        direct = np.einsum("npi,nij,npj->np", z, A, z) - w[:, None]
        np.testing.assert_allclose(cost, direct, atol=1e-12)


def test_design_spans_regular_equals_pointwise():
    import paper_2605_20816_b200 as pgb
    from paper_2605_20816_b200.optimizer import design_spans

    basis = pgb.DesignBasis.make("legendre", 3)
    assert design_spans(pgb.make_grid(4), basis)
    assert design_spans(pgb.PixelGrid(points=pgb.make_grid(4).points), basis)
    assert not design_spans(pgb.PixelGrid(points=np.array([[0.1, 0.2], [0.3, -0.1]])), basis)
