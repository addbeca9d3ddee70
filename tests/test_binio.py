"""Binary sidecars of the grain-map / theta text formats (paper_2605_20816_b200/binio.py;
reference formats: fileio.py:36-44, 101-179).  CPU only."""

import os
import sys

import numpy as np
import pytest

import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import binio

REF_SRC = "/root/reference/pkg/src"


def _grain_map(rng, m=8, n=7, points=False):
    grid = pgb.make_grid(m)
    labels = rng.integers(1, n + 1, len(grid))
    labels[:n] = np.arange(1, n + 1)
    if points:
        pts = rng.uniform(-0.99, 0.99, (50, 2))
        return pgb.GrainMap(grid=pgb.PixelGrid(points=pts), labels=rng.integers(1, n + 1, 50), n_grains=n)
    return pgb.GrainMap(grid=grid, labels=labels, n_grains=n)


@pytest.mark.parametrize("points", [False, True])
def test_grain_map_round_trip(tmp_path, points):
    rng = np.random.default_rng(3)
    gm = _grain_map(rng, points=points)
    p = tmp_path / "map.pgxg"
    binio.write_grain_map_bin(p, gm)
    back = binio.read_grain_map_bin(p)
    assert back.n_grains == gm.n_grains and np.array_equal(back.labels, gm.labels)
    assert back.grid.resolution == gm.grid.resolution
    assert np.array_equal(back.grid.points, gm.grid.points)
    # 2 bytes per pixel on a regular grid (labels only)
    assert os.path.getsize(p) == 64 + 2 * len(gm) + (0 if not points else 16 * len(gm))


def test_grain_map_wide_labels_and_3d(tmp_path):
    rng = np.random.default_rng(4)
    grid = pgb.make_grid(4, 3)
    n = 70000
    labels = rng.integers(1, n + 1, len(grid))
    gm = pgb.GrainMap(grid=grid, labels=labels, n_grains=n)
    p = tmp_path / "vox.pgxg"
    binio.write_grain_map_bin(p, gm)
    back = binio.read_grain_map_bin(p)
    assert back.grid.dim == 3 and back.grid.resolution == 4 and np.array_equal(back.labels, labels)
    assert os.path.getsize(p) == 64 + 4 * len(grid)


def test_csv_and_bin_agree(tmp_path):
    rng = np.random.default_rng(5)
    gm = _grain_map(rng, m=6, n=5)
    binio.write_grain_map_csv(tmp_path / "m.csv", gm)
    got = binio.grain_map_csv_to_bin(tmp_path / "m.csv", tmp_path / "m.pgxg")
    assert got.grid.resolution == 6  # the canonical regular grid is recognised (fileio.py:89-98)
    back = binio.read_grain_map_bin(tmp_path / "m.pgxg")
    assert np.array_equal(back.labels, gm.labels) and np.array_equal(back.grid.points, gm.grid.points)
    th = pgb.ParamMatrix(rng.normal(size=(6, 5)), pgb.DesignBasis.make("legendre", 2))
    binio.write_theta_csv(tmp_path / "t.csv", th)
    th2 = binio.theta_csv_to_bin(tmp_path / "t.csv", tmp_path / "t.pgxt")
    th3 = binio.read_theta_bin(tmp_path / "t.pgxt")
    assert np.array_equal(th2.values, th.values) and np.array_equal(th3.values, th.values)  # bit-exact
    assert th3.basis.kind == "legendre" and th3.degree == 2 and th3.gauge == th.gauge


def test_theta_gauge_and_3d(tmp_path):
    rng = np.random.default_rng(6)
    vals = rng.normal(size=(10, 4))
    vals[:, -1] = 0.0
    th = pgb.ParamMatrix(vals, pgb.DesignBasis.make("monomial", 2, 3), gauge=pgb.GAUGE_LAST_ZERO)
    binio.write_theta_bin(tmp_path / "t.pgxt", th)
    back = binio.read_theta_bin(tmp_path / "t.pgxt")
    assert back.gauge == pgb.GAUGE_LAST_ZERO and back.basis.dim == 3 and np.array_equal(back.values, vals)


def test_malformed_files_raise(tmp_path):
    rng = np.random.default_rng(7)
    gm = _grain_map(rng)
    p = tmp_path / "map.pgxg"
    binio.write_grain_map_bin(p, gm)
    raw = bytearray(p.read_bytes())
    (tmp_path / "short.pgxg").write_bytes(raw[:-3])
    with pytest.raises(pgb.InputFormatError):
        binio.read_grain_map_bin(tmp_path / "short.pgxg")
    raw[70] ^= 0xFF
    (tmp_path / "flip.pgxg").write_bytes(raw)
    with pytest.raises(pgb.InputFormatError, match="checksum"):
        binio.read_grain_map_bin(tmp_path / "flip.pgxg")
    (tmp_path / "magic.pgxg").write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(pgb.InputFormatError, match="magic"):
        binio.read_grain_map_bin(tmp_path / "magic.pgxg")
    with pytest.raises(pgb.InputFormatError):
        binio.read_theta_bin(p)  # a grain map is not a theta file
    (tmp_path / "bad.csv").write_text("x1,x2,label\n0.1,0.2,0\n0.3,0.4,1\n")
    with pytest.raises(pgb.InputFormatError, match="1-based"):
        binio.read_grain_map_csv(tmp_path / "bad.csv")
    (tmp_path / "hdr.csv").write_text("a,b,c\n")
    with pytest.raises(pgb.InputFormatError, match="header"):
        binio.read_grain_map_csv(tmp_path / "hdr.csv")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="the reference tree exists only in the build container")
def test_reads_the_reference_writers_files(tmp_path):
    """Files written by the reference's own fileio are read identically, and files
    written here are read back by the reference."""
    sys.path.insert(0, REF_SRC)
    try:
        import polygrain
        from polygrain import fileio
    finally:
        sys.path.remove(REF_SRC)
    rng = np.random.default_rng(8)
    rgrid = polygrain.make_grid(5)
    labels = rng.integers(1, 5, len(rgrid.points))
    labels[:4] = [1, 2, 3, 4]
    rmap = polygrain.GrainMap(grid=rgrid, labels=labels, n_grains=4)
    fileio.write_grain_map_csv(tmp_path / "ref.csv", rmap)
    gm = binio.read_grain_map_csv(tmp_path / "ref.csv")
    assert gm.grid.resolution == 5 and np.array_equal(gm.labels, labels)
    assert np.array_equal(gm.grid.points, rgrid.points)
    binio.write_grain_map_csv(tmp_path / "ours.csv", gm)
    assert (tmp_path / "ours.csv").read_text() == (tmp_path / "ref.csv").read_text()
    rth = polygrain.ParamMatrix(values=rng.normal(size=(6, 4)), basis=polygrain.DesignBasis.make("legendre", 2))
    fileio.write_theta_csv(tmp_path / "ref_t.csv", rth)
    th = binio.read_theta_csv(tmp_path / "ref_t.csv")
    assert np.array_equal(th.values, rth.values)
    binio.write_theta_csv(tmp_path / "ours_t.csv", th)
    assert np.array_equal(fileio.read_theta_csv(tmp_path / "ours_t.csv").values, rth.values)
