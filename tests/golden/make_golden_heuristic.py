"""Golden vectors of the REFERENCE's moment heuristic (build container only).

    python tests/golden/make_golden_heuristic.py

Runs polygrain.heuristics.moments / heuristic_theta (read-only import from
/root/reference/pkg/src) on seeded label maps of regular grids: the c1 and c2
configs and a small map with empty, single-pixel and collinear grains.  The
.npz is committed; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import polygrain as pg  # noqa: E402  (the reference)

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
from paper_2605_20816_b200 import configs  # noqa: E402  (seeded input generator only)


def degenerate_map():
    """16 x 16 grid, 7 grains: 0 empty, 1 one pixel, 2 a single column, the rest random."""
    rng = np.random.default_rng(3)
    side = 16
    lab = rng.integers(3, 7, side * side)
    lab[lab == 4] = 5
    lab[5 * side + 7] = 1            # single pixel
    lab[np.arange(side) * side + 2] = 2  # one collinear column
    return 8, lab                     # M = 8; grain 0 and 4 empty


def main():
    out = {}
    w1 = configs.c1(labeler="host")
    w2 = configs.c2(labeler="host")
    m3, lab3 = degenerate_map()
    cases = [("c1", w1.M, w1.labels0, w1.n_grains, [(1, "legendre"), (2, "legendre"), (3, "monomial")]),
             ("c2", w2.M, w2.labels0, w2.n_grains, [(2, "legendre"), (4, "legendre")]),
             ("deg", m3, lab3, 7, [(1, "legendre"), (2, "legendre"), (2, "monomial")])]
    for name, m, lab0, n, specs in cases:
        grid = pg.make_grid(m)
        gm = pg.GrainMap(grid=grid, labels=np.asarray(lab0, dtype=np.int64) + 1, n_grains=n)
        mom = pg.heuristics.moments(gm)
        out[f"{name}_m"] = np.array(m)
        out[f"{name}_labels"] = np.asarray(lab0, dtype=np.uint16)
        out[f"{name}_n"] = np.array(n)
        out[f"{name}_counts"] = mom.counts
        out[f"{name}_centroids"] = mom.centroids
        out[f"{name}_second"] = mom.second_moments
        out[f"{name}_degenerate"] = mom.degenerate
        for d, kind in specs:
            th = pg.heuristics.heuristic_theta(gm, d, kind)
            out[f"{name}_theta_{d}_{kind}"] = th.values
    path = os.path.join(OUT, "heuristic.npz")
    np.savez_compressed(path, **out)
    print(f"heuristic: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
