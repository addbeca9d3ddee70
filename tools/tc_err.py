"""Worst tc-vs-exact errors (relative to the test tolerances' scales) over the
configs at the bench theta and a N(0,1) theta:  python tools/tc_err.py [c1 c2 ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import configs
names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
for name in names:
    w = configs.make(name, labeler="gpu")
    rng = np.random.default_rng(21)
    thetas = [np.asarray(w.theta_bench, dtype=np.float64), rng.normal(size=(w.K, w.n_grains))]
    ex = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision="exact")
    tc = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision="tc")
    for j, th in enumerate(thetas):
        r, _ = ex.eval(th, w.eps, lam=w.lam, want_assign=True)
        t, _ = tc.eval(th, w.eps, lam=w.lam, want_assign=True)
        print(f"{os.environ.get('PGX_LIB', 'lib')[-12:]} {name} theta{j}: phi {abs(t.phi - r.phi) / (1 + abs(r.phi)):.2e}"
              f" grad {np.abs(t.grad - r.grad).max() / np.abs(r.grad).max():.2e}")
    ex.close(); tc.close()
