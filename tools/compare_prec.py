"""Compare precision modes on one config: python tools/compare_prec.py c2 [fp64 tc exact]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2605_20816_b200 as pgb  # noqa: E402
from paper_2605_20816_b200 import configs  # noqa: E402

name = sys.argv[1]
modes = sys.argv[2:] or ["fp64", "tc"]
w = configs.make(name, labeler="host" if name in ("c1", "c2") else "gpu")
rng = np.random.default_rng(0)
thetas = {"bench": np.asarray(w.theta_bench, dtype=np.float64),
          "normal": rng.normal(size=(w.K, w.n_grains))}
res = {}
for mode in modes:
    prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=mode)
    for tn, th in thetas.items():
        r, st = prob.eval(th, w.eps, want_grad=True, want_assign=True)
        prob.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            prob.eval(th, w.eps, want_grad=True, want_assign=True)
        dt = (time.perf_counter() - t0) / 3
        res[(mode, tn)] = (r, st)
        print(f"{name} {mode:5s} theta={tn:6s} phi={r.phi:.12f} err={r.err:.6f} e0={r.e0:.8f} "
              f"amb={st.n_ambiguous} rescanned={st.n_rescanned} wall={1e3 * dt:.3f} ms")
    prob.close()
base = modes[0]
for mode in modes[1:]:
    for tn in thetas:
        a, sa = res[(base, tn)]
        b, sb = res[(mode, tn)]
        gr = np.abs(a.grad - b.grad).max() / np.abs(a.grad).max()
        gn = np.linalg.norm(a.grad - b.grad) / np.linalg.norm(a.grad)
        print(f"  {mode} vs {base} [{tn}]: dphi={abs(a.phi - b.phi) / (1 + abs(a.phi)):.2e} "
              f"dgrad_max={gr:.2e} dgrad_norm={gn:.2e} derr={abs(a.err - b.err) * w.n_points:.0f}px "
              f"de0={abs(a.e0 - b.e0):.2e}")
