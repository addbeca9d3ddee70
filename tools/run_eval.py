"""Run a few fused evaluations of one config (for ncu / compute-sanitizer captures).

    python tools/run_eval.py --config c2 --precision fp64 --iters 3
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2605_20816_b200 as pgb  # noqa: E402
from paper_2605_20816_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--theta", default="bench", choices=["bench", "normal"])
ap.add_argument("--assign", action="store_true", help="also run one hard assignment")
a = ap.parse_args()
w = configs.make(a.config, labeler="host" if a.config in ("c1", "c2", "paper140") else "gpu")
prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=a.precision)
th = w.theta_bench if a.theta == "bench" else np.random.default_rng(0).normal(size=(w.K, w.n_grains))
for _ in range(a.iters):
    t0 = time.perf_counter()
    res, st = prob.eval(th, w.eps, lam=w.lam, want_grad=True, want_assign=True)
    print(f"{a.config} {a.precision}: phi={res.phi:.12f} err={res.err:.6f} "
          f"amb={st.n_ambiguous} wall={1e3 * (time.perf_counter() - t0):.3f} ms")
if a.assign:
    lab = prob.assign(th)
    print(f"assign: {len(np.unique(lab))} distinct labels, kernels {[n for n, _ in prob.profile()]}")
prob.close()
