import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import configs
from paper_2605_20816_b200.optimizer import _DeviceState
cfg = sys.argv[1]
w = configs.make(cfg, labeler="host" if cfg in ("c1", "c2") else "gpu")
prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision="tc")
t0 = time.perf_counter(); dev = _DeviceState(prob, 10, w.lam); print("create", time.perf_counter() - t0)
th = np.zeros((w.K, w.n_grains))
def tm(name, f):
    t0 = time.perf_counter(); r = f(); print(f"{name}: {1e3 * (time.perf_counter() - t0):.3f} ms"); return r
tm("start", lambda: dev.start(th, w.eps))
for i in range(4):
    tm("iterate", lambda: dev.iterate(1.0, w.eps))
    tm("trial", lambda: dev.trial(0.5, w.eps))
    tm("trial", lambda: dev.trial(0.25, w.eps))
    tm("accept", lambda: dev.accept(True))
    tm("direction", lambda: dev.direction(0))
tm("theta", lambda: dev.theta())
tm("eval host", lambda: prob.eval(th, w.eps, lam=w.lam, want_grad=True, want_assign=True))
tm("eval host", lambda: prob.eval(th, w.eps, lam=w.lam, want_grad=True, want_assign=True))
