"""Wall time of fit() with the host-resident and the device-resident L-BFGS loop.
    python tools/fit_time.py c1 100 tc"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import configs
cfg = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prec = sys.argv[3] if len(sys.argv) > 3 else "tc"
w = configs.make(cfg, labeler="host" if cfg in ("c1", "c2") else "gpu")
gm = pgb.GrainMap(grid=w.grid, labels=w.labels0 + 1, n_grains=w.n_grains)
prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=prec)
for dev in (False, True, False, True):
    c = pgb.FitConfig(degree=w.degree, basis_kind=w.kind, eps=w.eps, lam=w.lam, max_iters=iters,
                      precision=prec, device_loop=dev)
    t0 = time.perf_counter()
    rep = pgb.fit(gm, c, problem=prob)
    dt = time.perf_counter() - t0
    print(f"{cfg} {prec} device_loop={dev}: {rep.iterations_run} iterations, {rep.evaluations} evaluations, "
          f"{dt:.3f} s ({1e3 * dt / max(1, rep.evaluations):.3f} ms/eval), phi {rep.phi_final:.12f}, stop {rep.stop_reason}")
