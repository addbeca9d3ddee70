"""Per-kernel times of one config (non-finite results tolerated, for experiments):
    python tools/ktime.py c5 tc [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import configs
cfg, prec = sys.argv[1], sys.argv[2]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
w = configs.make(cfg, labeler="host" if cfg in ("c1", "c2") else "gpu")
prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=prec)
acc = {}
for i in range(iters + 1):
    prob.set_profiling(True)
    try:
        prob.eval(w.theta_bench, w.eps, lam=w.lam, want_grad=True, want_assign=True)
    except Exception as e:  # noqa: BLE001
        err = type(e).__name__
    if i:
        for name, ms in prob.profile():
            acc[name] = acc.get(name, 0.0) + ms / iters
print(os.environ.get("PGX_DBG", "0"), cfg, prec, {k: round(v, 4) for k, v in acc.items()})
