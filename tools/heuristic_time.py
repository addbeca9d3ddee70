"""Wall time of the moment heuristic: device moments (pgx_label_moments) vs the
NumPy bincount path, on a config's label map.   python tools/heuristic_time.py c5 8"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import configs, heuristics
cfg = sys.argv[1]
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = configs.make(cfg, labeler="host" if cfg in ("c1", "c2") else "gpu")
gm = pgb.GrainMap(grid=w.grid, labels=w.labels0 + 1, n_grains=w.n_grains)
lab0 = np.asarray(w.labels0, dtype=np.int64)
heuristics.label_moment_sums(w.grid, lab0, w.n_grains)  # warm-up
t0 = time.perf_counter(); s = heuristics.label_moment_sums(w.grid, lab0, w.n_grains); t1 = time.perf_counter()
th = pgb.heuristic_theta(gm, deg); t2 = time.perf_counter()
pl = pgb.GrainMap(grid=pgb.PixelGrid(points=np.asarray(w.grid.points)), labels=w.labels0 + 1, n_grains=w.n_grains)
t3 = time.perf_counter(); th_cpu = pgb.heuristic_theta(pl, deg); t4 = time.perf_counter()
P = len(lab0)
print(f"{cfg}: P={P} N={w.n_grains} degree {deg}: device moments {1e3 * (t1 - t0):.2f} ms "
      f"({P / (t1 - t0) / 1e9:.2f} Gpixel/s incl. 8 B/pixel H2D), heuristic_theta {1e3 * (t2 - t1):.2f} ms; "
      f"NumPy bincount path {1e3 * (t4 - t3):.2f} ms; max |theta diff| {np.abs(th.values - th_cpu.values).max():.2e}")
