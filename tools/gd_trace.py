"""Pipeline trace of the tc pass-2 kernel (build with -DPGX_GD_TRACE=1):
    PGX_LIB=.../trace.so python tools/gd_trace.py c5"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_20816_b200 as pgb
from paper_2605_20816_b200 import _lib, configs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = configs.make(cfg, labeler="host" if cfg in ("c1", "c2") else "gpu")
prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision="tc")
for _ in range(3):
    try:
        prob.eval(w.theta_bench, w.eps, lam=w.lam, want_grad=True, want_assign=True)
    except Exception as exc:  # what-if builds produce garbage: only the stamps matter
        print("eval:", type(exc).__name__)
lib = _lib.load()
buf = np.zeros((14, 256), dtype=np.int64)
lib.pgx_debug_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.pgx_debug_trace(buf.ctypes.data))
t0 = buf[0, 8]
names = ["ep_S_ready", "ep_arrive", "mma_got_p", "mma_umma2_iss", "mma_umma1_iss", "ep_wait_start"]
for k in range(40, 72):
    print(k, " ".join(f"{names[e]}={buf[e, k] - t0:8d}" for e in (5, 0, 1, 2, 3, 4)))
sl = slice(40, 200)
print("per-item period (arrive k+1 - arrive k) median", np.median(np.diff(buf[1, sl])), "mean", np.diff(buf[1, sl]).mean())
print("epilogue wait for S (S_ready - wait_start) median", np.median(buf[0, sl] - buf[5, sl]), "mean", (buf[0, sl] - buf[5, sl]).mean())
print("epilogue work (arrive - S_ready) median", np.median(buf[1, sl] - buf[0, sl]))
print("arrive -> mma_got_p median", np.median(buf[2, sl] - buf[1, sl]))
print("mma_got_p -> umma2 issued median", np.median(buf[3, sl] - buf[2, sl]))
print("umma2 issued(k) -> umma1(k+3) issued median", np.median(buf[4, 43:203] - buf[3, sl]))
print("umma1(k) issued -> S(k) seen median", np.median(buf[0, sl] - buf[4, sl]))
print("next-item gap (wait_start(k+2) - arrive(k)) median", np.median(buf[5, 42:202] - buf[1, sl]))
for q in range(4):
    print(f"quarter {q}: S seen -> arrive median", np.median(buf[6 + q, sl] - buf[10 + q, sl]),
          " arrive - arrive(q0) median", np.median(buf[6 + q, sl] - buf[6, sl]),
          " S seen - S seen(q0) median", np.median(buf[10 + q, sl] - buf[10, sl]))
arr = buf[6:10, sl]
last = arr.max(axis=0)
print("last quarter arrive - first quarter arrive: median", np.median(last - arr.min(axis=0)), "mean", (last - arr.min(axis=0)).mean())
print("mma_got_p - last quarter arrive: median", np.median(buf[2, sl] - last), "mean", (buf[2, sl] - last).mean())
print("which quarter is last (counts)", np.bincount(arr.argmax(axis=0), minlength=4))
for k in range(40, 56):
    print(k, "arrive q0..q3", (buf[6:10, k] - t0).tolist(), "S seen q0..q3", (buf[10:14, k] - t0).tolist(), "got_p", buf[2, k] - t0)
