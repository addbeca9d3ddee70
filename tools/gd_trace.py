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
    prob.eval(w.theta_bench, w.eps, lam=w.lam, want_grad=True, want_assign=True)
lib = _lib.load()
buf = np.zeros((5, 256), dtype=np.int64)
lib.pgx_debug_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.pgx_debug_trace(buf.ctypes.data))
t0 = buf[0, 8]
names = ["ep_S_ready", "ep_arrive", "mma_got_p", "mma_umma2_done", "mma_umma1_done"]
for k in range(8, 40):
    print(k, " ".join(f"{names[e]}={buf[e, k] - t0:8d}" for e in range(5)),
          " chain(arrive->S(k+3) seen)=%d" % (buf[0, k + 3] - buf[1, k] if k + 3 < 256 else -1))
d = np.diff(buf[1, 20:200])
print("per-item epilogue period (even/odd interleaved):", np.median(d), "mean", d.mean())
print("arrive->mma_got_p median", np.median(buf[2, 20:200] - buf[1, 20:200]))
print("mma_got_p->umma2 issued median", np.median(buf[3, 20:200] - buf[2, 20:200]))
print("umma2->umma1(k+3) issued median", np.median(buf[4, 20:200] - buf[3, 20:200]))
print("umma1(k+3) issued -> S(k+3) seen median", np.median(buf[0, 23:203] - buf[4, 20:200]))
print("S seen -> arrive (epilogue item) median", np.median(buf[1, 20:200] - buf[0, 20:200]))
