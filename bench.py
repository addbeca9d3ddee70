"""Benchmark of the fused Phi + grad + assignment evaluation (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--precision tc]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

One "step" = one fused objective+gradient+assignment evaluation of the whole
workload (the unit ``fit`` calls per trial point, optimizer.py:215-219).
Default workload: c5, the largest single-GPU config of BASELINE.json (the
north_star's ">= 60% of roofline on the largest config").  Multi-GPU runs are replicas
(the north_star forbids multi-GPU data paths): every rank evaluates
the full workload; value = all ranks' logits / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

# The CPU legs (cpu_baseline, --impl reference) parallelise the NumPy oracle
# with a chunk thread pool; BLAS must then be single-threaded, and this has to
# be set before the first numpy import anywhere in the process.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pixel×grain logits/s for fused objective+gradient; % of roofline"
L2_FLUSH_BYTES = 256 << 20
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# B200 per-SM issue rates (CUDA programming guide arithmetic-throughput table)
MUFU_PER_CLK_SM = 16       # ex2 / lg2 results per clock per SM
DFMA_PER_CLK_SM = 64       # fp64 FMA per clock per SM
N_SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "paper140"])
    # tc: tcgen05 logits (3-product fp16 split, fp32 accumulate) -- the north-star
    # path, within the stated 1e-6 (phi) / 1e-5 (grad) tolerances; fp64 and exact
    # are the tighter modes
    ap.add_argument("--precision", default=os.environ.get("PGX_PRECISION", "tc"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    # the fp64 mode measured beside the headline mode (same problem, same theta)
    ap.add_argument("--also", default="fp64", help="comma list of extra precision modes ('' = none)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML polling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # noqa: BLE001
            self._nvml = None
            self.error = str(exc)

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nvml is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        if self._nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.error}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit]
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    return world, rank, local


def max_over_ranks(value: float, world: int, device) -> float:
    """Max of a per-rank float over all ranks (the contract's timing rule)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(world: int, steps: int, units_per_step: int, t_max: float) -> float:
    """Whole-job throughput of N independent replicas: every rank processed
    ``steps`` x ``units_per_step`` units; the job time is the slowest rank's."""
    return world * steps * units_per_step / t_max


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_measure(w, seconds: float, threads: int):
    """Time the CPU oracle (NumPy port of the reference, threads = pool size) on
    a bounded pixel-prefix sample of the workload; returns (logits/s, sample)."""
    import numpy as np

    import oracle

    pts = oracle.grid_points(w.M, w.dim)
    theta = np.asarray(w.theta_bench, dtype=np.float64)
    n = pts.shape[0]
    sample = n
    # size the sample so one evaluation is ~1/4 of the budget (probe on 8192 px)
    t0 = time.perf_counter()
    oracle.evaluate_problem(theta, w.kind, w.degree, pts, w.labels0, w.eps, want_grad=True,
                            want_assign=True, threads=threads, max_points=8192)
    per_px = (time.perf_counter() - t0) / 8192
    sample = int(min(n, max(8192, seconds / 4 / max(per_px, 1e-12))))
    sample = (sample // 8192) * 8192 or 8192
    reps, t_total = 0, 0.0
    while t_total < seconds and reps < 1000:
        t0 = time.perf_counter()
        oracle.evaluate_problem(theta, w.kind, w.degree, pts, w.labels0, w.eps, want_grad=True,
                                want_assign=True, threads=threads, lam=w.lam, max_points=sample)
        t_total += time.perf_counter() - t0
        reps += 1
    rate = reps * sample * w.n_grains / t_total
    desc = (f"{reps} x fused eval of the first {sample} of {n} pixels x {w.n_grains} grains "
            f"({w.name}, oracle NumPy port, threads={threads}, OPENBLAS_NUM_THREADS="
            f"{os.environ.get('OPENBLAS_NUM_THREADS', 'unset')})")
    return rate, desc, reps, t_total


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from paper_2605_20816_b200 import configs

    w = configs.make(args.config, labeler="host" if args.config in ("c1", "c2", "paper140") else "gpu")
    threads = os.cpu_count() or 1
    import numpy as np

    import oracle

    pts = oracle.grid_points(w.M, w.dim)
    theta = np.asarray(w.theta_bench, dtype=np.float64)
    # bounded sample per step: ~2 s of work
    t0 = time.perf_counter()
    oracle.evaluate_problem(theta, w.kind, w.degree, pts, w.labels0, w.eps, want_grad=True,
                            want_assign=True, threads=threads, max_points=8192)
    per_px = (time.perf_counter() - t0) / 8192
    sample = int(min(pts.shape[0], max(8192, 2.0 / max(per_px, 1e-12))))
    sample = (sample // 8192) * 8192 or 8192
    for _ in range(args.warmup):
        oracle.evaluate_problem(theta, w.kind, w.degree, pts, w.labels0, w.eps, want_grad=True,
                                want_assign=True, threads=threads, lam=w.lam, max_points=sample)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.evaluate_problem(theta, w.kind, w.degree, pts, w.labels0, w.eps, want_grad=True,
                                want_assign=True, threads=threads, lam=w.lam, max_points=sample)
    dt = time.perf_counter() - t0
    value = args.steps * sample * w.n_grains / dt
    desc = (f"fused eval of the first {sample} of {pts.shape[0]} pixels x {w.n_grains} grains "
            f"per step ({w.name}); oracle NumPy port of polygrain.evaluate_objective, "
            f"{threads}-thread chunk pool")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "logits/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "description": w.description, "P": w.n_points,
                   "N": w.n_grains, "K": w.K, "sample_pixels": sample},
        "cpu_baseline": {"value": value, "unit": "logits/s", "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "logits/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ roofline
FP64_DFMA_PER_CLK_SM = 59   # measured FP64 FMA rate on this pool's B200s (tools/)


def roofline_8d(P, N, K, precision, t_eval_s, peaks, sm_mhz):
    """T_roof = max(4PNK / F_mode, PN / E_exp, B / BW_HBM); frac = T_roof / t_eval.

    F_mode: tc = measured bf16 burst peak / 3 (the 3-product fp16 split), fp64 /
    exact = the FP64 FMA peak; E_exp = 16 MUFU ex2 /clk/SM x 148 x sm_max clock;
    B = the algorithmic minimum labels 4P + theta 4KN + grad 8KN (§8d)."""
    clk = sm_mhz * 1e6
    flops, exps, nbytes = 4.0 * P * N * K, float(P * N), 4.0 * P + 12.0 * K * N
    if precision == "tc":
        f_peak, f_name = peaks["bf16_tflops"] * 1e12 / 3.0, "tensor"
    else:
        f_peak, f_name = 2.0 * FP64_DFMA_PER_CLK_SM * N_SMS * clk, "fp64"
    e_peak = MUFU_PER_CLK_SM * N_SMS * clk
    bw = peaks["hbm_gbs"] * 1e9
    terms = {f_name: flops / f_peak, "mufu": exps / e_peak, "hbm": nbytes / bw}
    bound = max(terms, key=terms.get)
    t_roof = terms[bound]
    work = {f_name: (flops / 1e12, f_peak / 1e12, "TFLOP/s"), "mufu": (exps / 1e9, e_peak / 1e9, "Gexp/s"),
            "hbm": (nbytes / 1e9, bw / 1e9, "GB/s")}[bound]
    return {
        "bound": bound, "achieved": work[0] / t_eval_s, "peak": work[1], "unit": work[2],
        "frac": t_roof / t_eval_s, "t_roof_ms": 1e3 * t_roof, "t_eval_ms": 1e3 * t_eval_s,
        "terms_ms": {k: 1e3 * v for k, v in terms.items()},
        "fracs": {k: v / t_eval_s for k, v in terms.items()},
        "algorithmic": {"flops": flops, "exps": exps, "bytes": nbytes},
        "peaks": {"F_mode_tflops": f_peak / 1e12, "E_exp_gexps": e_peak / 1e9, "hbm_gbs": bw / 1e9,
                  "sm_mhz": sm_mhz},
    }


def kernel_roofline(name, ms, P, N, K, peaks, sm_mhz):
    """The dominant kernel's own fraction: pass 1 = 2PNK flops + PN exps,
    pass 2 = 2PNK flops + PN exps (each recomputes the logits; §8d splits the
    4PNK evenly), other kernels: bytes only."""
    t = ms / 1e3
    clk = sm_mhz * 1e6
    exps = float(P * N)
    e_peak = MUFU_PER_CLK_SM * N_SMS * clk
    f_peak = peaks["bf16_tflops"] * 1e12 / 3.0
    if "pass" in name or "sweep" in name or "grad" in name:
        return {"kernel": name, "ms": ms, "mufu_frac": exps / e_peak / t,
                "tensor_frac": 2.0 * P * N * K / f_peak / t}
    return {"kernel": name, "ms": ms}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


class _OracleProblem:
    """CPU stand-in for ``Problem`` in the cpu_baseline leg: the reference fit
    loop (optimizer.fit, a port of optimizer.py:195-342) evaluating through the
    NumPy oracle port of objective.evaluate_objective."""

    def __init__(self, w):
        import oracle

        self._o = oracle
        self.w = w
        self.pts = oracle.grid_points(w.M, w.dim)

    def eval(self, theta, eps, *, lam=0.0, want_grad=True, want_assign=False):
        r = self._o.evaluate_problem(theta, self.w.kind, self.w.degree, self.pts, self.w.labels0,
                                     eps, want_grad=want_grad, want_assign=want_assign, lam=lam)
        from paper_2605_20816_b200.objective import EvalResult

        return EvalResult(r.phi, r.grad, r.err, r.e0), None


def fit_c1(problem, precision=None, device_loop=False, repeats=1, method="lbfgs"):
    """The reference fit at c1: 100 L-BFGS iterations
    (the last of `repeats` runs on one problem is reported: a fit's first run on a
    fresh GPU problem pays the one-time set-up launches and graph captures)."""
    import paper_2605_20816_b200 as pgb
    from paper_2605_20816_b200 import configs

    w = configs.c1(labeler="host")
    gm = pgb.GrainMap(grid=w.grid, labels=w.labels0 + 1, n_grains=w.n_grains)
    # (BASELINE c1: eps = 0.05, lambda = 1e-4 with the ascent variant; the reference's own fit
    # is L-BFGS at lambda = 0)
    cfg = pgb.FitConfig(degree=w.degree, basis_kind=w.kind, eps=w.eps, max_iters=100,
                        precision=precision or "tc", device_loop=device_loop, method=method,
                        lam=w.lam if method == "ascent" else 0.0)
    prob = problem(w) if callable(problem) else problem
    if prob is None and repeats > 1:
        prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=precision or "tc")
    for _ in range(repeats):
        t0 = time.perf_counter()
        rep = pgb.fit(gm, cfg, problem=prob)
        dt = time.perf_counter() - t0
    return {"seconds": dt, "iterations": rep.iterations_run, "evaluations": rep.evaluations,
            "evals_per_s": rep.evaluations / dt, "phi_final": rep.phi_final, "stop": rep.stop_reason,
            "loop": "device-resident state + CUDA graphs" if device_loop else "host", "runs": repeats,
            "method": method}


def cpu_baseline_leg(w, seconds):
    """The oracle (NumPy port of polygrain.evaluate_objective) on this host's
    cores: all threads (the reported value) and 1 thread, plus the c1 fit."""
    threads = os.cpu_count() or 1
    rate, desc, _, _ = cpu_measure(w, seconds, threads)
    rate1, desc1, _, _ = cpu_measure(w, seconds / 2, 1)
    fit = fit_c1(_OracleProblem)
    return {"value": rate, "unit": "logits/s", "cores": threads, "kind": "port", "sample": desc,
            "cpu_model": cpu_model(), "nproc": threads,
            "single_thread": {"value": rate1, "unit": "logits/s", "cores": 1, "sample": desc1},
            "fit_c1": fit}


# ------------------------------------------------------------------ our arm
def time_mode(prob, step, flush, stream, steps, warmup, dev):
    """Device time per step (CUDA events on the problem's stream, L2 flushed
    between steps outside the events)."""
    import torch

    with torch.cuda.stream(stream):
        for _ in range(max(warmup, 0)):
            step()
        torch.cuda.synchronize(dev)
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        for i in range(steps):
            flush.zero_()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
    return [a.elapsed_time(b) for a, b in zip(starts, ends)]


def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2605_20816_b200 as pgb
    from paper_2605_20816_b200 import _lib, configs

    w = configs.make(args.config, labeler="host" if args.config in ("c1", "c2", "paper140") else "gpu")
    stream = torch.cuda.Stream(device=dev)
    prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0,
                       precision=args.precision, device=local, stream=stream.cuda_stream)
    K, N, P = w.K, w.n_grains, w.n_points
    f32 = w.theta_dtype == "f32"
    theta_d = torch.as_tensor(np.asarray(w.theta_bench), device=dev)
    grad_d = torch.empty((K, N), dtype=torch.float64, device=dev)
    stats_d = torch.empty(_lib.STATS_WORDS, dtype=torch.float64, device=dev)
    flags = _lib.PGX_WANT_GRAD | _lib.PGX_WANT_ASSIGN | (_lib.PGX_THETA_F32 if f32 else 0)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step():
        prob.eval_device(theta_d.data_ptr(), w.eps, w.lam, flags, grad_d.data_ptr(),
                         stats_d.data_ptr())

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 0)):
            step()
        torch.cuda.synchronize(dev)
        barrier(world)
        torch.cuda.synchronize(dev)
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        launches = 0
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                flush.zero_()  # L2 flush between timed steps (outside the events)
                starts[i].record(stream)
                step()
                ends[i].record(stream)
                launches += prob.last_launch_count()
            torch.cuda.synchronize(dev)
        barrier(world)
        torch.cuda.synchronize(dev)
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_rank = sum(step_ms) / 1000.0
    t_max = max_over_ranks(t_rank, world, dev)
    value = replica_value(world, args.steps, P * N, t_max)
    stats = stats_d.cpu().numpy()

    # ---- kernel-level timing with CUDA events on the problem's stream
    prob.set_profiling(True)
    per_kernel = {}
    with torch.cuda.stream(stream):
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            step()
            for name, ms in prob.profile():
                per_kernel.setdefault(name, []).append(ms)
    prob.set_profiling(False)
    avg = {k: sum(v) / len(v) for k, v in per_kernel.items()}
    top = max(avg, key=avg.get)

    # ---- e2e through the C ABI with HOST buffers (pinned), copies inside the timing
    theta_h = torch.empty(theta_d.shape, dtype=theta_d.dtype, pin_memory=True)
    theta_h.copy_(theta_d.cpu())
    grad_h = torch.empty((K, N), dtype=torch.float64, pin_memory=True)
    stats_h = torch.empty(_lib.STATS_WORDS, dtype=torch.float64, pin_memory=True)
    host_flags = flags & ~_lib.PGX_DEVICE_PTRS
    lib = _lib.load()

    def step_host():
        _lib.check(lib.pgx_eval(prob.handle, theta_h.data_ptr(), float(w.eps), float(w.lam),
                                host_flags, grad_h.data_ptr(), stats_h.data_ptr()))

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 1)):
            step_host()
        e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            step_host()
            e.record(stream)
            e.synchronize()
            e_ms.append(s.elapsed_time(e))
    t_e2e = max_over_ranks(sum(e_ms) / 1000.0, world, dev)
    e2e_value = replica_value(world, args.steps, P * N, t_e2e)
    h2d = K * N * (4 if f32 else 8)
    d2h = K * N * 8 + 8 * _lib.STATS_WORDS

    # ---- the other precision modes on the same workload (device-timed)
    modes = {}
    for m in [x for x in args.also.split(",") if x and x != args.precision]:
        pm = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0, precision=m,
                         device=local, stream=stream.cuda_stream)

        def step_m(pm=pm):
            pm.eval_device(theta_d.data_ptr(), w.eps, w.lam, flags, grad_d.data_ptr(),
                           stats_d.data_ptr())

        ms = time_mode(pm, step_m, flush, stream, max(3, args.steps // 4), 2, dev)
        t_m = sum(ms) / 1e3 / len(ms)
        modes[m] = {"ms_per_step": 1e3 * t_m, "value": P * N / t_m, "unit": "logits/s",
                    "dtype": DTYPE[m], "phi": float(stats_d[0].item())}
        pm.close()

    # ---- hard assignment (pgx_assign: hard_assign without the N x P costs), device-timed
    assign = None
    try:
        lab_d = torch.empty(P, dtype=torch.int64, device=dev)

        def step_a():
            prob.assign_device(theta_d.data_ptr(), flags & _lib.PGX_THETA_F32, lab_d.data_ptr())

        ms = time_mode(prob, step_a, flush, stream, max(3, args.steps // 4), 2, dev)
        prob.set_profiling(True)
        with torch.cuda.stream(stream):
            step_a()
            a_kern = {n: v for n, v in prob.profile()}
        prob.set_profiling(False)
        t_a = sum(ms) / 1e3 / len(ms)
        assign = {"ms_per_step": 1e3 * t_a, "value": P * N / t_a, "unit": "logits/s",
                  "kernels_ms": a_kern, "labels_checksum": int(lab_d.sum().item())}
    except Exception as exc:  # noqa: BLE001
        assign = {"error": repr(exc)}

    # ---- roofline (§8d, whole evaluation) + the dominant kernel
    peaks, peaks_kind = load_peaks()
    clocks = clk.summary()
    sm_peak = float(peaks.get("sm_max_mhz", 1965.0))
    t_eval = t_max / args.steps
    roofline = roofline_8d(P, N, K, args.precision, t_eval, peaks, sm_peak)
    traffic, traffic_src = measured_traffic(args.config, args.precision, top)
    roofline.update({
        "traffic": traffic, "traffic_source": traffic_src,
        "peak_kind": f"{peaks_kind} (MEASURED_PEAKS.json bf16 burst / 3; MUFU 16/clk/SM x 148 x "
                     f"sm_max {sm_peak:.0f} MHz; HBM copy)",
        "dominant": kernel_roofline(top, avg[top], P, N, K, peaks, sm_peak),
        "kernel_share": avg[top] / sum(avg.values()),
        "kernels_ms": avg,
    })

    cpu_baseline = None
    fit = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_baseline = cpu_baseline_leg(w, args.cpu_seconds)
    if rank == 0 and world == 1:
        try:
            fit = fit_c1(None, args.precision, repeats=2)
            fit["device_loop"] = fit_c1(None, args.precision, device_loop=True, repeats=2)
            fit["ascent_device_loop"] = fit_c1(None, args.precision, device_loop=True, repeats=2,
                                               method="ascent")
        except Exception as exc:  # noqa: BLE001
            fit = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "logits/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE[args.precision],
            "data": "synthetic (seeded; SURVEY.md §8d generators)",
            "config": {"workload": w.name, "description": w.description, "P": P, "N": N, "K": K,
                       "precision": args.precision, "theta_dtype": w.theta_dtype,
                       "parallelism": f"replicas x{world}",
                       "l2": "flushed between timed steps (256 MiB memset, outside the events)",
                       "nonempty_grains": w.n_nonempty},
            "evals_per_s": world * args.steps / t_max,
            "e2e": {"value": e2e_value, "unit": "logits/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": 1000 * t_e2e / args.steps,
                    "transfers": "theta: cudaMemcpyAsync H2D from pinned host memory; gradient + "
                                 "stats: D2H (or, <= 256 KB, stored by the tail kernel into mapped "
                                 "pinned host memory), then stream sync"},
            "roofline": roofline,
            "modes": modes,
            "assign": assign,
            "cpu_baseline": cpu_baseline,
            "fit_c1_gpu": fit,
            "gpu_launches": launches,
            "clocks": clocks,
            "result": {"phi": float(stats[0]), "err": float(stats[1]), "e0": float(stats[2]),
                       "n_rescanned": int(stats[3]),
                       "n_ambiguous": int(stats.view(np.int64)[6]),
                       "flags": int(stats.view(np.int64)[8])},
        }
        print(json.dumps(line), flush=True)
    prob.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def measured_traffic(config: str, precision: str, kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the latest committed
    ncu --set full capture (profiles/*_traffic.json, written from the .ncu-rep
    of tools/profile_round.sh), or (None, None)."""
    import glob
    for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                              "profiles", "*_traffic.json")), reverse=True):
        try:
            with open(path) as f:
                ent = json.load(f).get(f"{config}_{precision}:{kernel}")
        except (OSError, ValueError):
            continue
        if ent:
            return ent["dram_bytes_read"] + ent["dram_bytes_write"], os.path.relpath(path)
    return None, None


# arithmetic the path computes in, per precision mode
DTYPE = {"tc": "f16x3-f32", "fp64": "f64", "exact": "f64"}


def self_launch(args) -> bool:
    """`bench.py --gpus N` without torchrun: launch the N ranks ourselves
    (one process per GPU, the driver's own torchrun form)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
