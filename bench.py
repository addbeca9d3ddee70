"""Benchmark of the fused Phi + grad + assignment evaluation (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--precision fp64]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

One "step" = one fused objective+gradient+assignment evaluation of the whole
workload (the unit ``fit`` calls per trial point, optimizer.py:215-219).
Default workload: BASELINE.json configs[1] (c2).  Multi-GPU runs are replicas
(the north_star forbids multi-GPU data paths): every rank evaluates
the full workload; value = all ranks' logits / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

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
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    # tc: tcgen05 logits (3-product fp16 split, fp32 accumulate) -- the north-star
    # path, within the stated 1e-6 (phi) / 1e-5 (grad) tolerances; fp64 and exact
    # are the tighter modes
    ap.add_argument("--precision", default=os.environ.get("PGX_PRECISION", "tc"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
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

    w = configs.make(args.config, labeler="host" if args.config in ("c1", "c2") else "gpu")
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


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2605_20816_b200 as pgb
    from paper_2605_20816_b200 import _lib, configs

    w = configs.make(args.config, labeler="host" if args.config in ("c1", "c2") else "gpu")
    stream = torch.cuda.Stream(device=dev)
    prob = pgb.Problem(w.grid, w.kind, w.degree, w.n_grains, w.labels0,
                       precision=args.precision, device=local, stream=stream.cuda_stream)
    K, N, P = w.K, w.n_grains, w.n_points
    f32 = w.theta_dtype == "f32"
    theta_d = torch.as_tensor(np.asarray(w.theta_bench), device=dev)
    grad_d = torch.empty((K, N), dtype=torch.float64, device=dev)
    stats_d = torch.empty(8, dtype=torch.float64, device=dev)
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

    # ---- kernel-level timing (dominant kernel) with CUDA events, same stream
    prob.set_profiling(True)
    per_kernel = {}
    with torch.cuda.stream(stream):
        for _ in range(max(3, min(args.steps, 20))):
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
    stats_h = torch.empty(8, dtype=torch.float64, pin_memory=True)
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
    d2h = K * N * 8 + 64

    # ---- roofline of the dominant kernel
    peaks, peaks_kind = load_peaks()
    clocks = clk.summary()
    mhz = clocks["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    t_top = avg[top] / 1000.0
    logits = P * N
    flops_top = (2 if "pass1" in top else 4) * logits * K
    exps_top = logits
    bytes_top = P * 4 + K * N * 8 + (16 * P if "pass1" in top else 16 * P + 8 * K * N)
    tensor_peak = peaks["bf16_tflops"] * 1e12
    pipes = {
        "fp64": {"achieved": flops_top / t_top / 1e12,
                 "peak": 2 * DFMA_PER_CLK_SM * N_SMS * mhz * 1e6 / 1e12, "unit": "TFLOP/s"},
        "mufu_ex2": {"achieved": exps_top / t_top / 1e9,
                     "peak": MUFU_PER_CLK_SM * N_SMS * mhz * 1e6 / 1e9, "unit": "Gexp/s"},
        "hbm": {"achieved": bytes_top / t_top / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"},
        "tensor": {"achieved": flops_top / t_top / 1e12, "peak": tensor_peak / 1e12,
                   "unit": "TFLOP/s"},
    }
    for v in pipes.values():
        v["frac"] = v["achieved"] / v["peak"]
    binding = max(("fp64", "mufu_ex2") if args.precision != "tc" else ("tensor", "mufu_ex2"),
                  key=lambda k: pipes[k]["frac"])
    traffic, traffic_src = measured_traffic(args.config, args.precision, top)
    roofline = {
        "bound": "tensor", "achieved": pipes["tensor"]["achieved"], "peak": pipes["tensor"]["peak"],
        "unit": "TFLOP/s", "frac": pipes["tensor"]["frac"], "traffic": traffic,
        "traffic_source": traffic_src, "algorithmic_bytes": bytes_top,
        "kernel": top, "kernel_ms": avg[top], "kernel_share": avg[top] / (sum(avg.values())),
        "peak_kind": f"{peaks_kind} (bf16 burst, MEASURED_PEAKS.json)",
        "binding_pipe": binding, "binding_frac": pipes[binding]["frac"], "pipes": pipes,
        "kernels_ms": avg,
        "note": ("algorithmic work of the dominant kernel: pass1 = 2PNK flops + PN exps, "
                 "pass2 = 4PNK flops + PN exps; SFU/FP64 peaks = per-SM issue rate x 148 SMs x "
                 "median SM clock under load"),
    }

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        threads = os.cpu_count() or 1
        rate, desc, _, _ = cpu_measure(w, args.cpu_seconds, threads)
        cpu_baseline = {"value": rate, "unit": "logits/s", "cores": threads, "kind": "port",
                        "sample": desc}

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
                                 "stats: stored by the tail kernel into mapped pinned host memory "
                                 "(pgx_eval zero-copy results), then stream sync"},
            "roofline": roofline,
            "cpu_baseline": cpu_baseline,
            "gpu_launches": launches,
            "clocks": clocks,
            "result": {"phi": float(stats[0]), "err": float(stats[1]), "e0": float(stats[2]),
                       "n_rescanned": int(stats[3]),
                       "n_ambiguous": int(stats.view(np.int64)[6])},
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


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
