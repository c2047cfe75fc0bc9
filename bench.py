#!/usr/bin/env python
"""Benchmark of the shifted-Krylov hot path (one JSON line on rank 0).

A step is one full iteration of shifted COCG/BiCG (seed SpMV with
fused dot, scalar recurrences + retirement + seed switch, fused three-term update with the
next-iteration dots and the per-shift projected / full update) over the config's synthetic
input.  Default workload: C5 (BASELINE.json configs[4], the largest single-GPU config and the
north star's HBM / scaling config) — Heisenberg L=30, M=2^30, N_z=512, a=b projection, COCG,
complex128; `--config c1..c5` selects another (C2 is the latency-bound configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Timing: W untimed iterations, then three passes of K iterations, each step
bracketed by CUDA events on the solver's stream with L2 flushed (256 MiB write) before every
step outside the events; barrier + synchronize around each pass; max over ranks; `value` is the
median pass.  Clocks are sampled with NVML every 2 ms (nvidia-smi where NVML is missing) during
the timed passes.  A fourth pass of the same K flushed steps records CUDA events around every
kernel (on the solver's stream) for the per-kernel durations behind `roofline` (events between
the kernels cost the programmatic-launch overlap, so that pass is not the value).

CPU legs (the oracle, oracle/, test infrastructure timed as it stands): `cpu_baseline` runs the
OpenMP build on all host cores over the first iterations of the full-size workload (a bounded
sample, ~20 s); `cpu_baseline_1core` runs the one-thread build on a scaled instance of the same
config (16x fewer rows, same shifts) and extrapolates to the full size (the oracle's cost is
linear in M; labelled as such).  `--impl reference` times the OpenMP oracle on the workload itself
(the reference arm of this tier: the paper has no code).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "shift-iterations/sec (N_z x iters / s)"
UNIT = "shift-it/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def bytes_per_row(problem, kernel: str, plan=None) -> float:
    """Algorithmic bytes per row of one launch.

    With the bond split's fused r_{n-1} term (plan["split_fuse"]) the SpMV also
    reads r_{n-1} (+16) and the update no longer does (-16): the iteration's total is unchanged."""
    nseq = 2 if problem.method == "bicg" else 1
    shift = 16.0 if plan and plan.get("split_fuse") else 0.0
    if kernel == "spmv":
        return bytes_per_row(problem, "spmv_") + shift
    if kernel == "update":
        return bytes_per_row(problem, "update_") - shift
    if kernel == "spmv_":
        if problem.op["kind"] in ("heisenberg", "heisenberg_sz"):   # generated on the fly
            bh = 0.0
        else:
            nnz_row = problem.op["col"].shape[0] / problem.M
            vb = 8 if problem.op["kind"] == "csr_real" else 16
            bh = nnz_row * (vb + 4) + 8
        return bh + 32.0 * nseq
    if kernel == "update_":
        b = 64.0 * nseq + 16.0 * problem.n_left
        if problem.full_x:
            b += 64.0 * problem.n_shift   # all shifts active during the timed window
        return b
    raise KeyError(kernel)


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    NVML (pynvml) polled every 2 ms from a thread, so even a few-ms timed region gets several
    samples; nvidia-smi (-lms 100) where NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []     # (sm_mhz, sm_max_mhz, {reason names}) from NVML
        self.power = []       # board power samples (W), NVML
        self.power_limit = None
        self.stop = threading.Event()
        self.source = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.bits = [pynvml.nvmlClocksEventReasonHwSlowdown,
                         pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwPowerCap]
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.nvml, self.h = pynvml, h
            self._sample_nvml()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            self.source = "nvml"
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self.source = "nvidia-smi"
        except OSError:
            self.proc = None
        return self

    def _sample_nvml(self):
        nv = self.nvml
        sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((sm, self.smax, {n for n, b in zip(self.NAMES, self.bits) if r & b}))
        try:   # board power (W), to explain sw_power_cap (the enforced limit is recorded once)
            self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            if self.power_limit is None:
                self.power_limit = nv.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
        except Exception:
            pass

    def _poll(self):
        while not self.stop.wait(self.period):
            try:
                self._sample_nvml()
            except Exception:
                return

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=5)
            try:
                self._sample_nvml()      # the end of the timed region (after its synchronize)
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        for s_, m_, r_ in self.samples:
            sm.append(s_)
            smax = m_
            reasons |= r_
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "power_w": statistics.median(self.power) if self.power else None,
                "power_limit_w": self.power_limit,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


# ------------------------------------------------------------------------------ oracle legs

def oracle_sample(problem, budget_s: float, max_iters: int, omp: bool):
    """Time the CPU oracle (as it stands) on the first iterations of `problem` (at least one)."""
    import oracle
    o = oracle.Oracle(problem.method, problem.b, problem.z, left=problem.left,
                      full_x=problem.full_x, tol=problem.tol, itermax=problem.itermax, omp=omp)
    t0 = time.perf_counter()
    its = 0
    while its < max_iters:
        o.step(problem.op)
        its += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    o.close()
    return its, dt


def scaled_sample(name: str, problem):
    """A 16x smaller instance of the same config (same shifts, same generator recipe), for the
    one-thread oracle leg; None when the config has no size knob."""
    if name in ("c1", "c2", "c5"):
        return synth.make_problem(name, L=problem.op["L"] - 4)
    if name == "c3":
        return synth.make_problem(name, M=problem.M >> 4)
    if name == "c4":
        return synth.make_problem(name, W=int(round(math.sqrt(problem.M))) >> 2)
    return None


def cpu_legs(args, problem):
    """cpu_baseline (OpenMP, all cores, full size) and cpu_baseline_1core (scaled, extrapolated)."""
    import oracle
    out = {}
    its, dt = oracle_sample(problem, args.cpu_budget, 400, omp=True)
    out["cpu_baseline"] = {
        "value": problem.n_shift * its / dt, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle",
        "host": host_info(), "build": "OpenMP (static chunks, chunk partials combined in index order)",
        "sample": f"first {its} iterations of {problem.name} at full size (M={problem.M}), {dt:.1f} s "
                  f"on {oracle.threads()} threads"}
    base = problem.name.split("[")[0]
    small = scaled_sample(base, problem) if problem.M >= (1 << 22) else problem
    if small is not None:
        its1, dt1 = oracle_sample(small, args.cpu_budget, 400, omp=False)
        v = small.n_shift * its1 / dt1 * (small.M / problem.M)
        out["cpu_baseline_1core"] = {
            "value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_info(),
            "sample": (f"first {its1} iterations of {small.name} (M={small.M}), {dt1:.1f} s on one thread"
                       + ("" if small is problem else
                          f"; extrapolated to M={problem.M} by M_sample/M (oracle cost is linear in M)"))}
    return out


def run_reference(args, problem):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    o = oracle.Oracle(problem.method, problem.b, problem.z, left=problem.left,
                      full_x=problem.full_x, tol=problem.tol, itermax=problem.itermax, omp=True)
    for _ in range(args.warmup):
        o.step(problem.op)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.step(problem.op)
    dt = time.perf_counter() - t0
    o.close()
    val = problem.n_shift * args.steps / dt
    sample = (f"{problem.name}: oracle iterations {args.warmup}..{args.warmup + args.steps - 1} "
              f"of the full-size workload (M={problem.M}, N_z={problem.n_shift}), OpenMP on "
              f"{oracle.threads()} threads")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": config_dict(problem, 1),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle",
                             "sample": sample, "host": host_info()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_info():
    """CPU model and core count of the box the oracle baseline ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem = None
    try:
        with open("/proc/meminfo") as f:
            mem = round(int(f.readline().split()[1]) / 2 ** 20, 1)
    except (OSError, ValueError, IndexError):
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "ram_gib": mem}


def config_dict(problem, world):
    c = {"workload": f"{problem.name}: {synth.CONFIGS[problem.name.split('[')[0]]['desc']}",
         "M": problem.M, "n_shift": problem.n_shift, "n_left": problem.n_left,
         "method": problem.method, "full_x": problem.full_x,
         "parallelism": "single GPU" if world == 1 else
         f"rows sharded over {world} GPUs (top spin bits / contiguous row blocks); dots by NCCL "
         f"all-reduce; other ranks' rows read in place over NVLink (CUDA IPC)",
         "l2": "flushed before every timed step (256 MiB write, outside the events)"}
    return c


# ------------------------------------------------------------------------------ whole convergence

def run_converge(args, problem):
    """SURVEY §8(d.5) for C1/C2: the WHOLE convergence run (sk_run with status polled every 256
    iterations, graph-captured) timed with CUDA events on the solver's stream, median of
    `--repeats` runs on fresh contexts; one-time costs (module load, graph capture) are paid by a
    warm-up context first.  The OpenMP oracle's own full run beside it."""
    import torch
    from paper_2001_08707_b200 import shiftk
    from paper_2001_08707_b200.device import to_device
    dp = to_device(problem)
    st = torch.cuda.Stream()
    mk = lambda: shiftk.Solver(dp.op, problem.method, dp.b, problem.z, left=dp.left,
                               full_x=problem.full_x, tol=problem.tol, itermax=problem.itermax,
                               stream=st.cuda_stream)
    w = mk()
    w.run(256, poll_every=256)
    w.finalize()
    runs = []
    with ClockSampler(0) as clk:
        for _ in range(max(1, args.repeats)):
            s = mk()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                a.record(st)
                status = s.run(problem.itermax, poll_every=256)
                b.record(st)
            torch.cuda.synchronize()
            c = s.coefficients()
            _, _, ret = s.shift_state()
            runs.append((a.elapsed_time(b), status, c, ret, s.residuals()))
            s.finalize()
    runs.sort(key=lambda r: r[0])
    ms, status, c, ret, res = runs[len(runs) // 2]
    its = c["iterations"]
    line = {"metric": METRIC, "value": problem.n_shift * its / (ms * 1e-3), "unit": UNIT, "n_gpus": 1,
            "steps": its, "warmup": 256, "ms_per_step": ms / its, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": dict(config_dict(problem, 1), l2="not flushed (one continuous run)"),
            "mode": "whole convergence (SURVEY 8(d.5))",
            "converge": {"status": shiftk.STATUS_NAMES[status], "iterations": its, "switches": c["switches"],
                         "total_ms": ms, "runs_ms": [r[0] for r in runs],
                         "active_shift_iterations": int(sum(int(r) if r >= 0 else its for r in ret)),
                         "max_residual": float(np.max(res)), "tol": problem.tol},
            "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        import oracle
        o = oracle.Oracle(problem.method, problem.b, problem.z, left=problem.left,
                          full_x=problem.full_x, tol=problem.tol, itermax=problem.itermax, omp=True)
        t0 = time.perf_counter()
        ost = o.run(problem.op, problem.itermax)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": problem.n_shift * o.iterations / dt, "unit": UNIT,
                                "cores": oracle.threads(), "kind": "oracle", "host": host_info(),
                                "sample": f"the oracle's whole run of {problem.name}: {o.iterations} iterations "
                                          f"({oracle.STATUS_NAMES[ost]}) in {dt:.1f} s on {oracle.threads()} threads"}
        o.close()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU leg

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle time per CPU leg")
    ap.add_argument("--repeats", type=int, default=3, help="timed passes (value = the median)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--converge", action="store_true", help="time the whole convergence run (C1, C2)")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"
    rank, world, local = dist_env()
    problem = synth.make_problem(args.config)

    if args.impl == "reference":
        run_reference(args, problem)
        return
    if args.converge:
        run_converge(args, problem)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2001_08707_b200 import shiftk
    from paper_2001_08707_b200.device import to_device

    stream = torch.cuda.Stream()
    if world == 1:
        dp = to_device(problem, f"cuda:{local}")
        sl = None
    else:   # this rank's rows; the global problem is the same on every rank (strong scaling)
        from paper_2001_08707_b200 import dist as skdist
        dp, sl = skdist.to_device_slice(problem, world, rank, f"cuda:{local}")
    solver = shiftk.Solver(dp.op, problem.method, dp.b, problem.z, left=dp.left,
                           full_x=problem.full_x, tol=problem.tol, itermax=10 ** 9,
                           device=local, stream=stream.cuda_stream, rank=rank, world=world)
    if world > 1:
        skdist.connect(solver)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    with torch.cuda.stream(stream):
        solver.enqueue(args.warmup)
    torch.cuda.synchronize()

    def timed_pass(clk=None):
        """K steps, L2 flushed before each (outside the events); returns the summed step ms."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xff)
                starts[i].record(stream)
                solver.enqueue(1)
                ends[i].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))

    # passes 1..R (the value = the median pass): no instrumentation between the kernels
    n0 = solver.coefficients()["iterations"]   # (may launch the pending finish: before the count)
    launches0 = solver.profile()["launches"]
    passes = []
    with ClockSampler(local) as clk:
        for _ in range(max(1, args.repeats)):
            passes.append(timed_pass())
    launches = (solver.profile()["launches"] - launches0) // max(1, args.repeats)
    if world > 1:
        t = torch.tensor(passes, device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        passes = [float(v) for v in t.tolist()]
    total_ms = statistics.median(passes)
    # active shift-iterations of the timed windows: shift k is updated in
    # iteration m while m < retired_at[k] (per pass: the mean over the passes)
    n1 = solver.coefficients()["iterations"]
    _, _, ret = solver.shift_state()
    stop = np.where(ret >= 0, np.minimum(ret, n1), n1)
    active_its = int(np.clip(stop - n0, 0, None).sum()) / max(1, args.repeats)
    # pass 2 (the kernel shares): the same K steps with CUDA events around each kernel on the
    # solver's stream (the events cost the programmatic launch overlap, so not the value)
    solver.profile_enable(True)
    solver.profile(reset=True)
    prof_total_ms = timed_pass()
    prof = solver.profile(reset=True)
    solver.profile_enable(False)
    coeffs = solver.coefficients()
    value = problem.n_shift * args.steps / (total_ms * 1e-3)   # one global problem (strong scaling)

    # roofline of the dominant kernel (per launch: algorithmic bytes / mean device duration)
    peak, peak_src = measured_peaks()
    kernels = {"spmv": prof["ms_spmv"], "update": prof["ms_update"]}
    dom = max(kernels, key=kernels.get)
    per_launch_ms = kernels[dom] / max(prof["iterations"], 1)
    plan = solver.info()
    alg_bytes = bytes_per_row(problem, dom, plan) * problem.M / world   # this rank's rows
    achieved = alg_bytes / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"{problem.name}:{dom}")
    iter_bytes = (bytes_per_row(problem, "spmv") + bytes_per_row(problem, "update")) * problem.M / world
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(problem, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_launch": alg_bytes, "ms_per_launch": per_launch_ms,
                     "peak_source": peak_src},
        "profiled_pass_ms_per_step": prof_total_ms / args.steps,
        "kernel_ms_per_step": {k: v / max(prof["iterations"], 1) for k, v in
                               (("spmv", prof["ms_spmv"]), ("scalar", prof["ms_scalar"]),
                                ("update", prof["ms_update"]))},
        "iteration_gbs_model": iter_bytes / (total_ms / args.steps * 1e-3) / 1e9,
        "iteration_gbs_model_frac": iter_bytes / (total_ms / args.steps * 1e-3) / 1e9 / peak,
        "active_shift_iterations_per_s": active_its / (total_ms * 1e-3),
        "gpu_launches": launches,
        "passes_ms": passes,
        "plan": plan,
        "solver_state": {"iterations": coeffs["iterations"], "n_active": coeffs["n_active"],
                         "switches": coeffs["switches"]},
    }
    line["clocks"] = clk.summary()
    if world > 1:   # exchange volume of the SpMV: other ranks' rows read over NVLink (dist.py model)
        from paper_2001_08707_b200 import dist as skdist_model
        per = [skdist_model.remote_rows_per_spmv(problem, world, g) * 16 * (2 if problem.method == "bicg" else 1)
               for g in range(world)]
        line["nvlink_bytes_per_rank"] = {"max": max(per), "per_rank": per,
                                         "model": "element reads of other ranks' rows per iteration "
                                                  "(paper_2001_08707_b200/dist.py remote_rows_per_spmv)"}

    # the timed solver's arena (C5: 94 GB) is released before the end-to-end leg builds its own
    solver.finalize()
    torch.cuda.empty_cache()

    # end-to-end through the public API with HOST buffers (pinned b in, results out)
    if not args.no_e2e:
        src_b = problem.b if sl is None else sl.b
        src_left = problem.left if sl is None else sl.left
        b_host = torch.from_numpy(src_b).pin_memory()
        left_host = None if src_left is None else torch.from_numpy(src_left).pin_memory()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        s2 = shiftk.Solver(dp.op, problem.method, b_host, problem.z, left=left_host,
                           full_x=problem.full_x, tol=problem.tol, itermax=10 ** 9, device=local,
                           rank=rank, world=world)
        if world > 1:
            skdist.connect(s2)
        s2.run(args.steps, poll_every=max(args.steps, 1))
        y = s2.projections()
        res = s2.residuals()
        s2.finalize()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = src_b.nbytes + problem.z.nbytes + (0 if src_left is None else src_left.nbytes)
        d2h = y.nbytes + res.nbytes
        line["e2e"] = {"value": problem.n_shift * args.steps / e2e_s, "unit": UNIT,
                       "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                       "note": "sk_init(host b) + sk_run(K) + sk_get_projection/residual + finalize"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line.update(cpu_legs(args, problem))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
