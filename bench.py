#!/usr/bin/env python
"""Benchmark of the shifted-Krylov hot path (one JSON line on rank 0).

A step is one full iteration of shifted COCG/BiCG (seed SpMV with
fused dot, scalar recurrences + retirement + seed switch, fused three-term update with the
next-iteration dots and the per-shift projected / full update) over the config's synthetic
input.  Default workload: C2 (BASELINE.json configs[1]) — Heisenberg L=20, M=2^20, N_z=1024,
a=b projection, COCG, complex128.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Timing: W untimed iterations, then K iterations each bracketed by CUDA events on the solver's
stream, with L2 flushed (256 MiB write) before every step outside the events; barrier +
synchronize around the timed region; max over ranks.  Clocks are sampled with NVML every 2 ms
(nvidia-smi where NVML is missing) during the timed region.  `value` comes from a pass with nothing between the kernels; a second
pass of the same K flushed steps records CUDA events around every kernel (on the solver's
stream) for the per-kernel durations behind `roofline` (events between the kernels cost the
programmatic-launch overlap, ~10 us per step at C2, so that pass is not the value).  `--impl reference` times the CPU oracle (oracle/) on the same
workload (the reference arm of this tier: the paper has no code).
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


def bytes_per_row(problem, kernel: str) -> float:
    """Algorithmic bytes per row of one launch."""
    nseq = 2 if problem.method == "bicg" else 1
    if kernel == "spmv":
        if problem.op["kind"] in ("heisenberg", "heisenberg_sz"):   # generated on the fly
            bh = 0.0
        else:
            nnz_row = problem.op["col"].shape[0] / problem.M
            vb = 8 if problem.op["kind"] == "csr_real" else 16
            bh = nnz_row * (vb + 4) + 8
        return bh + 32.0 * nseq
    if kernel == "update":
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
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


# ------------------------------------------------------------------------------ oracle legs

def oracle_sample(problem, budget_s: float, max_iters: int):
    """Time the CPU oracle (as it stands) on the first iterations of the workload."""
    import oracle
    o = oracle.Oracle(problem.method, problem.b, problem.z, left=problem.left,
                      full_x=problem.full_x, tol=problem.tol, itermax=problem.itermax)
    t0 = time.perf_counter()
    its = 0
    while its < max_iters:
        o.step(problem.op)
        its += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return its, dt


def run_reference(args, problem):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    o = oracle.Oracle(problem.method, problem.b, problem.z, left=problem.left,
                      full_x=problem.full_x, tol=problem.tol, itermax=problem.itermax)
    for _ in range(args.warmup):
        o.step(problem.op)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.step(problem.op)
    dt = time.perf_counter() - t0
    val = problem.n_shift * args.steps / dt
    sample = (f"{problem.name}: oracle iterations {args.warmup}..{args.warmup + args.steps - 1} "
              f"of the full-size workload (M={problem.M}, N_z={problem.n_shift})")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": config_dict(problem, 1),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "host": host_info()},
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
    return {"cpu": model, "nproc": os.cpu_count()}


def config_dict(problem, world):
    c = {"workload": f"{problem.name}: {synth.CONFIGS[problem.name.split('[')[0]]['desc']}",
         "M": problem.M, "n_shift": problem.n_shift, "n_left": problem.n_left,
         "method": problem.method, "full_x": problem.full_x,
         "parallelism": "single GPU" if world == 1 else
         f"rows sharded over {world} GPUs (top spin bits / contiguous row blocks); dots by NCCL "
         f"all-reduce; other ranks' rows read in place over NVLink (CUDA IPC)",
         "l2": "flushed before every timed step (256 MiB write, outside the events)"}
    return c


# ------------------------------------------------------------------------------ GPU leg

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle time")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"
    rank, world, local = dist_env()
    problem = synth.make_problem(args.config)

    if args.impl == "reference":
        run_reference(args, problem)
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

    # pass 1 (the value): no instrumentation between the kernels
    n0 = solver.coefficients()["iterations"]   # (may launch the pending finish: before the count)
    launches0 = solver.profile()["launches"]
    with ClockSampler(local) as clk:
        total_ms = timed_pass()
    launches = solver.profile()["launches"] - launches0
    # active shift-iterations of the timed window: shift k is updated in
    # iteration m while m < retired_at[k]
    n1 = solver.coefficients()["iterations"]
    _, _, ret = solver.shift_state()
    stop = np.where(ret >= 0, np.minimum(ret, n1), n1)
    active_its = int(np.clip(stop - n0, 0, None).sum())
    # pass 2 (the kernel shares): the same K steps with CUDA events around each kernel on the
    # solver's stream (the events cost the programmatic launch overlap, so not the value)
    solver.profile_enable(True)
    solver.profile(reset=True)
    prof_total_ms = timed_pass()
    prof = solver.profile(reset=True)
    solver.profile_enable(False)
    coeffs = solver.coefficients()
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = problem.n_shift * args.steps / (total_ms * 1e-3)   # one global problem (strong scaling)

    # roofline of the dominant kernel (per launch: algorithmic bytes / mean device duration)
    peak, peak_src = measured_peaks()
    kernels = {"spmv": prof["ms_spmv"], "update": prof["ms_update"]}
    dom = max(kernels, key=kernels.get)
    per_launch_ms = kernels[dom] / max(prof["iterations"], 1)
    alg_bytes = bytes_per_row(problem, dom) * problem.M / world   # this rank's rows
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
        "solver_state": {"iterations": coeffs["iterations"], "n_active": coeffs["n_active"],
                         "switches": coeffs["switches"]},
    }
    line["clocks"] = clk.summary()

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
        its, dt = oracle_sample(problem, args.cpu_budget, 400)
        line["cpu_baseline"] = {"value": problem.n_shift * its / dt, "unit": UNIT, "cores": 1,
                                "host": host_info(),
                                "kind": "oracle",
                                "sample": f"first {its} iterations of {problem.name} (full size), "
                                          f"{dt:.1f} s single-threaded"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
