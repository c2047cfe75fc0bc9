"""Timing probe (run by hand on the GPU box): per-kernel times of one iteration under
different L2 conditions, and the cost breakdown of the host-buffer e2e path."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2001_08707_b200 import shiftk  # noqa: E402
from paper_2001_08707_b200.device import to_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = 100
p = synth.make_problem(cfg)
dp = to_device(p)
stream = torch.cuda.Stream()
out = {}


def solver():
    return shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol,
                         itermax=10 ** 9, stream=stream.cuda_stream)


wbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(64 << 20, dtype=torch.float32, device="cuda")   # 256 MiB
for mode in ("write_flush", "write_flush_noprof", "write_read_flush", "no_flush", "no_flush_noprof"):
    s = solver()
    prof = not mode.endswith("noprof")
    s.profile_enable(prof)
    with torch.cuda.stream(stream):
        s.enqueue(5)
    torch.cuda.synchronize()
    s.profile(reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e9 * 200e-6 * K))   # GPU busy until every launch is queued
        for i in range(K):
            if not mode.startswith("no_flush"):
                wbuf.fill_(i & 255)
            if mode == "write_read_flush":
                rbuf.sum()
            ev[i][0].record(stream)
            s.enqueue(1)
            ev[i][1].record(stream)
    torch.cuda.synchronize()
    step_us = 1e3 * sum(a.elapsed_time(b) for a, b in ev) / K
    if not prof:
        out[mode] = {"step_us": step_us}
        s.finalize()
        continue
    pr = s.profile(reset=True)
    out[mode] = {"step_us": step_us,
                 "spmv_us": 1e3 * pr["ms_spmv"] / pr["iterations"],
                 "scalar_us": 1e3 * pr["ms_scalar"] / pr["iterations"],
                 "update_us": 1e3 * pr["ms_update"] / pr["iterations"]}
    s.finalize()

# graph mode, back-to-back iterations (no flush)
s = solver()
with torch.cuda.stream(stream):
    s.enqueue(32)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(stream):
    torch.cuda._sleep(int(2e9 * 0.05))
    a.record(stream)
    s.enqueue(1024)
    b.record(stream)
torch.cuda.synchronize()
out["graph_back_to_back_us_per_iter"] = 1e3 * a.elapsed_time(b) / 1024
s.finalize()

# e2e breakdown
b_host = torch.from_numpy(p.b).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
s2 = shiftk.Solver(dp.op, p.method, b_host, p.z, tol=p.tol, itermax=10 ** 9)
t1 = time.perf_counter()
s2.run(200, poll_every=200)
t2 = time.perf_counter()
y = s2.projections()
t3 = time.perf_counter()
s2.finalize()
t4 = time.perf_counter()
out["e2e_ms"] = {"init": 1e3 * (t1 - t0), "run200": 1e3 * (t2 - t1), "get": 1e3 * (t3 - t2),
                 "finalize": 1e3 * (t4 - t3)}
print(json.dumps(out, indent=1))
