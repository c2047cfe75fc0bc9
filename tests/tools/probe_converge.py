"""Whole convergence runs (SURVEY 8(d.5) for C1/C2): sk_run to convergence, device-timed."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import synth
from paper_2001_08707_b200 import shiftk
from paper_2001_08707_b200.device import to_device
out = {}
for name in (sys.argv[1:] or ["c1", "c2"]):
    p = synth.make_problem(name)
    dp = to_device(p)
    st = torch.cuda.Stream()
    # one-time costs (lazy module loading, graph capture) outside the timed run
    w = shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol,
                      itermax=p.itermax, stream=st.cuda_stream)
    w.run(64, poll_every=64)
    w.finalize()
    s = shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol,
                      itermax=p.itermax, stream=st.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(st):
        a.record(st)
        status = s.run(p.itermax, poll_every=256)
        b.record(st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = a.elapsed_time(b)
    c = s.coefficients()
    _, act, ret = s.shift_state()
    out[name] = {"status": status, "iterations": c["iterations"], "switches": c["switches"],
                 "device_ms": round(ms, 3), "wall_ms": round(1e3 * wall, 3),
                 "us_per_iteration": round(1e3 * ms / max(c["iterations"], 1), 2),
                 "shift_its_per_s": p.n_shift * c["iterations"] / (ms * 1e-3),
                 "active_shift_its": int(sum(int(r) if r >= 0 else c["iterations"] for r in ret))}
    s.finalize()
print(json.dumps(out, indent=1))
