"""Per-iteration time of sk_run / sk_enqueue with the host far ahead of the device."""
import os, sys, json
sys.path.insert(0, '/root/repo')
import torch, synth
from paper_2001_08707_b200 import shiftk
from paper_2001_08707_b200.device import to_device
p = synth.make_problem(sys.argv[1] if len(sys.argv) > 1 else "c2")
dp = to_device(p)
out = {}
for mode in ("enqueue", "run256", "run1024", "enqueue_again"):
    st = torch.cuda.Stream()
    s = shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol, itermax=10**9, stream=st.cuda_stream)
    with torch.cuda.stream(st):
        s.enqueue(16)   # capture the graph
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        torch.cuda._sleep(int(1e8))
        a.record(st)
        if mode.startswith("enqueue"): s.enqueue(1024)
        elif mode == "run256": s.run(1024, poll_every=256)
        else: s.run(1024, poll_every=1024)
        b.record(st)
    torch.cuda.synchronize()
    out[mode] = round(1e3 * a.elapsed_time(b) / 1024, 2)
    s.finalize()
print(json.dumps(out))
