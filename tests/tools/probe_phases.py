"""Phase stamps (ns, relative to the first SpMV worker CTA) of one iteration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["SHIFTK_DEBUG_TS"] = "1"
import torch
import synth
from paper_2001_08707_b200.device import to_device, make_solver
p = synth.make_problem(sys.argv[1] if len(sys.argv) > 1 else "c2")
from paper_2001_08707_b200 import shiftk
dp = to_device(p)
st = torch.cuda.Stream()
g = shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol,
                  itermax=p.itermax, stream=st.cuda_stream)
g.run(20)
names = {0: "spmv_worker1_start", 1: "agent_start", 2: "finish_done", 3: "last_cta", 4: "seed_done",
         5: "shift_agent_start", 6: "shift_done", 7: "upd_worker1_start", 8: "upd_lastcta_end",
         9: "seed_reduced", 10: "commit_reduced", 11: "commit_seeded", 12: "finish_reduced",
         13: "upd_w0_enter", 14: "upd_w0_seeded"}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if "flush" in sys.argv else None
for i in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        if flush is not None:
            flush.fill_(i)
        a.record(st)
        g.enqueue(1)
        b.record(st)
    torch.cuda.synchronize()
    ts = g.debug_timestamps()
    t0 = ts[0]
    d = {names[k]: int(ts[k] - t0) for k in range(15)}
    d["event_step_ns"] = int(1e6 * a.elapsed_time(b))
    print(d)
