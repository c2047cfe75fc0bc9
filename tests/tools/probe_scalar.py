"""Phase timestamps of the scalar kernel (run on the GPU box with SHIFTK_DEBUG_TS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["SHIFTK_DEBUG_TS"] = "1"
import numpy as np, torch
import synth
from paper_2001_08707_b200.device import to_device, make_solver
p = synth.make_problem(sys.argv[1] if len(sys.argv) > 1 else "c2")
g = make_solver(to_device(p))
g.run(20)
for i in range(5):
    g.enqueue(1)
    ts = g.debug_timestamps()
    t0 = ts[0]
    print({k: int(ts[k] - t0) for k in (1, 2, 5, 6, 3, 4)})
