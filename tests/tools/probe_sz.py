"""Stand-alone Sz-sector Heisenberg SpMV timing (sk_apply_operator), L given, n = L/2."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2001_08707_b200 import shiftk
out = {}
for L in [int(x) for x in sys.argv[1:]] or [24, 28, 30]:
    n = L // 2
    D = math.comb(L, n)
    r = torch.randn(D, dtype=torch.complex128, device="cuda")
    q = torch.empty_like(r)
    op = shiftk.make_operator({"kind": "heisenberg_sz", "L": L, "J": 1.0, "n_up": n}, D)
    for _ in range(2):
        shiftk.apply_operator(op, r, q)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        shiftk.apply_operator(op, r, q)
    b.record(); torch.cuda.synchronize()
    us = 1e3 * a.elapsed_time(b) / 5
    out[L] = {"rows": D, "us": round(us, 1), "alg_GBps": round(32 * D / us / 1e3, 1)}
    del r, q
print(json.dumps(out))
