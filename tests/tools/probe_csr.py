"""Time the CSR SpMV (standalone sk_apply_operator) on a full-size config: python probe_csr.py c3|c4"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import synth
from paper_2001_08707_b200 import shiftk
from paper_2001_08707_b200.device import to_device
name = sys.argv[1]
p = synth.make_problem(name)
dp = to_device(p)
r = dp.b.clone()
q = torch.empty_like(r)
for _ in range(3):
    shiftk.apply_operator(dp.op, r, q)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    shiftk.apply_operator(dp.op, r, q)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
nnz = p.op["col"].shape[0]
vb = 8 if p.op["kind"] == "csr_real" else 16
alg = nnz * (vb + 4) + 8 * p.M + 32 * p.M
print(f"{name} mode={os.environ.get('SHIFTK_CSR_ROW', '1')} spmv {ms:.3f} ms  {alg / ms / 1e6:.0f} GB/s algorithmic")
