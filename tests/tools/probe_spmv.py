"""Stand-alone Heisenberg SpMV (sk_apply_operator) timing: warm (back-to-back) and cold (L2
flushed before each launch), for several chain lengths."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2001_08707_b200 import shiftk
Ls = [int(x) for x in sys.argv[1:]] or [16, 20, 24, 26]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for L in Ls:
    M = 1 << L
    r = torch.randn(M, dtype=torch.complex128, device="cuda")
    q = torch.empty_like(r)
    op = shiftk.make_operator({"kind": "heisenberg", "L": L, "J": 1.0}, M, None)
    for _ in range(3):
        shiftk.apply_operator(op, r, q)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n = 50
    ev[0].record()
    for _ in range(n):
        shiftk.apply_operator(op, r, q)
    ev[1].record(); torch.cuda.synchronize()
    warm = 1e3 * ev[0].elapsed_time(ev[1]) / n
    cold = []
    for i in range(10):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); shiftk.apply_operator(op, r, q); b.record(); torch.cuda.synchronize()
        cold.append(1e3 * a.elapsed_time(b))
    cold = sorted(cold)[len(cold) // 2]
    # cold data, warm code: flush, then the same kernel on another vector, then time on r
    r2 = torch.randn_like(r)
    q2 = torch.empty_like(r)
    colddata = []
    for i in range(10):
        flush.fill_(i)
        shiftk.apply_operator(op, r2, q2)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); shiftk.apply_operator(op, r, q); b.record(); torch.cuda.synchronize()
        colddata.append(1e3 * a.elapsed_time(b))
    colddata = sorted(colddata)[len(colddata) // 2]
    # graph of n back-to-back launches (no host overhead)
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        shiftk.apply_operator(op, r, q, st.cuda_stream)
        with torch.cuda.graph(gr, stream=st):
            for _ in range(n):
                shiftk.apply_operator(op, r, q, st.cuda_stream)
    torch.cuda.synchronize()
    gr.replay(); torch.cuda.synchronize()
    ev[0].record(); gr.replay(); ev[1].record(); torch.cuda.synchronize()
    graph = 1e3 * ev[0].elapsed_time(ev[1]) / n
    byt = 32 * M
    out[L] = {"graph_us": round(graph, 2), "graph_GBps": round(byt / graph / 1e3, 1), "warm_us": round(warm, 2), "cold_us": round(cold, 2), "colddata_us": round(colddata, 2),
              "warm_GBps": round(byt / warm / 1e3, 1), "cold_GBps": round(byt / cold / 1e3, 1)}
print(json.dumps(out, indent=1))
