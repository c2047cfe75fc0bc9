"""Floor of the bench harness: two trivial kernels after the 256 MiB L2 flush, bracketed by CUDA
events (graph replay vs direct launches)."""
import torch, json
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x = torch.zeros(1, device="cuda")
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    x.add_(1); x.add_(1)
    with torch.cuda.graph(g, stream=st):
        x.add_(1); x.add_(1)
torch.cuda.synchronize()
res = {}
for mode in ("graph2", "direct2"):
    ts = []
    for i in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            flush.fill_(i)
            a.record(st)
            if mode == "graph2": g.replay()
            else: x.add_(1); x.add_(1)
            b.record(st)
        torch.cuda.synchronize()
        ts.append(1e3 * a.elapsed_time(b))
    res[mode] = sorted(ts)[10]
print(json.dumps(res))
