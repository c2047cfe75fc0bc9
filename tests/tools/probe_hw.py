"""Calibration probe: copy bandwidth vs size (L2 flushed), and back-to-back tiny-kernel latency."""
import json, torch
out = {}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
rb = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
for mb in (4, 16, 64, 256, 1024):
    n = (mb << 20) // 16
    a = torch.randn(n, dtype=torch.complex128, device="cuda")
    b = torch.empty_like(a)
    ts = []
    for i in range(10):
        flush.fill_(i); rb.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); b.copy_(a); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = min(ts[2:])
    out[f"copy_{mb}MB"] = {"us": round(1e3 * t, 2), "GBps": round(2 * mb * 1.048576e6 / (t * 1e-3) / 1e9, 1)}
# tiny kernels back to back in a graph
x = torch.zeros(1, device="cuda")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    x.add_(1)
    with torch.cuda.graph(g, stream=s):
        for _ in range(100):
            x.add_(1)
torch.cuda.synchronize()
for _ in range(3): g.replay()
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); g.replay(); e.record(); torch.cuda.synchronize()
out["tiny_kernel_in_graph_us"] = round(1e3 * a.elapsed_time(e) / 100, 2)
a.record()
for _ in range(100): x.add_(1)
e.record(); torch.cuda.synchronize()
out["tiny_kernel_stream_us"] = round(1e3 * a.elapsed_time(e) / 100, 2)
print(json.dumps(out, indent=1))
