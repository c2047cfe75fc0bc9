"""Summarise an ncu --import-source report: per-CUDA-line stall samples (top N)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if "Source" in r and any("Sampling" in c for c in r))
hdr = rows[hdr_i]
si = next(i for i, c in enumerate(hdr) if c.startswith("Warp Stall Sampling (All"))
src_i = hdr.index("Source")
data = []
for r in rows[hdr_i + 1:]:
    if len(r) <= si:
        continue
    try:
        v = float(r[si])
    except ValueError:
        continue
    data.append((v, r))
tot = sum(v for v, _ in data) or 1
print("total samples", tot)
for v, r in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{100*v/tot:5.1f}% {r[0][:12]:12s} {r[src_i][:110]}")
