"""Key raw metrics of every kernel in an ncu report."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_op_read_hit_rate.pct",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "launch__registers_per_thread", "launch__grid_size"]
extra = sys.argv[2:]
for v in rows[2:]:
    for k in keys + extra:
        if k in h:
            i = h.index(k)
            print(f"{k:60s} {v[i]} {u[i]}")
    print()
